// Declarations of the reference-side B200 binding (gpu_eval.cpp).
#ifndef HFMM_GPU_EVAL_HPP
#define HFMM_GPU_EVAL_HPP
#include <vector>

#include "hfmm/traversal.hpp"

namespace hfmm {
// Drop-in for evaluate_with_setup (traversal.cpp:790-817) on one B200.
EvalResult evaluate_with_setup_b200(const GlobalSetup& s, int device = 0);
// Drop-in for evaluate_potential (traversal.cpp:819-823).
EvalResult evaluate_potential_b200(const std::vector<Particle>& ps, const RunConfig& cfg, int device = 0);
}  // namespace hfmm
#endif
