// Declarations of the reference-side B200 binding (gpu_eval.cpp): what a
// maintainer adds to proj/ so that callers of the reference's evaluation API
// (traversal.hpp:120-166) run on B200s through the C ABI (include/hfmm_gpu.h).
#ifndef HFMM_GPU_EVAL_HPP
#define HFMM_GPU_EVAL_HPP
#include <complex>
#include <memory>
#include <optional>
#include <vector>

#include "hfmm/traversal.hpp"

struct hfmm_setup;
struct hfmm_world;

namespace hfmm {

// Drop-in for evaluate_with_setup (traversal.cpp:790-817): the caller's
// GlobalSetup is imported as is (hfmm_setup_import: no build_setup, no
// re-sort), every logical rank of its partition runs on the given devices
// (rank r on devices[r % n]), and EvalResult carries the potentials in input
// order plus a CostLedger with one RankLedger per rank: device seconds per
// phase and the reference's flop charges (operators.hpp:16-20, interp_flops).
EvalResult evaluate_with_setup_b200(const GlobalSetup& s, std::vector<int> devices = {0});

// Drop-in for evaluate_potential (traversal.cpp:819-823): the B200 setup
// (bit-exact with build_setup) plus the same evaluation.
EvalResult evaluate_potential_b200(const std::vector<Particle>& ps, const RunConfig& cfg,
                                   std::vector<int> devices = {0});

// RankEngine phase seam (traversal.hpp:125-156) for every rank of a setup at
// once, the way run_world drives the reference's engines: each phase runs on
// all ranks with the exchanges it owns.  multipole / local_expansion return
// rank r's stored slice of a node (nullopt where the reference returns
// nullptr: the rank holds no slice of it).
class B200RankWorld {
 public:
  explicit B200RankWorld(const GlobalSetup& s, std::vector<int> devices = {0});
  ~B200RankWorld();
  B200RankWorld(const B200RankWorld&) = delete;
  B200RankWorld& operator=(const B200RankWorld&) = delete;

  void c2m_phase();
  void m2m_pass();
  void m2l_pass();
  void l2l_pass();
  // L2O + near field on every rank; potentials of all particles in INPUT order.
  std::vector<cplx> l2o_near_phase();

  std::optional<std::vector<cplx>> multipole(int rank, const MortonKey& key) const;
  std::optional<std::vector<cplx>> local_expansion(int rank, const MortonKey& key) const;

 private:
  std::optional<std::vector<cplx>> slice_of(int rank, int kind, const MortonKey& key) const;
  const GlobalSetup& s_;
  hfmm_setup* setup_ = nullptr;
  hfmm_world* world_ = nullptr;
};

// The caller's GlobalSetup imported into the B200 library (no build_setup).
hfmm_setup* import_setup_b200(const GlobalSetup& s);

}  // namespace hfmm
#endif
