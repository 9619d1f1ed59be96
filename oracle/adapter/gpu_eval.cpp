// proj/src/gpu_eval.cpp -- the reference-side binding a maintainer would add
// to route hfmm::evaluate_with_setup / evaluate_potential (traversal.cpp:790-823)
// to the B200 engine through the C ABI (include/hfmm_gpu.h).  Kept as a real
// source file so that it is compiled against the reference's own headers and
// run against the reference on the GPU (oracle/Makefile target adapter_check,
// tests/test_gpu_adapter.py); INTEGRATION.md shows the same code.
#include <stdexcept>
#include <string>
#include <vector>

#include "hfmm/traversal.hpp"
#include "hfmm_gpu.h"
#include "gpu_eval.hpp"

namespace hfmm {
namespace {
// Rethrow the C-ABI status as the exception type the reference throws
// (traversal.cpp:42-46, operators.cpp:43-50, kernel.cpp:11, operators.cpp:160).
void check(hfmm_status st) {
  if (st == HFMM_OK) return;
  std::string msg = hfmm_last_error();
  switch (st) {
    case HFMM_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case HFMM_ERR_OUT_OF_RANGE:     throw std::out_of_range(msg);
    case HFMM_ERR_DOMAIN:           throw std::domain_error(msg);
    case HFMM_ERR_LOGIC:            throw std::logic_error(msg);
    case HFMM_ERR_LENGTH:           throw std::length_error(msg);
    default:                        throw std::runtime_error(msg);
  }
}
hfmm_run_config to_c(const RunConfig& r) {
  hfmm_run_config c;
  hfmm_run_config_default(&c);
  c.lambda = r.lambda; c.digits = r.digits; c.leaf_lambda = r.leaf_lambda;
  c.num_ranks = r.num_ranks; c.buffer_limit = r.buffer_limit;
  c.policy = r.policy == AlignPolicy::Aligned ? HFMM_POLICY_ALIGNED : HFMM_POLICY_RANK_ORDERED;
  c.one_particle_per_leaf = r.one_particle_per_leaf; c.top_level = r.top_level;
  c.d_override = r.d_override; c.seed = r.seed;
  return c;
}
}  // namespace

// Drop-in for evaluate_with_setup (traversal.cpp:790-817) on one B200.
EvalResult evaluate_with_setup_b200(const GlobalSetup& s, int device) {
  const size_t n = s.particles.size();
  std::vector<double> xyz(3 * n), q(2 * n);
  for (size_t i = 0; i < n; ++i) {            // back to input order
    const size_t j = s.original_index[i];
    const Particle& p = s.particles[i];
    xyz[3 * j] = p.position.x; xyz[3 * j + 1] = p.position.y; xyz[3 * j + 2] = p.position.z;
    q[2 * j] = p.intensity.real(); q[2 * j + 1] = p.intensity.imag();
  }
  hfmm_run_config c = to_c(s.config);
  c.num_ranks = 1;                           // one GPU = one logical rank
  hfmm_setup* hs = nullptr;
  check(hfmm_setup_build(xyz.data(), q.data(), n, &c, &hs));
  hfmm_gpu* g = nullptr;
  hfmm_status st = hfmm_gpu_create(hs, device, 0, &g);
  if (st != HFMM_OK) { hfmm_setup_destroy(hs); check(st); }
  EvalResult out;
  out.potentials.resize(n);
  hfmm_gpu_timing t;
  st = hfmm_gpu_evaluate(g, nullptr, reinterpret_cast<double*>(out.potentials.data()), &t);
  hfmm_gpu_destroy(g);
  hfmm_setup_destroy(hs);
  check(st);
  return out;                                 // ledger left empty: the device has its own timing
}

// Drop-in for evaluate_potential (traversal.cpp:819-823).
EvalResult evaluate_potential_b200(const std::vector<Particle>& ps, const RunConfig& cfg, int device) {
  std::vector<double> xyz(3 * ps.size()), q(2 * ps.size());
  for (size_t i = 0; i < ps.size(); ++i) {
    xyz[3 * i] = ps[i].position.x; xyz[3 * i + 1] = ps[i].position.y; xyz[3 * i + 2] = ps[i].position.z;
    q[2 * i] = ps[i].intensity.real(); q[2 * i + 1] = ps[i].intensity.imag();
  }
  hfmm_run_config c = to_c(cfg);
  c.num_ranks = 1;
  EvalResult out;
  out.potentials.resize(ps.size());
  check(hfmm_evaluate_potential(xyz.data(), q.data(), ps.size(), &c, device,
                                reinterpret_cast<double*>(out.potentials.data())));
  return out;
}
}  // namespace hfmm
