// proj/src/gpu_eval.cpp -- the reference-side binding a maintainer would add
// to route hfmm::evaluate_with_setup / evaluate_potential and the RankEngine
// phases (traversal.hpp:120-166) to B200s through the C ABI
// (include/hfmm_gpu.h).  Kept as a real source file so that it is compiled
// against the reference's own headers and run against the reference on the
// GPU (oracle/Makefile target adapter_check, tests/test_gpu_adapter.py);
// INTEGRATION.md walks through it.
//
// The caller's GlobalSetup is IMPORTED (setup_flat.hpp -> hfmm_setup_import):
// the Morton sort, partition, slices, lists and plans the reference built
// are used as they are.  All logical ranks run in this process
// (hfmm_world), as the reference's run_world runs them.
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "gpu_eval.hpp"
#include "hfmm/operators.hpp"
#include "hfmm_gpu.h"
#include "setup_flat.hpp"

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
hfmm_world* make_world(hfmm_setup* hs, const std::vector<int>& devices) {
  hfmm_world* w = nullptr;
  check(hfmm_world_create(hs, devices.data(), int(devices.size()), &w));
  return w;
}

// The reference's flop charges per rank and phase (operators.hpp:16-20,
// traversal.cpp:306-788, interp_flops sphere_grid.cpp:220-226): exact for
// C2M, M2L, L2O and Near; M2M / L2L charge each child's interpolation to its
// owner (a plural child's to its users by their interpolation columns, the
// parallel_interpolate split) plus the shift and aggregation per parent slice.
void charge_flops(const GlobalSetup& s, CostLedger& led) {
  const int L = s.tree.levels, P = s.partition.num_ranks;
  const LevelSampling& sl = s.samplings[std::size_t(L)];
  auto add = [&](int r, Phase p, double f) { led.ranks[std::size_t(r)].at(p).flops += std::uint64_t(f); };
  for (int r = 0; r < P; ++r) {
    auto [lb, le] = s.partition.rank_ranges[std::size_t(r)];
    for (std::size_t li = lb; li < le; ++li) {
      auto [pb, pe] = s.leaf_particles[li];
      const double entries = double(pe - pb) * double(sl.num_samples());
      add(r, Phase::C2M, double(kC2MFlopsPerEntry) * entries);
      add(r, Phase::L2O, double(kL2OFlopsPerEntry) * entries);
      double srcs = 0.0;
      for (const MortonKey& nk : s.lists.near.at(s.leaves[li].packed())) {
        auto it = std::lower_bound(s.leaves.begin(), s.leaves.end(), nk);
        auto [sb, se] = s.leaf_particles[std::size_t(it - s.leaves.begin())];
        srcs += double(se - sb);
      }
      add(r, Phase::Near, double(kNearFlopsPerPair) * srcs * double(pe - pb));
    }
  }
  for (int l = s.top_level; l <= L; ++l) {
    const LevelSampling& sp = s.samplings[std::size_t(l)];
    for (const NodeInfo& o : s.levels[std::size_t(l)].nodes) {
      auto it = s.lists.far.find(o.key.packed());
      const double nfar = it == s.lists.far.end() ? 0.0 : double(it->second.size());
      for (const Slice& x : o.slices)
        add(x.rank, Phase::M2L, double(kM2LFlopsPerSample) * double(x.size()) * nfar);
      if (l == L) continue;
      const LevelSampling& sc = s.samplings[std::size_t(l + 1)];
      const double fi = interp_flops(sc.n_theta, sc.n_phi, sp.n_theta, sp.n_phi);
      const double Sp = double(sp.num_samples());
      for (std::size_t ci : o.children) {
        const NodeInfo& c = s.levels[std::size_t(l + 1)].nodes[ci];
        if (!c.plural) {
          for (Phase ph : {Phase::M2M, Phase::L2L}) add(c.first_user, ph, fi + kShiftFlopsPerSample * Sp);
        } else {
          const auto users = c.user_ranks();
          for (std::size_t u = 0; u < users.size(); ++u) {
            const double share = double(c.interp_layout.splits[u + 1] - c.interp_layout.splits[u]) /
                                 double(sp.n_theta);
            for (Phase ph : {Phase::M2M, Phase::L2L}) add(users[u], ph, share * (fi + kShiftFlopsPerSample * Sp));
          }
        }
      }
      for (const Slice& x : o.slices)
        for (Phase ph : {Phase::M2M, Phase::L2L}) add(x.rank, ph, 2.0 * double(x.size()) * double(o.children.size()));
    }
  }
}
}  // namespace

hfmm_setup* import_setup_b200(const GlobalSetup& s) {
  hfmm_run_config c = to_c(s.config);
  c.num_ranks = s.partition.num_ranks;
  hfmm_setup_import* im = nullptr;
  check(hfmm_setup_import_begin(&c, &im));
  try {
    flatten_setup(s, [&](const std::string& name, const auto& v) {
      check(hfmm_setup_import_put(im, name.c_str(), v.data(), v.size() * sizeof(v[0])));
    });
  } catch (...) {
    hfmm_setup_import_abort(im);
    throw;
  }
  hfmm_setup* hs = nullptr;
  check(hfmm_setup_import_end(im, &hs));  // consumes im
  return hs;
}

EvalResult evaluate_with_setup_b200(const GlobalSetup& s, std::vector<int> devices) {
  if (devices.empty()) devices = {0};
  hfmm_setup* hs = import_setup_b200(s);
  hfmm_world* w = nullptr;
  try {
    w = make_world(hs, devices);
  } catch (...) {
    hfmm_setup_destroy(hs);
    throw;
  }
  hfmm_setup_destroy(hs);  // the world shares ownership of the imported setup
  const int P = s.partition.num_ranks;
  EvalResult out;
  out.potentials.resize(s.particles.size());
  std::vector<double> ms(std::size_t(P) * kNumPhases, 0.0);
  hfmm_status st = hfmm_world_evaluate(w, nullptr, reinterpret_cast<double*>(out.potentials.data()), ms.data());
  hfmm_world_destroy(w);
  check(st);
  out.ledger.ranks.resize(std::size_t(P));
  out.ledger.virtual_time = false;  // device time (CUDA events), like the Threaded scheduler's wall clock
  for (int r = 0; r < P; ++r)
    for (int p = 0; p < kNumPhases; ++p)
      out.ledger.ranks[std::size_t(r)].phases[std::size_t(p)].seconds = 1e-3 * ms[std::size_t(r) * kNumPhases + std::size_t(p)];
  charge_flops(s, out.ledger);
  return out;
}

EvalResult evaluate_potential_b200(const std::vector<Particle>& ps, const RunConfig& cfg, std::vector<int> devices) {
  cfg.validate();  // the reference's error before any work (traversal.cpp:42-46)
  return evaluate_with_setup_b200(build_setup(ps, cfg), std::move(devices));
}

B200RankWorld::B200RankWorld(const GlobalSetup& s, std::vector<int> devices) : s_(s) {
  if (devices.empty()) devices = {0};
  setup_ = import_setup_b200(s);
  try {
    world_ = make_world(setup_, devices);
  } catch (...) {
    hfmm_setup_destroy(setup_);
    throw;
  }
}

B200RankWorld::~B200RankWorld() {
  hfmm_world_destroy(world_);
  hfmm_setup_destroy(setup_);
}

void B200RankWorld::c2m_phase() { check(hfmm_world_run_phase(world_, HFMM_PHASE_C2M)); }
void B200RankWorld::m2m_pass() { check(hfmm_world_run_phase(world_, HFMM_PHASE_M2M)); }
void B200RankWorld::m2l_pass() { check(hfmm_world_run_phase(world_, HFMM_PHASE_M2L)); }
void B200RankWorld::l2l_pass() { check(hfmm_world_run_phase(world_, HFMM_PHASE_L2L)); }

std::vector<cplx> B200RankWorld::l2o_near_phase() {
  check(hfmm_world_run_phase(world_, HFMM_PHASE_L2T));
  std::vector<cplx> pot(s_.particles.size());
  check(hfmm_world_potentials(world_, reinterpret_cast<double*>(pot.data())));
  return pot;
}

std::optional<std::vector<cplx>> B200RankWorld::slice_of(int rank, int kind, const MortonKey& key) const {
  if (key.level < s_.top_level || key.level > s_.tree.levels) return std::nullopt;
  const LevelTable& t = s_.levels[std::size_t(key.level)];
  const NodeInfo* n = t.find(key);
  if (!n) return std::nullopt;
  auto sl = n->slice_for(rank);
  if (!sl) return std::nullopt;
  const std::size_t S = s_.samplings[std::size_t(key.level)].num_samples();
  std::vector<cplx> all(t.nodes.size() * S);
  check(hfmm_world_get_expansion(world_, rank, kind, key.level, reinterpret_cast<double*>(all.data()), 2 * all.size()));
  const std::size_t i = t.index.at(key.packed());
  return std::vector<cplx>(all.begin() + std::ptrdiff_t(i * S + sl->first),
                           all.begin() + std::ptrdiff_t(i * S + sl->second));
}

std::optional<std::vector<cplx>> B200RankWorld::multipole(int rank, const MortonKey& key) const {
  return slice_of(rank, 0, key);
}
std::optional<std::vector<cplx>> B200RankWorld::local_expansion(int rank, const MortonKey& key) const {
  return slice_of(rank, 1, key);
}

}  // namespace hfmm
