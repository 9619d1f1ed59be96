// Runs the reference-side binding (gpu_eval.cpp) next to the reference's own
// CPU evaluation, through the reference's C++ API, on seeded inputs.  The
// checks follow the reference's traversal tests (proj/tests/test_traversal.cpp)
// with the B200 entry points in place of the CPU ones:
//   - evaluate_with_setup_b200(GlobalSetup) vs hfmm::evaluate_with_setup at
//     1 and 4 ranks (1e-10), the setup imported as built by the reference;
//     ledger flops of C2M / M2L / L2O / Near equal to the reference's ledger;
//   - evaluate_potential_b200 vs hfmm::evaluate_potential;
//   - single-rank evaluation vs the direct oracle at digits 3 (<= 1e-3,
//     test_traversal.cpp:78-86), zero intensities (:88-96), one particle per
//     leaf near-field ledger = 20 x pairs (:98-109);
//   - distributed upward pass reproduces the serial root multipole at 2, 3
//     and 5 ranks through the RankEngine seam (:111-172), and equals the
//     reference's root multipole;
//   - an invalid RunConfig raises the same std exception type on both paths.
// TEST INFRASTRUCTURE (tests/test_gpu_adapter.py); prints one line per check.
#include <cmath>
#include <complex>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "gpu_eval.hpp"
#include "hfmm/kernel.hpp"
#include "inputs.hpp"

using hfmm::cplx;

static int bad = 0;

static void expect(bool ok, const char* what, double v = 0.0) {
  std::printf("%-72s %s (%.3e)\n", what, ok ? "ok" : "FAILED", v);
  if (!ok) ++bad;
}

static double rel_l2(const std::vector<cplx>& a, const std::vector<cplx>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += std::norm(a[i] - b[i]);
    den += std::norm(b[i]);
  }
  return den > 0 ? std::sqrt(num / den) : std::sqrt(num);
}

static std::vector<hfmm::Particle> particles(int shape, size_t n, double ext, uint64_t seed) {
  std::vector<double> xyz(3 * n), q(2 * n);
  hfmm_b200::generate_inputs(shape, n, ext, seed, xyz.data(), q.data());
  std::vector<hfmm::Particle> ps(n);
  for (size_t i = 0; i < n; ++i) {
    ps[i].position = hfmm::Vec3{xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
    ps[i].intensity = cplx(q[2 * i], q[2 * i + 1]);
  }
  return ps;
}

static std::vector<hfmm::Particle> grid_particles(double extent, std::uint64_t seed = 7) {
  hfmm::GeometrySpec g;
  g.kind = hfmm::GeometryKind::PlanarGrid;
  g.extent = extent;
  g.spacing = 0.25;
  return hfmm::generate_geometry(g, 1.0, hfmm::IntensityRule::RandomSeeded, seed);
}

template <class F>
static std::string exception_kind(F f) {
  try {
    f();
  } catch (const std::invalid_argument&) {
    return "invalid_argument";
  } catch (const std::out_of_range&) {
    return "out_of_range";
  } catch (const std::domain_error&) {
    return "domain_error";
  } catch (const std::length_error&) {
    return "length_error";
  } catch (const std::logic_error&) {
    return "logic_error";
  } catch (const std::exception&) {
    return "exception";
  }
  return "none";
}

int main() {
  using namespace hfmm;
  char line[256];
  struct Case { int shape; size_t n; double ext; uint64_t seed; double digits; int ranks; };
  for (const Case& c : {Case{0, 20000, 3.0, 41, 3.0, 1}, Case{1, 30000, 2.0, 42, 4.0, 4},
                        Case{0, 100000, 4.0, 0, 3.0, 1}}) {
    const auto ps = particles(c.shape, c.n, c.ext, c.seed);
    RunConfig cfg;
    cfg.digits = c.digits;
    cfg.num_ranks = c.ranks;
    const GlobalSetup s = build_setup(ps, cfg);
    const EvalResult want = evaluate_with_setup(s);
    const EvalResult got = evaluate_with_setup_b200(s);
    const double e1 = rel_l2(got.potentials, want.potentials);
    std::snprintf(line, sizeof line, "shape=%d n=%zu digits=%.0f ranks=%d evaluate_with_setup_b200 vs reference",
                  c.shape, c.n, c.digits, c.ranks);
    expect(e1 < 1e-10, line, e1);
    bool ledger_ok = got.ledger.ranks.size() == size_t(c.ranks);
    for (Phase p : {Phase::C2M, Phase::M2L, Phase::L2O, Phase::Near})
      for (int r = 0; r < c.ranks && ledger_ok; ++r)
        ledger_ok = got.ledger.ranks[size_t(r)].at(p).flops == want.ledger.ranks[size_t(r)].at(p).flops;
    expect(ledger_ok && got.ledger.total(Phase::M2L).seconds > 0, "  ledger: per-rank C2M/M2L/L2O/Near flops equal the reference's");
    const EvalResult got2 = evaluate_potential_b200(ps, cfg);
    const double e2 = rel_l2(got2.potentials, want.potentials);
    expect(e2 < 1e-10, "  evaluate_potential_b200 vs reference", e2);
  }
  {  // test_traversal.cpp:78-86
    auto p = grid_particles(8.0);
    RunConfig cfg;
    cfg.digits = 3;
    EvalResult res = evaluate_potential_b200(p, cfg);
    std::vector<Vec3> obs;
    for (const auto& q : p) obs.push_back(q.position);
    const auto want = direct_potential(p, obs, Wavenumber::from_lambda(cfg.lambda));
    const double e = rel_l2(res.potentials, want);
    expect(e <= 1e-3 && res.ledger.grand_total().flops > 0, "32x32 grid, digits 3: B200 vs direct oracle <= 1e-3", e);
  }
  {  // :88-96
    auto p = grid_particles(4.0);
    for (auto& q : p) q.intensity = {0.0, 0.0};
    RunConfig cfg;
    EvalResult res = evaluate_potential_b200(p, cfg);
    bool zero = true;
    for (const auto& v : res.potentials) zero = zero && std::abs(v) == 0.0;
    expect(zero && res.ledger.total(Phase::Near).flops > 0, "zero intensities: zero potentials, populated ledger");
  }
  {  // :98-109
    auto p = grid_particles(4.0);
    RunConfig cfg;
    cfg.one_particle_per_leaf = true;
    GlobalSetup s = build_setup(p, cfg);
    EvalResult res = evaluate_with_setup_b200(s);
    std::uint64_t pairs = 0;
    for (const MortonKey& leaf : s.leaves) pairs += s.lists.near.at(leaf.packed()).size();
    expect(res.ledger.total(Phase::Near).flops == 20u * pairs, "one particle per leaf: Near flops == 20 x pairs",
           double(pairs));
  }
  {  // :111-172 through the RankEngine seam
    GeometrySpec g;
    g.kind = GeometryKind::CubicVolume;
    g.extent = 2.0;
    g.spacing = 1.0;
    auto p = generate_geometry(g, 1.0, IntensityRule::RandomSeeded, 5);
    RunConfig cfg;
    cfg.leaf_lambda = 1.0;
    cfg.top_level = 1;
    GlobalSetup serial_setup = build_setup(p, cfg);
    MortonKey root{1, 0};
    std::vector<cplx> serial_root, ref_root;
    {
      B200RankWorld w(serial_setup);
      w.c2m_phase();
      w.m2m_pass();
      serial_root = w.multipole(0, root).value();
    }
    {
      WorldOptions opt;
      opt.num_ranks = 1;
      run_world(opt, [&](Endpoint& ep) {
        RankEngine eng(serial_setup, ep);
        eng.c2m_phase();
        eng.m2m_pass();
        ref_root = *eng.multipole(root);
      });
    }
    const double er = rel_l2(serial_root, ref_root);
    expect(serial_setup.leaves.size() == 8u && er < 1e-10, "root multipole (8 leaves, top_level 1) vs reference", er);
    for (int ranks : {2, 3, 5}) {
      RunConfig cfgN = cfg;
      cfgN.num_ranks = ranks;
      GlobalSetup setup = build_setup(p, cfgN);
      B200RankWorld w(setup);
      w.c2m_phase();
      w.m2m_pass();
      const NodeInfo* node = setup.levels[1].find(root);
      std::vector<cplx> assembled(serial_root.size(), cplx(0, 0));
      for (int r = 0; r < ranks; ++r) {
        auto slice = node->slice_for(r);
        auto mp = w.multipole(r, root);
        if (!slice) continue;
        for (size_t i = 0; i < mp->size(); ++i) assembled[slice->first + i] = (*mp)[i];
      }
      const double e = rel_l2(assembled, serial_root);
      std::snprintf(line, sizeof line, "distributed upward pass, %d ranks: assembled root vs serial < 1e-12", ranks);
      expect(e < 1e-12, line, e);
    }
  }
  {
    const auto ps = particles(0, 1000, 1.0, 43);
    RunConfig cfg;
    cfg.digits = -1.0;  // RunConfig::validate rejects it
    const std::string a = exception_kind([&] { evaluate_potential(ps, cfg); });
    const std::string b = exception_kind([&] { evaluate_potential_b200(ps, cfg); });
    std::snprintf(line, sizeof line, "invalid config: reference throws %s, b200 binding throws %s", a.c_str(), b.c_str());
    expect(a == b && a != "none", line);
  }
  std::printf(bad ? "ADAPTER CHECK FAILED\n" : "ADAPTER CHECK OK\n");
  return bad ? 1 : 0;
}
