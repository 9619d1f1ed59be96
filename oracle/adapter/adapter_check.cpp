// Runs the reference-side binding (gpu_eval.cpp) next to the reference's own
// CPU evaluation, through the reference's C++ API, on seeded inputs:
//   - evaluate_with_setup_b200(build_setup(...)) vs hfmm::evaluate_with_setup
//   - evaluate_potential_b200 vs hfmm::evaluate_potential
//   - an invalid RunConfig raises the same std exception type on both paths.
// TEST INFRASTRUCTURE (tests/test_gpu_adapter.py); prints one line per check.
#include <cmath>
#include <complex>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "gpu_eval.hpp"
#include "inputs.hpp"

using hfmm::cplx;

static double rel_l2(const std::vector<cplx>& a, const std::vector<cplx>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    num += std::norm(a[i] - b[i]);
    den += std::norm(b[i]);
  }
  return std::sqrt(num / den);
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
  int bad = 0;
  struct Case { int shape; size_t n; double ext; uint64_t seed; double digits; };
  for (const Case& c : {Case{0, 20000, 3.0, 41, 3.0}, Case{1, 30000, 2.0, 42, 4.0}, Case{0, 100000, 4.0, 0, 3.0}}) {
    const auto ps = particles(c.shape, c.n, c.ext, c.seed);
    hfmm::RunConfig cfg;
    cfg.digits = c.digits;
    const hfmm::GlobalSetup s = hfmm::build_setup(ps, cfg);
    const hfmm::EvalResult want = hfmm::evaluate_with_setup(s);
    const hfmm::EvalResult got = hfmm::evaluate_with_setup_b200(s, 0);
    const double e1 = rel_l2(got.potentials, want.potentials);
    const hfmm::EvalResult got2 = hfmm::evaluate_potential_b200(ps, cfg, 0);
    const double e2 = rel_l2(got2.potentials, want.potentials);
    std::printf("case shape=%d n=%zu digits=%.1f evaluate_with_setup_b200 rel_l2=%.3e evaluate_potential_b200 rel_l2=%.3e\n",
                c.shape, c.n, c.digits, e1, e2);
    if (!(e1 < 1e-10) || !(e2 < 1e-10)) ++bad;
  }
  {
    const auto ps = particles(0, 1000, 1.0, 43);
    hfmm::RunConfig cfg;
    cfg.digits = -1.0;  // RunConfig::validate rejects it
    const std::string a = exception_kind([&] { hfmm::evaluate_potential(ps, cfg); });
    const std::string b = exception_kind([&] { hfmm::evaluate_potential_b200(ps, cfg, 0); });
    std::printf("invalid config: reference throws %s, b200 binding throws %s\n", a.c_str(), b.c_str());
    if (a != b || a == "none") ++bad;
  }
  std::printf(bad ? "ADAPTER CHECK FAILED\n" : "ADAPTER CHECK OK\n");
  return bad ? 1 : 0;
}
