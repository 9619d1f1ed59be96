// ref_driver.cpp -- C-ABI driver around the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  This file is compiled together with the
// reference sources where they lie (/root/reference/proj/src/*.cpp, see
// oracle/Makefile) into oracle/_ref/libhfmm_ref.so.  Only tests/, the
// smoke check and bench.py's reference / cpu_baseline legs load it, and only
// as the checker or the timed CPU baseline -- never on the product path.
//
// It exposes:
//   * ref_setup_*: build_setup (traversal.cpp:66-238) and a flat dump of the
//     resulting GlobalSetup under the same array names the product's
//     hfmm_setup_get() uses, so tests compare them byte for byte;
//   * ref_evaluate: evaluate_with_setup (traversal.cpp:790-817) with the
//     per-phase ledger seconds;
//   * ref_expansions: multipole / local expansions of one level after a
//     given RankEngine phase (traversal.hpp:129-143), assembled over ranks;
//   * operator-level entry points (green, c2m, l2o, translation_operator,
//     fft_interpolate, fft_anterpolate_adjoint, make_quadrature, ...);
//   * ref_direct: direct_potential (kernel.cpp:16-41) split over threads.
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hfmm/kernel.hpp"
#include "hfmm/operators.hpp"
#include "hfmm/sphere_grid.hpp"
#include "hfmm/traversal.hpp"
#include "hfmm_gpu.h"
#include "inputs.hpp"
#include "adapter/setup_flat.hpp"

using namespace hfmm;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return HFMM_ERR_INVALID_ARGUMENT;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return HFMM_ERR_OUT_OF_RANGE;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return HFMM_ERR_DOMAIN;
  } catch (const std::length_error& e) {
    g_err = e.what();
    return HFMM_ERR_LENGTH;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return HFMM_ERR_LOGIC;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HFMM_ERR_INTERNAL;
  }
}

RunConfig to_ref(const hfmm_run_config* c) {
  RunConfig r;
  r.lambda = c->lambda;
  r.digits = c->digits;
  r.leaf_lambda = c->leaf_lambda;
  r.num_ranks = c->num_ranks;
  r.buffer_limit = c->buffer_limit;
  r.policy = c->policy == HFMM_POLICY_RANK_ORDERED ? AlignPolicy::RankOrdered
                                                   : AlignPolicy::Aligned;
  r.one_particle_per_leaf = c->one_particle_per_leaf != 0;
  r.seed = c->seed;
  r.scheduler = c->scheduler == 2   ? SchedulerKind::Threaded
                : c->scheduler == 1 ? SchedulerKind::Adversarial
                                    : SchedulerKind::Deterministic;
  r.top_level = c->top_level;
  r.d_override = c->d_override;
  return r;
}

std::vector<Particle> to_particles(const double* xyz, const double* q, size_t n) {
  std::vector<Particle> p(n);
  for (size_t i = 0; i < n; ++i) {
    p[i].position = {xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]};
    p[i].intensity = {q[2 * i], q[2 * i + 1]};
  }
  return p;
}

struct Dump {
  std::map<std::string, std::vector<unsigned char>> arrays;
  template <class T>
  void put(const std::string& name, const std::vector<T>& v) {
    auto& a = arrays[name];
    a.resize(v.size() * sizeof(T));
    if (!v.empty()) std::memcpy(a.data(), v.data(), a.size());
  }
};

struct RefSetup {
  GlobalSetup s;
  Dump dump;
};

void make_dump(RefSetup& h) {
  flatten_setup(h.s, [&](const std::string& name, const auto& v) { h.dump.put(name, v); });
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_generate_inputs(int shape, size_t n, double extent, uint64_t seed,
                         double* xyz, double* q) {
  hfmm_b200::generate_inputs(shape, n, extent, seed, xyz, q);
}

// generate_geometry (geometry.cpp:75-127): kind 0 planar grid, 1 sphere
// (Fibonacci), 2 cubic volume; rule 0 unit, 1 seeded random intensities.
// Returns the point count; xyz/q (if non-null) must hold cap particles.
int ref_generate_geometry(int kind, double extent, double spacing, double lambda, int rule,
                          uint64_t seed, size_t cap, double* xyz, double* q, size_t* count) {
  return guard([&] {
    GeometrySpec g;
    g.kind = kind == 0 ? GeometryKind::PlanarGrid
             : kind == 1 ? GeometryKind::SphereSurface
                         : GeometryKind::CubicVolume;
    g.extent = extent;
    g.spacing = spacing;
    auto p = generate_geometry(g, lambda, rule ? IntensityRule::RandomSeeded : IntensityRule::Unit, seed);
    *count = p.size();
    if (xyz && q)
      for (size_t i = 0; i < std::min(cap, p.size()); ++i) {
        xyz[3 * i] = p[i].position.x;
        xyz[3 * i + 1] = p[i].position.y;
        xyz[3 * i + 2] = p[i].position.z;
        q[2 * i] = p[i].intensity.real();
        q[2 * i + 1] = p[i].intensity.imag();
      }
  });
}

int ref_setup_build(const double* xyz, const double* q, size_t n,
                    const hfmm_run_config* cfg, void** out) {
  return guard([&] {
    auto h = std::make_unique<RefSetup>();
    h->s = build_setup(to_particles(xyz, q, n), to_ref(cfg));
    make_dump(*h);
    *out = h.release();
  });
}

void ref_setup_destroy(void* h) { delete static_cast<RefSetup*>(h); }

int ref_setup_get(void* hv, const char* name, void* dst, size_t cap, size_t* nbytes) {
  return guard([&] {
    auto* h = static_cast<RefSetup*>(hv);
    auto it = h->dump.arrays.find(name);
    if (it == h->dump.arrays.end())
      throw std::invalid_argument(std::string("ref_setup_get: unknown array ") + name);
    *nbytes = it->second.size();
    if (dst && cap) std::memcpy(dst, it->second.data(), std::min(cap, it->second.size()));
  });
}

// evaluate_with_setup; pot: n*2 input order; phase_sec/phase_flops: 7 entries
// (ledger Phase order Setup, C2M, M2M, M2L, L2L, L2O, Near; max over ranks for
// seconds, sum for flops).
int ref_evaluate(void* hv, double* pot, double* phase_sec, double* phase_flops) {
  return guard([&] {
    auto* h = static_cast<RefSetup*>(hv);
    EvalResult r = evaluate_with_setup(h->s);
    for (size_t i = 0; i < r.potentials.size(); ++i) {
      pot[2 * i] = r.potentials[i].real();
      pot[2 * i + 1] = r.potentials[i].imag();
    }
    for (int p = 0; p < kNumPhases; ++p) {
      double mx = 0.0;
      double fl = 0.0;
      for (const RankLedger& rl : r.ledger.ranks) {
        mx = std::max(mx, rl.phases[p].seconds);
        fl += double(rl.phases[p].flops);
      }
      if (phase_sec) phase_sec[p] = mx;
      if (phase_flops) phase_flops[p] = fl;
    }
  });
}

// Runs the RankEngine phases C2M..stop_phase (1..5 = c2m, m2m, m2l, l2l,
// l2o_near) on every rank and assembles the kind (0 multipole, 1 local)
// expansions of all nodes at `level` into out (n_nodes * S * 2 doubles);
// samples no rank holds stay zero.  If stop_phase == 5, pot_sorted (n*2)
// receives the sorted-order potentials.
int ref_expansions(void* hv, int stop_phase, int kind, int level, double* out,
                   double* pot_sorted) {
  return guard([&] {
    auto* h = static_cast<RefSetup*>(hv);
    const GlobalSetup& s = h->s;
    const LevelTable& t = s.levels.at(size_t(level));
    const size_t S = s.samplings.at(size_t(level)).num_samples();
    if (out) std::memset(out, 0, t.nodes.size() * S * 2 * sizeof(double));
    WorldOptions opts;
    opts.num_ranks = s.partition.num_ranks;
    opts.scheduler = SchedulerKind::Deterministic;
    std::vector<std::vector<cplx>> pots(size_t(opts.num_ranks));
    std::vector<std::vector<std::pair<size_t, std::vector<cplx>>>> got(
        size_t(opts.num_ranks));
    run_world(opts, [&](Endpoint& ep) {
      RankEngine eng(s, ep);
      if (stop_phase >= 1) eng.c2m_phase();
      if (stop_phase >= 2) eng.m2m_pass();
      if (stop_phase >= 3) eng.m2l_pass();
      if (stop_phase >= 4) eng.l2l_pass();
      if (stop_phase >= 5) pots[size_t(ep.rank())] = eng.l2o_near_phase();
      for (size_t i = 0; i < t.nodes.size(); ++i) {
        const std::vector<cplx>* v = kind == 0 ? eng.multipole(t.nodes[i].key)
                                               : eng.local_expansion(t.nodes[i].key);
        if (!v) continue;
        got[size_t(ep.rank())].emplace_back(i, *v);
      }
    });
    if (out) {
      for (int r = 0; r < opts.num_ranks; ++r)
        for (auto& [i, v] : got[size_t(r)]) {
          auto sl = t.nodes[i].slice_for(r);
          size_t b = sl ? sl->first : 0;
          for (size_t j = 0; j < v.size(); ++j) {
            out[2 * (i * S + b + j)] = v[j].real();
            out[2 * (i * S + b + j) + 1] = v[j].imag();
          }
        }
    }
    if (pot_sorted && stop_phase >= 5) {
      for (int r = 0; r < opts.num_ranks; ++r) {
        size_t p0 = s.leaf_particles[s.partition.rank_ranges[size_t(r)].first].first;
        for (size_t i = 0; i < pots[size_t(r)].size(); ++i) {
          pot_sorted[2 * (p0 + i)] = pots[size_t(r)][i].real();
          pot_sorted[2 * (p0 + i) + 1] = pots[size_t(r)][i].imag();
        }
      }
    }
  });
}

// direct_potential over observers given as indices into the sources,
// observers split across nthreads std::threads (each calls the reference).
int ref_direct(const double* xyz, const double* q, size_t n, const int64_t* obs_idx,
               size_t m, double lambda, int nthreads, double* pot) {
  return guard([&] {
    auto src = to_particles(xyz, q, n);
    Wavenumber k = Wavenumber::from_lambda(lambda);
    if (nthreads < 1) nthreads = 1;
    std::vector<std::thread> th;
    std::vector<std::string> errs(static_cast<size_t>(nthreads));
    for (int t = 0; t < nthreads; ++t)
      th.emplace_back([&, t] {
        try {
          size_t b = m * size_t(t) / size_t(nthreads), e = m * size_t(t + 1) / size_t(nthreads);
          std::vector<Vec3> obs;
          for (size_t i = b; i < e; ++i) obs.push_back(src[size_t(obs_idx[i])].position);
          auto v = direct_potential(src, obs, k);
          for (size_t i = b; i < e; ++i) {
            pot[2 * i] = v[i - b].real();
            pot[2 * i + 1] = v[i - b].imag();
          }
        } catch (const std::exception& ex) {
          errs[size_t(t)] = ex.what();
        }
      });
    for (auto& x : th) x.join();
    for (auto& e : errs)
      if (!e.empty()) throw std::domain_error(e);
  });
}

// ---- operator-level known answers (operators.cpp, sphere_grid.cpp, kernel.cpp)

int ref_green(double k, const double* r, double* out) {
  return guard([&] {
    cplx g = green(Wavenumber::from_k(k), {r[0], r[1], r[2]});
    out[0] = g.real();
    out[1] = g.imag();
  });
}

int ref_truncation_order(double diameter, double k, double digits, int* out) {
  return guard([&] { *out = truncation_order(diameter, Wavenumber::from_k(k), digits); });
}

int ref_level_sampling(int level, double side, double lambda, double digits,
                       int64_t* out3) {
  return guard([&] {
    LevelSampling s = make_level_sampling(level, side, Wavenumber::from_lambda(lambda), digits);
    out3[0] = s.trunc_order;
    out3[1] = int64_t(s.n_theta);
    out3[2] = int64_t(s.n_phi);
  });
}

int ref_quadrature(size_t nt, size_t np, double* theta_w, double* phi_w) {
  return guard([&] {
    QuadratureRule q = make_quadrature(nt, np);
    std::memcpy(theta_w, q.theta_weight.data(), nt * sizeof(double));
    *phi_w = q.phi_weight;
  });
}

static LevelSampling mk_sampling(int trunc, size_t nt, size_t np) {
  LevelSampling s;
  s.level = 1;
  s.trunc_order = trunc;
  s.n_theta = nt;
  s.n_phi = np;
  return s;
}

int ref_translation_operator(int trunc, size_t nt, size_t np, const double* D,
                             double side, double k, double* out) {
  return guard([&] {
    auto v = translation_operator(mk_sampling(trunc, nt, np), {D[0], D[1], D[2]}, side,
                                  Wavenumber::from_k(k), 0, nt * np);
    std::memcpy(out, v.data(), v.size() * sizeof(cplx));
  });
}

int ref_c2m(const double* xyz, const double* q, size_t n, const double* center,
            size_t nt, size_t np, double k, double* out) {
  return guard([&] {
    auto p = to_particles(xyz, q, n);
    SphereGrid g = c2m(p, {center[0], center[1], center[2]}, mk_sampling(0, nt, np),
                       Wavenumber::from_k(k));
    std::memcpy(out, g.samples.data(), g.size() * sizeof(cplx));
  });
}

int ref_l2o(const double* local, size_t nt, size_t np, const double* center,
            const double* obs, size_t m, double k, double* out) {
  return guard([&] {
    SphereGrid g(nt, np);
    std::memcpy(g.samples.data(), local, nt * np * sizeof(cplx));
    std::vector<Vec3> o(m);
    for (size_t i = 0; i < m; ++i) o[i] = {obs[3 * i], obs[3 * i + 1], obs[3 * i + 2]};
    auto v = l2o(g, {center[0], center[1], center[2]}, o, make_quadrature(nt, np),
                 Wavenumber::from_k(k));
    std::memcpy(out, v.data(), v.size() * sizeof(cplx));
  });
}

int ref_shift(double* samples, size_t nt, size_t np, const double* disp, double k) {
  return guard([&] {
    std::vector<cplx> v(nt * np);
    std::memcpy(v.data(), samples, v.size() * sizeof(cplx));
    shift_expansion(v, mk_sampling(0, nt, np), 0, {disp[0], disp[1], disp[2]},
                    Wavenumber::from_k(k));
    std::memcpy(samples, v.data(), v.size() * sizeof(cplx));
  });
}

// mode 0: fft_interpolate, 1: fft_anterpolate, 2: fft_anterpolate_adjoint
int ref_resample_grid(int mode, const double* src, size_t nt, size_t np, size_t nt_dst,
                      size_t np_dst, double* out) {
  return guard([&] {
    SphereGrid g(nt, np);
    std::memcpy(g.samples.data(), src, nt * np * sizeof(cplx));
    SphereGrid r = mode == 0   ? fft_interpolate(g, nt_dst, np_dst)
                   : mode == 1 ? fft_anterpolate(g, nt_dst, np_dst)
                               : fft_anterpolate_adjoint(g, nt_dst, np_dst);
    std::memcpy(out, r.samples.data(), r.size() * sizeof(cplx));
  });
}

int ref_resample_circle(const double* in, size_t n_in, double shift_in, double* out,
                        size_t n_out, double shift_out) {
  return guard([&] {
    std::vector<cplx> a(n_in), b(n_out);
    std::memcpy(a.data(), in, n_in * sizeof(cplx));
    resample_circle(a, n_in, shift_in, b, n_out, shift_out);
    std::memcpy(out, b.data(), n_out * sizeof(cplx));
  });
}

}  // extern "C"
