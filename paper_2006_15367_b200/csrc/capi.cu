// C ABI (include/hfmm_gpu.h): status codes mirror the reference's exception
// types; every entry point is wrapped so no C++ exception crosses the ABI.
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.hpp"
#include "hfmm_gpu.h"
#include "inputs.hpp"
#include "interp.hpp"
#include "setup.hpp"
#include "world.hpp"

struct hfmm_setup {
  // shared with every engine created from it (hfmm_gpu_create)
  std::shared_ptr<hfmm_b200::Setup> sp = std::make_shared<hfmm_b200::Setup>();
  hfmm_b200::Setup& s = *sp;
};
struct hfmm_gpu {
  std::unique_ptr<hfmm_b200::Engine> eng;
};
struct hfmm_world {
  std::unique_ptr<hfmm_b200::World> w;
};

namespace {

thread_local std::string g_err;

struct CudaFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
hfmm_status guard(F&& f) {
  try {
    f();
    g_err.clear();
    return HFMM_OK;
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
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return std::string(e.what()).find("no CUDA device") != std::string::npos ? HFMM_ERR_NO_DEVICE
                                                                             : HFMM_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return HFMM_ERR_INTERNAL;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string(what) + ": null pointer");
}

}  // namespace

extern "C" {

void hfmm_run_config_default(hfmm_run_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof(*c));
  c->lambda = 1.0;
  c->digits = 3.0;
  c->leaf_lambda = 0.25;
  c->num_ranks = 1;
  c->policy = HFMM_POLICY_ALIGNED;
  c->buffer_limit = ~uint64_t(0);
  c->one_particle_per_leaf = 0;
  c->top_level = 3;
  c->d_override = 0;
  c->scheduler = 0;
  c->seed = 0;
  c->partition_weight = 0;
}

const char* hfmm_last_error(void) { return g_err.c_str(); }

hfmm_status hfmm_setup_build(const double* positions, const double* charges, size_t n,
                             const hfmm_run_config* cfg, hfmm_setup** out) {
  return guard([&] {
    need(cfg, "hfmm_setup_build(cfg)");
    need(out, "hfmm_setup_build(out)");
    if (n > 0) {
      need(positions, "hfmm_setup_build(positions)");
      need(charges, "hfmm_setup_build(charges)");
    }
    auto h = std::make_unique<hfmm_setup>();
    h->s = hfmm_b200::build_setup(positions, charges, n, *cfg);
    *out = h.release();
  });
}

void hfmm_setup_destroy(hfmm_setup* s) { delete s; }

hfmm_status hfmm_setup_get(const hfmm_setup* s, const char* name, void* dst, size_t cap,
                           size_t* nbytes) {
  return guard([&] {
    need(s, "hfmm_setup_get(setup)");
    need(name, "hfmm_setup_get(name)");
    auto v = hfmm_b200::setup_array(s->s, name);
    if (nbytes) *nbytes = v.size();
    if (dst && cap) std::memcpy(dst, v.data(), std::min(cap, v.size()));
  });
}

hfmm_status hfmm_setup_import_begin(const hfmm_run_config* cfg, hfmm_setup_import** out) {
  return guard([&] {
    need(cfg, "hfmm_setup_import_begin(cfg)");
    need(out, "hfmm_setup_import_begin(out)");
    if (!(cfg->lambda > 0) || !(cfg->digits > 0) || !(cfg->leaf_lambda > 0) || cfg->num_ranks < 1 ||
        cfg->buffer_limit == 0 || cfg->top_level < 1)
      throw std::invalid_argument("RunConfig: invalid fields");
    *out = reinterpret_cast<hfmm_setup_import*>(hfmm_b200::setup_import_begin(*cfg));
  });
}

hfmm_status hfmm_setup_import_put(hfmm_setup_import* im, const char* name, const void* data, size_t nbytes) {
  return guard([&] {
    need(im, "hfmm_setup_import_put(import)");
    need(name, "hfmm_setup_import_put(name)");
    hfmm_b200::setup_import_put(reinterpret_cast<hfmm_b200::SetupImport*>(im), name, data, nbytes);
  });
}

hfmm_status hfmm_setup_import_end(hfmm_setup_import* im, hfmm_setup** out) {
  auto* p = reinterpret_cast<hfmm_b200::SetupImport*>(im);
  hfmm_status st = guard([&] {
    need(im, "hfmm_setup_import_end(import)");
    need(out, "hfmm_setup_import_end(out)");
    auto h = std::make_unique<hfmm_setup>();
    h->s = hfmm_b200::setup_import_end(p);
    *out = h.release();
  });
  if (p) hfmm_b200::setup_import_abort(p);
  return st;
}

void hfmm_setup_import_abort(hfmm_setup_import* im) {
  if (im) hfmm_b200::setup_import_abort(reinterpret_cast<hfmm_b200::SetupImport*>(im));
}

hfmm_status hfmm_gpu_create(const hfmm_setup* s, int device, int rank, hfmm_gpu** out) {
  return guard([&] {
    need(s, "hfmm_gpu_create(setup)");
    need(out, "hfmm_gpu_create(out)");
    auto g = std::make_unique<hfmm_gpu>();
    g->eng = std::make_unique<hfmm_b200::Engine>(s->sp, device, rank);
    *out = g.release();
  });
}

void hfmm_gpu_destroy(hfmm_gpu* g) { delete g; }

hfmm_status hfmm_gpu_evaluate(hfmm_gpu* g, const double* charges, double* pot_out,
                              hfmm_gpu_timing* timing) {
  return guard([&] {
    need(g, "hfmm_gpu_evaluate(gpu)");
    need(pot_out, "hfmm_gpu_evaluate(pot_out)");
    double ms[8] = {0};
    int64_t l0 = g->eng->launches();
    g->eng->evaluate_host(charges, pot_out, ms);
    if (timing) {
      std::memcpy(timing->ms, ms, sizeof(ms));
      timing->kernel_launches = g->eng->launches() - l0;
    }
  });
}

hfmm_status hfmm_gpu_evaluate_device(hfmm_gpu* g, const double* d_q, double* d_pot, void* stream) {
  return guard([&] {
    need(g, "hfmm_gpu_evaluate_device(gpu)");
    g->eng->evaluate_device(d_q, d_pot, static_cast<cudaStream_t>(stream));
  });
}

hfmm_status hfmm_gpu_last_timing(hfmm_gpu* g, hfmm_gpu_timing* timing) {
  return guard([&] {
    need(g, "hfmm_gpu_last_timing(gpu)");
    need(timing, "hfmm_gpu_last_timing(timing)");
    g->eng->last_timing(timing->ms, &timing->kernel_launches);
  });
}

hfmm_status hfmm_gpu_set_charges(hfmm_gpu* g, const double* charges) {
  return guard([&] {
    need(g, "hfmm_gpu_set_charges(gpu)");
    need(charges, "hfmm_gpu_set_charges(charges)");
    g->eng->set_charges(charges);
  });
}

hfmm_status hfmm_gpu_run_phase(hfmm_gpu* g, int phase) {
  return guard([&] {
    need(g, "hfmm_gpu_run_phase(gpu)");
    g->eng->run_phase(phase);
  });
}

hfmm_status hfmm_gpu_get_expansion(hfmm_gpu* g, int kind, int level, double* out, size_t cap) {
  return guard([&] {
    need(g, "hfmm_gpu_get_expansion(gpu)");
    need(out, "hfmm_gpu_get_expansion(out)");
    g->eng->get_expansion(kind, level, out, cap);
  });
}

hfmm_status hfmm_gpu_get_potentials_sorted(hfmm_gpu* g, double* out, size_t cap) {
  return guard([&] {
    need(g, "hfmm_gpu_get_potentials_sorted(gpu)");
    need(out, "hfmm_gpu_get_potentials_sorted(out)");
    g->eng->get_potentials_sorted(out, cap);
  });
}

hfmm_status hfmm_gpu_exchange_sizes(hfmm_gpu* g, int kind, int peer, int level, int64_t* send_d,
                                    int64_t* recv_d) {
  return guard([&] {
    need(g, "hfmm_gpu_exchange_sizes(gpu)");
    need(send_d, "hfmm_gpu_exchange_sizes(send)");
    need(recv_d, "hfmm_gpu_exchange_sizes(recv)");
    g->eng->exchange_sizes(kind, peer, level, send_d, recv_d);
  });
}

hfmm_status hfmm_gpu_pack(hfmm_gpu* g, int kind, int peer, int level, double* d_send) {
  return guard([&] {
    need(g, "hfmm_gpu_pack(gpu)");
    g->eng->pack(kind, peer, level, d_send);
  });
}

hfmm_status hfmm_gpu_unpack(hfmm_gpu* g, int kind, int peer, int level, const double* d_recv) {
  return guard([&] {
    need(g, "hfmm_gpu_unpack(gpu)");
    g->eng->unpack(kind, peer, level, d_recv);
  });
}

hfmm_status hfmm_gpu_run_level(hfmm_gpu* g, int phase, int level) {
  return guard([&] {
    need(g, "hfmm_gpu_run_level(gpu)");
    g->eng->run_level(phase, level);
  });
}

hfmm_status hfmm_gpu_set_stream(hfmm_gpu* g, void* stream) {
  return guard([&] {
    need(g, "hfmm_gpu_set_stream(gpu)");
    g->eng->set_stream(static_cast<cudaStream_t>(stream));
  });
}

hfmm_status hfmm_gpu_synchronize(hfmm_gpu* g) {
  return guard([&] {
    need(g, "hfmm_gpu_synchronize(gpu)");
    g->eng->synchronize();
  });
}

hfmm_status hfmm_gpu_load_charges_device(hfmm_gpu* g, const double* d_q) {
  return guard([&] {
    need(g, "hfmm_gpu_load_charges_device(gpu)");
    need(d_q, "hfmm_gpu_load_charges_device(charges)");
    g->eng->load_charges_device(d_q);
  });
}

hfmm_status hfmm_gpu_particle_range(hfmm_gpu* g, int64_t* b, int64_t* e) {
  return guard([&] {
    need(g, "hfmm_gpu_particle_range(gpu)");
    *b = g->eng->particle_begin();
    *e = g->eng->particle_end();
  });
}

hfmm_status hfmm_gpu_store_potentials_device(hfmm_gpu* g, double* d_pot) {
  return guard([&] {
    need(g, "hfmm_gpu_store_potentials_device(gpu)");
    need(d_pot, "hfmm_gpu_store_potentials_device(pot)");
    g->eng->store_potentials_device(d_pot);
  });
}

hfmm_status hfmm_gpu_set_overlap(hfmm_gpu* g, int on) {
  return guard([&] {
    need(g, "hfmm_gpu_set_overlap(gpu)");
    g->eng->set_overlap(on != 0);
  });
}

hfmm_status hfmm_gpu_launch_count(hfmm_gpu* g, int64_t* n) {
  return guard([&] {
    need(g, "hfmm_gpu_launch_count(gpu)");
    need(n, "hfmm_gpu_launch_count(out)");
    *n = g->eng->launch_count();
  });
}

hfmm_status hfmm_world_create(const hfmm_setup* s, const int* devices, int ndev, hfmm_world** out) {
  return guard([&] {
    need(s, "hfmm_world_create(setup)");
    need(out, "hfmm_world_create(out)");
    std::vector<int> devs;
    if (devices && ndev > 0)
      devs.assign(devices, devices + ndev);
    else
      devs.push_back(0);
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
      throw std::runtime_error("no CUDA device available (the engine has no CPU fallback)");
    for (int d : devs)
      if (d < 0 || d >= count) throw std::invalid_argument("hfmm_world_create: bad device");
    auto w = std::make_unique<hfmm_world>();
    w->w = std::make_unique<hfmm_b200::World>(s->sp, devs);
    *out = w.release();
  });
}

void hfmm_world_destroy(hfmm_world* w) { delete w; }

hfmm_status hfmm_world_set_charges(hfmm_world* w, const double* charges) {
  return guard([&] {
    need(w, "hfmm_world_set_charges(world)");
    need(charges, "hfmm_world_set_charges(charges)");
    w->w->set_charges(charges);
  });
}

hfmm_status hfmm_world_run_phase(hfmm_world* w, int phase) {
  return guard([&] {
    need(w, "hfmm_world_run_phase(world)");
    w->w->run_phase(phase);
  });
}

hfmm_status hfmm_world_evaluate(hfmm_world* w, const double* charges, double* pot_out, double* rank_ms) {
  return guard([&] {
    need(w, "hfmm_world_evaluate(world)");
    need(pot_out, "hfmm_world_evaluate(pot_out)");
    w->w->evaluate(charges, pot_out);
    if (rank_ms)
      for (int r = 0; r < w->w->ranks(); ++r) w->w->rank_ms(r, rank_ms + size_t(r) * hfmm_b200::kLedgerPhases);
  });
}

hfmm_status hfmm_world_potentials(hfmm_world* w, double* pot_out) {
  return guard([&] {
    need(w, "hfmm_world_potentials(world)");
    need(pot_out, "hfmm_world_potentials(pot_out)");
    w->w->potentials(pot_out);
  });
}

hfmm_status hfmm_world_get_expansion(hfmm_world* w, int rank, int kind, int level, double* out, size_t cap) {
  return guard([&] {
    need(w, "hfmm_world_get_expansion(world)");
    need(out, "hfmm_world_get_expansion(out)");
    if (rank < 0 || rank >= w->w->ranks()) throw std::out_of_range("hfmm_world_get_expansion: bad rank");
    w->w->engine(rank).get_expansion(kind, level, out, cap);
  });
}

hfmm_status hfmm_evaluate_potential(const double* positions, const double* charges, size_t n,
                                    const hfmm_run_config* cfg, int device, double* pot_out) {
  return guard([&] {
    need(cfg, "hfmm_evaluate_potential(cfg)");
    need(pot_out, "hfmm_evaluate_potential(pot_out)");
    if (cfg->num_ranks != 1)
      throw std::invalid_argument("hfmm_evaluate_potential: one device evaluates num_ranks == 1");
    auto s = std::make_shared<hfmm_b200::Setup>(hfmm_b200::build_setup(positions, charges, n, *cfg));
    hfmm_b200::Engine e(s, device, 0);
    e.evaluate_host(nullptr, pot_out, nullptr);
  });
}

hfmm_status hfmm_gpu_direct(const double* positions, const double* charges, size_t n,
                            const int64_t* obs, size_t m, double k, int device, double* pot_out) {
  return guard([&] {
    need(positions, "hfmm_gpu_direct(positions)");
    need(charges, "hfmm_gpu_direct(charges)");
    need(obs, "hfmm_gpu_direct(observers)");
    need(pot_out, "hfmm_gpu_direct(pot_out)");
    hfmm_b200::direct_sum(positions, charges, n, obs, m, k, device, pot_out);
  });
}

hfmm_status hfmm_resample_matrix(int64_t n_in, double s_in, int64_t n_out, double s_out,
                                 double* out) {
  return guard([&] {
    need(out, "hfmm_resample_matrix(out)");
    if (n_in <= 0 || n_out <= 0) throw std::invalid_argument("resample_circle: bad sizes");
    auto m = hfmm_b200::resample_matrix(n_in, s_in, n_out, s_out);
    std::memcpy(out, m.data(), m.size() * sizeof(double));
  });
}

hfmm_status hfmm_m2m_operands(int nc, int np, double* bphi, double* vphi, double* bth, double* vth,
                              int dims[4]) {
  return guard([&] {
    need(dims, "hfmm_m2m_operands(dims)");
    if (nc <= 0 || np <= 0 || nc % 2 || np % 2) throw std::invalid_argument("hfmm_m2m_operands: grids must be even");
    using namespace hfmm_b200;
    const RealRank1 uphi = real_rank1(nc, 0.0, np, 0.0);
    const RealRank1 uf = fold_columns(uphi, nc, np);
    const EvenOdd ue = even_odd(real_rank1(2 * nc, 0.5, 2 * np, 0.5), 2 * nc, 2 * np);
    dims[0] = uf.K;
    dims[1] = uf.N;
    dims[2] = ue.KH4;
    dims[3] = ue.NH;
    if (bphi) std::memcpy(bphi, uf.B.data(), uf.B.size() * sizeof(double));
    if (vphi) std::memcpy(vphi, uf.v.data(), uf.v.size() * sizeof(double));
    if (bth) std::memcpy(bth, ue.B.data(), ue.B.size() * sizeof(double));
    if (vth) std::memcpy(vth, ue.v.data(), ue.v.size() * sizeof(double));
  });
}

hfmm_status hfmm_l2l_operands(int nc, int np, const double* row_scale, const double* col_scale,
                              double* bth, double* vth, double* bphi, double* vphi, int dims[4]) {
  return guard([&] {
    need(dims, "hfmm_l2l_operands(dims)");
    need(row_scale, "hfmm_l2l_operands(row_scale)");
    need(col_scale, "hfmm_l2l_operands(col_scale)");
    if (nc <= 0 || np <= 0 || nc % 2 || np % 2) throw std::invalid_argument("hfmm_l2l_operands: grids must be even");
    using namespace hfmm_b200;
    const std::vector<double> rs(row_scale, row_scale + 2 * nc), cs(col_scale, col_scale + 2 * np);
    const EvenOdd de = even_odd(real_rank1(2 * np, 0.5, 2 * nc, 0.5, &rs, &cs), 2 * np, 2 * nc);
    const RealRank1 du = unfold_rows(real_rank1(np, 0.0, nc, 0.0), np, nc);
    dims[0] = de.KH4;
    dims[1] = de.NH;
    dims[2] = du.K;
    dims[3] = du.N;
    if (bth) std::memcpy(bth, de.B.data(), de.B.size() * sizeof(double));
    if (vth) std::memcpy(vth, de.v.data(), de.v.size() * sizeof(double));
    if (bphi) std::memcpy(bphi, du.B.data(), du.B.size() * sizeof(double));
    if (vphi) std::memcpy(vphi, du.v.data(), du.v.size() * sizeof(double));
  });
}

void hfmm_generate_inputs(int shape, size_t n, double extent, uint64_t seed, double* positions,
                          double* charges) {
  hfmm_b200::generate_inputs(shape, n, extent, seed, positions, charges);
}

}  // extern "C"
