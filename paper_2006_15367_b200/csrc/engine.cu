// Device engine host side: setup upload and per-phase launches.
#include "engine.hpp"

#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "interp.hpp"
#include "kernels.cuh"
#include "m2l.cuh"
#include "p2p.cuh"
#include "leaf.cuh"
#include "m2l_tc.cuh"
#include "interp_rb.cuh"
#include "interp_fused.cuh"
#include "interp_big.cuh"

namespace hfmm_b200 {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();  // a non-sticky error must not resurface at the next launch check
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }
}

inline int slot_of(long ox, long oy, long oz) {
  return int((ox + 3) * 49 + (oy + 3) * 7 + (oz + 3));
}

inline uint32_t cell_axis(uint64_t code, int level, int axis) {
  uint32_t v = 0;
  for (int t = 0; t < level - 1; ++t) v |= uint32_t((code >> (3 * t + axis)) & 1) << t;
  return v;
}

}  // namespace

template <class T>
T* Engine::alloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  ck(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
  allocs_.push_back(p);
  return static_cast<T*>(p);
}

template <class T>
T* Engine::upload_vec(const std::vector<T>& v) {
  T* d = alloc<T>(v.size());
  if (!v.empty()) ck(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st_), "upload");
  return d;
}

Engine::Engine(std::shared_ptr<const Setup> sp, int device, int rank)
    : keep_(std::move(sp)), s_(*keep_), dev_(device), rank_(rank) {
  const Setup& s = s_;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw std::runtime_error("no CUDA device available (the engine has no CPU fallback)");
  if (device < 0 || device >= ndev) throw std::invalid_argument("hfmm_gpu_create: bad device");
  if (rank < 0 || rank >= s.P) throw std::invalid_argument("hfmm_gpu_create: bad rank");
  dist_ = s.P > 1;
  ck(cudaSetDevice(device), "cudaSetDevice");
  ck(cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device), "sm count");
  // Test hooks (tests/test_gpu_paths.py): route every level pair through the
  // general kernels that otherwise serve only the largest grids or leaves.
  hook_no_rb_ = std::getenv("HFMM_NO_RB") != nullptr;    // no compile-time-shaped M2M/L2L pairs
  hook_no_rbl_ = std::getenv("HFMM_NO_RBL") != nullptr;  // no runtime-shaped streaming M2M/L2L
  hook_no_quad_ = std::getenv("HFMM_NO_QUAD") != nullptr;  // generic C2M / L2T instead of quad kernels
  ck(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "stream");
  for (auto& e : ev_) ck(cudaEventCreate(&e), "event");
  // Side stream for the near field.  (Giving the far-field chain a higher
  // stream priority measured slower on cfg 2 and cfg 3: equal priorities.)
  ck(cudaStreamCreateWithFlags(&st2_, cudaStreamNonBlocking), "stream2");
  {
    int least = 0, greatest = 0;
    ck(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priorities");
    ck(cudaStreamCreateWithPriority(&st_hi_, cudaStreamNonBlocking, greatest), "stream hi");
    ck(cudaStreamCreateWithPriority(&st_lo_, cudaStreamNonBlocking, least), "stream lo");
    for (cudaEvent_t* e : {&ev_ofork_, &ev_ojoin_, &ev_c2m_, &ev_m2l_leaf_})
      ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    for (cudaEvent_t* e : {&ev_lf0_, &ev_lf1_, &ev_la_, &ev_lb_}) ck(cudaEventCreate(e), "event");
  }
  ck(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming), "event");
  ck(cudaEventCreate(&ev_near0_), "event");
  ck(cudaEventCreate(&ev_near1_), "event");
  ck(cudaStreamCreateWithFlags(&st_cp_, cudaStreamNonBlocking), "copy stream");
  ck(cudaEventCreateWithFlags(&ev_q_, cudaEventDisableTiming), "event");
  ck(cudaEventCreateWithFlags(&ev_cp_order_, cudaEventDisableTiming), "event");
  if (dist_) {  // rank plan first: it sizes the compact per-rank storage
    rp_ = std::make_unique<RankPlan>(build_rank_plan(s, rank));
    rows_.assign(size_t(s.L + 1), {});
    for (int l = s.top; l <= s.L; ++l) {
      auto& ro = rows_[size_t(l)];
      ro.assign(s.levels[size_t(l)].num_nodes(), -1);
      int r = 0;
      for (int n : rp_->held[size_t(l)]) ro[size_t(n)] = r++;
      for (int n : rp_->halo[size_t(l)]) ro[size_t(n)] = r++;
    }
  }
  upload();
  if (dist_) upload_rank_plan();
  // Parent descriptors of the M2M / L2L work loops (rb::PDesc), per parent level.
  pdesc_.assign(size_t(s.L + 1), nullptr);
  for (int l = s.top; l < s.L; ++l) {
    const DevLevel& P = lv_[size_t(l)];
    const RankLevel* R = dist_ ? &rl_[size_t(l)] : nullptr;
    const int n_par = R ? R->n_par : P.n_nodes;
    int4* d = alloc<int4>(size_t(3) * size_t(std::max(n_par, 1)));
    if (n_par > 0)
      k_build_pdesc<<<(n_par + 127) / 128, 128, 0, st_>>>(n_par, R ? R->plist : nullptr, R ? R->child_off : P.child_off,
                                                         R ? R->children : P.children, oct_[size_t(l + 1)], d);
    pdesc_[size_t(l)] = d;
  }
  ck(cudaGetLastError(), "k_build_pdesc");
  ck(cudaStreamSynchronize(st_), "upload sync");
}

Engine::~Engine() {
  cudaSetDevice(dev_);
  for (cudaStream_t s : {st_, st2_, st_hi_, st_lo_, st_cp_})  // every stream idle before the buffers go
    if (s) cudaStreamSynchronize(s);
  for (void* p : allocs_) cudaFree(p);
  for (auto& e : ev_)
    if (e) cudaEventDestroy(e);
  if (st_ && owns_stream_) cudaStreamDestroy(st_);
  if (st2_) cudaStreamDestroy(st2_);
  for (cudaStream_t s : {st_hi_, st_lo_, st_cp_})
    if (s) cudaStreamDestroy(s);
  if (ev_q_) cudaEventDestroy(ev_q_);
  if (ev_cp_order_) cudaEventDestroy(ev_cp_order_);
  for (cudaEvent_t e : {ev_ofork_, ev_ojoin_, ev_c2m_, ev_m2l_leaf_, ev_lf0_, ev_lf1_, ev_la_, ev_lb_})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : {ev_fork_, ev_join_, ev_near0_, ev_near1_})
    if (e) cudaEventDestroy(e);
}

namespace {
int lda_for(int K) { return (K % 8 == 4) ? K : K + 4; }  // row stride == 4 (mod 8) double2
void set_dims(int* d, int K, int N, bool with_ldo) {
  d[0] = K;
  d[1] = N;
  d[2] = lda_for(K);
  d[3] = with_ldo ? N + 4 : 0;
}
PassDims to_dims(const int* d) { return PassDims{d[0], d[1], d[2], d[3]}; }
}  // namespace

// Real + rank-1 matrices of the DMMA M2M / L2L passes of parent level P over
// child level C, and the launch plan of the two-stage large-grid kernels.
void Engine::setup_interp(DevLevel& P, const DevLevel& C, const LevelData& tp, const LevelData& tc) {
  const int nc = C.nt, np = P.nt, half = np / 2;
  // M2M: phi n_c -> n_p (shift 0), theta 2 n_c -> 2 n_p (shift 0.5)
  RealRank1 uphi = real_rank1(nc, 0.0, np, 0.0);
  RealRank1 uth = real_rank1(2 * nc, 0.5, 2 * np, 0.5);
  set_dims(P.up_phi, uphi.K, uphi.N, false);
  set_dims(P.up_th, uth.K, uth.N, true);
  P.up_phi_B = upload_vec(uphi.B);
  P.up_phi_v = upload_vec(uphi.v);
  P.up_th_B = upload_vec(uth.B);
  P.up_th_v = upload_vec(uth.v);
  // L2L: theta 2 n_p -> 2 n_c with w_p (cols) and scale / w_c (rows); phi n_p -> n_c
  std::vector<double> wp(size_t(2 * np)), wc(size_t(2 * nc));
  const double scale = (double(P.S) / double(C.S)) * tp.phi_w / tc.phi_w;
  for (int i = 0; i < 2 * np; ++i) wp[size_t(i)] = tp.theta_w[size_t(i < np ? i : 2 * np - 1 - i)];
  for (int j = 0; j < 2 * nc; ++j) wc[size_t(j)] = scale / tc.theta_w[size_t(j < nc ? j : 2 * nc - 1 - j)];
  RealRank1 dth = real_rank1(2 * np, 0.5, 2 * nc, 0.5, &wc, &wp);
  RealRank1 dphi = real_rank1(np, 0.0, nc, 0.0);
  set_dims(P.dn_th, dth.K, dth.N, false);
  set_dims(P.dn_phi, dphi.K, dphi.N, false);
  P.dn_th_B = upload_vec(dth.B);
  P.dn_th_v = upload_vec(dth.v);
  P.dn_phi_B = upload_vec(dphi.B);
  P.dn_phi_v = upload_vec(dphi.v);
  // Even / odd form of the theta passes, with the fold / unfold baked into the
  // phi matrices (interp.hpp): what the fused and compile-time-shaped kernels take.
  if (nc % 2 == 0 && np % 2 == 0) {
    const EvenOdd ue = even_odd(uth, 2 * nc, 2 * np), de = even_odd(dth, 2 * np, 2 * nc);
    const RealRank1 uf = fold_columns(uphi, nc, np), du = unfold_rows(dphi, np, nc);
    P.up_phi_Bf = upload_vec(uf.B);
    P.up_th_Be = upload_vec(ue.B);
    P.up_th_ve = upload_vec(ue.v);
    P.dn_th_Be = upload_vec(de.B);
    P.dn_th_ve = upload_vec(de.v);
    P.dn_phi_Bu = upload_vec(du.B);
    P.dn_phi_vu = upload_vec(du.v);
  }
  // Two-stage large-grid plans.
  {
    const int ldf = P.up_th[2];
    const size_t per_circle = (size_t(kBigCB) * ldf + size_t(2 * np)) * sizeof(double2);
    P.big_m2m_cp = int(std::max<size_t>(1, std::min<size_t>(size_t(half), (110 * 1024) / per_circle)));
    const size_t row_budget = 96 * 1024;
    P.big_rc[0] = int(std::max<size_t>(1, std::min<size_t>(size_t(nc), row_budget / (size_t(P.up_phi[2]) * sizeof(double2)))));
    P.big_smem[0] = size_t(P.big_rc[0]) * P.up_phi[2] * sizeof(double2);
    P.big_smem[1] = size_t(P.big_m2m_cp) * per_circle;
    const size_t per_c2 = size_t(P.dn_th[2]) * sizeof(double2);
    P.big_l2l_cp = int(std::max<size_t>(1, std::min<size_t>(size_t(half), (72 * 1024) / per_c2)));
    P.big_smem[2] = size_t(P.big_l2l_cp) * per_c2;
    P.big_rc[1] = int(std::max<size_t>(1, std::min<size_t>(size_t(nc), row_budget / (size_t(P.dn_phi[2]) * sizeof(double2)))));
    P.big_smem[3] = size_t(P.big_rc[1]) * P.dn_phi[2] * sizeof(double2);
    P.big_ldn = P.dn_phi[2];
    tmp_need_ = std::max(tmp_need_, std::max(size_t(C.n_rows) * half * ldf, size_t(C.n_rows) * nc * P.big_ldn));
  }
}

void Engine::upload() {
  const Setup& s = s_;
  const int L = s.L;
  const size_t n = s.n;
  leaf_b_ = int64_t(s.rank_begin[size_t(rank_)]);
  leaf_e_ = int64_t(s.rank_end[size_t(rank_)]);
  part_b_ = int64_t(s.leaf_start[size_t(leaf_b_)]);
  part_e_ = int64_t(s.leaf_start[size_t(leaf_e_)]);

  std::vector<double> x(n), y(n), z(n);
  for (size_t i = 0; i < n; ++i) {
    x[i] = s.xyz[3 * i];
    y[i] = s.xyz[3 * i + 1];
    z[i] = s.xyz[3 * i + 2];
  }
  d_x = upload_vec(x);
  d_y = upload_vec(y);
  d_z = upload_vec(z);
  d_q = alloc<double2>(n);
  ck(cudaMemcpyAsync(d_q, s.q.data(), n * sizeof(double2), cudaMemcpyHostToDevice, st_), "q");
  d_pot = alloc<double2>(n);
  d_pot_near = alloc<double2>(n);
  d_q_in = alloc<double2>(n);
  d_pot_in = alloc<double2>(n);
  std::vector<int64_t> orig(s.original_index.begin(), s.original_index.end());
  d_orig = upload_vec(orig);
  std::vector<int64_t> ls(s.leaf_start.begin(), s.leaf_start.end());
  d_leaf_start = upload_vec(ls);
  std::vector<int64_t> no(s.near_off.begin(), s.near_off.end());
  d_near_off = upload_vec(no);
  std::vector<int> nr(s.near.begin(), s.near.end());
  d_near = upload_vec(nr);
  // P2P launch lists: own leaves by population (k_p2p_leaf2 for <= 32, k_p2p_sym2 above)
  {
    // tiny (<= 8: warp per leaf), small (<= 32: CTA per leaf), dense (symmetric)
    std::vector<int> tiny, small, dense;
    for (int64_t li = leaf_b_; li < leaf_e_; ++li) {
      const uint64_t pop = s.leaf_start[size_t(li) + 1] - s.leaf_start[size_t(li)];
      (pop <= 8 ? tiny : pop <= 32 ? small : dense).push_back(int(li));
    }
    n_tiny_ = int(tiny.size());
    n_small_ = int(small.size());
    n_dense_ = int(dense.size());
    d_tiny_leaves_ = upload_vec(tiny);
    d_small_leaves_ = upload_vec(small);
    d_dense_leaves_ = upload_vec(dense);
    {  // leaves with <= 32 particles (L2T lanes-over-quads kernel)
      std::vector<int> sp(tiny);
      sp.insert(sp.end(), small.begin(), small.end());
      std::sort(sp.begin(), sp.end());
      n_sparse_ = int(sp.size());
      d_sparse_leaves_ = upload_vec(sp);
    }
    // Leaf phase table (sincos_l): |A| <= k side / sqrt 2, |B| <= k side / 2
    // for particles in their leaf; larger leaves (or the HFMM_LEAF_POLY test
    // hook) use the sincos polynomials.
    {
      const double amax = s.k * s.leaf_side / std::sqrt(2.0);
      const int nh = int(std::ceil(amax * 128.0)) + 2;
      if (nh <= kLeafTabMax && std::getenv("HFMM_LEAF_POLY") == nullptr) {
        std::vector<double2> tab(static_cast<size_t>(2 * nh + 1));
        for (int i = -nh; i <= nh; ++i) tab[size_t(i + nh)] = make_double2(std::cos(i / 128.0), std::sin(i / 128.0));
        d_ltab_ = upload_vec(tab);
        ltab_half_ = nh;
      }
    }
    // Near-field phase table (green_tab): r' = k r <= k 2 sqrt(3) leaf side
    // between particles of adjacent leaves; larger leaves (or the
    // HFMM_P2P_POLY test hook) use the sincos polynomials.
    {
      const double rmax = s.k * 2.0 * std::sqrt(3.0) * s.leaf_side;
      const int ntab = int(std::ceil(rmax * 128.0)) + 2;
      if (ntab <= kPhaseTabMax && std::getenv("HFMM_P2P_POLY") == nullptr) {
        std::vector<double2> tab(static_cast<size_t>(ntab));
        for (int i = 0; i < ntab; ++i) tab[size_t(i)] = make_double2(std::cos(i / 128.0), -std::sin(i / 128.0));
        d_ptab_ = upload_vec(tab);
        ptab_max_ = ntab - 1;
      }
    }
    // symmetric pair lists among own dense leaves (k_p2p_sym2 / k_p2p_gather).
    // k_p2p_sym2 runs one CTA per (leaf, pass of 128 observers): each pass
    // writes its own scratch rows (no read-modify-write across CTAs), and
    // the gather adds them in (sender leaf, pass) order, so sums are
    // deterministic.
    const int obs_pass = 32 * kSymObs;
    auto pop = [&](int64_t lf) { return int64_t(s.leaf_start[size_t(lf) + 1] - s.leaf_start[size_t(lf)]); };
    std::vector<int> pos(s.num_leaves(), -1);
    for (size_t i = 0; i < dense.size(); ++i) pos[size_t(dense[i])] = int(i);
    std::vector<int> poff{0}, pl, soff{0}, sl;
    std::vector<int64_t> sscr, srows;
    std::vector<std::vector<std::pair<std::pair<int, int>, int64_t>>> incoming(dense.size());
    std::vector<std::pair<int64_t, int2>> items[4];  // by slots per lane - 1: (cost, {leaf idx, pass})
    int64_t scr = 0;
    for (size_t i = 0; i < dense.size(); ++i) {
      const int a = dense[i];
      const int64_t na = pop(a);
      const int npass = int((na + obs_pass - 1) / obs_pass);
      int64_t rows = 0, plain_src = 0;
      const size_t sb = sl.size();
      for (uint64_t z2 = s.near_off[size_t(a)]; z2 < s.near_off[size_t(a) + 1]; ++z2) {
        const int b = int(s.near[z2]);
        // k_p2p_sym2 takes the self leaf as a symmetric entry (pairs o < t once)
        if (b >= a && pos[size_t(b)] >= 0) {
          sl.push_back(b);
          sscr.push_back(scr + rows);
          rows += pop(b);
        } else if (b == a || pos[size_t(b)] < 0) {
          pl.push_back(b);
          plain_src += pop(b);
        }
      }
      for (size_t jj = sb; jj < sl.size(); ++jj)
        for (int p = 0; p < npass; ++p)
          incoming[size_t(pos[size_t(sl[jj])])].push_back({{a, p}, sscr[jj] + int64_t(p) * rows});
      for (int p = 0; p < npass; ++p) {
        const int64_t no = std::min<int64_t>(na - int64_t(p) * obs_pass, obs_pass);
        const int nc = int((no + 31) / 32);
        items[nc - 1].push_back({int64_t(nc) * (plain_src + rows), make_int2(int(i), p)});
      }
      srows.push_back(rows);
      scr += int64_t(npass) * rows;
      poff.push_back(int(pl.size()));
      soff.push_back(int(sl.size()));
    }
    std::vector<int> ioff{0};
    std::vector<int64_t> iscr;
    for (auto& v : incoming) {  // senders in ascending (leaf, pass) order: deterministic sums
      std::sort(v.begin(), v.end());
      for (auto& e : v) iscr.push_back(e.second);
      ioff.push_back(int(iscr.size()));
    }
    // work items per slot count, most expensive first (LPT order)
    std::vector<int2> it;
    for (int c = 3; c >= 0; --c) {
      std::stable_sort(items[c].begin(), items[c].end(),
                       [](const std::pair<int64_t, int2>& u, const std::pair<int64_t, int2>& v) {
                         return u.first > v.first;
                       });
      p2p_items_b_[c] = int(it.size());
      for (auto& e : items[c]) it.push_back(e.second);
      p2p_items_n_[c] = int(items[c].size());
    }
    d_p2p_items_ = upload_vec(it);
    d_sym_rows_ = upload_vec(srows);
    d_plain_off_ = upload_vec(poff);
    d_plain_ = upload_vec(pl);
    d_sym_off_ = upload_vec(soff);
    d_sym_ = upload_vec(sl);
    d_sym_scr_ = upload_vec(sscr);
    d_in_off_ = upload_vec(ioff);
    d_in_scr_ = upload_vec(iscr);
    d_p2p_scratch_ = alloc<double2>(size_t(std::max<int64_t>(scr, 1)));
  }

  lv_.assign(size_t(L + 1), DevLevel{});
  std::vector<std::vector<double>> hdir(size_t(L + 1));
  size_t tmp = 0;
  for (int l = s.top; l <= L; ++l) {
    const LevelData& t = s.levels[size_t(l)];
    DevLevel& d = lv_[size_t(l)];
    d.level = l;
    d.nt = int(t.nt);
    d.np = int(t.np);
    d.trunc = t.trunc;
    d.S = t.samples();
    d.n_nodes = int(t.num_nodes());
    // rows: every node (one rank), or held + halo + one zero row (distributed mode)
    d.n_rows = dist_ ? int(rp_->held[size_t(l)].size() + rp_->halo[size_t(l)].size()) + 1 : d.n_nodes;
    d.side = t.side;
    // Directions exactly as LevelSampling::direction (sphere_grid.cpp:25-37).
    std::vector<double> dir(size_t(3 * d.S)), wq(size_t(d.S));
    for (int64_t sidx = 0; sidx < d.S; ++sidx) {
      const int64_t i = sidx / d.np, j = sidx % d.np;
      const double th = (double(i) + 0.5) * M_PI / double(d.nt);
      const double ph = double(j) * 2.0 * M_PI / double(d.np);
      const double st = std::sin(th);
      dir[size_t(3 * sidx)] = st * std::cos(ph);
      dir[size_t(3 * sidx + 1)] = st * std::sin(ph);
      dir[size_t(3 * sidx + 2)] = std::cos(th);
      wq[size_t(sidx)] = t.theta_w[size_t(i)] * t.phi_w;
    }
    d.dir = upload_vec(dir);
    hdir[size_t(l)] = dir;
    d.wq = upload_vec(wq);
    d.centers = upload_vec(t.centers);
    d.mp = alloc<double2>(size_t(d.n_rows) * size_t(d.S));
    d.loc = alloc<double2>(size_t(d.n_rows) * size_t(d.S));
    ck(cudaMemsetAsync(d.mp, 0, size_t(d.n_rows) * size_t(d.S) * sizeof(double2), st_), "memset mp");
    ck(cudaMemsetAsync(d.loc, 0, size_t(d.n_rows) * size_t(d.S) * sizeof(double2), st_), "memset loc");
    // Far lists as (source, offset slot) and the used slots.
    std::vector<int64_t> foff(t.far_off.begin(), t.far_off.end());
    std::vector<int2> far(t.far.size());
    std::vector<uint8_t> used(kSlots, 0);
    for (size_t o = 0; o < t.num_nodes(); ++o)
      for (uint64_t f = t.far_off[o]; f < t.far_off[o + 1]; ++f) {
        const uint32_t src = t.far[f];
        long ox = long(cell_axis(t.codes[o], l, 0)) - long(cell_axis(t.codes[src], l, 0));
        long oy = long(cell_axis(t.codes[o], l, 1)) - long(cell_axis(t.codes[src], l, 1));
        long oz = long(cell_axis(t.codes[o], l, 2)) - long(cell_axis(t.codes[src], l, 2));
        const int sl = slot_of(ox, oy, oz);
        far[f] = make_int2(int(src), sl);
        used[size_t(sl)] = 1;
      }
    d.n_far = int64_t(far.size());
    if (dist_) {  // far-list CSR over the held observers (rows 0..H-1), sources as rows
      const int zero_row = d.n_rows - 1;  // absent sources (outside every needed slice) read zeros
      std::vector<int64_t> fo{0};
      std::vector<int2> fr;
      for (int o : rp_->held[size_t(l)]) {
        for (uint64_t f = t.far_off[size_t(o)]; f < t.far_off[size_t(o) + 1]; ++f) {
          const int r = row(l, int(far[f].x));
          fr.push_back(make_int2(r >= 0 ? r : zero_row, far[f].y));
        }
        fo.push_back(int64_t(fr.size()));
      }
      foff.swap(fo);
      far.swap(fr);
    }
    d.far_off = upload_vec(foff);
    d.far = upload_vec(far);
    d.slot_used = upload_vec(used);
    // Translation-operator coefficients (operators.cpp:52-63), host libstdc++
    // special functions exactly as the reference evaluates them.
    std::vector<double2> coef(size_t(kSlots) * size_t(d.trunc + 1), make_double2(0, 0));
    for (int sl = 0; sl < kSlots; ++sl) {
      if (!used[size_t(sl)]) continue;
      const double Dx = double(sl / 49 - 3) * t.side, Dy = double((sl / 7) % 7 - 3) * t.side,
                   Dz = double(sl % 7 - 3) * t.side;
      const double dist = std::sqrt(Dx * Dx + Dy * Dy + Dz * Dz);
      if (dist < 2.0 * t.side * (1.0 - 1e-12))
        throw std::invalid_argument("translation_operator: boxes not well separated (|D| < 2 * side)");
      const double xk = s.k * dist;
      std::complex<double> mj_pow(1.0, 0.0);
      const std::complex<double> mj(0.0, -1.0);
      for (int ll = 0; ll <= d.trunc; ++ll) {
        std::complex<double> h2(std::sph_bessel(unsigned(ll), xk), -std::sph_neumann(unsigned(ll), xk));
        std::complex<double> c = mj_pow * double(2 * ll + 1) * h2;
        coef[size_t(sl * (d.trunc + 1) + ll)] = make_double2(c.real(), c.imag());
        mj_pow *= mj;
      }
    }
    d.tcoef = upload_vec(coef);
    // Dense cell lookup for well-populated levels (stencil M2L).
    d.G = 1 << (l - 1);
    const double cells = double(d.G) * d.G * d.G;
    // (grids smaller than one 8^3 observer block -- level 3 -- leave the block
    // mostly empty: far-list CSR kernel there)
    if (d.n_far > 0 && d.G >= m2l::MB && d.G <= 512 && double(d.n_nodes) >= 0.25 * cells) {
      // row-major cell -> node table padded by a 3-cell halo of -1 (m2l.cuh)
      const size_t GP = size_t(std::max(d.G, m2l::MB)) + 6;
      std::vector<int> lk(GP * GP * GP, -1);
      for (size_t i = 0; i < t.num_nodes(); ++i) {
        const uint64_t c = t.codes[i];
        const size_t gx = cell_axis(c, l, 0) + 3, gy = cell_axis(c, l, 1) + 3, gz = cell_axis(c, l, 2) + 3;
        lk[(gz * GP + gy) * GP + gx] = row(l, int(i));  // -1: not stored on this rank (zero-filled)
      }
      d.lookup = upload_vec(lk);
      d.dense = true;
    }
    d.T = alloc<double2>(size_t(kSlots) * size_t(d.S));
    // Child CSR, parent links and octants.
    if (l < L) {
      std::vector<int> coff(t.child_off.begin(), t.child_off.end());
      std::vector<int> ch(t.children.begin(), t.children.end());
      d.child_off = upload_vec(coff);
      d.children = upload_vec(ch);
    }
    if (l > s.top) {  // parent row of every row
      const LevelData& pt = s.levels[size_t(l - 1)];
      std::vector<int> par(size_t(d.n_rows), -1);
      for (size_t p = 0; p < pt.num_nodes(); ++p)
        for (uint64_t z2 = pt.child_off[p]; z2 < pt.child_off[p + 1]; ++z2) {
          const int rc = row(l, int(pt.children[z2]));
          if (rc >= 0) par[size_t(rc)] = row(l - 1, int(p));
        }
      d.parent = upload_vec(par);
    }
  }
  // Octant per node (child side of every parent/child pair).
  std::vector<uint8_t*> octs(size_t(L + 1), nullptr);
  for (int l = s.top; l <= L; ++l) {
    const LevelData& t = s.levels[size_t(l)];
    std::vector<uint8_t> oc(size_t(lv_[size_t(l)].n_rows), 0);  // per row
    for (size_t i = 0; i < t.num_nodes(); ++i) {
      const int r = row(l, int(i));
      if (r >= 0) oc[size_t(r)] = uint8_t(t.codes[i] & 7);
    }
    octs[size_t(l)] = upload_vec(oc);
  }
  oct_ = octs;
  // Interpolation matrices and shift tables per parent level.
  for (int l = s.top; l < L; ++l) {
    DevLevel& P = lv_[size_t(l)];
    const DevLevel& C = lv_[size_t(l + 1)];
    const LevelData& tp = s.levels[size_t(l)];
    const LevelData& tc = s.levels[size_t(l + 1)];
    const int nc = C.nt, np = P.nt;
    if (C.np != nc || P.np != np) throw std::logic_error("non-square sampling");
    // Shift tables on the parent grid: disp = c_child - c_parent = (b - 1/2) side_c.
    const std::vector<double>& dir = hdir[size_t(l)];
    std::vector<double2> up(size_t(8 * P.S)), dn(size_t(8 * P.S));
    for (int o = 0; o < 8; ++o) {
      const double dx = ((o & 1) ? 0.5 : -0.5) * C.side, dy = ((o & 2) ? 0.5 : -0.5) * C.side,
                   dz = ((o & 4) ? 0.5 : -0.5) * C.side;
      for (int64_t sidx = 0; sidx < P.S; ++sidx) {
        const double a = s.k * (dir[size_t(3 * sidx)] * dx + dir[size_t(3 * sidx + 1)] * dy +
                                dir[size_t(3 * sidx + 2)] * dz);
        up[size_t(o * P.S + sidx)] = make_double2(std::cos(a), std::sin(a));
        const double b = s.k * (dir[size_t(3 * sidx)] * (-dx) + dir[size_t(3 * sidx + 1)] * (-dy) +
                                dir[size_t(3 * sidx + 2)] * (-dz));
        dn[size_t(o * P.S + sidx)] = make_double2(std::cos(b), std::sin(b));
      }
    }
    P.shift_up = upload_vec(up);
    P.shift_dn = upload_vec(dn);
    setup_interp(P, C, tp, tc);
    tmp = std::max(tmp, size_t(C.n_rows) * size_t(nc) * size_t(np));
    tmp = std::max(tmp, rb_m2m_scratch(C.n_rows, nc, np));
    tmp = std::max(tmp, rb_l2l_scratch(C.n_rows, nc, np));
  }
  tmp_elems_ = std::max(tmp, tmp_need_);
  d_tmp = alloc<double2>(tmp_elems_);
}

void Engine::set_charges(const double* q_in) {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  const int64_t n = int64_t(s_.n);
  ck(cudaMemcpyAsync(d_q_in, q_in, size_t(n) * sizeof(double2), cudaMemcpyHostToDevice, st_), "H2D q");
  if (dist_) {
    const int64_t cnt = part_e_ - part_b_;
    if (cnt > 0) k_gather_q_range<<<unsigned((cnt + 255) / 256), 256, 0, st_>>>(part_b_, part_e_, d_orig, d_q_in, d_q);
  } else {
    k_gather_q<<<unsigned((n + 255) / 256), 256, 0, st_>>>(n, d_orig, d_q_in, d_q);
  }
  ++launches_;
  ck(cudaGetLastError(), "k_gather_q");
}

void Engine::build_T() {
  for (int l = s_.top; l <= s_.L; ++l) {
    DevLevel& d = lv_[size_t(l)];
    if (d.n_far == 0) continue;
    dim3 grid(unsigned((d.S + 127) / 128), kSlots);
    k_tbuild<<<grid, 128, 2 * size_t(d.trunc + 1) * sizeof(double2), st_>>>(d.S, d.trunc, d.dir, d.side,
                                                                         d.tcoef, d.slot_used, d.T);
    ++launches_;
  }
  ck(cudaGetLastError(), "k_tbuild");
}

namespace {
// Quad-symmetric leaf kernels need an even, square grid with n/2 <= kQuadHalfMax.
bool quad_ok(const DevLevel& d, bool hook_generic) {
  return d.nt == d.np && d.nt % 2 == 0 && d.nt / 2 <= kQuadHalfMax && !hook_generic;
}
}  // namespace

void Engine::phase_c2m() {
  const DevLevel& d = lv_[size_t(s_.L)];
  const int64_t nl = leaf_e_ - leaf_b_;
  if (quad_ok(d, hook_no_quad_)) {
    const int quads = int(d.nt / 2) * int(d.nt / 2);
    // quads per lane: fewest lane slots (passes x R), ties to fewer passes; R <= 4
    // keeps 4 CTAs/SM (R = 6 needs 208 registers and measured slower at config 2)
    int r = 1, best = INT32_MAX;
    for (int rr = 1; rr <= 4; ++rr) {
      const int cost = (quads + 32 * rr - 1) / (32 * rr) * rr;
      if (cost <= best) {
        best = cost;
        r = rr;
      }
    }
    const unsigned g = unsigned((nl + 3) / 4);
#define HFMM_C2M(RR, HN)                                                                                    \
  k_c2m_quad2<RR, HN><<<g, 128, 0, st_>>>(leaf_b_, nl, d_leaf_start, d_x, d_y, d_z, d_q, d.centers, d.dir, d.nt, \
                                          s_.k, d.mp)
    const int hn = int(d.nt / 2);
    if (r == 3 && hn == 9) HFMM_C2M(3, 9);        // n = 18 (configs 1, 3, 4)
    else if (r == 4 && hn == 11) HFMM_C2M(4, 11);  // n = 22 (config 5)
    else if (r == 3 && hn == 13) HFMM_C2M(3, 13);  // n = 26 (config 2)
    else
      switch (r) {
        case 1: HFMM_C2M(1, 0); break;
        case 2: HFMM_C2M(2, 0); break;
        case 3: HFMM_C2M(3, 0); break;
        default: HFMM_C2M(4, 0); break;
      }
#undef HFMM_C2M
  } else  // leaf grids past kQuadHalfMax: generic kernel
    k_c2m<<<unsigned(nl), 128, 0, st_>>>(leaf_b_, d_leaf_start, d_x, d_y, d_z, d_q, d.centers, d.dir, d.S, s_.k,
                                         d.mp);
  ++launches_;
  ck(cudaGetLastError(), "k_c2m");
}

namespace {
// Runtime-shaped streaming kernels: any even grid pair (the host B layouts
// K = round4(n_in + 1), N = round8(n_out) are what they expect).
#ifndef HFMM_RBL_SMEM_KB
#define HFMM_RBL_SMEM_KB 100
#endif
constexpr int kRblSmemLim = HFMM_RBL_SMEM_KB * 1024;  // two CTAs per SM at the default
// n8 tiles per CTA column block of a theta pass with n_in inputs and n_out outputs per
// half circle: the most that fit shared memory, in even blocks of a multiple of `mult` tiles
int rbl_chb(int n_in, int n_out, int mult) {
  const int rows = 2 * rb::r4(n_in + 1), nt = rb::r8(n_out) / 8;
  int chb = (nt + mult - 1) / mult * mult;
  while (chb > mult && rows * rb::blk_ldb(8 * chb) * 8 > kRblSmemLim) chb -= mult;
  const int nblk = (nt + chb - 1) / chb;
  return ((nt + nblk - 1) / nblk + mult - 1) / mult * mult;
}
int l2l_rbl_chb(int nc, int np) { return rbl_chb(np, nc, 1); }
int m2m_rbl_chb(int nc, int np) { return rbl_chb(nc, np, rb::kChunkEO); }
bool rbl_ok(int nc, int np) {
  // shared-memory B: whole phi matrices and one theta column block must fit
  const int lim = kRblSmemLim, lim_phi = 225 * 1024;
  const bool fits = rb::r4(nc + 1) * rb::blk_ldb(rb::r8(np)) * 8 <= lim_phi && rb::r4(np + 1) * rb::blk_ldb(rb::r8(nc)) * 8 <= lim_phi &&
                    2 * rb::r4(nc + 1) * rb::blk_ldb(8 * m2m_rbl_chb(nc, np)) * 8 <= lim &&
                    2 * rb::r4(np + 1) * rb::blk_ldb(8 * l2l_rbl_chb(nc, np)) * 8 <= lim;
  return nc % 2 == 0 && np % 2 == 0 && fits;
}
}  // namespace

void Engine::phase_m2m() {
  for (int l = s_.L - 1; l >= s_.top; --l) {
    DevLevel& P = lv_[size_t(l)];
    DevLevel& C = lv_[size_t(l + 1)];
    const int nc = C.nt, np = P.nt;
    const RankLevel* R = dist_ ? &rl_[size_t(l)] : nullptr;
    const RbLaunch rl{R ? R->n_par : P.n_nodes, R ? R->plist : nullptr, R ? R->child_off : P.child_off,
                      R ? R->children : P.children, dist_ ? R->n_children : int64_t(C.n_nodes),
                      oct_[size_t(l + 1)], pdesc_[size_t(l)], 2 * sms_, st_, kPhiCtas * sms_};
    if (rl.n_par == 0) continue;
    // 0. fused single-kernel pair (folded circles stay in shared memory)
#ifndef HFMM_NO_FZ
    if (!hook_no_rb_ && fz_pair(nc, np)) {
      launch_m2m_fz2(rl, sms_, C.mp, P.mp, P.up_phi_Bf, P.up_phi_v, P.up_th_Be, P.up_th_ve, P.shift_up);
      ++launches_;
      ck(cudaGetLastError(), "k_m2m_fz");
      continue;
    }
#endif
    // 1. compile-time-shaped streaming pairs (the BASELINE leaf-side pairs)
    if (!hook_no_rb_ && rb_pair(nc, np) &&
        launch_m2m_rb(nc, np, rl, C.mp, P.mp, P.up_phi_Bf, P.up_phi_v, P.up_th_Be, P.up_th_ve, P.shift_up, d_tmp)) {
      launches_ += 2;
      ck(cudaGetLastError(), "k_m2m_rb");
      continue;
    }
    // 2. runtime-shaped streaming kernels (B matrices fit shared memory)
    if (!hook_no_rbl_ && rbl_ok(nc, np)) {
      const int s_phi = rb::r4(nc + 1) * rb::blk_ldb(rb::r8(np)) * 8;
      const int chb = m2m_rbl_chb(nc, np), nchunk = (rb::r8(np) / 8 + chb - 1) / chb;
      const int s_th = 2 * rb::r4(nc + 1) * rb::blk_ldb(8 * chb) * 8;
      ck(cudaFuncSetAttribute(k_m2m_phi_rbl, cudaFuncAttributeMaxDynamicSharedMemorySize, s_phi), "attr");
      ck(cudaFuncSetAttribute(k_m2m_theta_rbl, cudaFuncAttributeMaxDynamicSharedMemorySize, s_th), "attr");
      if (rl.nch > 0)
        k_m2m_phi_rbl<<<2 * sms_, rb::kThreads, s_phi, st_>>>(nc, np, rl.nch, rl.children, C.mp, P.up_phi_Bf, P.up_phi_v,
                                                              d_tmp);
      const int per_sm_u = std::max(1, std::min(2, (220 * 1024) / (s_th + 1024)));
      const dim3 gth(unsigned(std::max(1, per_sm_u * sms_ / nchunk)), unsigned(nchunk));
      k_m2m_theta_rbl<<<gth, rb::kThreads, s_th, st_>>>(nc, np, chb, rl.n_par, rl.pdesc, d_tmp, P.up_th_Be, P.up_th_ve, P.shift_up, P.mp);
      launches_ += 2;
      ck(cudaGetLastError(), "k_m2m_rbl");
      continue;
    }
    // 3. two-stage large-grid kernels (any grid; B streams from L2)
    const int* clist = nullptr;  // children rows 0..ncl-1 (held rows come first)
    const int ncl = dist_ ? held_cnt_[size_t(l + 1)] : C.n_nodes;
    ck(cudaFuncSetAttribute(k_m2m_big_phi, cudaFuncAttributeMaxDynamicSharedMemorySize, int(P.big_smem[0])), "attr");
    ck(cudaFuncSetAttribute(k_m2m_big_theta, cudaFuncAttributeMaxDynamicSharedMemorySize, int(P.big_smem[1])), "attr");
    if (ncl > 0) {
      dim3 g0(unsigned(ncl), unsigned((nc + P.big_rc[0] - 1) / P.big_rc[0]));
      k_m2m_big_phi<<<g0, kBigThreads, P.big_smem[0], st_>>>(nc, np, to_dims(P.up_phi), P.up_th[2], P.big_rc[0], clist,
                                                             C.mp, P.up_phi_B, P.up_phi_v, d_tmp);
      ++launches_;
    }
    dim3 grid(unsigned(rl.n_par), unsigned((np / 2 + P.big_m2m_cp - 1) / P.big_m2m_cp));
    k_m2m_big_theta<<<grid, kBigThreads, P.big_smem[1], st_>>>(nc, np, P.big_m2m_cp, to_dims(P.up_th), rl.plist,
                                                               rl.child_off, rl.children, rl.oct_c, d_tmp, P.up_th_B,
                                                               P.up_th_v, P.shift_up, P.mp);
    ++launches_;
    ck(cudaGetLastError(), "m2m big");
  }
}

void Engine::phase_m2l(int lo, int hi) {
  if (lo < 0) lo = s_.top;
  if (hi < 0) hi = s_.L;
  ck(cudaFuncSetAttribute(k_m2l_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, m2l::SMEM_BYTES), "attr");
  for (int l = lo; l <= hi; ++l) {
    DevLevel& d = lv_[size_t(l)];
    // distributed mode: only the observers this rank holds (the multipole
    // exchange completed exactly their far sources)
    if (d.dense) {
      const int nb = (d.G + m2l::MB - 1) / m2l::MB;
      const int nblk = dist_ ? d.m2l_nblk : nb * nb * nb;
      if (nblk == 0) continue;
      const int ppc = m2l_pairs_per_cta(nblk, d.S, sms_);
      dim3 grid(unsigned(nblk), unsigned((d.S / 2 + ppc - 1) / ppc));
      k_m2l_dmma<<<grid, 128, m2l::SMEM_BYTES, st_>>>(d.G, nb, d.S, ppc, dist_ ? d.m2l_blk : nullptr, d.lookup, d.T,
                                                      d.mp, d.loc);
    } else {
      const int nobs = dist_ ? held_cnt_[size_t(l)] : int(d.n_nodes);
      if (nobs == 0) continue;
      dim3 grid(unsigned(nobs), unsigned((d.S + 127) / 128));
      k_m2l<<<grid, 128, 0, st_>>>(d.S, 0, nullptr, d.far_off, d.far, d.T, d.mp, d.loc);  // rows 0..nobs-1
    }
    ++launches_;
  }
  ck(cudaGetLastError(), "m2l");
}

void Engine::phase_l2l(int lo, int hi) {
  if (lo < 0) lo = s_.top;
  if (hi < 0) hi = s_.L - 1;
  for (int l = lo; l <= hi; ++l) {
    DevLevel& P = lv_[size_t(l)];
    DevLevel& C = lv_[size_t(l + 1)];
    const int nc = C.nt, np = P.nt;
    const RankLevel* R = dist_ ? &rl_[size_t(l)] : nullptr;
    const RbLaunch rl{R ? R->n_par : P.n_nodes, R ? R->plist : nullptr, R ? R->child_off : P.child_off,
                      R ? R->children : P.children, dist_ ? R->n_children : int64_t(C.n_nodes),
                      oct_[size_t(l + 1)], pdesc_[size_t(l)], 2 * sms_, st_, kPhiCtas * sms_};
    if (rl.n_par == 0) continue;
    // 1. compile-time-shaped streaming pairs
    if (!hook_no_rb_ && rb_pair(nc, np) &&
        launch_l2l_rb(nc, np, rl, P.loc, C.loc, P.dn_th_Be, P.dn_th_ve, P.dn_phi_Bu, P.dn_phi_vu, P.shift_dn, d_tmp)) {
      launches_ += 2;
      ck(cudaGetLastError(), "k_l2l_rb");
      continue;
    }
    // 2. runtime-shaped streaming kernels
    if (!hook_no_rbl_ && rbl_ok(nc, np)) {
      const int s_phi = rb::r4(np + 1) * rb::blk_ldb(rb::r8(nc)) * 8;
      ck(cudaFuncSetAttribute(k_l2l_phi_rbl, cudaFuncAttributeMaxDynamicSharedMemorySize, s_phi), "attr");
      const int chb = l2l_rbl_chb(nc, np), nblk = (rb::r8(nc) / 8 + chb - 1) / chb;
      const int s_th = 2 * rb::r4(np + 1) * rb::blk_ldb(8 * chb) * 8;
      ck(cudaFuncSetAttribute(k_l2l_theta_rbl, cudaFuncAttributeMaxDynamicSharedMemorySize, s_th), "attr");
      const int per_sm = std::max(1, std::min(2, (220 * 1024) / (s_th + 1024)));
      const dim3 gth(unsigned(std::max(1, per_sm * sms_ / nblk)), unsigned(nblk));
      k_l2l_theta_rbl<<<gth, rb::kThreads, s_th, st_>>>(nc, np, chb, rl.n_par, rl.pdesc, P.loc, P.dn_th_Be, P.dn_th_ve, P.shift_dn, d_tmp);
      if (rl.nch > 0)
        k_l2l_phi_rbl<<<2 * sms_, rb::kThreads, s_phi, st_>>>(nc, np, rl.nch, rl.children, d_tmp, P.dn_phi_Bu, P.dn_phi_vu,
                                                              C.loc);
      launches_ += 2;
      ck(cudaGetLastError(), "k_l2l_rbl");
      continue;
    }
    // 3. two-stage large-grid kernels
    const int* clist = nullptr;  // children rows 0..ncl-1 (held rows come first)
    const int ncl = dist_ ? held_cnt_[size_t(l + 1)] : C.n_nodes;
    if (ncl == 0) continue;
    ck(cudaFuncSetAttribute(k_l2l_big_theta, cudaFuncAttributeMaxDynamicSharedMemorySize, int(P.big_smem[2])), "attr");
    ck(cudaFuncSetAttribute(k_l2l_big_phi, cudaFuncAttributeMaxDynamicSharedMemorySize, int(P.big_smem[3])), "attr");
    dim3 grid(unsigned(ncl), unsigned((np / 2 + P.big_l2l_cp - 1) / P.big_l2l_cp));
    k_l2l_big_theta<<<grid, kBigThreads, P.big_smem[2], st_>>>(nc, np, P.big_l2l_cp, to_dims(P.dn_th), P.big_ldn, clist,
                                                               C.parent, rl.oct_c, P.loc, P.shift_dn, P.dn_th_B,
                                                               P.dn_th_v, d_tmp);
    ++launches_;
    dim3 g3(unsigned(ncl), unsigned((nc + P.big_rc[1] - 1) / P.big_rc[1]));
    k_l2l_big_phi<<<g3, kBigThreads, P.big_smem[3], st_>>>(nc, np, to_dims(P.dn_phi), P.big_ldn, P.big_rc[1], clist,
                                                           d_tmp, P.dn_phi_B, P.dn_phi_v, C.loc);
    ++launches_;
    ck(cudaGetLastError(), "l2l big");
  }
}

void Engine::phase_l2t() {
  const DevLevel& d = lv_[size_t(s_.L)];
  const int64_t nl = leaf_e_ - leaf_b_;
  if (quad_ok(d, hook_no_quad_)) {
    const size_t smem = 4 * size_t(kQuadP * (d.nt / 2)) * sizeof(double2);
    {
      // (n / 2 <= kQuadHalfMax keeps the table under 48 KB: no attribute needed)
      auto l2t_quads = [&](unsigned grid, int64_t lb, int64_t cnt, const int* list) {
        const int hn = int(d.nt / 2);
        // quads per lane: fewest lane slots (chunks x R), ties to fewer chunks; R <= 4
        const int quads = hn * hn;
        int r = 1, best = INT32_MAX;
        for (int rr = 1; rr <= 4; ++rr) {
          const int cost = (quads + 32 * rr - 1) / (32 * rr) * rr;
          if (cost <= best) {
            best = cost;
            r = rr;
          }
        }
#define HFMM_L2T3(RR, HN)                                                                                        \
  do {                                                                                                            \
    if (d_ltab_)                                                                                                  \
      k_l2t_quad3<RR, HN, true><<<grid, 128, 0, st_>>>(lb, cnt, list, d_leaf_start, d_x, d_y, d_z, d.centers, d.dir, \
                                                       d.wq, d.nt, s_.k, d.loc, d_pot, d_ltab_, ltab_half_);        \
    else                                                                                                          \
      k_l2t_quad3<RR, HN, false><<<grid, 128, 0, st_>>>(lb, cnt, list, d_leaf_start, d_x, d_y, d_z, d.centers,      \
                                                        d.dir, d.wq, d.nt, s_.k, d.loc, d_pot);                     \
  } while (0)
        if (r == 3 && hn == 9) HFMM_L2T3(3, 9);        // n = 18 (configs 1, 3, 4)
        else if (r == 4 && hn == 11) HFMM_L2T3(4, 11);  // n = 22 (config 5)
        else if (r == 3 && hn == 13) HFMM_L2T3(3, 13);  // n = 26 (config 2)
        else
          switch (r) {
            case 1: HFMM_L2T3(1, 0); break;
            case 2: HFMM_L2T3(2, 0); break;
            case 3: HFMM_L2T3(3, 0); break;
            default: HFMM_L2T3(4, 0); break;
          }
#undef HFMM_L2T3
      };
      if (n_dense_ > 0) {  // populous leaves: lane per observer, the rest: lanes over quads
        const int quads = int(d.nt / 2) * int(d.nt / 2);
        const size_t so = 4 * size_t(quads) * 5 * sizeof(double2);
        const int hn = int(d.nt / 2);
#define HFMM_L2TO(HN)                                                                                          \
  do {                                                                                                         \
    if (so > 24 * 1024) {                                                                                      \
      ck(cudaFuncSetAttribute(k_l2t_obs<HN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(so)), "a"); \
      ck(cudaFuncSetAttribute(k_l2t_obs<HN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(so)), "a"); \
    }                                                                                                          \
    if (d_ltab_)                                                                                               \
      k_l2t_obs<HN, true><<<unsigned((n_dense_ + 3) / 4), 128, so, st_>>>(                                      \
          leaf_b_, n_dense_, d_dense_leaves_, d_leaf_start, d_x, d_y, d_z, d.centers, d.dir, d.wq, d.nt, s_.k, d.loc, d_pot, \
          d_ltab_, ltab_half_);                                                                                \
    else                                                                                                       \
      k_l2t_obs<HN, false><<<unsigned((n_dense_ + 3) / 4), 128, so, st_>>>(                                     \
          leaf_b_, n_dense_, d_dense_leaves_, d_leaf_start, d_x, d_y, d_z, d.centers, d.dir, d.wq, d.nt, s_.k, d.loc, d_pot); \
  } while (0)
        if (hn == 9) HFMM_L2TO(9);
        else if (hn == 11) HFMM_L2TO(11);
        else if (hn == 13) HFMM_L2TO(13);
        else HFMM_L2TO(0);
#undef HFMM_L2TO
        ++launches_;
        if (n_sparse_ > 0) l2t_quads(unsigned((n_sparse_ + 3) / 4), leaf_b_, n_sparse_, d_sparse_leaves_);  // rows start at leaf_b_
      } else {
        l2t_quads(unsigned((nl + 3) / 4), leaf_b_, nl, nullptr);
      }
    }
  } else {  // leaf grids past kQuadHalfMax: generic kernel
    k_l2t<<<unsigned(nl), 128, 0, st_>>>(leaf_b_, d_leaf_start, d_x, d_y, d_z, d.centers, d.dir, d.wq, d.S, s_.k,
                                         d.loc, d_pot);
  }
  ++launches_;
  ck(cudaGetLastError(), "k_l2t");
}

// Near field on the side stream: waits for everything issued so far on the
// main stream (charges, ghosts), accumulates into d_pot_near.
void Engine::near_start() {
  const DevLevel& d = lv_[size_t(s_.L)];
  ck(cudaEventRecord(ev_fork_, st_), "fork");
  ck(cudaStreamWaitEvent(st2_, ev_fork_, 0), "fork wait");
  cudaEventRecord(ev_near0_, st2_);
  const int64_t cnt = part_e_ - part_b_;
  if (cnt > 0)
    ck(cudaMemsetAsync(d_pot_near + part_b_, 0, size_t(cnt) * sizeof(double2), st2_), "memset near");
  if (n_tiny_ + n_small_ > 0) {  // leaves with <= 32 particles: one warp per leaf
    const int nl = n_tiny_ + n_small_;
    if (d_ptab_)
      k_p2p_leaf2<true><<<unsigned((nl + 3) / 4), 128, 0, st2_>>>(nl, d_sparse_leaves_, d_leaf_start, d_near_off,
                                                                  d_near, d.centers, d_x, d_y, d_z, d_q, s_.k,
                                                                  d_pot_near, d_ptab_, ptab_max_);
    else
      k_p2p_leaf2<false><<<unsigned((nl + 3) / 4), 128, 0, st2_>>>(nl, d_sparse_leaves_, d_leaf_start, d_near_off,
                                                                   d_near, d.centers, d_x, d_y, d_z, d_q, s_.k,
                                                                   d_pot_near);
    ++launches_;
  }
  if (n_dense_ > 0) {
    for (int c = 3; c >= 0; --c) {
        if (p2p_items_n_[c] == 0) continue;
        const int2* itm = d_p2p_items_ + p2p_items_b_[c];
        const unsigned g = unsigned(p2p_items_n_[c]);
#define HFMM_SYM2(NC, TB)                                                                                          \
  k_p2p_sym2<NC, TB><<<g, 128, 0, st2_>>>(itm, d_dense_leaves_, d_leaf_start, d_plain_off_, d_plain_, d_sym_off_,     \
                                          d_sym_, d_sym_scr_, d_sym_rows_, d.centers, d_x, d_y, d_z, d_q, s_.k,      \
                                          d_pot_near, d_p2p_scratch_, d_ptab_, ptab_max_)
        if (d_ptab_) {
          if (c == 3) HFMM_SYM2(4, true); else if (c == 2) HFMM_SYM2(3, true);
          else if (c == 1) HFMM_SYM2(2, true); else HFMM_SYM2(1, true);
        } else {
          if (c == 3) HFMM_SYM2(4, false); else if (c == 2) HFMM_SYM2(3, false);
          else if (c == 1) HFMM_SYM2(2, false); else HFMM_SYM2(1, false);
        }
#undef HFMM_SYM2
        ++launches_;
      }
    k_p2p_gather<<<unsigned(n_dense_), 128, 0, st2_>>>(d_dense_leaves_, d_leaf_start, d_in_off_, d_in_scr_,
                                                       d_p2p_scratch_, d_pot_near);
    ++launches_;
  }
  ck(cudaGetLastError(), "k_p2p");
  cudaEventRecord(ev_near1_, st2_);
  ck(cudaEventRecord(ev_join_, st2_), "join");
  near_started_ = true;
}

// Joins the near field into the potentials (after L2T wrote the far field).
void Engine::phase_near() {
  if (!near_started_) near_start();
  ck(cudaStreamWaitEvent(st_, ev_join_, 0), "join wait");
  const int64_t cnt = part_e_ - part_b_;
  if (cnt > 0) {
    k_add_pot<<<unsigned((cnt + 255) / 256), 256, 0, st_>>>(part_b_, part_e_, d_pot_near, d_pot);
    ++launches_;
  }
  ck(cudaGetLastError(), "k_add_pot");
  near_started_ = false;
}

void Engine::run_phase(int phase) {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  switch (phase) {
    case HFMM_PHASE_C2M:
      phase_c2m();
      break;
    case HFMM_PHASE_M2M:
      phase_m2m();
      break;
    case HFMM_PHASE_M2L:
      build_T();
      phase_m2l();
      break;
    case HFMM_PHASE_L2L:
      phase_l2l();
      break;
    case HFMM_PHASE_L2T:
      phase_l2t();
      break;
    case HFMM_PHASE_NEAR:
      phase_near();
      break;
    case HFMM_PHASE_NEAR_START:
      near_start();
      break;
    case HFMM_PHASE_T_BUILD:
      build_T();
      break;
    default:
      throw std::invalid_argument("hfmm_gpu_run_phase: unknown phase");
  }
  ck(cudaGetLastError(), "run_phase");
}

void Engine::evaluate(double* ms) {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  evaluate_device(nullptr, nullptr, nullptr);
  ck(cudaStreamSynchronize(st_), "evaluate");
  if (ms) last_timing(ms, nullptr);
}

void Engine::last_timing(double* ms, int64_t* launches) {
  if (!timed_) throw std::logic_error("last_timing: no evaluation recorded");
  ck(cudaEventSynchronize(ev_[7]), "event sync");
  float f = 0.f;
  for (int i = 0; i < 7; ++i) {
    cudaEventElapsedTime(&f, ev_[i], ev_[i + 1]);
    ms[i] = f;
  }
  if (cudaEventElapsedTime(&f, ev_near0_, ev_near1_) == cudaSuccess) ms[6] = f;  // side stream
  if (overlapped_) {
    // M2L = upper levels on the chain + the leaf level's own duration on its
    // stream; L2L = the chain's L2L segments without the wait for that leaf M2L.
    float a = 0.f, b = 0.f;
    if (cudaEventElapsedTime(&a, ev_lf0_, ev_lf1_) == cudaSuccess) ms[3] += a;
    if (cudaEventElapsedTime(&a, ev_[4], ev_la_) == cudaSuccess && cudaEventElapsedTime(&b, ev_lb_, ev_[5]) == cudaSuccess)
      ms[4] = a + b;
  }
  cudaEventElapsedTime(&f, ev_[0], ev_[7]);
  ms[7] = f;
  if (launches) *launches = last_launches_;
}

void Engine::evaluate_device(const double* d_q_sorted, double* d_pot_sorted, cudaStream_t st) {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  if (dist_)
    throw std::logic_error("evaluate_device: num_ranks > 1 runs phase by phase with exchanges");
  cudaStream_t saved = st_;
  if (st) st_ = st;
  const int64_t l0 = launches_;
  const int64_t n = int64_t(s_.n);
  if (d_q_sorted && d_q_sorted != reinterpret_cast<const double*>(d_q))
    ck(cudaMemcpyAsync(d_q, d_q_sorted, size_t(n) * sizeof(double2), cudaMemcpyDeviceToDevice, st_), "q");
  // Schedule autotune (overlap mode): the leaf-level M2L beside the chain
  // helps configs 2 and 3 and costs configs 4 and 5 (measured); evaluation 1
  // runs it beside the chain, evaluation 2 inside it, and from evaluation 3
  // on the faster of the two (each timed by its own ev_[0] -> ev_[7]).
  if (overlap_ && !tune_done_) {
    if (tune_evals_ == 2 || tune_evals_ == 3) {
      float f = 0.f;
      ck(cudaEventSynchronize(ev_[7]), "tune sync");
      ck(cudaEventElapsedTime(&f, ev_[0], ev_[7]), "tune time");
      tune_ms_[tune_evals_ - 2] = f;
    }
    if (tune_evals_ == 1) {
      m2l_seq_ = false;
    } else if (tune_evals_ == 2) {
      m2l_seq_ = true;
    } else if (tune_evals_ == 3) {
      m2l_seq_ = tune_ms_[1] < tune_ms_[0];
      tune_done_ = true;
    }
    ++tune_evals_;
  }
  cudaEventRecord(ev_[0], st_);
  // The far-field chain runs on a high-priority stream; the leaf-level M2L
  // (it needs only C2M's multipoles and is consumed only by the last L2L
  // step) runs beside it on a low-priority stream and fills the SMs that the
  // small upper-level kernels leave idle.  Dependencies are unchanged.
  const bool overlap = overlap_ && s_.L > s_.top && !m2l_seq_;
  cudaStream_t user = st_;
  overlapped_ = overlap;
  if (overlap) {
    ck(cudaEventRecord(ev_ofork_, user), "fork");
    ck(cudaStreamWaitEvent(st_hi_, ev_ofork_, 0), "fork wait");
    st_ = st_hi_;
  }
  // Charges still in flight on the copy stream (evaluate_host): the T build,
  // which does not read them, goes first.
  const bool t_first = q_pending_;
  if (t_first) {
    build_T();
    ck(cudaStreamWaitEvent(st_, ev_q_, 0), "q wait");
    q_pending_ = false;
  }
  // Near field: side stream, overlapped with the far-field chain; in the
  // sequential mode (set_overlap off) it runs after L2T, inside phase_near.
  if (overlap_) near_start();
  if (!t_first) build_T();
  cudaEventRecord(ev_[1], st_);
  phase_c2m();
  cudaEventRecord(ev_[2], st_);
  if (overlap) {
    ck(cudaEventRecord(ev_c2m_, st_), "c2m");
    ck(cudaStreamWaitEvent(st_lo_, ev_c2m_, 0), "c2m wait");
    cudaStream_t keep = st_;
    st_ = st_lo_;
    cudaEventRecord(ev_lf0_, st_);
    phase_m2l(s_.L, s_.L);
    cudaEventRecord(ev_lf1_, st_);
    ck(cudaEventRecord(ev_m2l_leaf_, st_), "m2l leaf");
    st_ = keep;
  }
  phase_m2m();
  cudaEventRecord(ev_[3], st_);
  if (overlap) {
    phase_m2l(s_.top, s_.L - 1);
    cudaEventRecord(ev_[4], st_);
    phase_l2l(s_.top, s_.L - 2);
    cudaEventRecord(ev_la_, st_);
    ck(cudaStreamWaitEvent(st_, ev_m2l_leaf_, 0), "m2l leaf wait");
    cudaEventRecord(ev_lb_, st_);
    phase_l2l(s_.L - 1, s_.L - 1);
  } else {
    phase_m2l();
    cudaEventRecord(ev_[4], st_);
    phase_l2l();
  }
  cudaEventRecord(ev_[5], st_);
  phase_l2t();
  cudaEventRecord(ev_[6], st_);
  phase_near();
  cudaEventRecord(ev_[7], st_);
  if (overlap) {
    ck(cudaEventRecord(ev_ojoin_, st_), "join");
    ck(cudaStreamWaitEvent(user, ev_ojoin_, 0), "join wait");
    st_ = user;
  }
  if (d_pot_sorted)
    ck(cudaMemcpyAsync(d_pot_sorted, d_pot, size_t(n) * sizeof(double2), cudaMemcpyDeviceToDevice, st_), "pot");
  last_launches_ = launches_ - l0;
  timed_ = true;
  st_ = saved;
}

void Engine::evaluate_host(const double* q_in, double* pot_out, double* ms) {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  if (dist_)
    throw std::logic_error(
        "evaluate: num_ranks > 1 needs the exchanges of the distributed driver "
        "(paper_2006_15367_b200.distributed)");
  if (q_in) {
    // charges H2D + Morton gather on the copy stream; evaluate_device builds
    // T meanwhile and joins before the first phase that reads them
    const int64_t n = int64_t(s_.n);
    // d_q_in / d_q may still be in use by work already queued on st_ (and,
    // through st_'s joins, on the side streams): order the copy after it.
    ck(cudaEventRecord(ev_cp_order_, st_), "cp order");
    ck(cudaStreamWaitEvent(st_cp_, ev_cp_order_, 0), "cp order wait");
    ck(cudaMemcpyAsync(d_q_in, q_in, size_t(n) * sizeof(double2), cudaMemcpyHostToDevice, st_cp_), "H2D q");
    k_gather_q<<<unsigned((n + 255) / 256), 256, 0, st_cp_>>>(n, d_orig, d_q_in, d_q);
    ++launches_;
    ck(cudaGetLastError(), "k_gather_q");
    ck(cudaEventRecord(ev_q_, st_cp_), "q ready");
    q_pending_ = true;
  }
  evaluate_device(nullptr, nullptr, nullptr);
  const int64_t cnt = part_e_ - part_b_;
  if (cnt > 0) {
    k_scatter_pot<<<unsigned((cnt + 255) / 256), 256, 0, st_>>>(part_b_, part_e_, d_orig, d_pot, d_pot_in);
    ++launches_;
  }
  ck(cudaGetLastError(), "scatter");
  if (s_.P == 1) {
    ck(cudaMemcpyAsync(pot_out, d_pot_in, s_.n * sizeof(double2), cudaMemcpyDeviceToHost, st_), "D2H pot");
  } else {
    throw std::logic_error("evaluate_host: multi-rank gather not supported here");
  }
  ck(cudaStreamSynchronize(st_), "evaluate_host");
  if (ms) last_timing(ms, nullptr);
}

void Engine::get_expansion(int kind, int level, double* out, size_t cap) {
  if (level < s_.top || level > s_.L) throw std::out_of_range("get_expansion: level not computed");
  const DevLevel& d = lv_[size_t(level)];
  const size_t cnt = size_t(d.n_nodes) * size_t(d.S) * 2;
  if (cap < cnt) throw std::invalid_argument("get_expansion: buffer too small");
  ck(cudaStreamSynchronize(st_), "sync");
  const double2* src = kind == 0 ? d.mp : d.loc;
  if (rows_.empty()) {
    ck(cudaMemcpy(out, src, cnt * sizeof(double), cudaMemcpyDeviceToHost), "D2H exp");
    return;
  }
  // distributed mode: rows -> node order; nodes not stored here read as zero
  std::vector<double2> tmp(size_t(d.n_rows) * size_t(d.S));
  ck(cudaMemcpy(tmp.data(), src, tmp.size() * sizeof(double2), cudaMemcpyDeviceToHost), "D2H exp");
  std::memset(out, 0, cnt * sizeof(double));
  for (int n = 0; n < d.n_nodes; ++n) {
    const int r = row(level, n);
    if (r >= 0) std::memcpy(out + size_t(n) * size_t(d.S) * 2, tmp.data() + size_t(r) * size_t(d.S), size_t(d.S) * 16);
  }
}

void Engine::get_potentials_sorted(double* out, size_t cap) {
  if (cap < 2 * s_.n) throw std::invalid_argument("get_potentials_sorted: buffer too small");
  ck(cudaStreamSynchronize(st_), "sync");
  ck(cudaMemcpy(out, d_pot, s_.n * sizeof(double2), cudaMemcpyDeviceToHost), "D2H pot");
}


void Engine::store_potentials_host(double* host_sorted) {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  ck(cudaStreamSynchronize(st_), "sync");
  if (part_e_ > part_b_)
    ck(cudaMemcpy(host_sorted + 2 * part_b_, d_pot + part_b_, size_t(part_e_ - part_b_) * sizeof(double2),
                  cudaMemcpyDeviceToHost),
       "D2H pot");
}

void Engine::upload_rank_plan() {
  const Setup& s = s_;
  const int L = s.L, P = s.P;
  const RankPlan& rp = *rp_;
  // Every index the kernels see is a ROW of the compact per-rank storage.
  auto rows_of = [&](int l, const std::vector<int>& nodes) {
    std::vector<int> v(nodes.size());
    for (size_t i = 0; i < nodes.size(); ++i) v[i] = row(l, nodes[i]);
    return v;
  };
  rl_.assign(size_t(L + 1), RankLevel{});
  for (int l = s.top; l < L; ++l) {
    RankLevel& R = rl_[size_t(l)];
    R.n_par = int(rp.held[size_t(l)].size());
    R.plist = upload_vec(rows_of(l, rp.held[size_t(l)]));  // 0..H-1
    R.child_off = upload_vec(rp.child_off[size_t(l)]);
    R.children = upload_vec(rows_of(l + 1, rp.children[size_t(l)]));
    R.n_children = int64_t(rp.children[size_t(l)].size());
  }
  held_.assign(size_t(L + 1), nullptr);
  held_cnt_.assign(size_t(L + 1), 0);
  for (int l = s.top; l <= L; ++l) {
    held_cnt_[size_t(l)] = int(rp.held[size_t(l)].size());
    held_[size_t(l)] = upload_vec(rows_of(l, rp.held[size_t(l)]));
    DevLevel& d = lv_[size_t(l)];
    if (d.dense) {  // the 8^3 observer blocks (Morton subtrees) holding held nodes
      const int nb = (d.G + m2l::MB - 1) / m2l::MB;
      std::vector<int> blk;
      for (int node : rp.held[size_t(l)]) {
        const uint64_t c = s.levels[size_t(l)].codes[size_t(node)];
        blk.push_back((int(cell_axis(c, l, 2)) / m2l::MB * nb + int(cell_axis(c, l, 1)) / m2l::MB) * nb +
                      int(cell_axis(c, l, 0)) / m2l::MB);
      }
      std::sort(blk.begin(), blk.end());
      blk.erase(std::unique(blk.begin(), blk.end()), blk.end());
      d.m2l_nblk = int(blk.size());
      d.m2l_blk = upload_vec(blk);
    }
  }
  peers_.assign(size_t(P), PeerPlan{});
  for (int q = 0; q < P; ++q) {
    if (q == rank_) continue;
    PeerPlan& pp = peers_[size_t(q)];
    for (int kind : {int(kXHalo), int(kXReduce), int(kXGather)})
      for (int dir = 0; dir < 2; ++dir) {
        const std::vector<RowItem>& items = dir == 0 ? rp.send[kind][size_t(q)] : rp.recv[kind][size_t(q)];
        RowXfer& x = dir == 0 ? pp.send[kind] : pp.recv[kind];
        x.items.assign(size_t(L + 1), nullptr);
        x.cnt.assign(size_t(L + 1), 0);
        x.len.assign(size_t(L + 1), 0);
        x.maxlen.assign(size_t(L + 1), 0);
        std::vector<std::vector<int64_t>> per(size_t(L + 1));
        for (const RowItem& it : items) {  // (level, node, begin) order
          auto& v = per[size_t(it.level)];
          const int64_t len = it.end - it.begin;
          const int r = row(it.level, it.node);
          if (r < 0) throw std::logic_error("exchange plan: node not stored on this rank");
          v.insert(v.end(), {int64_t(r), it.begin, len, x.len[size_t(it.level)]});
          x.len[size_t(it.level)] += len;
          x.maxlen[size_t(it.level)] = std::max(x.maxlen[size_t(it.level)], len);
        }
        for (int l = s.top; l <= L; ++l) {
          x.cnt[size_t(l)] = int(per[size_t(l)].size() / 4);
          if (x.cnt[size_t(l)]) x.items[size_t(l)] = upload_vec(per[size_t(l)]);
          x.total += x.len[size_t(l)];
        }
      }
    // ghosts: leaves r owns that q needs, and leaves q owns that r needs (comm_plan.cpp:84-109)
    for (int dir = 0; dir < 2; ++dir) {
      const auto& leaves = dir == 0 ? s.near_send[size_t(rank_) * P + size_t(q)] : s.near_send[size_t(q) * P + size_t(rank_)];
      std::vector<int64_t> idx;
      for (uint64_t li : leaves)
        for (uint64_t p = s.leaf_start[li]; p < s.leaf_start[li + 1]; ++p) idx.push_back(int64_t(p));
      (dir == 0 ? pp.n_gh_send : pp.n_gh_recv) = int64_t(idx.size());
      (dir == 0 ? pp.gh_send_idx : pp.gh_recv_idx) = upload_vec(idx);
    }
  }
}

namespace {
void check_level(int level, int top, int L) {
  if (level != -1 && (level < top || level > L)) throw std::out_of_range("exchange: level not computed");
}
}  // namespace

void Engine::exchange_sizes(int kind, int peer, int level, int64_t* send_d, int64_t* recv_d) const {
  if (!dist_) throw std::logic_error("exchange: single-rank engine");
  if (peer < 0 || peer >= s_.P || peer == rank_) throw std::out_of_range("exchange: bad peer");
  const PeerPlan& pp = peers_[size_t(peer)];
  if (kind == kXGhost) {
    *send_d = 5 * pp.n_gh_send;
    *recv_d = 5 * pp.n_gh_recv;
    return;
  }
  if (kind != kXHalo && kind != kXReduce && kind != kXGather) throw std::invalid_argument("exchange: bad kind");
  check_level(level, s_.top, s_.L);
  const RowXfer& sx = pp.send[kind];
  const RowXfer& rx = pp.recv[kind];
  *send_d = 2 * (level < 0 ? sx.total : sx.len[size_t(level)]);
  *recv_d = 2 * (level < 0 ? rx.total : rx.len[size_t(level)]);
}

void Engine::pack(int kind, int peer, int level, double* d_buf) {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  int64_t sd = 0, rd = 0;
  exchange_sizes(kind, peer, level, &sd, &rd);
  const PeerPlan& pp = peers_[size_t(peer)];
  if (kind == kXGhost) {
    if (pp.n_gh_send > 0) {
      k_pack_particles<<<unsigned((pp.n_gh_send + 255) / 256), 256, 0, st_>>>(pp.n_gh_send, pp.gh_send_idx, d_x, d_y,
                                                                             d_z, d_q, d_buf);
      ++launches_;
    }
  } else {
    const RowXfer& x = pp.send[kind];
    double2* buf = reinterpret_cast<double2*>(d_buf);
    for (int l = level < 0 ? s_.top : level; l <= (level < 0 ? s_.L : level); ++l) {
      if (x.cnt[size_t(l)] > 0) {
        const DevLevel& d = lv_[size_t(l)];
        dim3 grid(unsigned(x.cnt[size_t(l)]), unsigned(std::min<int64_t>((x.maxlen[size_t(l)] + 255) / 256, 64)));
        k_pack_items<<<grid, 256, 0, st_>>>(kind == kXGather ? d.loc : d.mp, d.S, x.items[size_t(l)], buf);
        ++launches_;
      }
      buf += x.len[size_t(l)];
    }
  }
  ck(cudaGetLastError(), "pack");
}

void Engine::unpack(int kind, int peer, int level, const double* d_buf) {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  int64_t sd = 0, rd = 0;
  exchange_sizes(kind, peer, level, &sd, &rd);
  const PeerPlan& pp = peers_[size_t(peer)];
  if (kind == kXGhost) {
    if (pp.n_gh_recv > 0) {
      k_unpack_particles<<<unsigned((pp.n_gh_recv + 255) / 256), 256, 0, st_>>>(pp.n_gh_recv, pp.gh_recv_idx, d_buf,
                                                                               d_x, d_y, d_z, d_q);
      ++launches_;
    }
  } else {
    const RowXfer& x = pp.recv[kind];
    const double2* buf = reinterpret_cast<const double2*>(d_buf);
    for (int l = level < 0 ? s_.top : level; l <= (level < 0 ? s_.L : level); ++l) {
      if (x.cnt[size_t(l)] > 0) {
        DevLevel& d = lv_[size_t(l)];
        dim3 grid(unsigned(x.cnt[size_t(l)]), unsigned(std::min<int64_t>((x.maxlen[size_t(l)] + 255) / 256, 64)));
        if (kind == kXReduce)  // partial sums of the peer, added in the caller's (rank) order
          k_unpack_items<true><<<grid, 256, 0, st_>>>(d.mp, d.S, x.items[size_t(l)], buf);
        else
          k_unpack_items<false><<<grid, 256, 0, st_>>>(kind == kXGather ? d.loc : d.mp, d.S, x.items[size_t(l)], buf);
        ++launches_;
      }
      buf += x.len[size_t(l)];
    }
  }
  ck(cudaGetLastError(), "unpack");
}

void Engine::run_level(int phase, int level) {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  if (phase == HFMM_PHASE_M2L) {
    if (level < s_.top || level > s_.L) throw std::out_of_range("run_level: M2L level not computed");
    phase_m2l(level, level);
  } else if (phase == HFMM_PHASE_L2L) {
    if (level < s_.top || level >= s_.L) throw std::out_of_range("run_level: L2L parent level not computed");
    phase_l2l(level, level);
  } else {
    throw std::invalid_argument("run_level: phase must be M2L or L2L");
  }
  ck(cudaGetLastError(), "run_level");
}

void Engine::set_stream(cudaStream_t st) {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  ck(cudaStreamSynchronize(st_), "sync");
  if (owns_stream_) cudaStreamDestroy(st_);
  owns_stream_ = st == nullptr;
  if (st == nullptr)
    ck(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "stream");
  else
    st_ = st;
}

void Engine::synchronize() {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  ck(cudaStreamSynchronize(st_), "sync");
}

void Engine::load_charges_device(const double* d_q_sorted) {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  const int64_t b = dist_ ? part_b_ : 0, e = dist_ ? part_e_ : int64_t(s_.n);
  if (e > b)
    ck(cudaMemcpyAsync(d_q + b, reinterpret_cast<const double2*>(d_q_sorted) + b, size_t(e - b) * sizeof(double2),
                       cudaMemcpyDeviceToDevice, st_),
       "charges");
}

void Engine::store_potentials_device(double* d_pot_sorted) {
  ck(cudaSetDevice(dev_), "cudaSetDevice");
  const int64_t b = dist_ ? part_b_ : 0, e = dist_ ? part_e_ : int64_t(s_.n);
  if (e > b)
    ck(cudaMemcpyAsync(reinterpret_cast<double2*>(d_pot_sorted) + b, d_pot + b, size_t(e - b) * sizeof(double2),
                       cudaMemcpyDeviceToDevice, st_),
       "potentials");
}

void direct_sum(const double* positions, const double* charges, size_t n, const int64_t* obs,
                size_t m, double k, int device, double* pot_out) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw std::runtime_error("no CUDA device available (the engine has no CPU fallback)");
    auto ck = [](cudaError_t e, const char* w) {
      if (e != cudaSuccess) throw std::runtime_error(std::string(w) + ": " + cudaGetErrorString(e));
    };
    ck(cudaSetDevice(device), "cudaSetDevice");
    for (size_t i = 0; i < m; ++i)
      if (obs[i] < 0 || size_t(obs[i]) >= n) throw std::out_of_range("hfmm_gpu_direct: observer index");
    std::vector<double> x(n), y(n), z(n);
    for (size_t i = 0; i < n; ++i) {
      x[i] = positions[3 * i];
      y[i] = positions[3 * i + 1];
      z[i] = positions[3 * i + 2];
    }
    double *dx, *dy, *dz;
    double2 *dq, *dout;
    int64_t* dobs;
    int* derr;
    ck(cudaMalloc(&dx, n * 8), "malloc");
    ck(cudaMalloc(&dy, n * 8), "malloc");
    ck(cudaMalloc(&dz, n * 8), "malloc");
    ck(cudaMalloc(&dq, n * 16), "malloc");
    ck(cudaMalloc(&dout, m * 16 + 16), "malloc");
    ck(cudaMalloc(&dobs, m * 8 + 8), "malloc");
    ck(cudaMalloc(&derr, sizeof(int)), "malloc");
    cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, y.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dz, z.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dq, charges, n * 16, cudaMemcpyHostToDevice);
    cudaMemcpy(dobs, obs, m * 8, cudaMemcpyHostToDevice);
    cudaMemset(derr, 0, sizeof(int));
    if (m > 0) k_direct<<<unsigned(m), 256>>>(int64_t(n), dx, dy, dz, dq, dobs, k, dout, derr);
    cudaError_t le = cudaGetLastError();
    int err = 0;
    cudaMemcpy(&err, derr, sizeof(int), cudaMemcpyDeviceToHost);
    cudaError_t e2 = cudaMemcpy(pot_out, dout, m * 16, cudaMemcpyDeviceToHost);
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(dz);
    cudaFree(dq);
    cudaFree(dout);
    cudaFree(dobs);
    cudaFree(derr);
    ck(le, "k_direct");
    ck(e2, "k_direct D2H");
    if (err) throw std::domain_error("direct_potential: coincident source and observer");
}

}  // namespace hfmm_b200
