// Fused M2M for the leaf-side level pair (18, 28) of the BASELINE cubes
// (configs 1, 3, 4 leaf level): one CTA per parent (persistent over parents),
// both passes of the separable resampling in one kernel with the folded
// circles F of the phi pass in SHARED memory -- they never touch HBM (the
// two-kernel streaming form, interp_rb.cuh, writes and re-reads them: 27.8 GB
// + 25.9 GB per evaluation at config 4; fused, the kernel moves the compulsory
// 14.2 GB).  Same algebra and the same device helpers as interp_rb.cuh (real +
// rank-1 matrices on DMMA, complex-row warp tiles, child sum as a
// reduce-scatter); traversal.cpp:322-429, sphere_grid.cpp:183-192.  Each CTA
// prefetches its NEXT parent's children into L2 with the Blackwell bulk-copy
// engine (cp.async.bulk.prefetch.L2, bulk.cuh) while the current parent
// computes.  (The mirrored fused L2L measured 1.3 ms slower than the
// two-kernel form at config 4 and was dropped.)
#ifndef HFMM_B200_INTERP_FUSED_CUH
#define HFMM_B200_INTERP_FUSED_CUH

#include "bulk.cuh"
#include "interp_rb.cuh"

namespace hfmm_b200 {
namespace fz {

constexpr int kThreads = 224;  // 7 warps: the 14 theta circles of a parent split evenly
__host__ __device__ constexpr int pad4mod8(int x) { return x + ((4 - x % 8) + 8) % 8; }  // stride == 4 (mod 8) double2

template <int NC, int NP>
struct Lay {
  using D = rb::Dims<NC, NP>;
  // M2M: F[c][p][..] (c = child slot, p < HALF; x_e at [0, NC), x_o at [4 UTH_KH, ..)), child stride CSF
  static constexpr int CSF = pad4mod8(D::HALF * D::LDF);
  static constexpr int BPHI = D::UPHI_K * D::UPHI_LDB, BTH = D::UTH_K * D::UTH_LDB;  // doubles
  static constexpr int M2M_SMEM = (BPHI + BTH) * 8 + 8 * CSF * 16;
};

// L2 prefetch of a parent's children block (children of a parent are
// consecutive nodes, so their expansions are one contiguous block).
__device__ __forceinline__ void prefetch_children(int par, int n_par, const int* __restrict__ child_off,
                                                  const int* __restrict__ children, const double2* base, int S) {
  if (par >= n_par) return;
  const int cb = child_off[par], n = child_off[par + 1] - cb;
  if (n <= 0) return;
  const int c0 = children[cb];
  if (children[cb + n - 1] - c0 != n - 1) return;  // not contiguous: no hint
  bulk::prefetch_l2(base + int64_t(c0) * S, uint32_t(n) * uint32_t(S) * 16u);
}

}  // namespace fz

template <int NC, int NP>
__global__ void __launch_bounds__(fz::kThreads, 2) k_m2m_fz(int n_par, const int* __restrict__ plist,
                                                            const int* __restrict__ child_off,
                                                            const int* __restrict__ children,
                                                            const uint8_t* __restrict__ oct_c,
                                                            const double2* __restrict__ mp_c,
                                                            const double* __restrict__ Bphi,
                                                            const double* __restrict__ vphi,
                                                            const double* __restrict__ Bth,
                                                            const double* __restrict__ vth,
                                                            const double2* __restrict__ shift_up,
                                                            double2* __restrict__ mp_p) {
  using D = rb::Dims<NC, NP>;
  using Y = fz::Lay<NC, NP>;
  constexpr int KSP = D::UPHI_K / 4, NTP = D::UPHI_N / 8;
  constexpr int HALF = D::HALF, SP = D::SP, SC = D::SC;
  extern __shared__ __align__(16) double fz_smem[];
  double* Bp = fz_smem;
  double* Bt = Bp + Y::BPHI;
  double2* Fs = reinterpret_cast<double2*>(Bt + Y::BTH);
  rb::stage_b<D::UPHI_K, D::UPHI_N, D::UPHI_LDB>(Bp, Bphi);
  rb::stage_b<D::UTH_K, D::UTH_N, D::UTH_LDB>(Bt, Bth);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  constexpr int NW = fz::kThreads / 32;
  for (int par = blockIdx.x; par < n_par; par += gridDim.x) {
    const int cb = child_off[par], nch = child_off[par + 1] - cb;
    if (threadIdx.x == 0) fz::prefetch_children(par + gridDim.x, n_par, child_off, children, mp_c, SC);
    // phi pass: rows (child c, theta row i) -> folded circles in shared memory
    const int rows = nch * NC, tiles = (rows + 7) / 8;
    for (int t = warp; t < tiles; t += NW) {
      const int R = t * 8 + g;
      const bool ok = R < rows;
      const int c = ok ? R / NC : 0, i = ok ? R - c * NC : 0;
      const double2* x = mp_c + int64_t(children[cb + c]) * SC + i * NC;
      double are[KSP], aim[KSP];
#pragma unroll
      for (int kk = 0; kk < KSP; ++kk) {
        const int k = 4 * kk + tq;
        const double2 xv = (ok && k < NC) ? __ldg(x + k) : make_double2(0.0, 0.0);
        are[kk] = xv.x;
        aim[kk] = xv.y;
      }
      rb::rank1_inject<KSP, NC>(are, aim, vphi);
      double cre[NTP][2] = {}, cim[NTP][2] = {};
      rb::tile_mma<KSP, NTP, D::UPHI_LDB>(are, aim, Bp, cre, cim);
      if (ok) {
        double2* Fc = Fs + c * Y::CSF;
#pragma unroll
        for (int jn = 0; jn < NTP; ++jn)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = 8 * jn + 2 * tq + q;  // column 2 p + h: circle p, part e / o
            if (n < NP) Fc[(n >> 1) * D::LDF + (n & 1) * 4 * D::UTH_KH + i] = make_double2(cre[jn][q], cim[jn][q]);
          }
      }
    }
    __syncthreads();
    // theta pass + shift + child sum: item = circle p, tile rows = child slots
    const bool ok = g < nch;
    const double2* sh = shift_up + int64_t(ok ? oct_c[children[cb + g]] : 0) * SP;
    double2* out = mp_p + int64_t(plist ? plist[par] : par) * SP;
    for (int p = warp; p < HALF; p += NW) {
      const double2* frow = Fs + (ok ? g : 0) * Y::CSF + p * D::LDF;
      rb::m2m_theta_item<NC, NP>([&](int k) { return frow[k]; }, ok, sh, out, p, Bt, vth);
    }
    __syncthreads();
  }
}

// Pairs served by the fused kernel (two CTAs per SM fit its shared memory).
inline bool fz_pair(int nc, int np) { return nc == 18 && np == 28; }

inline void launch_m2m_fz(const RbLaunch& L, int sms, const double2* mp_c, double2* mp_p, const double* Bphi,
                          const double* vphi, const double* Bth, const double* vth, const double2* shift_up) {
  constexpr int smem = fz::Lay<18, 28>::M2M_SMEM;
  cudaFuncSetAttribute(k_m2m_fz<18, 28>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = std::min(L.n_par, 2 * sms);
  k_m2m_fz<18, 28><<<grid, fz::kThreads, smem, L.st>>>(L.n_par, L.plist, L.child_off, L.children, L.oct_c, mp_c, Bphi,
                                                       vphi, Bth, vth, shift_up, mp_p);
}


// ---------------------------------------------------------------------------
// Version 2 of the fused (18, 28) M2M: one CTA per SM, 14 warps, and NO global
// load inside the two passes.  The children of a parent arrive as bulk
// asynchronous copies (cp.async.bulk, mbarrier completion) into a
// double-buffered shared-memory block, issued a whole parent ahead; the shift
// factors come from a quarter table in shared memory (the sphere grid's
// symmetries theta -> pi - theta and phi -> phi + pi map a sample of octant o
// to the mirrored sample of octant o ^ 4 / o ^ 3, so rows < NP / 2 and columns
// < NP / 2 of the 8 octant tables suffice: 25 KB instead of 100 KB); the rank-1
// vectors sit in shared memory as well.  ncu on the first version showed
// long-scoreboard stalls on the child and shift loads at 14 warps per SM
// (43% tensor pipe); here both passes read shared memory only.
namespace fz2 {

constexpr int kWarps = 14, kThreads = 32 * kWarps;

template <int NC, int NP>
struct Lay {
  using D = rb::Dims<NC, NP>;
  static constexpr int H = NP / 2, SC = NC * NC;
  // folded circles: x_e at [0, NC), x_o at [4 KH, 4 KH + NC) of a row of LDF
  // complex; LDF == 2 (mod 8) spreads the phi pass's 16-byte stores over the banks
  static constexpr int LDF = D::UTH_K + 2;
  static constexpr int CSF = fz::pad4mod8(H * LDF);
  static constexpr int BPHI = D::UPHI_K * D::UPHI_LDB, BTH = D::UTH_K * D::UTH_LDB;  // doubles
  static constexpr int VPHI = D::UPHI_K, VTH = D::UTH_K;                               // doubles
  static constexpr int SHROW = H + 1, SHOCT = H * SHROW + 1;                           // double2 (padded)
  static constexpr int OFF_SH = (BPHI + BTH + VPHI + VTH) * 8;
  static constexpr int OFF_F = OFF_SH + 8 * SHOCT * 16;
  static constexpr int OFF_CH = OFF_F + 8 * CSF * 16;
  static constexpr int OFF_BAR = OFF_CH + 2 * 8 * SC * 16;
  static constexpr int SMEM = OFF_BAR + 16;
  static_assert(OFF_SH % 16 == 0 && H % 2 == 0, "layout");
};

}  // namespace fz2

template <int NC, int NP>
__global__ void __launch_bounds__(fz2::kThreads, 1) k_m2m_fz2(int n_par, const int* __restrict__ plist,
                                                              const int* __restrict__ child_off,
                                                              const int* __restrict__ children,
                                                              const uint8_t* __restrict__ oct_c,
                                                              const double2* __restrict__ mp_c,
                                                              const double* __restrict__ Bphi,
                                                              const double* __restrict__ vphi,
                                                              const double* __restrict__ Bth,
                                                              const double* __restrict__ vth,
                                                              const double2* __restrict__ shift_up,
                                                              double2* __restrict__ mp_p) {
  using D = rb::Dims<NC, NP>;
  using Y = fz2::Lay<NC, NP>;
  constexpr int KSP = D::UPHI_K / 4, HALF = D::HALF, SP = D::SP, SC = D::SC, H = Y::H;
  constexpr int NW = fz2::kWarps;
  extern __shared__ __align__(16) unsigned char fz2_smem[];
  double* Bp = reinterpret_cast<double*>(fz2_smem);
  double* Bt = Bp + Y::BPHI;
  double* vp = Bt + Y::BTH;
  double* vt = vp + Y::VPHI;
  double2* shq = reinterpret_cast<double2*>(fz2_smem + Y::OFF_SH);
  double2* Fs = reinterpret_cast<double2*>(fz2_smem + Y::OFF_F);
  double2* Ch = reinterpret_cast<double2*>(fz2_smem + Y::OFF_CH);
  uint64_t* bar = reinterpret_cast<uint64_t*>(fz2_smem + Y::OFF_BAR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;

  // children of parent `par` -> buffer b (one bulk copy per child: rows need not be contiguous)
  auto issue = [&](int par, int b) {
    const int cb = child_off[par], n = child_off[par + 1] - cb;
    bulk::mbar_expect_tx(bar + b, uint32_t(n) * uint32_t(SC) * 16u);
    for (int c = 0; c < n; ++c)
      bulk::copy_g2s(Ch + (b * 8 + c) * SC, mp_c + int64_t(children[cb + c]) * SC, uint32_t(SC) * 16u, bar + b);
  };
  if (threadIdx.x == 0) {
    bulk::mbar_init(bar, 1);
    bulk::mbar_init(bar + 1, 1);
    bulk::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && int(blockIdx.x) < n_par) issue(blockIdx.x, 0);
  for (int t = threadIdx.x; t < Y::VPHI; t += blockDim.x) vp[t] = t < NC ? vphi[t] : 0.0;
  for (int t = threadIdx.x; t < Y::VTH; t += blockDim.x) vt[t] = vth[t];
  for (int t = threadIdx.x; t < 8 * H * H; t += blockDim.x) {
    const int o = t / (H * H), r = t - o * H * H, n = r / H, pc = r - n * H;
    shq[o * Y::SHOCT + n * Y::SHROW + pc] = shift_up[int64_t(o) * SP + n * NP + pc];
  }
  rb::stage_b<D::UPHI_K, D::UPHI_N, D::UPHI_LDB>(Bp, Bphi);
  rb::stage_b<D::UTH_K, D::UTH_N, D::UTH_LDB>(Bt, Bth);  // (ends with a CTA barrier)

  int it = 0;
  for (int par = blockIdx.x; par < n_par; par += gridDim.x, ++it) {
    const int b = it & 1;
    const int cb = child_off[par], nch = child_off[par + 1] - cb;
    // buffer b ^ 1 was last read by the phi pass of the previous parent, which
    // every warp left before that parent's theta pass
    if (threadIdx.x == 0 && par + int(gridDim.x) < n_par) issue(par + gridDim.x, b ^ 1);
    bulk::mbar_wait(bar + b, uint32_t(it >> 1) & 1u);
    const double2* ch = Ch + b * 8 * SC;
    // phi pass: item = (row tile, half of the output columns) -> folded circles
    const int rows = nch * NC, tiles = (rows + 7) / 8;
    for (int item = warp; item < 2 * tiles; item += NW) {
      const int t = item >> 1, hh = item & 1;
      const int R = t * 8 + g;
      const bool ok = R < rows;
      const int c = ok ? R / NC : 0, i = ok ? R - c * NC : 0;
      const double2* x = ch + c * SC + i * NC;
      double are[KSP], aim[KSP];
#pragma unroll
      for (int kk = 0; kk < KSP; ++kk) {
        const int k = 4 * kk + tq;
        const double2 xv = (ok && k < NC) ? x[k] : make_double2(0.0, 0.0);
        are[kk] = xv.x;
        aim[kk] = xv.y;
      }
      rb::rank1_inject_f<KSP, NC>(are, aim, [&](int k) { return vp[k]; });
      constexpr int NTH = D::UPHI_N / 16;  // n8 tiles per half
      static_assert(D::UPHI_N % 16 == 0, "phi output tiles split in two halves");
      double cre[NTH][2] = {}, cim[NTH][2] = {};
      rb::tile_mma<KSP, NTH, D::UPHI_LDB>(are, aim, Bp + 8 * NTH * hh, cre, cim);
      if (ok) {
        double2* Fc = Fs + c * Y::CSF;
#pragma unroll
        for (int jn = 0; jn < NTH; ++jn)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = 8 * (NTH * hh + jn) + 2 * tq + q;  // column 2 p + h: circle p, part e / o
            if (n < NP) Fc[(n >> 1) * Y::LDF + (n & 1) * 4 * D::UTH_KH + i] = make_double2(cre[jn][q], cim[jn][q]);
          }
      }
    }
    __syncthreads();
    // theta pass + shift + child sum: item = circle p, tile rows = child slots
    const bool ok = g < nch;
    const int oct = ok ? oct_c[children[cb + g]] : 0;
    double2* out = mp_p + int64_t(plist ? plist[par] : par) * SP;
    for (int p = warp; p < HALF; p += NW) {
      const double2* frow = Fs + (ok ? g : 0) * Y::CSF + p * Y::LDF;
      rb::m2m_theta_item_f<NC, NP>(
          [&](int k) { return frow[k]; }, ok,
          [&](int n, int back) {
            const int up = n >= H;  // mirrored theta row: octant with z flipped
            const int o = oct ^ (up ? 4 : 0) ^ (back ? 3 : 0);
            return shq[o * Y::SHOCT + (up ? NP - 1 - n : n) * Y::SHROW + p];
          },
          out, p, Bt, [&](int k) { return vt[k]; });
    }
    __syncthreads();
  }
}

inline void launch_m2m_fz2(const RbLaunch& L, int sms, const double2* mp_c, double2* mp_p, const double* Bphi,
                           const double* vphi, const double* Bth, const double* vth, const double2* shift_up) {
  constexpr int smem = fz2::Lay<18, 28>::SMEM;
  static_assert(smem <= 227 * 1024, "fused M2M v2 shared memory");
  cudaFuncSetAttribute(k_m2m_fz2<18, 28>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = std::min(L.n_par, sms);
  k_m2m_fz2<18, 28><<<grid, fz2::kThreads, smem, L.st>>>(L.n_par, L.plist, L.child_off, L.children, L.oct_c, mp_c, Bphi,
                                                         vphi, Bth, vth, shift_up, mp_p);
}

// ---------------------------------------------------------------------------
// Fused (18, 28) L2L, same construction (traversal.cpp:583-707,
// sphere_grid.cpp:194-214): the parent local arrives by bulk copies (one per
// theta row, into rows padded for conflict-free fragment loads), one parent
// ahead; the theta pass (even / odd form) reads it and the quarter shift table
// from shared memory and leaves the narrow rows (Ye, Yo pairs) in shared
// memory; the phi pass adds into the child locals, whose old values it loads
// at the top of each work item (the children block was pulled into L2 by a
// bulk prefetch while the previous parent computed).  The two-kernel form
// writes and re-reads the narrow rows through HBM (20 + 41 GB per evaluation
// at config 4); fused, the kernel moves the parent locals once and the child
// locals twice (read-add-write).
namespace fz2 {

template <int NC, int NP>
struct LayD {
  using D = rb::Dims<NC, NP>;
  static constexpr int H = NP / 2, SC = NC * NC;
  static constexpr int BTH = D::DTH_K * D::DTH_LDB, BPHI = D::DPHI_K * D::DPHI_LDB;  // doubles
  static constexpr int VTH = D::DTH_K, VPHI = D::DPHI_K;
  static constexpr int SHROW = H + 4, SHOCT = H * SHROW;  // double2; row stride == 2 (mod 8)
  static constexpr int LROW = NP + 2;                     // parent local row stride == 6 (mod 8)
  static constexpr int LDN = fz::pad4mod8(D::DPHI_K);     // narrow-row stride == 4 (mod 8)
  static constexpr int OFF_SH = (BTH + BPHI + VTH + VPHI) * 8;
  static constexpr int OFF_L = OFF_SH + 8 * SHOCT * 16;
  static constexpr int OFF_NB = OFF_L + 2 * NP * LROW * 16;
  static constexpr int OFF_BAR = OFF_NB + 8 * NC * LDN * 16;
  static constexpr int SMEM = OFF_BAR + 16;
  static_assert(OFF_SH % 16 == 0 && SHROW % 8 == 2 && LROW % 8 == 6, "layout");
};

}  // namespace fz2

template <int NC, int NP>
__global__ void __launch_bounds__(fz2::kThreads, 1) k_l2l_fz2(int n_par, const int* __restrict__ plist,
                                                              const int* __restrict__ child_off,
                                                              const int* __restrict__ children,
                                                              const uint8_t* __restrict__ oct_c,
                                                              const double2* __restrict__ loc_p,
                                                              const double* __restrict__ Bth,
                                                              const double* __restrict__ vth,
                                                              const double* __restrict__ Bphi,
                                                              const double* __restrict__ vphi,
                                                              const double2* __restrict__ shift_dn,
                                                              double2* __restrict__ loc_c) {
  using D = rb::Dims<NC, NP>;
  using Y = fz2::LayD<NC, NP>;
  constexpr int KH = D::DTH_KH, NT = D::DTH_N / 8, HALF = D::HALF, SP = D::SP, SC = D::SC, H = Y::H;
  constexpr int KSP = D::DPHI_K / 4, NTP = D::DPHI_N / 8;
  constexpr int NW = fz2::kWarps;
  extern __shared__ __align__(16) unsigned char fz2_smem[];
  double* Bt = reinterpret_cast<double*>(fz2_smem);
  double* Bp = Bt + Y::BTH;
  double* vt = Bp + Y::BPHI;
  double* vp = vt + Y::VTH;
  double2* shq = reinterpret_cast<double2*>(fz2_smem + Y::OFF_SH);
  double2* Ls = reinterpret_cast<double2*>(fz2_smem + Y::OFF_L);
  double2* Nbs = reinterpret_cast<double2*>(fz2_smem + Y::OFF_NB);
  uint64_t* bar = reinterpret_cast<uint64_t*>(fz2_smem + Y::OFF_BAR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;

  // parent local of `par` -> buffer b (one bulk copy per theta row: padded rows),
  // and its children block -> L2
  auto issue = [&](int par, int b) {
    const double2* src = loc_p + int64_t(plist ? plist[par] : par) * SP;
    bulk::mbar_expect_tx(bar + b, uint32_t(SP) * 16u);
    for (int r = 0; r < NP; ++r)
      bulk::copy_g2s(Ls + (b * NP + r) * Y::LROW, src + r * NP, uint32_t(NP) * 16u, bar + b);
    fz::prefetch_children(par, n_par, child_off, children, loc_c, SC);
  };
  if (threadIdx.x == 0) {
    bulk::mbar_init(bar, 1);
    bulk::mbar_init(bar + 1, 1);
    bulk::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0 && int(blockIdx.x) < n_par) issue(blockIdx.x, 0);
  for (int t = threadIdx.x; t < Y::VTH; t += blockDim.x) vt[t] = vth[t];
  for (int t = threadIdx.x; t < Y::VPHI; t += blockDim.x) vp[t] = t < NP ? vphi[t] : 0.0;
  for (int t = threadIdx.x; t < 8 * H * H; t += blockDim.x) {
    const int o = t / (H * H), r = t - o * H * H, n = r / H, pc = r - n * H;
    shq[o * Y::SHOCT + n * Y::SHROW + pc] = shift_dn[int64_t(o) * SP + n * NP + pc];
  }
  rb::stage_b<D::DTH_K, D::DTH_N, D::DTH_LDB>(Bt, Bth);
  rb::stage_b<D::DPHI_K, D::DPHI_N, D::DPHI_LDB>(Bp, Bphi);  // (ends with a CTA barrier)

  int it = 0;
  for (int par = blockIdx.x; par < n_par; par += gridDim.x, ++it) {
    const int b = it & 1;
    const int cb = child_off[par], nch = child_off[par + 1] - cb;
    if (threadIdx.x == 0 && par + int(gridDim.x) < n_par) issue(par + gridDim.x, b ^ 1);
    bulk::mbar_wait(bar + b, uint32_t(it >> 1) & 1u);
    const double2* L = Ls + b * NP * Y::LROW;
    // theta pass: tile rows rho = (child slot c, circle p) -> narrow rows in shared memory
    const int ttiles = (nch * HALF + 7) / 8;
    for (int tile = warp; tile < ttiles; tile += NW) {
      const int rho = tile * 8 + g, c = rho / HALF, p = rho - c * HALF;
      const bool ok = c < nch;
      const int oct = ok ? oct_c[children[cb + c]] : 0;
      double er[KH], ei[KH], qr[KH], qi[KH];
#pragma unroll
      for (int kk = 0; kk < KH; ++kk) {
        const int k = 4 * kk + tq;
        double2 f = make_double2(0.0, 0.0), bk = f;
        if (ok && k < NP) {
          const int up = k >= H, kr = up ? NP - 1 - k : k;
          const int of = oct ^ (up ? 4 : 0);
          f = cmul(L[k * Y::LROW + p], shq[of * Y::SHOCT + kr * Y::SHROW + p]);
          bk = cmul(L[k * Y::LROW + p + HALF], shq[(of ^ 3) * Y::SHOCT + kr * Y::SHROW + p]);
        }
        er[kk] = f.x + bk.x;
        ei[kk] = f.y + bk.y;
        qr[kk] = f.x - bk.x;
        qi[kk] = f.y - bk.y;
      }
      rb::rank1_inject_eo_f<KH, NP>(er, ei, qr, qi, [&](int k) { return vt[k]; });
      double2* Nc = Nbs + (ok ? c : 0) * NC * Y::LDN;
      constexpr int NTC = 2;
#pragma unroll
      for (int j0 = 0; j0 < NT; j0 += NTC) {
        double cer[NTC][2] = {}, cei[NTC][2] = {}, cqr[NTC][2] = {}, cqi[NTC][2] = {};
        const double* bp = Bt + tq * D::DTH_LDB + g + 8 * j0;
#pragma unroll
        for (int kk = 0; kk < KH; ++kk)
#pragma unroll
          for (int jc = 0; jc < NTC; ++jc)
            if (j0 + jc < NT) {
              const double be = bp[4 * kk * D::DTH_LDB + 8 * jc];
              dmma884(cer[jc][0], cer[jc][1], er[kk], be);
              dmma884(cei[jc][0], cei[jc][1], ei[kk], be);
              const double bo = bp[4 * (KH + kk) * D::DTH_LDB + 8 * jc];
              dmma884(cqr[jc][0], cqr[jc][1], qr[kk], bo);
              dmma884(cqi[jc][0], cqi[jc][1], qi[kk], bo);
            }
        if (ok) {
#pragma unroll
          for (int jc = 0; jc < NTC; ++jc)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int n = 8 * (j0 + jc) + 2 * tq + q;
              if (j0 + jc < NT && n < NC) {
                double2* d = Nc + n * Y::LDN + 2 * p;
                d[0] = make_double2(cer[jc][q], cei[jc][q]);
                d[1] = make_double2(cqr[jc][q], cqi[jc][q]);
              }
            }
        }
      }
    }
    __syncthreads();
    // phi pass: item = (row tile of (c, i), n8 tile of the child's columns); added to the child locals
    const int rows = nch * NC, ptiles = (rows + 7) / 8;
    for (int item = warp; item < ptiles * NTP; item += NW) {
      const int t = item / NTP, jn = item - t * NTP;
      const int R = t * 8 + g;
      const bool ok = R < rows;
      const int c = ok ? R / NC : 0, i = ok ? R - c * NC : 0;
      double2* dst = loc_c + int64_t(children[cb + c]) * SC + i * NC;
      double2 old[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int n = 8 * jn + 2 * tq + q;
        old[q] = (ok && n < NC) ? dst[n] : make_double2(0.0, 0.0);
      }
      const double2* a = Nbs + (c * NC + i) * Y::LDN;
      double are[KSP], aim[KSP];
#pragma unroll
      for (int kk = 0; kk < KSP; ++kk) {
        const int k = 4 * kk + tq;
        const double2 xv = (ok && k < NP) ? a[k] : make_double2(0.0, 0.0);
        are[kk] = xv.x;
        aim[kk] = xv.y;
      }
      rb::rank1_inject_f<KSP, NP>(are, aim, [&](int k) { return vp[k]; });
      double cre[1][2] = {}, cim[1][2] = {};
      rb::tile_mma<KSP, 1, D::DPHI_LDB>(are, aim, Bp + 8 * jn, cre, cim);
      if (ok) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int n = 8 * jn + 2 * tq + q;
          if (n < NC) dst[n] = make_double2(old[q].x + cre[0][q], old[q].y + cim[0][q]);
        }
      }
    }
    __syncthreads();
  }
}

inline void launch_l2l_fz2(const RbLaunch& L, int sms, const double2* loc_p, double2* loc_c, const double* Bth,
                           const double* vth, const double* Bphi, const double* vphi, const double2* shift_dn) {
  constexpr int smem = fz2::LayD<18, 28>::SMEM;
  static_assert(smem <= 227 * 1024, "fused L2L v2 shared memory");
  cudaFuncSetAttribute(k_l2l_fz2<18, 28>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = std::min(L.n_par, sms);
  k_l2l_fz2<18, 28><<<grid, fz2::kThreads, smem, L.st>>>(L.n_par, L.plist, L.child_off, L.children, L.oct_c, loc_p, Bth,
                                                         vth, Bphi, vphi, shift_dn, loc_c);
}

}  // namespace hfmm_b200

#endif
