// Fused M2M / L2L for the leaf-side level pair (18, 28) of the BASELINE cubes
// (configs 1, 3, 4 leaf level): one CTA per parent (persistent over parents),
// both passes of the separable resampling in one kernel with the
// intermediate in SHARED memory -- the folded circles F of the M2M phi pass
// and the narrow rows Nb of the L2L theta pass never touch HBM (the two-kernel
// streaming form, interp_rb.cuh, writes and re-reads them: at config 4 that
// is 27.8 GB + 25.9 GB for M2M and 24.1 GB + 41.0 GB for L2L per evaluation).
// Same algebra and the same device helpers as interp_rb.cuh (real + rank-1
// matrices on DMMA, complex-row warp tiles, child sum as a reduce-scatter);
// traversal.cpp:322-429 (M2M) and :583-707 (L2L), sphere_grid.cpp:183-214.
// Data movement uses the Blackwell bulk-copy engine (bulk.cuh): the L2L
// parent local is staged into shared memory by one cp.async.bulk with an
// mbarrier, and each M2M CTA prefetches its NEXT parent's children into L2
// with cp.async.bulk.prefetch while the current parent computes.
#ifndef HFMM_B200_INTERP_FUSED_CUH
#define HFMM_B200_INTERP_FUSED_CUH

#include "bulk.cuh"
#include "interp_rb.cuh"

namespace hfmm_b200 {
namespace fz {

constexpr int kThreads = 224;  // 7 warps: the 14 theta circles (M2M) / tiles (L2L) of a parent split evenly
__host__ __device__ constexpr int pad4mod8(int x) { return x + ((4 - x % 8) + 8) % 8; }  // stride == 4 (mod 8) double2

template <int NC, int NP>
struct Lay {
  using D = rb::Dims<NC, NP>;
  // M2M: F[c][p][ii] (c = child slot, p < HALF, ii < LDF), child stride CSF
  static constexpr int CSF = pad4mod8(D::HALF * D::LDF);
  static constexpr int BPHI = D::UPHI_K * D::UPHI_LDB, BTH = D::UTH_K * D::UTH_LDB;  // doubles
  static constexpr int M2M_SMEM = (BPHI + BTH) * 8 + 8 * CSF * 16;
  // L2L: Nb[c][row][col] (row < NC, col < LDN), child stride CSN
  static constexpr int CSN = pad4mod8(NC * D::LDN);
  static constexpr int BDTH = D::DTH_K * D::DTH_LDB, BDPHI = D::DPHI_K * D::DPHI_LDB;
  static constexpr int L2L_SMEM = (BDTH + BDPHI) * 8 + 8 * CSN * 16 + D::SP * 16;  // + the parent local
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
  constexpr int KST = D::UTH_K / 4, NTT = D::UTH_N / 8, HALF = D::HALF, SP = D::SP, SC = D::SC;
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
            const int n = 8 * jn + 2 * tq + q;
            if (n < NP) {
              const int p = n < HALF ? n : n - HALF;
              const int ii = n < HALF ? i : 2 * NC - 1 - i;
              Fc[p * D::LDF + ii] = make_double2(cre[jn][q], cim[jn][q]);
            }
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
      double are[KST], aim[KST];
#pragma unroll
      for (int kk = 0; kk < KST; ++kk) {
        const int k = 4 * kk + tq;
        const double2 fv = (ok && k < 2 * NC) ? frow[k] : make_double2(0.0, 0.0);
        are[kk] = fv.x;
        aim[kk] = fv.y;
      }
      rb::rank1_inject<KST, 2 * NC>(are, aim, vth);
      constexpr int NTC = 4;
#pragma unroll
      for (int j0 = 0; j0 < NTT; j0 += NTC) {
        double2 shv[NTC][2];
#pragma unroll
        for (int jc = 0; jc < NTC; ++jc)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = 8 * (j0 + jc) + 2 * tq + q;
            const int s = n < NP ? n * NP + p : (2 * NP - 1 - n) * NP + p + HALF;
            shv[jc][q] = (ok && j0 + jc < NTT && n < 2 * NP) ? __ldg(sh + s) : make_double2(0.0, 0.0);
          }
        double cre[NTC][2] = {}, cim[NTC][2] = {};
        const double* bp = Bt + tq * D::UTH_LDB + g + 8 * j0;
#pragma unroll
        for (int kk = 0; kk < KST; ++kk)
#pragma unroll
          for (int jc = 0; jc < NTC; ++jc)
            if (j0 + jc < NTT) {
              const double b = bp[4 * kk * D::UTH_LDB + 8 * jc];
              dmma884(cre[jc][0], cre[jc][1], are[kk], b);
              dmma884(cim[jc][0], cim[jc][1], aim[kk], b);
            }
        double v[16];
#pragma unroll
        for (int jc = 0; jc < NTC; ++jc)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const double2 f = shv[jc][q];
            v[(2 * jc + q) * 2] = cre[jc][q] * f.x - cim[jc][q] * f.y;
            v[(2 * jc + q) * 2 + 1] = cre[jc][q] * f.y + cim[jc][q] * f.x;
          }
        const double2 val = rb::child_sum_scatter(v);
        const int jt = j0 + (g >> 1), n = 8 * jt + 2 * tq + (g & 1);
        if (jt < NTT && n < 2 * NP) {
          const int s = n < NP ? n * NP + p : (2 * NP - 1 - n) * NP + p + HALF;
          out[s] = val;
        }
      }
    }
    __syncthreads();
  }
}

template <int NC, int NP>
__global__ void __launch_bounds__(fz::kThreads, 2) k_l2l_fz(int n_par, const int* __restrict__ plist,
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
  using Y = fz::Lay<NC, NP>;
  constexpr int KST = D::DTH_K / 4, NTT = D::DTH_N / 8, HALF = D::HALF, SP = D::SP, SC = D::SC;
  constexpr int KSP = D::DPHI_K / 4, NTP = D::DPHI_N / 8;
  extern __shared__ __align__(16) double fz_smem[];
  double* Bt = fz_smem;
  double* Bp = Bt + Y::BDTH;
  double2* Ns = reinterpret_cast<double2*>(Bp + Y::BDPHI);
  double2* Ls = Ns + 8 * Y::CSN;  // the parent's local expansion, staged per parent
  __shared__ __align__(8) uint64_t lbar;  // completion of the parent-local bulk copy
  if (threadIdx.x == 0) {
    bulk::mbar_init(&lbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  rb::stage_b<D::DTH_K, D::DTH_N, D::DTH_LDB>(Bt, Bth);
  rb::stage_b<D::DPHI_K, D::DPHI_N, D::DPHI_LDB>(Bp, Bphi);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  constexpr int NW = fz::kThreads / 32;
  uint32_t phase = 0;
  for (int par = blockIdx.x; par < n_par; par += gridDim.x, phase ^= 1u) {
    const int cb = child_off[par], nch = child_off[par + 1] - cb;
    if (threadIdx.x == 0) {  // the parent local: one bulk copy
      bulk::mbar_expect_tx(&lbar, uint32_t(SP) * 16u);
      bulk::copy_g2s(Ls, loc_p + int64_t(plist ? plist[par] : par) * SP, uint32_t(SP) * 16u, &lbar);
    }
    bulk::mbar_wait(&lbar, phase);
    const double2* L = Ls;
    // theta pass: rows (child c, circle p) built on the fly from the shifted
    // parent local -> narrow rows in shared memory
    const int trows = nch * HALF, ttiles = (trows + 7) / 8;
    for (int t = warp; t < ttiles; t += NW) {
      const int rho = t * 8 + g;
      const bool ok = rho < trows;
      const int c = ok ? rho / HALF : 0, p = ok ? rho - c * HALF : 0;
      const double2* sh = shift_dn + int64_t(ok ? oct_c[children[cb + c]] : 0) * SP;
      double are[KST], aim[KST];
#pragma unroll
      for (int kk = 0; kk < KST; ++kk) {
        const int k = 4 * kk + tq;
        double2 f = make_double2(0.0, 0.0);
        if (ok && k < 2 * NP) {
          const int s = k < NP ? k * NP + p : (2 * NP - 1 - k) * NP + p + HALF;
          f = cmul(L[s], __ldg(sh + s));
        }
        are[kk] = f.x;
        aim[kk] = f.y;
      }
      rb::rank1_inject<KST, 2 * NP>(are, aim, vth);
      double2* Nc = Ns + c * Y::CSN;
      constexpr int NTC = 4;
#pragma unroll
      for (int j0 = 0; j0 < NTT; j0 += NTC) {
        double cre[NTC][2] = {}, cim[NTC][2] = {};
        const double* bp = Bt + tq * D::DTH_LDB + g + 8 * j0;
#pragma unroll
        for (int kk = 0; kk < KST; ++kk)
#pragma unroll
          for (int jc = 0; jc < NTC; ++jc)
            if (j0 + jc < NTT) {
              const double b = bp[4 * kk * D::DTH_LDB + 8 * jc];
              dmma884(cre[jc][0], cre[jc][1], are[kk], b);
              dmma884(cim[jc][0], cim[jc][1], aim[kk], b);
            }
        if (ok) {
#pragma unroll
          for (int jc = 0; jc < NTC; ++jc)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int n = 8 * (j0 + jc) + 2 * tq + q;
              if (j0 + jc < NTT && n < 2 * NC) {
                const int row = n < NC ? n : 2 * NC - 1 - n;
                const int col = n < NC ? p : p + HALF;
                Nc[row * D::LDN + col] = make_double2(cre[jc][q], cim[jc][q]);
              }
            }
        }
      }
    }
    __syncthreads();
    // phi pass of every narrow row, added into the child's local expansion
    const int rows = nch * NC, tiles = (rows + 7) / 8;
    for (int t = warp; t < tiles; t += NW) {
      const int R = t * 8 + g;
      const bool ok = R < rows;
      const int c = ok ? R / NC : 0, row = ok ? R - c * NC : 0;
      const double2* a = Ns + c * Y::CSN + row * D::LDN;
      double2* dst = loc_c + int64_t(children[cb + c]) * SC + row * NC;
      double2 old[NTP][2];
#pragma unroll
      for (int jn = 0; jn < NTP; ++jn)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int n = 8 * jn + 2 * tq + q;
          old[jn][q] = (ok && n < NC) ? dst[n] : make_double2(0.0, 0.0);
        }
      double are[KSP], aim[KSP];
#pragma unroll
      for (int kk = 0; kk < KSP; ++kk) {
        const int k = 4 * kk + tq;
        const double2 xv = (ok && k < NP) ? a[k] : make_double2(0.0, 0.0);
        are[kk] = xv.x;
        aim[kk] = xv.y;
      }
      rb::rank1_inject<KSP, NP>(are, aim, vphi);
      double cre[NTP][2] = {}, cim[NTP][2] = {};
      rb::tile_mma<KSP, NTP, D::DPHI_LDB>(are, aim, Bp, cre, cim);
      if (ok) {
#pragma unroll
        for (int jn = 0; jn < NTP; ++jn)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = 8 * jn + 2 * tq + q;
            if (n < NC) dst[n] = make_double2(old[jn][q].x + cre[jn][q], old[jn][q].y + cim[jn][q]);
          }
      }
    }
    __syncthreads();
  }
}

// Pairs served by the fused kernels (two CTAs per SM fit their shared memory).
inline bool fz_pair(int nc, int np) { return nc == 18 && np == 28; }

inline void launch_m2m_fz(const RbLaunch& L, int sms, const double2* mp_c, double2* mp_p, const double* Bphi,
                          const double* vphi, const double* Bth, const double* vth, const double2* shift_up) {
  constexpr int smem = fz::Lay<18, 28>::M2M_SMEM;
  cudaFuncSetAttribute(k_m2m_fz<18, 28>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = std::min(L.n_par, 2 * sms);
  k_m2m_fz<18, 28><<<grid, fz::kThreads, smem, L.st>>>(L.n_par, L.plist, L.child_off, L.children, L.oct_c, mp_c, Bphi,
                                                       vphi, Bth, vth, shift_up, mp_p);
}

inline void launch_l2l_fz(const RbLaunch& L, int sms, const double2* loc_p, double2* loc_c, const double* Bth,
                          const double* vth, const double* Bphi, const double* vphi, const double2* shift_dn) {
  constexpr int smem = fz::Lay<18, 28>::L2L_SMEM;
  cudaFuncSetAttribute(k_l2l_fz<18, 28>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = std::min(L.n_par, 2 * sms);
  k_l2l_fz<18, 28><<<grid, fz::kThreads, smem, L.st>>>(L.n_par, L.plist, L.child_off, L.children, L.oct_c, loc_p, Bth,
                                                       vth, Bphi, vphi, shift_dn, loc_c);
}

}  // namespace hfmm_b200

#endif
