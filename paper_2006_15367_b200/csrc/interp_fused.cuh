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

}  // namespace hfmm_b200

#endif
