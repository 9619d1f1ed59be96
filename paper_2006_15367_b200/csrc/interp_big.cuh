// M2M / L2L for large sphere grids (upper levels) on DMMA.
//
// Same real + rank-1 passes as interp_tc.cuh, split in two kernels so that a
// CTA never needs a whole parent grid on chip:
//   M2M: k_m2m_big_phi   one CTA per child: phi pass, folded circles -> HBM (F)
//        k_m2m_big_theta one CTA per (parent, circle chunk): theta pass over
//                        the children (rows = circle, child, re/im), shift,
//                        in-warp child reduction, parent samples of the chunk
//   L2L: k_l2l_big_theta one CTA per (child, circle chunk): shifted + folded
//                        parent circles, theta anterpolation -> narrow rows (HBM)
//        k_l2l_big_phi   one CTA per child: phi anterpolation, += child local
// The B matrices stream from L2 (they are shared by every CTA of a level).
#ifndef HFMM_B200_INTERP_BIG_CUH
#define HFMM_B200_INTERP_BIG_CUH

#include "dmma.cuh"

namespace hfmm_b200 {

// ---------------------------------------------------------------------------
// M2M phi pass: X (n_c x n_c) of one child -> F rows [p][ii] (half rows of
// stride ldf, columns 0 .. 2 n_c - 1; the rank-1 column is added later).
__global__ void __launch_bounds__(256) k_m2m_big_phi(int n_c, int n_p, PassDims phi, int ldf, int RC,
                                                     const int* __restrict__ clist,
                                                     const double2* __restrict__ mp_c,
                                                     const double* __restrict__ RphiT,
                                                     const double* __restrict__ vphi, double2* __restrict__ F) {
  extern __shared__ double2 X[];
  const int half = n_p / 2, Sc = n_c * n_c;
  const int64_t child = clist ? clist[blockIdx.x] : blockIdx.x;
  const int i0 = blockIdx.y * RC, nr = min(RC, n_c - i0);  // rows (theta) of this CTA
  for (int t = threadIdx.x; t < nr * phi.lda; t += blockDim.x) {
    const int i = t / phi.lda, k = t - i * phi.lda;
    cp_async16(X + t, k < n_c ? mp_c + child * Sc + (i0 + i) * n_c + k : mp_c, k < n_c);
  }
  cp_async_wait_all();
  __syncthreads();
  rank1_column(nr, n_c, vphi, [&](int r) { return X + r * phi.lda; });
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  double2* Fc = F + child * half * ldf;
  warp_gemm_rc(nr * 2, phi.N, phi.K, [&](int r) { return X + r * phi.lda; }, RphiT,
               [&](int m0, int n0, double v0, double v1) {
                 const int r = m0 + g, i = i0 + (r >> 1);
                 if ((r >> 1) >= nr) return;
#pragma unroll
                 for (int q = 0; q < 2; ++q) {
                   const int n = n0 + 2 * tq + q;
                   if (n < n_p) {
                     const int p = n < half ? n : n - half;
                     const int ii = n < half ? i : 2 * n_c - 1 - i;
                     set_part(Fc + p * ldf + ii, r & 1, q ? v1 : v0);
                   }
                 }
               });
}

// M2M theta pass + shift + sum over children for circles [p0, p0 + CP).
// F rows of child c live at F + c * half * ldf (global child index).
constexpr int kBigCB = 4;
__global__ void __launch_bounds__(256) k_m2m_big_theta(int n_c, int n_p, int CP, PassDims th,
                                                       const int* __restrict__ plist,
                                                       const int* __restrict__ child_off,
                                                       const int* __restrict__ children,
                                                       const uint8_t* __restrict__ oct_c,
                                                       const double2* __restrict__ F,
                                                       const double* __restrict__ RthT,
                                                       const double* __restrict__ vth,
                                                       const double2* __restrict__ shift_up,
                                                       double2* __restrict__ mp_p) {
  extern __shared__ double2 sm[];
  const int half = n_p / 2, Sp = n_p * n_p, ldf = th.lda;
  const int par_i = blockIdx.x;
  const int64_t par = plist ? plist[par_i] : par_i;
  const int p0 = blockIdx.y * CP, ncirc = min(CP, half - p0);
  double2* Fs = sm;                            // [c][pl][k], rows of stride ldf
  double2* Sacc = sm + kBigCB * CP * ldf;      // [pl][n], 2 n_p per circle
  const int cb = child_off[par_i], ce = child_off[par_i + 1];
  for (int t = threadIdx.x; t < CP * 2 * n_p; t += blockDim.x) Sacc[t] = make_double2(0.0, 0.0);
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  constexpr int CB = kBigCB, R2 = 2 * kBigCB;
  for (int b0 = cb; b0 < ce; b0 += CB) {
    const int nb = min(CB, ce - b0);
    __syncthreads();
    for (int t = threadIdx.x; t < CB * CP * ldf; t += blockDim.x) {
      const int row = t / ldf, k = t - row * ldf;
      const int c = row / CP, pl = row - c * CP;
      const bool ok = c < nb && pl < ncirc && k < 2 * n_c;
      const double2* src = ok ? F + (int64_t(children[b0 + c]) * half + p0 + pl) * ldf + k : F;
      cp_async16(Fs + t, src, ok);
    }
    cp_async_wait_all();
    __syncthreads();
    rank1_column(CB * CP, 2 * n_c, vth, [&](int r) { return Fs + r * ldf; });
    __syncthreads();
    int octs[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) octs[c] = c < nb ? oct_c[children[b0 + c]] : 0;
    warp_gemm_rc(CP * R2, th.N, th.K,
                 [&](int row) {
                   const int pl = row / CB, c = row - pl * CB;
                   return Fs + (c * CP + pl) * ldf;
                 },
                 RthT, [&](int m0, int n0, double v0, double v1) {
                   const int r = m0 + g, part = r & 1, c = (r >> 1) % CB, pl = r / R2;
                   const double o0 = __shfl_xor_sync(0xffffffffu, v0, 4);
                   const double o1 = __shfl_xor_sync(0xffffffffu, v1, 4);
                   const bool live = c < nb && pl < ncirc;
                   const double2* sh = shift_up + octs[c] * Sp;
                   double cr[2], cim[2];
#pragma unroll
                   for (int q = 0; q < 2; ++q) {
                     const int n = n0 + 2 * tq + q, p = p0 + pl;
                     const double re = part ? (q ? o1 : o0) : (q ? v1 : v0);
                     const double im = part ? (q ? v1 : v0) : (q ? o1 : o0);
                     double2 f = make_double2(0.0, 0.0);
                     if (live && n < 2 * n_p) {
                       const int s = n < n_p ? n * n_p + p : (2 * n_p - 1 - n) * n_p + p + half;
                       f = __ldg(sh + s);
                     }
                     cr[q] = re * f.x - im * f.y;
                     cim[q] = re * f.y + im * f.x;
                   }
#pragma unroll
                   for (int q = 0; q < 2; ++q) {
                     cr[q] += __shfl_xor_sync(0xffffffffu, cr[q], 8);
                     cim[q] += __shfl_xor_sync(0xffffffffu, cim[q], 8);
                     cr[q] += __shfl_xor_sync(0xffffffffu, cr[q], 16);
                     cim[q] += __shfl_xor_sync(0xffffffffu, cim[q], 16);
                   }
                   if (part == 0 && c == 0 && pl < ncirc) {
#pragma unroll
                     for (int q = 0; q < 2; ++q) {
                       const int n = n0 + 2 * tq + q;
                       if (n < 2 * n_p) {
                         double2 a = Sacc[pl * 2 * n_p + n];
                         a.x += cr[q];
                         a.y += cim[q];
                         Sacc[pl * 2 * n_p + n] = a;
                       }
                     }
                   }
                 });
  }
  __syncthreads();
  for (int t = threadIdx.x; t < ncirc * 2 * n_p; t += blockDim.x) {
    const int pl = t / (2 * n_p), n = t - pl * 2 * n_p, p = p0 + pl;
    const int s = n < n_p ? n * n_p + p : (2 * n_p - 1 - n) * n_p + p + half;
    mp_p[par * Sp + s] = Sacc[t];
  }
}

// ---------------------------------------------------------------------------
// L2L theta pass for circles [p0, p0 + CP) of one child: fold(Lp * shift)
// -> theta anterpolation -> narrow rows Nb[child][row][col] (stride ldn).
__global__ void __launch_bounds__(256) k_l2l_big_theta(int n_c, int n_p, int CP, PassDims th, int ldn,
                                                       const int* __restrict__ clist,
                                                       const int* __restrict__ parent_c,
                                                       const uint8_t* __restrict__ oct_c,
                                                       const double2* __restrict__ loc_p,
                                                       const double2* __restrict__ shift_dn,
                                                       const double* __restrict__ RthT,
                                                       const double* __restrict__ vth, double2* __restrict__ Nb) {
  extern __shared__ double2 Fs[];
  const int half = n_p / 2, Sp = n_p * n_p;
  const int64_t child = clist ? clist[blockIdx.x] : blockIdx.x;
  const int64_t par = parent_c[child];
  const int p0 = blockIdx.y * CP, ncirc = min(CP, half - p0);
  const double2* lp = loc_p + par * Sp;
  const double2* sh = shift_dn + int64_t(oct_c[child]) * Sp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  for (int row = warp; row < CP; row += nwarp) {
    double2* f = Fs + row * th.lda;
    const int p = p0 + row;
    for (int i = lane; i < th.lda; i += 32) {
      double2 v = make_double2(0.0, 0.0);
      if (row < ncirc && i < 2 * n_p) {
        const int s = i < n_p ? i * n_p + p : (2 * n_p - 1 - i) * n_p + p + half;
        v = cmul(__ldg(lp + s), __ldg(sh + s));
      }
      f[i] = v;
    }
  }
  __syncthreads();
  rank1_column(CP, 2 * n_p, vth, [&](int r) { return Fs + r * th.lda; });
  __syncthreads();
  const int g = lane >> 2, tq = lane & 3;
  double2* Nc = Nb + child * n_c * ldn;
  warp_gemm_rc(CP * 2, th.N, th.K, [&](int r) { return Fs + r * th.lda; }, RthT,
               [&](int m0, int n0, double v0, double v1) {
                 const int r = m0 + g, pl = r >> 1;
                 if (pl >= ncirc) return;
                 const int p = p0 + pl;
#pragma unroll
                 for (int q = 0; q < 2; ++q) {
                   const int n = n0 + 2 * tq + q;
                   if (n < 2 * n_c) {
                     const int row = n < n_c ? n : 2 * n_c - 1 - n;
                     const int col = n < n_c ? p : p + half;
                     set_part(Nc + row * ldn + col, r & 1, q ? v1 : v0);
                   }
                 }
               });
}

// L2L phi pass of one child: narrow rows (n_c x n_p) -> += child local.
__global__ void __launch_bounds__(256) k_l2l_big_phi(int n_c, int n_p, PassDims phi, int ldn, int RC,
                                                     const int* __restrict__ clist,
                                                     const double2* __restrict__ Nb,
                                                     const double* __restrict__ RphiT,
                                                     const double* __restrict__ vphi,
                                                     double2* __restrict__ loc_c) {
  extern __shared__ double2 Ns[];
  const int Sc = n_c * n_c;
  const int64_t child = clist ? clist[blockIdx.x] : blockIdx.x;
  const int i0 = blockIdx.y * RC, nr = min(RC, n_c - i0);  // narrow rows of this CTA
  const double2* Nc = Nb + child * n_c * ldn + int64_t(i0) * ldn;
  for (int t = threadIdx.x; t < nr * phi.lda; t += blockDim.x) {
    const int row = t / phi.lda, k = t - row * phi.lda;
    cp_async16(Ns + t, k < n_p ? Nc + row * ldn + k : Nc, k < n_p);
  }
  cp_async_wait_all();
  __syncthreads();
  rank1_column(nr, n_p, vphi, [&](int r) { return Ns + r * phi.lda; });
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  double* lc = reinterpret_cast<double*>(loc_c) + 2 * (child * Sc + int64_t(i0) * n_c);
  warp_gemm_rc(nr * 2, phi.N, phi.K, [&](int r) { return Ns + r * phi.lda; }, RphiT,
               [&](int m0, int n0, double v0, double v1) {
                 const int r = m0 + g, row = r >> 1;
                 if (row >= nr) return;
#pragma unroll
                 for (int q = 0; q < 2; ++q) {
                   const int n = n0 + 2 * tq + q;
                   if (n < n_c) lc[2 * (row * n_c + n) + (r & 1)] += q ? v1 : v0;
                 }
               });
}

}  // namespace hfmm_b200

#endif
