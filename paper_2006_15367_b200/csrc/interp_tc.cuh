// Fused M2M / L2L on FP64 tensor cores (DMMA, mma.sync m8n8k4 f64).
//
// The reference resamples with FFTs (sphere_grid.cpp:128-214).  On B200 the
// per-level resampling maps are applied as dense matrices: a phi pass per
// theta row and a theta pass per folded great circle.  Each map
// M = Re(M) + i u v^T splits into a REAL matrix plus a rank-1 imaginary part
// (the unpaired Nyquist mode of the asymmetric window, sphere_grid.cpp:140-150),
// so y = M x = [Re(M) | u] [x ; i (v . x)]: one extra input column turns the
// complex-matrix product into a real-matrix x complex-data product -- half the
// flops -- which maps onto DMMA as a real GEMM whose rows are the real and
// imaginary parts of the data rows.
//
// One CTA (8 warps) owns one parent node and processes its children in
// batches of CB (1, 2 or 4).  Child samples stream in with cp.async (double
// buffered when shared memory allows); the M2M theta pass orders its rows
// (circle, child, re/im) so one 8-row DMMA tile holds every child of a
// circle: the epilogue combines re/im across lanes, applies each child's
// shift and sums the children with warp shuffles straight into the parent
// accumulator -- no intermediate grid ever leaves shared memory.
#ifndef HFMM_B200_INTERP_TC_CUH
#define HFMM_B200_INTERP_TC_CUH

#include "kernels.cuh"

namespace hfmm_b200 {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Shape of one pass, computed on the host (strides in double2).
struct PassDims {
  int K;    // padded reduction length (multiple of 4): n_in + 1 (rank-1 column) rounded up
  int N;    // padded output length (multiple of 8)
  int lda;  // smem row stride of the input rows (== 4 mod 8: conflict-free fragment loads)
  int ldo;  // unused (kept for layout stability)
};

// Warp-tiled real GEMM over complex smem rows, DMMA m8n8k4:
//   C(r, n) = sum_{k<K} A(r, k) B(k, n),   r < M (padded to 16), n < N.
// A(r, k) = part (r & 1) of element k of complex row rowp(r >> 1) (smem);
// B is K x N row-major in global memory (L1 resident).  The epilogue gets
// the 8x8 tile origin and both accumulators of the lane:
//   epi(m0, n0, c0, c1): lane holds C(m0 + g, n0 + 2 tq) and C(.., +1),
// and is called by all 32 lanes (warp-uniform), so it may shuffle.
template <class RowPtr, class Epi>
__device__ __forceinline__ void warp_gemm_rc(int M, int N, int K, RowPtr rowp, const double* __restrict__ B,
                                             Epi epi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int mt = (M + 15) >> 4, nt = (N + 15) >> 4;
  for (int w = warp; w < mt * nt; w += nwarp) {
    const int m0 = (w / nt) << 4, n0 = (w % nt) << 4;
    double c[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
    const int r0 = m0 + g, r1 = m0 + 8 + g;
    // Unconditional loads: rows past M read row 0 and a missing second n8
    // block re-reads the first (finite values in outputs the epilogue drops),
    // so the k-loop has no predicated loads.
    const double* a0p = reinterpret_cast<const double*>(rowp(r0 < M ? r0 >> 1 : 0)) + (r0 < M ? r0 & 1 : 0);
    const double* a1p = reinterpret_cast<const double*>(rowp(r1 < M ? r1 >> 1 : 0)) + (r1 < M ? r1 & 1 : 0);
    const double* bp = B + tq * N + n0 + g;
    const double* bp1 = n0 + 8 < N ? bp + 8 : bp;
#pragma unroll 4
    for (int k = 0; k < K; k += 4) {
      const int kk = k + tq;
      const double a0 = a0p[2 * kk];
      const double a1 = a1p[2 * kk];
      const double b0 = __ldg(bp + k * N);
      const double b1 = __ldg(bp1 + k * N);
      dmma884(c[0][0][0], c[0][0][1], a0, b0);
      dmma884(c[0][1][0], c[0][1][1], a0, b1);
      dmma884(c[1][0][0], c[1][0][1], a1, b0);
      dmma884(c[1][1][0], c[1][1][1], a1, b1);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (n0 + 8 * j < N) epi(m0 + 8 * i, n0 + 8 * j, c[i][j][0], c[i][j][1]);
  }
}

// x[row][kin] = i * (v . x[row][0:kin]) for `rows` complex rows: four lanes
// per row, eight rows per warp pass, two shuffle levels.
template <class RowPtr>
__device__ __forceinline__ void rank1_column(int rows, int kin, const double* __restrict__ v, RowPtr rowp) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  const int sub = lane & 3;
  const int rup = (rows + 7) & ~7;  // whole warps iterate together (shuffles)
  for (int r = warp * 8 + (lane >> 2); r < rup; r += nwarp * 8) {
    const bool live = r < rows;
    double sr = 0.0, si = 0.0;
    double2* x = rowp(live ? r : 0);
    for (int k = sub; k < kin; k += 4) {
      const double vk = __ldg(v + k);
      const double2 xv = x[k];
      sr = fma(vk, xv.x, sr);
      si = fma(vk, xv.y, si);
    }
    sr += __shfl_xor_sync(0xffffffffu, sr, 1);
    si += __shfl_xor_sync(0xffffffffu, si, 1);
    sr += __shfl_xor_sync(0xffffffffu, sr, 2);
    si += __shfl_xor_sync(0xffffffffu, si, 2);
    if (live && sub == 0) x[kin] = make_double2(-si, sr);
  }
}

__device__ __forceinline__ void set_part(double2* p, int part, double v) {
  reinterpret_cast<double*>(p)[part] = v;
}

constexpr int kFusedThreads = 256;

// Launch plan of a fused pass (host-computed).
struct FusedPlan {
  int CB;    // children per batch (1, 2, 4)
  int dbuf;  // M2M: double-buffer the child rows; L2L: keep the parent in smem
  int smem_bytes;
};

// ---------------------------------------------------------------------------
// M2M for one parent: phi upsample (n_c -> n_p per theta row), fold, theta
// upsample (2 n_c -> 2 n_p per great circle), unfold, shift, sum over the
// children (traversal.cpp:322-429, sphere_grid.cpp:183-192).
__global__ void __launch_bounds__(kFusedThreads) k_m2m_fused(
    int n_c, int n_p, FusedPlan plan, const int* __restrict__ plist, PassDims phi, PassDims th, const int* __restrict__ child_off,
    const int* __restrict__ children, const uint8_t* __restrict__ oct_c, const double2* __restrict__ mp_c,
    double2* __restrict__ mp_p, const double* __restrict__ RphiT, const double* __restrict__ vphi,
    const double* __restrict__ RthT, const double* __restrict__ vth, const double2* __restrict__ shift_up) {
  extern __shared__ double2 sm[];
  const int CB = plan.CB;
  const int half = n_p / 2, Sc = n_c * n_c, Sp = n_p * n_p;
  const int xsz = CB * n_c * phi.lda;
  double2* Xb0 = sm;
  double2* Xb1 = plan.dbuf ? sm + xsz : sm;
  double2* Fs = sm + (plan.dbuf ? 2 : 1) * xsz;
  double2* Sacc = Fs + CB * half * th.lda;
  const int par = blockIdx.x;
  const int cb = child_off[par], ce = child_off[par + 1];

  // Child rows [c][i][k] (k < n_c data, k == n_c rank-1 column, zero padding):
  // one 16-byte cp.async per element, padding zero-filled by the copy.
  auto issue_load = [&](double2* X, int b0) {
    const int nb = min(CB, ce - b0);
    for (int t = threadIdx.x; t < CB * n_c * phi.lda; t += blockDim.x) {
      const int row = t / phi.lda, k = t - row * phi.lda;
      const int c = row / n_c, i = row - c * n_c;
      const bool ok = c < nb && k < n_c;
      cp_async16(X + t, ok ? mp_c + int64_t(children[b0 + c]) * Sc + i * n_c + k : mp_c, ok);
    }
    cp_async_commit();
  };

  for (int t = threadIdx.x; t < CB * half * th.lda; t += blockDim.x) Fs[t] = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < Sp; t += blockDim.x) Sacc[t] = make_double2(0.0, 0.0);
  issue_load(Xb0, cb);

  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int R2 = 2 * CB;  // theta rows per circle: (child, re/im)
  int it = 0;
  for (int b0 = cb; b0 < ce; b0 += CB, ++it) {
    const int nb = min(CB, ce - b0);
    double2* X = (it & 1) ? Xb1 : Xb0;
    if (plan.dbuf && b0 + CB < ce) {
      issue_load((it & 1) ? Xb0 : Xb1, b0 + CB);
      cp_async_wait<1>();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    rank1_column(CB * n_c, n_c, vphi, [&](int r) { return X + r * phi.lda; });
    __syncthreads();
    // phi pass: rows (child, theta row, re/im) -> folded circles Fs[c][p][ii]
    warp_gemm_rc(CB * n_c * 2, phi.N, phi.K, [&](int r) { return X + r * phi.lda; }, RphiT,
                 [&](int m0, int n0, double v0, double v1) {
                   const int r = m0 + g, ci = r >> 1, c = ci / n_c, i = ci - c * n_c;
                   double2* base = Fs + c * half * th.lda;
#pragma unroll
                   for (int q = 0; q < 2; ++q) {
                     const int n = n0 + 2 * tq + q;
                     if (n < n_p && c < CB) {
                       const int p = n < half ? n : n - half;
                       const int ii = n < half ? i : 2 * n_c - 1 - i;
                       set_part(base + p * th.lda + ii, r & 1, q ? v1 : v0);
                     }
                   }
                 });
    __syncthreads();
    if (!plan.dbuf && b0 + CB < ce) issue_load(Xb0, b0 + CB);  // X is free: overlap with theta
    rank1_column(CB * half, 2 * n_c, vth, [&](int r) { return Fs + r * th.lda; });
    __syncthreads();
    // theta pass: rows (circle, child, re/im); an 8-row tile holds 8 / R2
    // whole circles, so the children of a circle reduce inside the warp.
    int octs[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) octs[c] = c < nb ? oct_c[children[b0 + c]] : 0;
    warp_gemm_rc(half * R2, th.N, th.K,
                 [&](int row) {  // complex row -> (circle, child)
                   const int p = row / CB, c = row - p * CB;
                   return Fs + (c * half + p) * th.lda;
                 },
                 RthT, [&](int m0, int n0, double v0, double v1) {
                   const int r = m0 + g, part = r & 1, c = (r >> 1) % CB, p = r / R2;
                   const double o0 = __shfl_xor_sync(0xffffffffu, v0, 4);  // the other part
                   const double o1 = __shfl_xor_sync(0xffffffffu, v1, 4);
                   const int o = octs[c];
                   const bool live = c < nb && p < half;
                   double cr[2], cim[2];
#pragma unroll
                   for (int q = 0; q < 2; ++q) {
                     const int n = n0 + 2 * tq + q;
                     const double re = part ? (q ? o1 : o0) : (q ? v1 : v0);
                     const double im = part ? (q ? v1 : v0) : (q ? o1 : o0);
                     double2 sh = make_double2(0.0, 0.0);
                     if (live && n < 2 * n_p) {
                       const int s = n < n_p ? n * n_p + p : (2 * n_p - 1 - n) * n_p + p + half;
                       sh = __ldg(shift_up + o * Sp + s);
                     }
                     cr[q] = re * sh.x - im * sh.y;
                     cim[q] = re * sh.y + im * sh.x;
                   }
                   // sum the children of the circle: lanes differing in the child bits of g
#pragma unroll
                   for (int q = 0; q < 2; ++q) {
                     if (CB >= 2) {
                       cr[q] += __shfl_xor_sync(0xffffffffu, cr[q], 8);
                       cim[q] += __shfl_xor_sync(0xffffffffu, cim[q], 8);
                     }
                     if (CB >= 4) {
                       cr[q] += __shfl_xor_sync(0xffffffffu, cr[q], 16);
                       cim[q] += __shfl_xor_sync(0xffffffffu, cim[q], 16);
                     }
                   }
                   if (part == 0 && c == 0 && p < half) {
#pragma unroll
                     for (int q = 0; q < 2; ++q) {
                       const int n = n0 + 2 * tq + q;
                       if (n < 2 * n_p) {
                         const int s = n < n_p ? n * n_p + p : (2 * n_p - 1 - n) * n_p + p + half;
                         double2 a = Sacc[s];
                         a.x += cr[q];
                         a.y += cim[q];
                         Sacc[s] = a;
                       }
                     }
                   }
                 });
    __syncthreads();
  }
  const int64_t gpar = plist ? plist[par] : par;
  for (int t = threadIdx.x; t < Sp; t += blockDim.x) mp_p[gpar * Sp + t] = Sacc[t];
}

// ---------------------------------------------------------------------------
// L2L for one parent's children: shift the parent local to each child,
// fold, weighted theta anterpolation (2 n_p -> 2 n_c), unfold, phi
// anterpolation (n_p -> n_c), accumulate into the child locals
// (traversal.cpp:583-661; the quadrature weights and the adjoint scale are
// folded into the theta matrix).
__global__ void __launch_bounds__(kFusedThreads) k_l2l_fused(
    int n_c, int n_p, FusedPlan plan, const int* __restrict__ plist, PassDims th, PassDims phi, const int* __restrict__ child_off,
    const int* __restrict__ children, const uint8_t* __restrict__ oct_c, const double2* __restrict__ loc_p,
    double2* __restrict__ loc_c, const double* __restrict__ RthT, const double* __restrict__ vth,
    const double* __restrict__ RphiT, const double* __restrict__ vphi, const double2* __restrict__ shift_dn) {
  extern __shared__ double2 sm[];
  const int CB = plan.CB;
  const int half = n_p / 2, Sc = n_c * n_c, Sp = n_p * n_p;
  const int par = blockIdx.x;
  const int cb = child_off[par], ce = child_off[par + 1];
  if (cb == ce) return;
  double2* Lp = sm;
  double2* Fs = plan.dbuf ? sm + Sp : sm;
  double2* Ns = Fs + CB * half * th.lda;
  const double2* lpg = loc_p + int64_t(plist ? plist[par] : par) * Sp;
  if (plan.dbuf) {
    for (int t = threadIdx.x; t < Sp; t += blockDim.x) cp_async16(Lp + t, lpg + t, true);
    cp_async_commit();
  }
  for (int t = threadIdx.x; t < CB * half * th.lda; t += blockDim.x) Fs[t] = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < CB * n_c * phi.lda; t += blockDim.x) Ns[t] = make_double2(0.0, 0.0);
  cp_async_wait_all();
  __syncthreads();
  const double2* L = plan.dbuf ? Lp : lpg;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  double* lc = reinterpret_cast<double*>(loc_c);

  for (int b0 = cb; b0 < ce; b0 += CB) {
    const int nb = min(CB, ce - b0);
    // 1. shifted parent, folded: Fs[c][p][i] (warp per circle row, lanes over i)
    for (int row = warp; row < CB * half; row += nwarp) {
      const int c = row / half, p = row - c * half;
      double2* f = Fs + row * th.lda;
      if (c < nb) {
        const double2* sh = shift_dn + int64_t(oct_c[children[b0 + c]]) * Sp;
        for (int i = lane; i < 2 * n_p; i += 32) {
          const int s = i < n_p ? i * n_p + p : (2 * n_p - 1 - i) * n_p + p + half;
          f[i] = cmul(L[s], __ldg(sh + s));
        }
      } else {
        for (int i = lane; i < 2 * n_p; i += 32) f[i] = make_double2(0.0, 0.0);
      }
    }
    __syncthreads();
    rank1_column(CB * half, 2 * n_p, vth, [&](int r) { return Fs + r * th.lda; });
    __syncthreads();
    // 2. theta pass: rows (child, circle, re/im), unfolded into Ns[c][row][col]
    warp_gemm_rc(CB * half * 2, th.N, th.K, [&](int r) { return Fs + r * th.lda; }, RthT,
                 [&](int m0, int n0, double v0, double v1) {
                   const int r = m0 + g, ci = r >> 1, c = ci / half, p = ci - c * half;
                   if (c >= CB) return;
                   double2* base = Ns + c * n_c * phi.lda;
#pragma unroll
                   for (int q = 0; q < 2; ++q) {
                     const int n = n0 + 2 * tq + q;
                     if (n < 2 * n_c) {
                       const int row = n < n_c ? n : 2 * n_c - 1 - n;
                       const int col = n < n_c ? p : p + half;
                       set_part(base + row * phi.lda + col, r & 1, q ? v1 : v0);
                     }
                   }
                 });
    __syncthreads();
    rank1_column(CB * n_c, n_p, vphi, [&](int r) { return Ns + r * phi.lda; });
    __syncthreads();
    // 3. phi pass, accumulated into the child locals
    warp_gemm_rc(CB * n_c * 2, phi.N, phi.K, [&](int r) { return Ns + r * phi.lda; }, RphiT,
                 [&](int m0, int n0, double v0, double v1) {
                   const int r = m0 + g, ci = r >> 1, c = ci / n_c, row = ci - c * n_c;
                   if (c >= nb) return;
                   double* dst = lc + 2 * (int64_t(children[b0 + c]) * Sc + row * n_c) + (r & 1);
#pragma unroll
                   for (int q = 0; q < 2; ++q) {
                     const int n = n0 + 2 * tq + q;
                     if (n < n_c) dst[2 * n] += q ? v1 : v0;
                   }
                 });
    __syncthreads();
  }
}

}  // namespace hfmm_b200

#endif
