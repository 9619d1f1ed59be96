// FP64 tensor-core building blocks shared by the resampling (M2M / L2L) and
// M2L kernels: DMMA (mma.sync m8n8k4 f64, SASS DMMA.8x8x4) and a warp-tiled
// real GEMM over complex rows.
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
#ifndef HFMM_B200_DMMA_CUH
#define HFMM_B200_DMMA_CUH

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

}  // namespace hfmm_b200

#endif
