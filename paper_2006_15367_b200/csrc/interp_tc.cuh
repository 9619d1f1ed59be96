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
// batches of CB: everything between the child samples in HBM and the parent
// accumulators stays in shared memory / registers.
#ifndef HFMM_B200_INTERP_TC_CUH
#define HFMM_B200_INTERP_TC_CUH

#include "kernels.cuh"

namespace hfmm_b200 {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// Shape of one fused pass, computed on the host (all strides in double2).
struct PassDims {
  int K;    // padded reduction length (multiple of 4): n_in + 1 (rank-1 column) rounded up
  int N;    // padded output length (multiple of 8)
  int lda;  // smem row stride of the input rows (== 4 mod 8 to avoid bank conflicts)
  int ldo;  // smem row stride of the output rows (theta pass of M2M only)
};

// C(r, n) = sum_k A(r, k) B(k, n) for r < M (real rows, padded to 16),
// n < N, k < K; B is a K x N row-major real matrix in global memory (L1
// resident, shared by all CTAs).  A(r, k) is part (r & 1) of the complex
// element at row (r >> 1), column k of a double2 smem array with row stride
// lda.  Warp tile 16 x 16 (2 x 2 DMMA tiles), warps stride over tiles.
template <class Store>
__device__ __forceinline__ void warp_gemm_rc(int M, int N, int K, const double2* __restrict__ A, int lda,
                                             const double* __restrict__ B, Store store) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int mt = (M + 15) >> 4, nt = (N + 15) >> 4;
  const double* Ad = reinterpret_cast<const double*>(A);
  for (int w = warp; w < mt * nt; w += nwarp) {
    const int m0 = (w / nt) << 4, n0 = (w % nt) << 4;
    double c[2][2][2] = {{{0.0, 0.0}, {0.0, 0.0}}, {{0.0, 0.0}, {0.0, 0.0}}};
    const int r0 = m0 + g, r1 = m0 + 8 + g;
    const double* a0p = Ad + 2 * (r0 >> 1) * lda + (r0 & 1);
    const double* a1p = Ad + 2 * (r1 >> 1) * lda + (r1 & 1);
    const bool bn1 = n0 + 8 < N;
    for (int k = 0; k < K; k += 4) {
      const int kk = k + tq;
      const double a0 = r0 < M ? a0p[2 * kk] : 0.0;
      const double a1 = r1 < M ? a1p[2 * kk] : 0.0;
      const double b0 = __ldg(B + kk * N + n0 + g);
      const double b1 = bn1 ? __ldg(B + kk * N + n0 + 8 + g) : 0.0;
      dmma884(c[0][0][0], c[0][0][1], a0, b0);
      dmma884(c[0][1][0], c[0][1][1], a0, b1);
      dmma884(c[1][0][0], c[1][0][1], a1, b0);
      dmma884(c[1][1][0], c[1][1][1], a1, b1);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = m0 + 8 * i + g, n = n0 + 8 * j + 2 * tq;
        if (r < M && n < N) {  // N is a multiple of 8: n and n + 1 are both in range
          store(r, n, c[i][j][0]);
          store(r, n + 1, c[i][j][1]);
        }
      }
  }
}

// x[row][K_in] = i * (v . x[row][0:K_in]) for `rows` complex rows (warp per row).
__device__ __forceinline__ void rank1_column(double2* X, int rows, int ld, int kin, const double* __restrict__ v) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  for (int r = warp; r < rows; r += nwarp) {
    double sr = 0.0, si = 0.0;
    double2* x = X + r * ld;
    for (int k = lane; k < kin; k += 32) {
      const double vk = __ldg(v + k);
      sr = fma(vk, x[k].x, sr);
      si = fma(vk, x[k].y, si);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      sr += __shfl_xor_sync(0xffffffffu, sr, off);
      si += __shfl_xor_sync(0xffffffffu, si, off);
    }
    if (lane == 0) x[kin] = make_double2(-si, sr);
  }
}

__device__ __forceinline__ void set_part(double2* p, int part, double v) {
  reinterpret_cast<double*>(p)[part] = v;
}

constexpr int kFusedThreads = 256;
constexpr int kFusedE = 12;  // parent samples per thread (S_p <= 3072)

// ---------------------------------------------------------------------------
// M2M for one parent: phi upsample (n_c -> n_p per theta row), fold, theta
// upsample (2 n_c -> 2 n_p per great circle), unfold, shift, sum over the
// children in child order (traversal.cpp:322-429, sphere_grid.cpp:183-192).
__global__ void __launch_bounds__(kFusedThreads) k_m2m_fused(
    int n_c, int n_p, int CB, PassDims phi, PassDims th, const int* __restrict__ child_off,
    const int* __restrict__ children, const uint8_t* __restrict__ oct_c, const double2* __restrict__ mp_c,
    double2* __restrict__ mp_p, const double* __restrict__ RphiT, const double* __restrict__ vphi,
    const double* __restrict__ RthT, const double* __restrict__ vth, const double2* __restrict__ shift_up) {
  extern __shared__ double2 sm[];
  const int half = n_p / 2, Sc = n_c * n_c, Sp = n_p * n_p;
  const int xs_size = CB * n_c * phi.lda, gs_size = CB * half * th.ldo;
  double2* U = sm;                                       // X rows, later G rows
  double2* Fs = sm + (xs_size > gs_size ? xs_size : gs_size);
  const int par = blockIdx.x;
  const int cb = child_off[par], ce = child_off[par + 1];

  // Fs padding columns (beyond 2 n_c + 1) stay zero for the whole kernel.
  for (int t = threadIdx.x; t < CB * half * th.lda; t += blockDim.x) Fs[t] = make_double2(0.0, 0.0);

  double2 acc[kFusedE];
#pragma unroll
  for (int r = 0; r < kFusedE; ++r) acc[r] = make_double2(0.0, 0.0);

  for (int b0 = cb; b0 < ce; b0 += CB) {
    const int nb = min(CB, ce - b0);
    __syncthreads();
    // 1. child samples -> X rows [c][i][0:n_c], zero padding
    for (int t = threadIdx.x; t < CB * n_c * phi.lda; t += blockDim.x) {
      const int c = t / (n_c * phi.lda), rem = t % (n_c * phi.lda);
      const int i = rem / phi.lda, k = rem % phi.lda;
      double2 v = make_double2(0.0, 0.0);
      if (c < nb && k < n_c) v = mp_c[int64_t(children[b0 + c]) * Sc + i * n_c + k];
      U[t] = v;
    }
    __syncthreads();
    rank1_column(U, CB * n_c, phi.lda, n_c, vphi);
    __syncthreads();
    // 2. phi pass, stored folded into Fs[c][p][ii]
    warp_gemm_rc(CB * n_c * 2, phi.N, phi.K, U, phi.lda, RphiT, [&](int r, int n, double v) {
      if (n >= n_p) return;
      const int ci = r >> 1, c = ci / n_c, i = ci % n_c;
      const int p = n < half ? n : n - half;
      const int ii = n < half ? i : 2 * n_c - 1 - i;
      set_part(Fs + (c * half + p) * th.lda + ii, r & 1, v);
    });
    __syncthreads();
    rank1_column(Fs, CB * half, th.lda, 2 * n_c, vth);
    __syncthreads();
    // 3. theta pass into G rows [c][p][n] (aliases the X rows)
    warp_gemm_rc(CB * half * 2, th.N, th.K, Fs, th.lda, RthT, [&](int r, int n, double v) {
      set_part(U + (r >> 1) * th.ldo + n, r & 1, v);
    });
    __syncthreads();
    // 4. unfold, shift, accumulate in child order
#pragma unroll
    for (int r = 0; r < kFusedE; ++r) {
      const int s = threadIdx.x + r * kFusedThreads;
      if (s < Sp) {
        const int row = s / n_p, col = s % n_p;
        const int p = col < half ? col : col - half;
        const int n = col < half ? row : 2 * n_p - 1 - row;
        for (int c = 0; c < nb; ++c) {
          const double2 g = U[(c * half + p) * th.ldo + n];
          const double2 sh = shift_up[oct_c[children[b0 + c]] * Sp + s];
          acc[r].x += g.x * sh.x - g.y * sh.y;
          acc[r].y += g.x * sh.y + g.y * sh.x;
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kFusedE; ++r) {
    const int s = threadIdx.x + r * kFusedThreads;
    if (s < Sp) mp_p[int64_t(par) * Sp + s] = acc[r];
  }
}

// ---------------------------------------------------------------------------
// L2L for one parent's children: shift the parent local to each child,
// fold, weighted theta anterpolation (2 n_p -> 2 n_c), unfold, phi
// anterpolation (n_p -> n_c), accumulate into the child locals
// (traversal.cpp:583-661; the quadrature weights and the adjoint scale are
// folded into the theta matrix).
__global__ void __launch_bounds__(kFusedThreads) k_l2l_fused(
    int n_c, int n_p, int CB, PassDims th, PassDims phi, const int* __restrict__ child_off,
    const int* __restrict__ children, const uint8_t* __restrict__ oct_c, const double2* __restrict__ loc_p,
    double2* __restrict__ loc_c, const double* __restrict__ RthT, const double* __restrict__ vth,
    const double* __restrict__ RphiT, const double* __restrict__ vphi, const double2* __restrict__ shift_dn) {
  extern __shared__ double2 sm[];
  const int half = n_p / 2, Sc = n_c * n_c, Sp = n_p * n_p;
  double2* Lp = sm;
  double2* Fs = Lp + Sp;
  double2* Ns = Fs + CB * half * th.lda;
  const int par = blockIdx.x;
  const int cb = child_off[par], ce = child_off[par + 1];
  if (cb == ce) return;
  for (int t = threadIdx.x; t < Sp; t += blockDim.x) Lp[t] = loc_p[int64_t(par) * Sp + t];
  for (int t = threadIdx.x; t < CB * half * th.lda; t += blockDim.x) Fs[t] = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < CB * n_c * phi.lda; t += blockDim.x) Ns[t] = make_double2(0.0, 0.0);

  for (int b0 = cb; b0 < ce; b0 += CB) {
    const int nb = min(CB, ce - b0);
    __syncthreads();
    // 1. shifted parent, folded: Fs[c][p][i], i < 2 n_p
    for (int t = threadIdx.x; t < CB * half * 2 * n_p; t += blockDim.x) {
      const int c = t / (half * 2 * n_p), rem = t % (half * 2 * n_p);
      const int p = rem / (2 * n_p), i = rem % (2 * n_p);
      double2 v = make_double2(0.0, 0.0);
      if (c < nb) {
        const int s = i < n_p ? i * n_p + p : (2 * n_p - 1 - i) * n_p + p + half;
        v = cmul(Lp[s], shift_dn[oct_c[children[b0 + c]] * Sp + s]);
      }
      Fs[(c * half + p) * th.lda + i] = v;
    }
    __syncthreads();
    rank1_column(Fs, CB * half, th.lda, 2 * n_p, vth);
    __syncthreads();
    // 2. theta pass, unfolded into narrow rows Ns[c][row][col] (n_c x n_p)
    warp_gemm_rc(CB * half * 2, th.N, th.K, Fs, th.lda, RthT, [&](int r, int n, double v) {
      if (n >= 2 * n_c) return;
      const int ci = r >> 1, c = ci / half, p = ci % half;
      const int row = n < n_c ? n : 2 * n_c - 1 - n;
      const int col = n < n_c ? p : p + half;
      set_part(Ns + (c * n_c + row) * phi.lda + col, r & 1, v);
    });
    __syncthreads();
    rank1_column(Ns, CB * n_c, phi.lda, n_p, vphi);
    __syncthreads();
    // 3. phi pass, accumulated into the child locals
    double* lc = reinterpret_cast<double*>(loc_c);
    warp_gemm_rc(CB * n_c * 2, phi.N, phi.K, Ns, phi.lda, RphiT, [&](int r, int n, double v) {
      if (n >= n_c) return;
      const int ci = r >> 1, c = ci / n_c, row = ci % n_c;
      if (c >= nb) return;
      double* dst = lc + 2 * (int64_t(children[b0 + c]) * Sc + row * n_c + n) + (r & 1);
      *dst += v;
    });
  }
}

}  // namespace hfmm_b200

#endif
