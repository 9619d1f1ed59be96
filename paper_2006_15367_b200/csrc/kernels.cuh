// sm_100a kernels of the MLFMA evaluation phase.  FP64 throughout (the
// reference is FP64; parity is 1e-10 relative L2).  Each kernel cites the
// reference loop it replaces.
#ifndef HFMM_B200_KERNELS_CUH
#define HFMM_B200_KERNELS_CUH

#include <cuda_runtime.h>

#include <cstdint>

namespace hfmm_b200 {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

constexpr int kSlots = 343;  // (ox, oy, oz) in [-3, 3]^3

// sin and cos of a moderate argument (|x| < 2^20): Cody-Waite reduction by
// pi/2 with the round-to-nearest quadrant taken from a 1.5*2^52 magic add,
// then Taylor polynomials on [-pi/4, pi/4] (truncation < 6e-17).  No slow
// path: the arguments on this path are phases k |r| of a few radians.
__device__ __forceinline__ void sincos_fast(double x, double* sp, double* cp) {
  const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  const double t = fma(x, 0.63661977236758138, kMagic);
  const int quad = __double2loint(t);
  const double n = t - kMagic;
  double y = fma(n, -1.5707963267948966, x);
  y = fma(n, -6.123233995736766e-17, y);
  const double y2 = y * y;
  double ps = -7.6471637318198164759e-13;            // -1/15!
  ps = fma(ps, y2, 1.6059043836821614599e-10);        //  1/13!
  ps = fma(ps, y2, -2.5052108385441718775e-08);       // -1/11!
  ps = fma(ps, y2, 2.7557319223985890653e-06);        //  1/9!
  ps = fma(ps, y2, -1.9841269841269841270e-04);       // -1/7!
  ps = fma(ps, y2, 8.3333333333333333333e-03);        //  1/5!
  ps = fma(ps, y2, -1.6666666666666666667e-01);       // -1/3!
  const double sn = fma(ps * y2, y, y);
  double pc = 4.7794773323873852974e-14;              //  1/16!
  pc = fma(pc, y2, -1.1470745597729724714e-11);       // -1/14!
  pc = fma(pc, y2, 2.0876756987868098979e-09);        //  1/12!
  pc = fma(pc, y2, -2.7557319223985890653e-07);       // -1/10!
  pc = fma(pc, y2, 2.4801587301587301587e-05);        //  1/8!
  pc = fma(pc, y2, -1.3888888888888888889e-03);       // -1/6!
  pc = fma(pc, y2, 4.1666666666666666667e-02);        //  1/4!
  pc = fma(pc, y2, -0.5);
  const double cs = fma(pc, y2, 1.0);
  const double s1 = (quad & 1) ? cs : sn;
  const double c1 = (quad & 1) ? sn : cs;
  *sp = (quad & 2) ? -s1 : s1;
  *cp = ((quad + 1) & 2) ? -c1 : c1;
}

// cp.async (Ampere+ LDGSTS) 16-byte copy; src-size 0 zero-fills the destination.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }  // (ox, oy, oz) in [-3, 3]^3

// ---------------------------------------------------------------------------
// Translation operators T[slot][s] (operators.cpp:39-80): Legendre series with
// host-computed coefficients (-i)^l (2l+1) h_l^(2)(k|D|).
__global__ void k_tbuild(int64_t S, int trunc, const double* __restrict__ dir, double side,
                         const double2* __restrict__ tcoef, const uint8_t* __restrict__ used,
                         double2* __restrict__ T) {
  const int slot = blockIdx.y;
  if (!used[slot]) return;
  extern __shared__ double2 coef[];
  for (int l = threadIdx.x; l <= trunc; l += blockDim.x) coef[l] = tcoef[slot * (trunc + 1) + l];
  __syncthreads();
  const int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const double Dx = double(slot / 49 - 3) * side, Dy = double((slot / 7) % 7 - 3) * side,
               Dz = double(slot % 7 - 3) * side;
  const double dist = sqrt(Dx * Dx + Dy * Dy + Dz * Dz);
  const double inv = 1.0 / dist;
  const double hx = Dx * inv, hy = Dy * inv, hz = Dz * inv;
  const double u = dir[3 * s] * hx + dir[3 * s + 1] * hy + dir[3 * s + 2] * hz;
  double pm1 = 0.0, p0 = 1.0;
  double2 acc = coef[0];
  for (int l = 1; l <= trunc; ++l) {
    const double p1 = (double(2 * l - 1) * u * p0 - double(l - 1) * pm1) / double(l);
    pm1 = p0;
    p0 = p1;
    acc.x = fma(coef[l].x, p0, acc.x);
    acc.y = fma(coef[l].y, p0, acc.y);
  }
  T[slot * S + s] = acc;
}

// ---------------------------------------------------------------------------
// C2M (operators.cpp:15-26, driver traversal.cpp:306-320): one CTA per leaf,
// threads over samples (R per thread), particles staged through shared memory.
constexpr int kC2MChunk = 256;
constexpr int kC2MR = 4;
__global__ void __launch_bounds__(128) k_c2m(int64_t leaf_b, const int64_t* __restrict__ leaf_start,
                                             const double* __restrict__ x, const double* __restrict__ y,
                                             const double* __restrict__ z, const double2* __restrict__ q,
                                             const double* __restrict__ centers,
                                             const double* __restrict__ dir, int64_t S, double k,
                                             double2* __restrict__ mp) {
  __shared__ double sx[kC2MChunk], sy[kC2MChunk], sz[kC2MChunk];
  __shared__ double2 sq[kC2MChunk];
  const int64_t leaf = leaf_b + blockIdx.x;
  const int64_t p0 = leaf_start[leaf], p1 = leaf_start[leaf + 1];
  const double cx = centers[3 * leaf], cy = centers[3 * leaf + 1], cz = centers[3 * leaf + 2];
  for (int64_t sb = 0; sb < S; sb += int64_t(blockDim.x) * kC2MR) {
    double2 acc[kC2MR];
    double kx[kC2MR], ky[kC2MR], kz[kC2MR];
#pragma unroll
    for (int r = 0; r < kC2MR; ++r) {
      acc[r] = make_double2(0.0, 0.0);
      const int64_t s = sb + threadIdx.x + int64_t(r) * blockDim.x;
      const bool ok = s < S;
      kx[r] = ok ? dir[3 * s] : 0.0;
      ky[r] = ok ? dir[3 * s + 1] : 0.0;
      kz[r] = ok ? dir[3 * s + 2] : 0.0;
    }
    for (int64_t pb = p0; pb < p1; pb += kC2MChunk) {
      const int n = int(p1 - pb < kC2MChunk ? p1 - pb : kC2MChunk);
      __syncthreads();
      for (int t = threadIdx.x; t < n; t += blockDim.x) {
        sx[t] = x[pb + t] - cx;
        sy[t] = y[pb + t] - cy;
        sz[t] = z[pb + t] - cz;
        sq[t] = q[pb + t];
      }
      __syncthreads();
      for (int t = 0; t < n; ++t) {
        const double dx = sx[t], dy = sy[t], dz = sz[t];
        const double2 qq = sq[t];
#pragma unroll
        for (int r = 0; r < kC2MR; ++r) {
          double sn, cs;
          sincos_fast(k * (kx[r] * dx + ky[r] * dy + kz[r] * dz), &sn, &cs);
          acc[r].x += qq.x * cs - qq.y * sn;
          acc[r].y += qq.x * sn + qq.y * cs;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kC2MR; ++r) {
      const int64_t s = sb + threadIdx.x + int64_t(r) * blockDim.x;
      if (s < S) mp[leaf * S + s] = acc[r];
    }
  }
}

// ---------------------------------------------------------------------------
// M2M phi pass + fold (sphere_grid.cpp:164-171 then fold_transpose :72-83):
// W[i][jj] = sum_j P_up[jj][j] X[i][j]; stored folded F[p][ii] (n_p/2 circles
// of length 2 n_c).  One CTA per child.
__global__ void k_m2m_phi(int n_c, int n_p, int64_t child_b, const double2* __restrict__ mp_c,
                          const double2* __restrict__ PuT, double2* __restrict__ F) {
  extern __shared__ double2 sX[];
  const int64_t child = child_b + blockIdx.x;
  const int Sc = n_c * n_c;
  for (int t = threadIdx.x; t < Sc; t += blockDim.x) sX[t] = mp_c[child * Sc + t];
  __syncthreads();
  const int half = n_p / 2;
  double2* Fc = F + (child - child_b) * int64_t(n_p) * n_c;
  for (int e = threadIdx.x; e < n_c * n_p; e += blockDim.x) {
    const int i = e / n_p, jj = e % n_p;
    double2 acc = make_double2(0.0, 0.0);
    for (int j = 0; j < n_c; ++j) cmac(acc, PuT[j * n_p + jj], sX[i * n_c + j]);
    const int p = jj < half ? jj : jj - half;
    const int ii = jj < half ? i : 2 * n_c - 1 - i;
    Fc[p * (2 * n_c) + ii] = acc;
  }
}

// M2M theta pass + unfold + shift + ordered aggregation (sphere_grid.cpp:173-181,
// :85-102; operators.cpp:28-37; traversal.cpp:392-425).  Grid (parent, circle
// chunk); each thread keeps E parent samples in registers over the children.
constexpr int kThetaE = 8;
__global__ void __launch_bounds__(256) k_m2m_theta(int n_c, int n_p, int CP, int64_t par_b,
                                                   int64_t child_b,
                                                   const int* __restrict__ child_off,
                                                   const int* __restrict__ children,
                                                   const uint8_t* __restrict__ oct_c,
                                                   const double2* __restrict__ F,
                                                   const double2* __restrict__ TuT,
                                                   const double2* __restrict__ shift_up,
                                                   double2* __restrict__ mp_p) {
  extern __shared__ double2 sF[];
  const int64_t par = par_b + blockIdx.x;
  const int half = n_p / 2, Lc = 2 * n_c, Lp = 2 * n_p;
  const int64_t Sp = int64_t(n_p) * n_p;
  const int p0 = blockIdx.y * CP, p1 = min(half, p0 + CP), ncirc = p1 - p0;
  const int nout = ncirc * Lp;
  double2 acc[kThetaE];
  int sidx[kThetaE];
#pragma unroll
  for (int r = 0; r < kThetaE; ++r) {
    acc[r] = make_double2(0.0, 0.0);
    const int e = threadIdx.x + r * blockDim.x;
    int s = -1;
    if (e < nout) {
      const int pl = e / Lp, j = e % Lp, p = p0 + pl;
      s = j < n_p ? j * n_p + p : (Lp - 1 - j) * n_p + p + half;
    }
    sidx[r] = s;
  }
  for (int kk = child_off[par]; kk < child_off[par + 1]; ++kk) {
    const int64_t ch = children[kk];
    const int o = oct_c[ch];
    const double2* Fc = F + (ch - child_b) * int64_t(n_p) * n_c + int64_t(p0) * Lc;
    __syncthreads();
    for (int t = threadIdx.x; t < ncirc * Lc; t += blockDim.x) sF[t] = Fc[t];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kThetaE; ++r) {
      const int e = threadIdx.x + r * blockDim.x;
      if (e < nout) {
        const int pl = e / Lp, j = e % Lp;
        double2 g = make_double2(0.0, 0.0);
        const double2* f = sF + pl * Lc;
        for (int i = 0; i < Lc; ++i) cmac(g, TuT[i * Lp + j], f[i]);
        const double2 sh = shift_up[o * Sp + sidx[r]];
        const double2 v = cmul(g, sh);
        acc[r].x += v.x;
        acc[r].y += v.y;
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kThetaE; ++r)
    if (sidx[r] >= 0) mp_p[par * Sp + sidx[r]] = acc[r];
}

// ---------------------------------------------------------------------------
// M2L (operators.cpp:82-87, traversal.cpp:443-581): L_o[s] = sum_far T[o-src][s] M_src[s].
__global__ void k_m2l(int64_t S, int64_t node_b, const int64_t* __restrict__ far_off,
                      const int2* __restrict__ far, const double2* __restrict__ T,
                      const double2* __restrict__ mp, double2* __restrict__ loc) {
  const int64_t o = node_b + blockIdx.x;
  const int64_t s = int64_t(blockIdx.y) * blockDim.x + threadIdx.x;
  if (s >= S) return;
  double2 acc = make_double2(0.0, 0.0);
  for (int64_t f = far_off[o]; f < far_off[o + 1]; ++f) {
    const int2 e = far[f];
    cmac(acc, mp[int64_t(e.x) * S + s], T[int64_t(e.y) * S + s]);
  }
  loc[o * S + s] = acc;
}

// ---------------------------------------------------------------------------
// L2L theta pass (fold, weighted theta anterpolation 2n_p -> 2n_c, unfold;
// traversal.cpp:648-661 with sphere_grid.cpp:194-214).  Grid (child, circle
// chunk); parent samples are shifted (operators.cpp:28-37) while staged.
__global__ void k_l2l_theta(int n_c, int n_p, int CP, int64_t child_b,
                            const int* __restrict__ parent_c, const uint8_t* __restrict__ oct_c,
                            const double2* __restrict__ loc_p, const double2* __restrict__ shift_dn,
                            const double2* __restrict__ TdT, double2* __restrict__ Nb) {
  extern __shared__ double2 sZ[];
  const int64_t child = child_b + blockIdx.x;
  const int64_t par = parent_c[child];
  const int o = oct_c[child];
  const int half = n_p / 2, Lc = 2 * n_c, Lp = 2 * n_p;
  const int64_t Sp = int64_t(n_p) * n_p;
  const int p0 = blockIdx.y * CP, p1 = min(half, p0 + CP), ncirc = p1 - p0;
  for (int t = threadIdx.x; t < ncirc * Lp; t += blockDim.x) {
    const int pl = t / Lp, i = t % Lp, p = p0 + pl;
    const int64_t s = i < n_p ? int64_t(i) * n_p + p : int64_t(Lp - 1 - i) * n_p + p + half;
    sZ[t] = cmul(loc_p[par * Sp + s], shift_dn[o * Sp + s]);
  }
  __syncthreads();
  double2* Nc = Nb + (child - child_b) * int64_t(n_c) * n_p;
  for (int e = threadIdx.x; e < ncirc * Lc; e += blockDim.x) {
    const int pl = e / Lc, j = e % Lc, p = p0 + pl;
    double2 g = make_double2(0.0, 0.0);
    const double2* f = sZ + pl * Lp;
    for (int i = 0; i < Lp; ++i) cmac(g, TdT[i * Lc + j], f[i]);
    const int row = j < n_c ? j : Lc - 1 - j;
    const int col = j < n_c ? p : p + half;
    Nc[row * n_p + col] = g;
  }
}

// L2L phi pass (n_p -> n_c per theta row) and accumulation into the child
// locals (traversal.cpp:658-660).  One CTA per child.
__global__ void k_l2l_phi(int n_c, int n_p, int64_t child_b, const double2* __restrict__ Nb,
                          const double2* __restrict__ PdT, double2* __restrict__ loc_c) {
  extern __shared__ double2 sN[];
  const int64_t child = child_b + blockIdx.x;
  const double2* Nc = Nb + (child - child_b) * int64_t(n_c) * n_p;
  for (int t = threadIdx.x; t < n_c * n_p; t += blockDim.x) sN[t] = Nc[t];
  __syncthreads();
  const int64_t Sc = int64_t(n_c) * n_c;
  for (int e = threadIdx.x; e < n_c * n_c; e += blockDim.x) {
    const int r = e / n_c, jc = e % n_c;
    double2 v = make_double2(0.0, 0.0);
    for (int jp = 0; jp < n_p; ++jp) cmac(v, PdT[jp * n_c + jc], sN[r * n_p + jp]);
    double2 cur = loc_c[child * Sc + e];
    cur.x += v.x;
    cur.y += v.y;
    loc_c[child * Sc + e] = cur;
  }
}

// ---------------------------------------------------------------------------
// L2T (operators.cpp:89-108, driver traversal.cpp:717-728): one CTA per leaf,
// one warp per observer, lanes over samples, warp-shuffle reduction.
__global__ void __launch_bounds__(128) k_l2t(int64_t leaf_b, const int64_t* __restrict__ leaf_start,
                                             const double* __restrict__ x, const double* __restrict__ y,
                                             const double* __restrict__ z,
                                             const double* __restrict__ centers,
                                             const double* __restrict__ dir,
                                             const double* __restrict__ wq, int64_t S, double k,
                                             const double2* __restrict__ loc,
                                             double2* __restrict__ pot) {
  extern __shared__ double2 sL[];
  double* sd = reinterpret_cast<double*>(sL + S);
  const int64_t leaf = leaf_b + blockIdx.x;
  for (int64_t s = threadIdx.x; s < S; s += blockDim.x) {
    const double2 v = loc[leaf * S + s];
    const double w = wq[s];
    sL[s] = make_double2(w * v.x, w * v.y);
    sd[3 * s] = dir[3 * s];
    sd[3 * s + 1] = dir[3 * s + 1];
    sd[3 * s + 2] = dir[3 * s + 2];
  }
  __syncthreads();
  const int64_t p0 = leaf_start[leaf], p1 = leaf_start[leaf + 1];
  const double cx = centers[3 * leaf], cy = centers[3 * leaf + 1], cz = centers[3 * leaf + 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const double c = -k / (16.0 * M_PI * M_PI);  // norm = (0, c)
  for (int64_t p = p0 + warp; p < p1; p += nw) {
    const double dx = x[p] - cx, dy = y[p] - cy, dz = z[p] - cz;
    double ar = 0.0, ai = 0.0;
    for (int64_t s = lane; s < S; s += 32) {
      double sn, cs;
      sincos_fast(-k * (sd[3 * s] * dx + sd[3 * s + 1] * dy + sd[3 * s + 2] * dz), &sn, &cs);
      const double2 v = sL[s];
      ar += v.x * cs - v.y * sn;
      ai += v.x * sn + v.y * cs;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      ar += __shfl_down_sync(0xffffffffu, ar, off);
      ai += __shfl_down_sync(0xffffffffu, ai, off);
    }
    if (lane == 0) pot[p] = make_double2(-c * ai, c * ar);
  }
}

// ---------------------------------------------------------------------------
// Near-field P2P (operators.cpp:110-122 with green kernel.cpp:9-14, driver
// traversal.cpp:768-786): one CTA per observer leaf; the near leaves'
// particles are streamed through shared memory as one concatenated list; G
// threads cooperate on one observer (G adapts to the leaf population) and
// reduce by warp shuffles.
constexpr int kP2PChunk = 512;
__global__ void __launch_bounds__(128) k_p2p(int64_t leaf_b, const int64_t* __restrict__ leaf_start,
                                             const int64_t* __restrict__ near_off,
                                             const int* __restrict__ near,
                                             const double* __restrict__ x, const double* __restrict__ y,
                                             const double* __restrict__ z,
                                             const double2* __restrict__ q, double k,
                                             double2* __restrict__ pot) {
  __shared__ double sx[kP2PChunk], sy[kP2PChunk], sz[kP2PChunk];
  __shared__ double2 sq[kP2PChunk];
  __shared__ int64_t pref[28], nbeg[27];
  const int64_t leaf = leaf_b + blockIdx.x;
  const int64_t p0 = leaf_start[leaf], p1 = leaf_start[leaf + 1];
  const int n_o = int(p1 - p0);
  const int64_t nb = near_off[leaf];
  const int nn = int(near_off[leaf + 1] - nb);
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int j = 0; j < nn; ++j) {
      const int lf = near[nb + j];
      pref[j] = run;
      nbeg[j] = leaf_start[lf];
      run += leaf_start[lf + 1] - leaf_start[lf];
    }
    pref[nn] = run;
  }
  __syncthreads();
  const int64_t total = pref[nn];
  int G = 32;
  while (G > 1 && G * n_o > int(blockDim.x)) G >>= 1;
  const int groups = blockDim.x / G;
  const int j = threadIdx.x % G;
  const double inv4pi = 1.0 / (4.0 * M_PI);
  for (int ob = 0; ob < n_o; ob += groups) {
    const int o = ob + threadIdx.x / G;
    const bool valid = o < n_o;
    const double xo = valid ? x[p0 + o] : 0.0, yo = valid ? y[p0 + o] : 0.0,
                 zo = valid ? z[p0 + o] : 0.0;
    double ar = 0.0, ai = 0.0;
    for (int64_t cb = 0; cb < total; cb += kP2PChunk) {
      const int n = int(total - cb < kP2PChunk ? total - cb : kP2PChunk);
      __syncthreads();
      for (int t = threadIdx.x; t < n; t += blockDim.x) {
        const int64_t v = cb + t;
        int jj = 0;
        while (pref[jj + 1] <= v) ++jj;
        const int64_t src = nbeg[jj] + (v - pref[jj]);
        sx[t] = x[src];
        sy[t] = y[src];
        sz[t] = z[src];
        sq[t] = q[src];
      }
      __syncthreads();
      if (valid) {
        for (int t = j; t < n; t += G) {
          const double dx = xo - sx[t], dy = yo - sy[t], dz = zo - sz[t];
          if (dx == 0.0 && dy == 0.0 && dz == 0.0) continue;  // self pair
          const double r = sqrt(dx * dx + dy * dy + dz * dz);
          double sn, cs;
          sincos_fast(-k * r, &sn, &cs);
          const double w = inv4pi / r;
          const double gr = cs * w, gi = sn * w;
          const double2 qq = sq[t];
          ar += gr * qq.x - gi * qq.y;
          ai += gr * qq.y + gi * qq.x;
        }
      }
    }
    for (int off = G >> 1; off > 0; off >>= 1) {
      ar += __shfl_down_sync(0xffffffffu, ar, off, G);
      ai += __shfl_down_sync(0xffffffffu, ai, off, G);
    }
    if (valid && j == 0) {
      double2 cur = pot[p0 + o];
      cur.x += ar;
      cur.y += ai;
      pot[p0 + o] = cur;
    }
  }
}

// ---------------------------------------------------------------------------
// Permutations between input order and Morton order (traversal.cpp:108-110, :809-815).
__global__ void k_gather_q(int64_t n, const int64_t* __restrict__ orig, const double2* __restrict__ q_in,
                           double2* __restrict__ q_sorted) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) q_sorted[i] = q_in[orig[i]];
}
__global__ void k_scatter_pot(int64_t b, int64_t e, const int64_t* __restrict__ orig,
                              const double2* __restrict__ pot_sorted, double2* __restrict__ pot_in) {
  const int64_t i = b + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < e) pot_in[orig[i]] = pot_sorted[i];
}

// ---------------------------------------------------------------------------
// Exchange packing (distributed mode): whole expansion rows and ghost particles.
__global__ void k_pack_rows(const double2* __restrict__ src, const int* __restrict__ nodes, int64_t S,
                            double2* __restrict__ dst) {
  const int64_t i = blockIdx.x;
  const int64_t node = nodes[i];
  for (int64_t s = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; s < S; s += int64_t(gridDim.y) * blockDim.x)
    dst[i * S + s] = src[node * S + s];
}
__global__ void k_add_rows(double2* __restrict__ dst, const int* __restrict__ nodes, int64_t S,
                           const double2* __restrict__ src) {
  const int64_t i = blockIdx.x;
  const int64_t node = nodes[i];
  for (int64_t s = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; s < S; s += int64_t(gridDim.y) * blockDim.x) {
    double2 a = dst[node * S + s];
    const double2 b = src[i * S + s];
    a.x += b.x;
    a.y += b.y;
    dst[node * S + s] = a;
  }
}
__global__ void k_zero_rows(double2* __restrict__ dst, const int* __restrict__ nodes, int64_t S) {
  const int64_t node = nodes[blockIdx.x];
  for (int64_t s = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; s < S; s += int64_t(gridDim.y) * blockDim.x)
    dst[node * S + s] = make_double2(0.0, 0.0);
}
__global__ void k_pack_particles(int64_t n, const int64_t* __restrict__ idx, const double* __restrict__ x,
                                 const double* __restrict__ y, const double* __restrict__ z,
                                 const double2* __restrict__ q, double* __restrict__ buf) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t p = idx[i];
  buf[5 * i] = x[p];
  buf[5 * i + 1] = y[p];
  buf[5 * i + 2] = z[p];
  buf[5 * i + 3] = q[p].x;
  buf[5 * i + 4] = q[p].y;
}
__global__ void k_unpack_particles(int64_t n, const int64_t* __restrict__ idx, const double* __restrict__ buf,
                                   double* __restrict__ x, double* __restrict__ y, double* __restrict__ z,
                                   double2* __restrict__ q) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t p = idx[i];
  x[p] = buf[5 * i];
  y[p] = buf[5 * i + 1];
  z[p] = buf[5 * i + 2];
  q[p] = make_double2(buf[5 * i + 3], buf[5 * i + 4]);
}
__global__ void k_gather_q_range(int64_t b, int64_t e, const int64_t* __restrict__ orig,
                                 const double2* __restrict__ q_in, double2* __restrict__ q_sorted) {
  const int64_t i = b + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < e) q_sorted[i] = q_in[orig[i]];
}

// ---------------------------------------------------------------------------
// Direct O(N M) sum (kernel.cpp:16-41): one CTA per observer; the first exact
// coincidence is the self term; a second one flags an error.
__global__ void k_direct(int64_t n, const double* __restrict__ x, const double* __restrict__ y,
                         const double* __restrict__ z, const double2* __restrict__ q,
                         const int64_t* __restrict__ obs, double k, double2* __restrict__ out,
                         int* __restrict__ err) {
  __shared__ double rr[32], ri[32];
  __shared__ int rc[32];
  const int64_t m = obs[blockIdx.x];
  const double xo = x[m], yo = y[m], zo = z[m];
  double ar = 0.0, ai = 0.0;
  int zeros = 0;
  const double inv4pi = 1.0 / (4.0 * M_PI);
  for (int64_t s = threadIdx.x; s < n; s += blockDim.x) {
    const double dx = xo - x[s], dy = yo - y[s], dz = zo - z[s];
    if (dx == 0.0 && dy == 0.0 && dz == 0.0) {
      ++zeros;
      continue;
    }
    const double r = sqrt(dx * dx + dy * dy + dz * dz);
    double sn, cs;
    sincos(-k * r, &sn, &cs);
    const double w = inv4pi / r;
    const double2 qq = q[s];
    ar += (cs * w) * qq.x - (sn * w) * qq.y;
    ai += (cs * w) * qq.y + (sn * w) * qq.x;
  }
  for (int off = 16; off > 0; off >>= 1) {
    ar += __shfl_down_sync(0xffffffffu, ar, off);
    ai += __shfl_down_sync(0xffffffffu, ai, off);
    zeros += __shfl_down_sync(0xffffffffu, zeros, off);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    rr[w] = ar;
    ri[w] = ai;
    rc[w] = zeros;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    int c = 0;
    for (int i = 0; i < int(blockDim.x >> 5); ++i) {
      a += rr[i];
      b += ri[i];
      c += rc[i];
    }
    out[blockIdx.x] = make_double2(a, b);
    if (c > 1) atomicExch(err, 1);
  }
}

}  // namespace hfmm_b200

#endif
