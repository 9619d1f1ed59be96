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
// then the published minimax kernels of fdlibm (__kernel_sin / __kernel_cos,
// degree 13 / 14 on [-pi/4, pi/4], error < 2^-58).  No slow path: the
// arguments on this path are phases k |r| of a few radians.  Coefficients
// live in the constant bank (64-bit immediates cannot be encoded in DFMA).
__constant__ double kSinCos[14] = {
    1.58969099521155010221e-10, -2.50507602534068634195e-08, 2.75573137070700676789e-06,
    -1.98412698298579493134e-04, 8.33333333332248946124e-03, -1.66666666666666324348e-01,  // S6..S1
    -1.13596475577881948265e-11, 2.08757232129817482790e-09, -2.75573143513906633035e-07,
    2.48015872894767294178e-05, -1.38888888888741095749e-03, 4.16666666666666019037e-02,   // C6..C1
    0.63661977236758138, -6.123233995736766e-17};  // 2/pi, -(pi/2)_lo
// cos(y) = 1 - y^2/2 + y^4 Q(y^2) on |y| <= pi/4 with a degree-4 Q (our own
// Remez fit in 50-digit arithmetic, tools/remez_cos.py): max error 7.7e-17,
// below half an ulp of 1, one FMA shorter than fdlibm's degree-5 Q.
__constant__ double kCos5[5] = {2.0647738026849685246e-9, -2.7555567133567867496e-7, 2.480158097168681492e-5,
                                -1.3888888878274371275e-3, 4.1666666666602257401e-2};

__device__ __forceinline__ void sincos_fast(double x, double* sp, double* cp) {
  const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  const double t = fma(x, kSinCos[12], kMagic);
  const int quad = __double2loint(t);
  const double n = t - kMagic;
  double y = fma(n, -1.5707963267948966, x);
  y = fma(n, kSinCos[13], y);
  const double y2 = y * y;
  double ps = kSinCos[0];
#pragma unroll
  for (int i = 1; i < 6; ++i) ps = fma(ps, y2, kSinCos[i]);
  const double sn = fma(ps * y2, y, y);
  double pc = kSinCos[6];
#pragma unroll
  for (int i = 7; i < 12; ++i) pc = fma(pc, y2, kSinCos[i]);
  const double cs = fma(pc, y2 * y2, fma(-0.5, y2, 1.0));
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
  // coefficients + Legendre recurrence factors a_l = (2l-1)/l, b_l = (l-1)/l
  // (one division per l per CTA instead of one per l per sample)
  extern __shared__ double2 coef[];
  double2* ab = coef + (trunc + 1);
  for (int l = threadIdx.x; l <= trunc; l += blockDim.x) {
    coef[l] = tcoef[slot * (trunc + 1) + l];
    ab[l] = l > 0 ? make_double2(double(2 * l - 1) / double(l), double(l - 1) / double(l)) : make_double2(0.0, 0.0);
  }
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
    const double2 f = ab[l];
    const double p1 = fma(f.x * u, p0, -f.y * pm1);
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
      if (s < S) mp[int64_t(blockIdx.x) * S + s] = acc[r];  // row: leaf - leaf_b
    }
  }
}

// ---------------------------------------------------------------------------
// M2L (operators.cpp:82-87, traversal.cpp:443-581): L_o[s] = sum_far T[o-src][s] M_src[s].
// nodes != nullptr (distributed mode): blockIdx.x indexes the held observers.
__global__ void k_m2l(int64_t S, int64_t node_b, const int* __restrict__ nodes, const int64_t* __restrict__ far_off,
                      const int2* __restrict__ far, const double2* __restrict__ T,
                      const double2* __restrict__ mp, double2* __restrict__ loc) {
  const int64_t o = nodes ? int64_t(nodes[blockIdx.x]) : node_b + blockIdx.x;
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
// Quad-symmetric C2M / L2T.  The sample grid (sphere_grid.cpp:25-50) is
// symmetric: theta_{n-1-i} = pi - theta_i and phi_{j+n/2} = phi_j + pi, so the
// four samples (i, j), (n-1-i, j), (i, j+n/2), (n-1-i, j+n/2) of a quad have
// phases  A + B, A - B, -A + B, -A - B  with
//   A = k sin(theta_i) (x cos(phi_j) + y sin(phi_j)),  B = k z cos(theta_i)
// (A, B read from the direction table of sample (i, j)).  One sincos of A per
// quad and one of B per theta pair and particle give all four exponentials
// (a quarter of the direct sincos count); the phases equal the reference's
// per-sample ones to rounding.  One warp per leaf.
constexpr int kQuadHalfMax = 16;  // n/2 <= 16 (leaf grids of the BASELINE configs: n <= 26)
constexpr int kQuadP = 32;        // particles per B-table chunk


// ---------------------------------------------------------------------------
// L2T (operators.cpp:89-108, driver traversal.cpp:717-728): one CTA per leaf,
// one warp per observer, lanes over samples, warp-shuffle reduction.
constexpr int kL2TChunk = 1024;  // samples staged per pass (40 KB of shared memory)
__global__ void __launch_bounds__(128) k_l2t(int64_t leaf_b, const int64_t* __restrict__ leaf_start,
                                             const double* __restrict__ x, const double* __restrict__ y,
                                             const double* __restrict__ z,
                                             const double* __restrict__ centers,
                                             const double* __restrict__ dir,
                                             const double* __restrict__ wq, int64_t S, double k,
                                             const double2* __restrict__ loc,
                                             double2* __restrict__ pot) {
  __shared__ double2 sL[kL2TChunk];
  __shared__ double sd[3 * kL2TChunk];
  const int64_t leaf = leaf_b + blockIdx.x;
  const int64_t p0 = leaf_start[leaf], p1 = leaf_start[leaf + 1];
  const double cx = centers[3 * leaf], cy = centers[3 * leaf + 1], cz = centers[3 * leaf + 2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const double c = -k / (16.0 * M_PI * M_PI);  // norm = (0, c)
  // Samples in chunks of kL2TChunk (any leaf grid); a particle stays with one
  // warp, which adds the chunk sums in chunk order (deterministic).
  for (int64_t sb = 0; sb < S; sb += kL2TChunk) {
    const int ns = int(S - sb < kL2TChunk ? S - sb : kL2TChunk);
    __syncthreads();
    for (int t = threadIdx.x; t < ns; t += blockDim.x) {
      const double2 v = loc[int64_t(blockIdx.x) * S + sb + t];  // row: leaf - leaf_b
      const double w = wq[sb + t];
      sL[t] = make_double2(w * v.x, w * v.y);
      sd[3 * t] = dir[3 * (sb + t)];
      sd[3 * t + 1] = dir[3 * (sb + t) + 1];
      sd[3 * t + 2] = dir[3 * (sb + t) + 2];
    }
    __syncthreads();
    for (int64_t p = p0 + warp; p < p1; p += nw) {
      const double dx = x[p] - cx, dy = y[p] - cy, dz = z[p] - cz;
      double ar = 0.0, ai = 0.0;
      for (int s = lane; s < ns; s += 32) {
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
      if (lane == 0) {
        const double2 v = make_double2(-c * ai, c * ar);
        if (sb == 0) {
          pot[p] = v;
        } else {
          double2 cur = pot[p];
          pot[p] = make_double2(cur.x + v.x, cur.y + v.y);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Near-field P2P (operators.cpp:110-122 with green kernel.cpp:9-14, driver
// traversal.cpp:768-786): one CTA per observer leaf; the near leaves'
// particles stream through shared memory as one concatenated list (a source
// finds its leaf by binary search in the prefix sums).  Coordinates are
// staged relative to the observer leaf centre and scaled by k, and the
// charges by k / (4 pi), so a pair costs rsqrt + sincos + 4 FMA:
//   g = exp(-i k r) / (4 pi r) = (k / 4 pi) exp(-i r') / r',  r' = k r.
// The exact-zero separation (self pair, operators.cpp:118) is masked.
// Two launch shapes over two leaf lists: SMALL leaves (<= 32 observers) let
// G threads cooperate per observer; DENSE leaves give every warp all
// observers of a pass (lane l holds l, l + 32, ...) and a quarter of each
// staged chunk, so warps do equal work, then combine across warps.
constexpr int kP2PChunk = 512;
constexpr int kP2PObsPerLane = 4;  // dense leaves: 32 x 4 observers per pass (measured best of 2..8)

// exp(-i r') / r' from r'^2 > 0 (finite): (gr, gi).
__device__ __forceinline__ void green_scaled(double r2, double& gr, double& gi) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(r2));
  const double t = r2 * y0;
  const double e = fma(-t, y0, 1.0);  // 1 - r2 y0^2
  const double p = fma(e, 0.375, 0.5);
  const double ri = fma(y0 * e, p, y0);  // 1 / r'
  const double x = r2 * ri;             // r'
  const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  const double tq = fma(x, kSinCos[12], kMagic);
  const int quad = __double2loint(tq);
  const double n = tq - kMagic;
  double y = fma(n, -1.5707963267948966, x);
  y = fma(n, kSinCos[13], y);
  const double y2 = y * y;
  double ps = kSinCos[0];
#pragma unroll
  for (int i = 1; i < 6; ++i) ps = fma(ps, y2, kSinCos[i]);
  const double sn = fma(ps * y2, y, y);
  double pc = kCos5[0];
#pragma unroll
  for (int i = 1; i < 5; ++i) pc = fma(pc, y2, kCos5[i]);
  const double cs = fma(pc, y2 * y2, fma(-0.5, y2, 1.0));
  // exp(-i (y + quad pi/2)) = (cos y - i sin y) (-i)^quad:
  //   quad 0: ( c, -s)   1: (-s, -c)   2: (-c,  s)   3: ( s,  c)
  const bool swap = quad & 1;
  const double mr = swap ? sn : cs, mi = swap ? cs : sn;
  const unsigned q30 = unsigned(quad) << 30;
  const unsigned sr = (q30 + 0x40000000u) & 0x80000000u;  // re < 0 for quad 1, 2
  const unsigned si = ~q30 & 0x80000000u;                 // im < 0 for quad 0, 1
  const int rhi = __double2hiint(ri), rlo = __double2loint(ri);
  gr = mr * __hiloint2double(rhi ^ int(sr), rlo);
  gi = mi * __hiloint2double(rhi ^ int(si), rlo);
}

// exp(-i r') / r' with a table instead of the sincos polynomials, for the
// bounded near-field range r' <= k 2 sqrt(3) leaf side: tab[n] = (cos(n/128),
// -sin(n/128)) (host libm), n = round(128 r') (magic add), and the residual
// d = r' - n/128 (exact, |d| <= 1/256) through short Taylor kernels (omitted
// terms < 1e-17): 21 FP64 instructions instead of 27.  Indices are clamped
// to [0, tmax] (idle slots sit at far points with zero charge).
constexpr int kPhaseTabMax = 1024;
__device__ __forceinline__ void green_tab(double r2, const double2* __restrict__ tab, int tmax, double& gr,
                                          double& gi) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(r2));
  const double t = r2 * y0;
  const double e = fma(-t, y0, 1.0);
  const double p = fma(e, 0.375, 0.5);
  const double ri = fma(y0 * e, p, y0);  // 1 / r'
  const double x = r2 * ri;             // r'
  const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  // table index from the unrefined r' (t = r2 y0, relative error ~2^-22): the
  // table load does not wait for the Newton step; |d| <= 1/256 + 2e-6 still
  // keeps the omitted Taylor terms below 1e-17
  const double tq = fma(t, 128.0, kMagic);
  const int n = min(max(__double2loint(tq), 0), tmax);
  const double d = fma(tq - kMagic, -0.0078125, x);  // r' - n / 128, exact
  const double d2 = d * d;
  const double sn = fma(d * d2, fma(d2, 8.3333333333333333e-3, -1.6666666666666667e-1), d);
  const double cs = fma(d2, fma(d2, 4.1666666666666667e-2, -0.5), 1.0);
  const double2 c0 = tab[n];  // (cos x0, -sin x0); shared (symmetric kernel) or global (small leaves)
  // exp(-i (x0 + d)) = (cos x0 - i sin x0)(cos d - i sin d)
  gr = fma(c0.x, cs, c0.y * sn) * ri;
  gi = fma(c0.y, cs, -(c0.x * sn)) * ri;
}

// green_tab without the index clamp, for callers whose r' is always inside
// the table (real observer and source particles of adjacent leaves).
__device__ __forceinline__ void green_tab_nc(double r2, const double2* __restrict__ tab, double& gr, double& gi) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(r2));
  const double t = r2 * y0;
  const double e = fma(-t, y0, 1.0);
  const double p = fma(e, 0.375, 0.5);
  const double ri = fma(y0 * e, p, y0);
  const double x = r2 * ri;
  const double kMagic = 6755399441055744.0;
  const double tq = fma(t, 128.0, kMagic);
  const int n = __double2loint(tq);
  const double d = fma(tq - kMagic, -0.0078125, x);
  const double d2 = d * d;
  const double sn = fma(d * d2, fma(d2, 8.3333333333333333e-3, -1.6666666666666667e-1), d);
  const double cs = fma(d2, fma(d2, 4.1666666666666667e-2, -0.5), 1.0);
  const double2 c0 = tab[n];
  gr = fma(c0.x, cs, c0.y * sn) * ri;
  gi = fma(c0.y, cs, -(c0.x * sn)) * ri;
}

template <bool TAB = false>
__device__ __forceinline__ void p2p_pair(double xo, double yo, double zo, double sx, double sy, double sz,
                                         double2 qq, double& ar, double& ai, const double2* __restrict__ tab = nullptr,
                                         int tmax = 0) {
  const double dx = xo - sx, dy = yo - sy, dz = zo - sz;
  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const bool self = r2 == 0.0;  // exact-zero separation (operators.cpp:118)
  double gr, gi;
  if constexpr (TAB) green_tab(self ? 1.0 : r2, tab, tmax, gr, gi); else green_scaled(self ? 1.0 : r2, gr, gi);
  gr = self ? 0.0 : gr;
  gi = self ? 0.0 : gi;
  ar = fma(gr, qq.x, fma(-gi, qq.y, ar));
  ai = fma(gr, qq.y, fma(gi, qq.x, ai));
}

struct P2PShared {
  double sx[kP2PChunk], sy[kP2PChunk], sz[kP2PChunk];
  double2 sq[kP2PChunk];
  int64_t pref[28], nbeg[28];
  int nn;
};

// Prefix sums of the near leaves of `leaf` into smem; returns the total.
__device__ __forceinline__ int64_t p2p_prepare(P2PShared& sh, int64_t leaf, const int64_t* __restrict__ leaf_start,
                                               const int64_t* __restrict__ near_off, const int* __restrict__ near) {
  if (threadIdx.x == 0) {
    const int64_t nb = near_off[leaf];
    const int nn = int(near_off[leaf + 1] - nb);
    int64_t run = 0;
    for (int j = 0; j < nn; ++j) {
      const int lf = near[nb + j];
      sh.pref[j] = run;
      sh.nbeg[j] = leaf_start[lf];
      run += leaf_start[lf + 1] - leaf_start[lf];
    }
    sh.pref[nn] = run;
    sh.nn = nn;
  }
  __syncthreads();
  return sh.pref[sh.nn];
}

// Stage concatenated sources [cb, cb + n): relative to (cx, cy, cz), scaled.
__device__ __forceinline__ void p2p_stage(P2PShared& sh, int64_t cb, int n, const double* __restrict__ x,
                                          const double* __restrict__ y, const double* __restrict__ z,
                                          const double2* __restrict__ q, double cx, double cy, double cz, double k,
                                          double qs) {
  const int nn = sh.nn;
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
    const int64_t v = cb + t;
    int lo = 0, hi = nn;  // largest j with pref[j] <= v
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (sh.pref[mid] <= v) lo = mid; else hi = mid;
    }
    const int64_t src = sh.nbeg[lo] + (v - sh.pref[lo]);
    sh.sx[t] = k * (x[src] - cx);
    sh.sy[t] = k * (y[src] - cy);
    sh.sz[t] = k * (z[src] - cz);
    const double2 qq = q[src];
    sh.sq[t] = make_double2(qs * qq.x, qs * qq.y);
  }
}

// ---------------------------------------------------------------------------
// Adds the scratch rows other dense leaves wrote for leaf B (fixed order).
__global__ void k_p2p_gather(const int* __restrict__ leaves, const int64_t* __restrict__ leaf_start,
                             const int* __restrict__ in_off, const int64_t* __restrict__ in_scr,
                             const double2* __restrict__ scratch, double2* __restrict__ pot) {
  const int i = blockIdx.x;
  const int64_t leaf = leaves[i];
  const int64_t p0 = leaf_start[leaf], n = leaf_start[leaf + 1] - p0;
  for (int64_t t = threadIdx.x; t < n; t += blockDim.x) {
    double2 acc = pot[p0 + t];
    for (int j = in_off[i]; j < in_off[i + 1]; ++j) {
      const double2 v = scratch[in_scr[j] + t];
      acc.x += v.x;
      acc.y += v.y;
    }
    pot[p0 + t] = acc;
  }
}

// ---------------------------------------------------------------------------
// Permutations between input order and Morton order (traversal.cpp:108-110, :809-815).
__global__ void k_gather_q(int64_t n, const int64_t* __restrict__ orig, const double2* __restrict__ q_in,
                           double2* __restrict__ q_sorted) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) q_sorted[i] = q_in[orig[i]];
}
__global__ void k_add_pot(int64_t b, int64_t e, const double2* __restrict__ add, double2* __restrict__ pot) {
  const int64_t i = b + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < e) {
    double2 a = pot[i];
    const double2 v = add[i];
    a.x += v.x;
    a.y += v.y;
    pot[i] = a;
  }
}
__global__ void k_scatter_pot(int64_t b, int64_t e, const int64_t* __restrict__ orig,
                              const double2* __restrict__ pot_sorted, double2* __restrict__ pot_in) {
  const int64_t i = b + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < e) pot_in[orig[i]] = pot_sorted[i];
}

// ---------------------------------------------------------------------------
// Exchange packing (distributed mode): whole expansion rows and ghost particles.
// Row exchanges of the distributed mode (setup.hpp, RankPlan kinds 0, 2, 3):
// item i = {node, begin, length, buffer offset} (int64, double2 units);
// one CTA row per item, grid.y strides over its samples.
__global__ void k_pack_items(const double2* __restrict__ src, int64_t S, const int64_t* __restrict__ items,
                             double2* __restrict__ buf) {
  const int64_t* it = items + 4 * int64_t(blockIdx.x);
  const int64_t node = it[0], b = it[1], len = it[2], off = it[3];
  for (int64_t s = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; s < len; s += int64_t(gridDim.y) * blockDim.x)
    buf[off + s] = src[node * S + b + s];
}
template <bool ADD>
__global__ void k_unpack_items(double2* __restrict__ dst, int64_t S, const int64_t* __restrict__ items,
                               const double2* __restrict__ buf) {
  const int64_t* it = items + 4 * int64_t(blockIdx.x);
  const int64_t node = it[0], b = it[1], len = it[2], off = it[3];
  for (int64_t s = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; s < len; s += int64_t(gridDim.y) * blockDim.x) {
    const double2 v = buf[off + s];
    if (ADD) {
      double2 a = dst[node * S + b + s];
      a.x += v.x;
      a.y += v.y;
      dst[node * S + b + s] = a;
    } else {
      dst[node * S + b + s] = v;
    }
  }
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
