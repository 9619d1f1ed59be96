// Quad-symmetric C2M and L2T with factored phase sums (operators.cpp:15-26
// and :89-108; drivers traversal.cpp:306-320 and :717-728).
//
// The four samples of a quad, (i, j), (n-1-i, j), (i, j+n/2), (n-1-i, j+n/2),
// have phases +-A +-B with A = k sin(theta_i)(x cos(phi_j) + y sin(phi_j))
// and B = k z cos(theta_i) (see k_c2m_quad, kernels.cuh).  B depends only on
// the particle and the theta row, so each kernel folds it into a per-warp
// table first and spends per (quad, particle) one sincos of A plus 8 FMA:
//
//  C2M: with Q+ = q e^{iB}, Q- = q e^{-iB} (table per particle and row),
//       M(i,j) = sum Q+ e^{iA}, M(n-1-i,j) = sum Q- e^{iA},
//       M(i,j+n/2) = sum Q+ e^{-iA}, M(n-1-i,j+n/2) = sum Q- e^{-iA};
//       accumulating Re(Q.) e^{iA} and Im(Q.) e^{iA} separately gives all
//       four from 8 real FMA (vs 16 for four complex MACs).
//  L2T: with G = L1+L2+L3+L4, H = L2-L1+L4-L3, G' = L3+L4-L1-L2,
//       H' = L1-L2-L3+L4 (weighted locals of the quad, formed once per
//       observer pass),  sum_quad = cos B (cos A G + i sin A G')
//                                 + sin B (i cos A H - sin A H').
//
// The sincos here applies the quadrant signs by XOR on the high word
// (integer pipe) instead of FP64 negations.  FP64 per (quad, particle):
// 2 (argument) + 20 (sincos) + 8 (C2M) or 12 (L2T), against 48 before.
#ifndef HFMM_B200_LEAF_CUH
#define HFMM_B200_LEAF_CUH

#include "kernels.cuh"

namespace hfmm_b200 {

__device__ __forceinline__ double xor_sign(double v, unsigned s) {
  return __hiloint2double(__double2hiint(v) ^ int(s), __double2loint(v));
}

// sin, cos of |x| < 2^20 (same reduction as sincos_fast; cos kernel kCos5).
__device__ __forceinline__ void sincos_q(double x, double& sp, double& cp) {
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
  double pc = kCos5[0];
#pragma unroll
  for (int i = 1; i < 5; ++i) pc = fma(pc, y2, kCos5[i]);
  const double cs = fma(pc, y2 * y2, fma(-0.5, y2, 1.0));
  const bool swap = quad & 1;
  const unsigned q30 = unsigned(quad) << 30;
  sp = xor_sign(swap ? cs : sn, q30 & 0x80000000u);                  // sin < 0 for quad 2, 3
  cp = xor_sign(swap ? sn : cs, (q30 + 0x40000000u) & 0x80000000u);  // cos < 0 for quad 1, 2
}

// sin, cos for the bounded leaf-level phases (|x| <= k side / sqrt 2 for A,
// k side / 2 for B) from a table tab[n] = (cos(n/128), sin(n/128)),
// n in [-nh, nh] (tab points at n = 0), with the exact residual
// |d| <= 1/256 through short Taylor kernels: 13 FP64 instructions instead
// of 19.  TAB = false: the polynomial sincos_q.
constexpr int kLeafTabMax = 256;  // |phase| <= 2 (leaf side <= 0.45 wavelengths)
template <bool TAB>
__device__ __forceinline__ void sincos_l(double x, const double2* __restrict__ tab, int nh, double& sp, double& cp) {
  if constexpr (!TAB) {
    sincos_q(x, sp, cp);
  } else {
    const double kMagic = 6755399441055744.0;  // 1.5 * 2^52
    const double tq = fma(x, 128.0, kMagic);
    const int n = min(max(__double2loint(tq), -nh), nh);
    const double d = fma(tq - kMagic, -0.0078125, x);  // x - n / 128, exact
    const double d2 = d * d;
    const double sd = fma(d * d2, fma(d2, 8.3333333333333333e-3, -1.6666666666666667e-1), d);
    const double cd = fma(d2, fma(d2, 4.1666666666666667e-2, -0.5), 1.0);
    const double2 c0 = __ldg(tab + n);
    sp = fma(c0.y, cd, c0.x * sd);
    cp = fma(c0.x, cd, -(c0.y * sd));
  }
}

// HFMM_LEAF_MINB (dev knob): CTAs per SM the register budget of the quad C2M /
// L2T kernels is sized for; unset = the compiler's choice (measured best).
#ifdef HFMM_LEAF_MINB
#define HFMM_LEAF_LB __launch_bounds__(128, HFMM_LEAF_MINB)
#else
#define HFMM_LEAF_LB __launch_bounds__(128)
#endif
constexpr int kQuadP2 = 16;  // particles per table chunk
#ifndef HFMM_C2M_UNROLL
#define HFMM_C2M_UNROLL 1
#endif
#ifndef HFMM_L2T_UNROLL
#define HFMM_L2T_UNROLL 1
#endif
constexpr int kC2MUnroll = HFMM_C2M_UNROLL;  // particle loop unroll (C2M)
constexpr int kL2TUnroll = HFMM_L2T_UNROLL;  // quad loop unroll (populous-leaf L2T)

// R quads per lane: the launch picks R = ceil(quads / 32) (<= 6), so a leaf
// is one pass and its (Q+, Q-) table is built once.
// HN > 0: n / 2 known at compile time (the BASELINE leaf grids n = 18, 22, 26),
// so quad indices and table rows need no integer division at run time.
template <int R, int HN = 0, bool TAB = false>
__global__ void HFMM_LEAF_LB k_c2m_quad2(int64_t leaf_b, int64_t nl, const int64_t* __restrict__ leaf_start,
                                                   const double* __restrict__ x, const double* __restrict__ y,
                                                   const double* __restrict__ z, const double2* __restrict__ q,
                                                   const double* __restrict__ centers, const double* __restrict__ dir,
                                                   int n, double k, double2* __restrict__ mp,
                                                   const double2* __restrict__ ltab = nullptr, int nh = 0) {
  __shared__ double4 sQ[4][kQuadP2][kQuadHalfMax];  // (Q+, Q-) per particle and theta row
  __shared__ double2 sR[4][kQuadP2];                 // (x - cx, y - cy) per particle
  const double2* tb = TAB ? ltab + nh : nullptr;  // read through L1 (small CTAs: no staging)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t li = int64_t(blockIdx.x) * 4 + warp;
  if (li >= nl) return;  // whole warp
  const int64_t leaf = leaf_b + li;
  const int half = HN > 0 ? HN : n / 2, quads = half * half, nphi = HN > 0 ? 2 * HN : n;
  const int64_t S = int64_t(n) * n;
  const int64_t p0 = leaf_start[leaf], p1 = leaf_start[leaf + 1];
  const double cx = centers[3 * leaf], cy = centers[3 * leaf + 1], cz = centers[3 * leaf + 2];
  double4 (*Qt)[kQuadHalfMax] = sQ[warp];
  double2* Rt = sR[warp];
  // Grids needing several quad passes (n = 26: 169 quads over 96 lane slots):
  // a leaf with <= kQuadP2 particles builds its tables once for all passes.
  // (Single-pass grids keep the build inside the particle loop: fewer live
  // registers, measured faster at n = 18.)
  constexpr bool kMultiPass = HN == 0 || HN * HN > 32 * R;
  const bool one_chunk = kMultiPass && p1 - p0 <= kQuadP2;
  auto build = [&](int64_t pc, int np) {
    __syncwarp();
    for (int t = lane; t < np * half; t += 32) {
      const int pp = t / half, i = t - pp * half;
      double sb, cb;
      sincos_l<TAB>(k * dir[3 * int64_t(i) * nphi + 2] * (z[pc + pp] - cz), tb, nh, sb, cb);
      const double2 qq = q[pc + pp];
      Qt[pp][i] = make_double4(fma(qq.x, cb, -qq.y * sb), fma(qq.x, sb, qq.y * cb),   // q e^{iB}
                               fma(qq.x, cb, qq.y * sb), fma(qq.y, cb, -qq.x * sb));  // q e^{-iB}
    }
    if (lane < np) Rt[lane] = make_double2(x[pc + lane] - cx, y[pc + lane] - cy);
    __syncwarp();
  };
  if (one_chunk) build(p0, int(p1 - p0));
  for (int qc = 0; qc < quads; qc += 32 * R) {
    double ax[R], ay[R];
    int qi[R];
    double upx[R], upy[R], vpx[R], vpy[R];
    double umx[R], umy[R], vmx[R], vmy[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int qd = qc + lane + 32 * r;
      const int i = qd < quads ? qd / half : 0, j = qd < quads ? qd - (qd / half) * half : 0;
      qi[r] = i;
      const int64_t s1 = int64_t(i) * nphi + j;
      ax[r] = k * dir[3 * s1];
      ay[r] = k * dir[3 * s1 + 1];
      upx[r] = upy[r] = vpx[r] = vpy[r] = umx[r] = umy[r] = vmx[r] = vmy[r] = 0.0;
    }
    for (int64_t pc = p0; pc < p1; pc += kQuadP2) {
      const int np = int(p1 - pc < kQuadP2 ? p1 - pc : kQuadP2);
      if (!one_chunk) build(pc, np);
#pragma unroll kC2MUnroll
      for (int pp = 0; pp < np; ++pp) {
        const double2 rr = Rt[pp];  // shared memory: no global load in the particle loop
#pragma unroll
        for (int r = 0; r < R; ++r) {
          double sa, ca;
          sincos_l<TAB>(fma(ax[r], rr.x, ay[r] * rr.y), tb, nh, sa, ca);
          const double4 Q = Qt[pp][qi[r]];
          upx[r] = fma(Q.x, ca, upx[r]);
          upy[r] = fma(Q.x, sa, upy[r]);
          vpx[r] = fma(Q.y, ca, vpx[r]);
          vpy[r] = fma(Q.y, sa, vpy[r]);
          umx[r] = fma(Q.z, ca, umx[r]);
          umy[r] = fma(Q.z, sa, umy[r]);
          vmx[r] = fma(Q.w, ca, vmx[r]);
          vmy[r] = fma(Q.w, sa, vmy[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int qd = qc + lane + 32 * r;
      if (qd < quads) {
        const int i = qd / half, j = qd - i * half;
        double2* m = mp + li * S;  // row of the leaf: leaf - leaf_b (engine rows, world.hpp)
        const int64_t s1 = int64_t(i) * nphi + j, s2 = int64_t(n - 1 - i) * nphi + j;
        m[s1] = make_double2(upx[r] - vpy[r], upy[r] + vpx[r]);         // A + B
        m[s2] = make_double2(umx[r] - vmy[r], umy[r] + vmx[r]);         // A - B   (pi - theta)
        m[s1 + half] = make_double2(upx[r] + vpy[r], vpx[r] - upy[r]);  // -A + B  (phi + pi)
        m[s2 + half] = make_double2(umx[r] + vmy[r], vmx[r] - umy[r]);  // -A - B
      }
    }
  }
}

constexpr int kQuadOB = 4;  // observers per L2T pass
// Multi-chunk grids (n = 26: 169 quads over 96 lane slots) for k_l2t_quad3:
// particle chunks outside (tables built once per chunk), quad chunks inside,
// one observer per pass (fewest live registers; measured fastest there).
template <int R, int HN, bool TAB, class Build>
__device__ __forceinline__ void l2t_quad3_multi(int64_t p0, int64_t p1, int half, int quads, int nphi, int n, double k,
                                                double c, const double2* __restrict__ lc,
                                                const double* __restrict__ wq, const double* __restrict__ dir,
                                                const double2* __restrict__ tb, int nh,
                                                double2 (*Bt)[kQuadHalfMax], double2* Rt, Build& build,
                                                double2* __restrict__ pot) {
  const int lane = threadIdx.x & 31;
  for (int64_t pc = p0; pc < p1; pc += kQuadP2) {
    const int np = int(p1 - pc < kQuadP2 ? p1 - pc : kQuadP2);
    build(pc, np);
    for (int qc = 0; qc < quads; qc += 32 * R) {
      double2 G[R], Gp[R], H[R], Hp[R];
      double dx[R], dy[R];
      int qi[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int qd = qc + lane + 32 * r;
        const bool live = qd < quads;
        const int i = live ? qd / half : 0, j = live ? qd - i * half : 0;
        qi[r] = i;
        const int64_t s1 = int64_t(i) * nphi + j, s2 = int64_t(n - 1 - i) * nphi + j;
        auto lw = [&](int64_t s) {
          const double2 v = __ldg(lc + s);
          const double w = live ? __ldg(wq + s) : 0.0;
          return make_double2(w * v.x, w * v.y);
        };
        const double2 l1 = lw(s1), l2 = lw(s2), l3 = lw(s1 + half), l4 = lw(s2 + half);
        const double2 s12 = make_double2(l1.x + l2.x, l1.y + l2.y), s34 = make_double2(l3.x + l4.x, l3.y + l4.y);
        const double2 d12 = make_double2(l2.x - l1.x, l2.y - l1.y), d34 = make_double2(l4.x - l3.x, l4.y - l3.y);
        G[r] = make_double2(s12.x + s34.x, s12.y + s34.y);
        Gp[r] = make_double2(s34.x - s12.x, s34.y - s12.y);
        H[r] = make_double2(d12.x + d34.x, d12.y + d34.y);
        Hp[r] = make_double2(d34.x - d12.x, d34.y - d12.y);
        dx[r] = dir[3 * s1];
        dy[r] = dir[3 * s1 + 1];
      }
      for (int pp = 0; pp < np; ++pp) {
        const double2 rr = Rt[pp];
        double ar = 0.0, ai = 0.0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          double sa, ca;
          sincos_l<TAB>(fma(dx[r], rr.x, dy[r] * rr.y), tb, nh, sa, ca);
          const double2 eb = Bt[pp][qi[r]];
          const double u = eb.x * ca, v = eb.x * sa, w = eb.y * ca, zz = eb.y * sa;
          ar = fma(u, G[r].x, fma(-v, Gp[r].y, fma(-w, H[r].y, fma(-zz, Hp[r].x, ar))));
          ai = fma(u, G[r].y, fma(v, Gp[r].x, fma(w, H[r].x, fma(-zz, Hp[r].y, ai))));
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          ar += __shfl_xor_sync(0xffffffffu, ar, off);
          ai += __shfl_xor_sync(0xffffffffu, ai, off);
        }
        if (lane == 0) {
          const double2 v = make_double2(-c * ai, c * ar);
          if (qc == 0) {
            pot[pc + pp] = v;
          } else {
            const double2 cur = pot[pc + pp];
            pot[pc + pp] = make_double2(cur.x + v.x, cur.y + v.y);
          }
        }
      }
    }
  }
}

// L2T for small leaves, one warp per leaf, lanes over quads: each lane keeps
// the weighted quad combinations (G, G', H, H') and k (dir_x, dir_y) of its R
// quads in registers (built once per leaf and quad chunk), the particles are
// staged per chunk in shared memory with their e^{iB} rows, so the
// observer loop reads no global memory; kQuadOB observers per pass, one
// shuffle reduction each.  Leaf grids with more than 32 R quads take several
// quad chunks per particle chunk (the tables are built once), whose sums lane
// 0 adds in chunk order (deterministic).
// L2T for small leaves, one warp per leaf, lanes over quads: each lane keeps
// the weighted quad combinations (G, G', H, H') and k (dir_x, dir_y) of its R
// quads in registers (built once per leaf and quad chunk), the particles are
// staged in shared memory with their e^{iB} rows, so the observer loop reads
// no global memory; kQuadOB observers per pass, one shuffle reduction each.
// Leaf grids with more than 32 R quads take several quad chunks
// (l2t_quad3_multi), whose sums lane 0 adds in chunk order (deterministic).
template <int R, int HN = 0, bool TAB = false>
__global__ void HFMM_LEAF_LB k_l2t_quad3(int64_t leaf_b, int64_t nl, const int* __restrict__ leaves,
                                         const int64_t* __restrict__ leaf_start, const double* __restrict__ x,
                                         const double* __restrict__ y, const double* __restrict__ z,
                                         const double* __restrict__ centers, const double* __restrict__ dir,
                                         const double* __restrict__ wq, int n, double k,
                                         const double2* __restrict__ loc, double2* __restrict__ pot,
                                         const double2* __restrict__ ltab = nullptr, int nh = 0) {
  __shared__ double2 sB[4][kQuadP2][kQuadHalfMax];  // e^{iB} per particle and theta row
  __shared__ double2 sR[4][kQuadP2];                // k (x - cx), k (y - cy)
  const double2* tb = TAB ? ltab + nh : nullptr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = HN > 0 ? HN : n / 2, quads = half * half, nphi = HN > 0 ? 2 * HN : n;
  const int64_t S = int64_t(n) * n;
  const int64_t li = int64_t(blockIdx.x) * 4 + warp;
  if (li >= nl) return;
  const int64_t leaf = leaves ? int64_t(leaves[li]) : leaf_b + li;
  const int64_t p0 = leaf_start[leaf], p1 = leaf_start[leaf + 1];
  const double cx = centers[3 * leaf], cy = centers[3 * leaf + 1], cz = centers[3 * leaf + 2];
  const double c = -k / (16.0 * M_PI * M_PI);  // norm = (0, c)
  const double2* lc = loc + (leaf - leaf_b) * S;  // leaf rows start at leaf_b
  double2 (*Bt)[kQuadHalfMax] = sB[warp];
  double2* Rt = sR[warp];
  auto build = [&](int64_t pc, int np) {
    __syncwarp();
    for (int t = lane; t < np * half; t += 32) {
      const int pp = t / half, i = t - pp * half;
      double sn, cs;
      sincos_l<TAB>(k * dir[3 * int64_t(i) * nphi + 2] * (z[pc + pp] - cz), tb, nh, sn, cs);
      Bt[pp][i] = make_double2(cs, sn);
    }
    if (lane < np) Rt[lane] = make_double2(k * (x[pc + lane] - cx), k * (y[pc + lane] - cy));
    __syncwarp();
  };
  constexpr bool kMultiPass = HN == 0 || HN * HN > 32 * R;
  if constexpr (kMultiPass) {  // several quad chunks: particle chunks outside, one observer per pass
    l2t_quad3_multi<R, HN, TAB>(p0, p1, half, quads, nphi, n, k, c, lc, wq, dir, tb, nh, Bt, Rt, build, pot);
    return;
  }
  for (int qc = 0; qc < quads; qc += 32 * R) {
    double2 G[R], Gp[R], H[R], Hp[R];
    double dx[R], dy[R];
    int qi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int qd = qc + lane + 32 * r;
      const bool live = qd < quads;
      const int i = live ? qd / half : 0, j = live ? qd - i * half : 0;
      qi[r] = i;
      const int64_t s1 = int64_t(i) * nphi + j, s2 = int64_t(n - 1 - i) * nphi + j;
      auto lw = [&](int64_t s) {
        const double2 v = __ldg(lc + s);
        const double w = live ? __ldg(wq + s) : 0.0;
        return make_double2(w * v.x, w * v.y);
      };
      const double2 l1 = lw(s1), l2 = lw(s2), l3 = lw(s1 + half), l4 = lw(s2 + half);
      const double2 s12 = make_double2(l1.x + l2.x, l1.y + l2.y), s34 = make_double2(l3.x + l4.x, l3.y + l4.y);
      const double2 d12 = make_double2(l2.x - l1.x, l2.y - l1.y), d34 = make_double2(l4.x - l3.x, l4.y - l3.y);
      G[r] = make_double2(s12.x + s34.x, s12.y + s34.y);
      Gp[r] = make_double2(s34.x - s12.x, s34.y - s12.y);
      H[r] = make_double2(d12.x + d34.x, d12.y + d34.y);
      Hp[r] = make_double2(d34.x - d12.x, d34.y - d12.y);
      dx[r] = dir[3 * s1];
      dy[r] = dir[3 * s1 + 1];
    }
    for (int64_t pc = p0; pc < p1; pc += kQuadP2) {
      const int np = int(p1 - pc < kQuadP2 ? p1 - pc : kQuadP2);
      build(pc, np);
      for (int pb = 0; pb < np; pb += kQuadOB) {
        double ar[kQuadOB], ai[kQuadOB];
#pragma unroll
        for (int o = 0; o < kQuadOB; ++o) {
          const int pp = pb + o < np ? pb + o : pb;  // idle slots repeat a live observer
          const double2 rr = Rt[pp];
          ar[o] = 0.0;
          ai[o] = 0.0;
#pragma unroll
          for (int r = 0; r < R; ++r) {
            double sa, ca;
            sincos_l<TAB>(fma(dx[r], rr.x, dy[r] * rr.y), tb, nh, sa, ca);
            const double2 eb = Bt[pp][qi[r]];
            const double u = eb.x * ca, v = eb.x * sa, w = eb.y * ca, zz = eb.y * sa;
            ar[o] = fma(u, G[r].x, fma(-v, Gp[r].y, fma(-w, H[r].y, fma(-zz, Hp[r].x, ar[o]))));
            ai[o] = fma(u, G[r].y, fma(v, Gp[r].x, fma(w, H[r].x, fma(-zz, Hp[r].y, ai[o]))));
          }
        }
#pragma unroll
        for (int o = 0; o < kQuadOB; ++o) {
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            ar[o] += __shfl_xor_sync(0xffffffffu, ar[o], off);
            ai[o] += __shfl_xor_sync(0xffffffffu, ai[o], off);
          }
          if (lane == 0 && pb + o < np) {
            const double2 v = make_double2(-c * ai[o], c * ar[o]);
            if (qc == 0) {
              pot[pc + pb + o] = v;
            } else {
              const double2 cur = pot[pc + pb + o];
              pot[pc + pb + o] = make_double2(cur.x + v.x, cur.y + v.y);
            }
          }
        }
      }
    }
  }
}

// L2T for populous leaves (> 32 particles): one warp per leaf, one LANE per
// observer, quads looped with their (G, G', H, H') and (dir_x, dir_y) staged
// once per leaf in shared memory (warp broadcasts).  The e^{iB} factor is
// taken out of the row sum: per row i, X = sum_j (cos A G + i sin A G') and
// Y = sum_j (i cos A H - sin A H') (8 FMA per quad), then
// acc += cos B_i X + sin B_i Y.  No cross-lane reduction.
// Shared memory per warp: quads x (4 + 1) double2.
template <int HN = 0, bool TAB = false>
__global__ void __launch_bounds__(128) k_l2t_obs(int64_t row0, int64_t nl, const int* __restrict__ leaves,
                                                 const int64_t* __restrict__ leaf_start, const double* __restrict__ x,
                                                 const double* __restrict__ y, const double* __restrict__ z,
                                                 const double* __restrict__ centers, const double* __restrict__ dir,
                                                 const double* __restrict__ wq, int n, double k,
                                                 const double2* __restrict__ loc, double2* __restrict__ pot,
                                                 const double2* __restrict__ ltab = nullptr, int nh = 0) {
  extern __shared__ double2 osm[];
  const double2* tb = TAB ? ltab + nh : nullptr;  // read through L1 (small CTAs: no staging)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int half = HN > 0 ? HN : n / 2, quads = half * half, nphi = HN > 0 ? 2 * HN : n;
  const int64_t S = int64_t(n) * n;
  double2* qt = osm + int64_t(warp) * quads * 5;  // per quad: G, G', H, H', (k dir_x, k dir_y)
  const int64_t li = int64_t(blockIdx.x) * 4 + warp;
  if (li >= nl) return;
  const int64_t leaf = leaves[li];
  const int64_t p0 = leaf_start[leaf], p1 = leaf_start[leaf + 1];
  const double cx = centers[3 * leaf], cy = centers[3 * leaf + 1], cz = centers[3 * leaf + 2];
  const double c = -k / (16.0 * M_PI * M_PI);  // norm = (0, c)
  const double2* lc = loc + (leaf - row0) * S;  // leaf rows start at the rank's first leaf
  for (int qd = lane; qd < quads; qd += 32) {
    const int i = qd / half, j = qd - i * half;
    const int64_t s1 = int64_t(i) * nphi + j, s2 = int64_t(n - 1 - i) * nphi + j;
    auto lw = [&](int64_t s) {
      const double2 v = __ldg(lc + s);
      const double w = __ldg(wq + s);
      return make_double2(w * v.x, w * v.y);
    };
    const double2 l1 = lw(s1), l2 = lw(s2), l3 = lw(s1 + half), l4 = lw(s2 + half);
    const double2 s12 = make_double2(l1.x + l2.x, l1.y + l2.y), s34 = make_double2(l3.x + l4.x, l3.y + l4.y);
    const double2 d12 = make_double2(l2.x - l1.x, l2.y - l1.y), d34 = make_double2(l4.x - l3.x, l4.y - l3.y);
    qt[5 * qd + 0] = make_double2(s12.x + s34.x, s12.y + s34.y);  // G
    qt[5 * qd + 1] = make_double2(s34.x - s12.x, s34.y - s12.y);  // G'
    qt[5 * qd + 2] = make_double2(d12.x + d34.x, d12.y + d34.y);  // H
    qt[5 * qd + 3] = make_double2(d34.x - d12.x, d34.y - d12.y);  // H'
    qt[5 * qd + 4] = make_double2(k * dir[3 * s1], k * dir[3 * s1 + 1]);
  }
  __syncwarp();
  for (int64_t ob = p0; ob < p1; ob += 32) {
    const int64_t o = ob + lane;
    const bool valid = o < p1;
    const int64_t oo = valid ? o : p0;
    const double rx = x[oo] - cx, ry = y[oo] - cy, rz = z[oo] - cz;
    double ar = 0.0, ai = 0.0;
    for (int i = 0; i < half; ++i) {
      double xr = 0.0, xi = 0.0, yr = 0.0, yi = 0.0;
      const double2* q = qt + 5 * i * half;
#pragma unroll kL2TUnroll
      for (int j = 0; j < half; ++j, q += 5) {
        const double2 a = q[4];
        double sa, ca;
        sincos_l<TAB>(fma(a.x, rx, a.y * ry), tb, nh, sa, ca);
        const double2 G = q[0], Gp = q[1], H = q[2], Hp = q[3];
        xr = fma(ca, G.x, fma(-sa, Gp.y, xr));
        xi = fma(ca, G.y, fma(sa, Gp.x, xi));
        yr = fma(-ca, H.y, fma(-sa, Hp.x, yr));
        yi = fma(ca, H.x, fma(-sa, Hp.y, yi));
      }
      double sb, cb;
      sincos_l<TAB>(k * dir[3 * int64_t(i) * nphi + 2] * rz, tb, nh, sb, cb);
      ar = fma(cb, xr, fma(sb, yr, ar));
      ai = fma(cb, xi, fma(sb, yi, ai));
    }
    if (valid) pot[o] = make_double2(-c * ai, c * ar);
  }
}

}  // namespace hfmm_b200

#endif  // HFMM_B200_LEAF_CUH
