// Near-field P2P, symmetric dense-leaf kernel (operators.cpp:110-122 with
// green kernel.cpp:9-14, driver traversal.cpp:768-786).  Same pair algebra
// and leaf schedule as k_p2p_sym (kernels.cuh), organised for the FP64 pipe:
//
//  * the scaled kernel g' = exp(-i r') / r' (r' = k r) costs 41 FP64
//    instructions: 6 for r'^2, 6 for 1/r' and r' (MUFU.RSQ64H + one cubic
//    Newton step, no special-case branch: r'^2 > 0 here), 19 for sincos
//    (Cody-Waite by pi/2, fdlibm's degree-13 sin, a degree-12 cos fit), 2 for g' and 8
//    for the two complex multiply-adds (A <- B and B <- A).  The quadrant
//    swap is a select and the quadrant signs are XORed into 1/r' (integer
//    pipe), so no FP64 negations;
//  * each lane evaluates its NC observers in lockstep (independent chains
//    side by side for the scheduler), NC a template parameter so a pass with
//    fewer than 4 observer slots does no padded work;
//  * a warp takes M partner sources per iteration and reduces their M
//    B-side sums with one split butterfly (M - 1 + 5 - log2 M shuffle steps
//    instead of 5 M).
#ifndef HFMM_B200_P2P_CUH
#define HFMM_B200_P2P_CUH

#include "kernels.cuh"

namespace hfmm_b200 {

#ifndef HFMM_P2P_SYMOBS
#define HFMM_P2P_SYMOBS 4
#endif
constexpr int kSymObs = HFMM_P2P_SYMOBS;  // observer slots per lane (pass = 32 kSymObs observers)


// green_scaled (exp(-i r') / r') lives in kernels.cuh next to p2p_pair.

// Sources [b0, b0 + nb) (staged kP2PChunk at a time, relative to the leaf
// centre) against the lane's NC observers; both sides accumulate: A's in
// ar/ai, each source's B-side sum (over the CTA's observers of this warp)
// is reduced across the warp and written to scr[source - b0].
// SELF: the sources are this leaf's particles from the pass's first
// observer on (source index s relative to the pass; slot tile u = s / 32):
// slots c < u are symmetric pairs, slot c == u only lanes with o < s (the
// diagonal tile, exact-zero self pair excluded), slots c > u are skipped --
// those pairs are taken when the roles are swapped.
template <int NC, int M, bool SELF, bool TAB>
__device__ __forceinline__ void sym_block(P2PShared& sh, const double2* __restrict__ tab, int tmax, double k,
                                          double cx, double cy, double cz, double qs,
                                          int64_t b0, int64_t nbp, double2* __restrict__ scr,
                                          const double* __restrict__ x, const double* __restrict__ y,
                                          const double* __restrict__ z, const double2* __restrict__ q,
                                          const double (&xo)[NC], const double (&yo)[NC], const double (&zo)[NC],
                                          const double (&qr)[NC], const double (&qi)[NC], double (&ar)[NC],
                                          double (&ai)[NC]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  for (int64_t cb = 0; cb < nbp; cb += kP2PChunk) {
    const int n = int(nbp - cb < kP2PChunk ? nbp - cb : kP2PChunk);
    const int npad = (n + M - 1) / M * M;
    __syncthreads();
    for (int t = threadIdx.x; t < npad; t += blockDim.x) {
      if (t < n) {
        const int64_t src = b0 + cb + t;
        sh.sx[t] = k * (x[src] - cx);
        sh.sy[t] = k * (y[src] - cy);
        sh.sz[t] = k * (z[src] - cz);
        const double2 qq = q[src];
        sh.sq[t] = make_double2(qs * qq.x, qs * qq.y);
      } else {  // padding source: far, zero charge
        sh.sx[t] = -1.0e4;
        sh.sy[t] = 0.0;
        sh.sz[t] = 0.0;
        sh.sq[t] = make_double2(0.0, 0.0);
      }
    }
    __syncthreads();
    for (int t = warp * M; t < npad; t += nwarp * M) {
      double br[M], bi[M];
#pragma unroll
      for (int m = 0; m < M; ++m) {
        const double px = sh.sx[t + m], py = sh.sy[t + m], pz = sh.sz[t + m];
        const double2 qq = sh.sq[t + m];
        const int srel = int(cb) + t + m, u = srel >> 5;  // SELF: source's slot tile
        br[m] = 0.0;
        bi[m] = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          if (SELF && c > u) continue;  // warp-uniform
          const double dx = xo[c] - px, dy = yo[c] - py, dz = zo[c] - pz;
          double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
          const bool keep = !SELF || c < u || lane < (srel & 31);
          if (SELF) r2 = keep ? r2 : 1.0;
          double gr, gi;
          if constexpr (TAB) green_tab(r2, tab, tmax, gr, gi); else green_scaled(r2, gr, gi);
          if (SELF) {
            gr = keep ? gr : 0.0;
            gi = keep ? gi : 0.0;
          }
          ar[c] = fma(gr, qq.x, fma(-gi, qq.y, ar[c]));
          ai[c] = fma(gr, qq.y, fma(gi, qq.x, ai[c]));
          br[m] = fma(gr, qr[c], fma(-gi, qi[c], br[m]));
          bi[m] = fma(gr, qi[c], fma(gi, qr[c], bi[m]));
        }
      }
      // split butterfly: after the first log2(M) steps lane group g holds
      // the partial of source g, then a plain butterfly over the rest
      int width = 16;
      int cnt = M;
#pragma unroll
      for (int s = 0; (1 << s) < M; ++s) {
        const bool hi = lane & width;
        cnt >>= 1;
#pragma unroll
        for (int m = 0; m < M; ++m) {
          if (m >= cnt) break;
          const double sr = hi ? br[m] : br[m + cnt], si = hi ? bi[m] : bi[m + cnt];
          const double kr = hi ? br[m + cnt] : br[m], ki = hi ? bi[m + cnt] : bi[m];
          br[m] = kr + __shfl_xor_sync(0xffffffffu, sr, width);
          bi[m] = ki + __shfl_xor_sync(0xffffffffu, si, width);
        }
        width >>= 1;
      }
      double vr = br[0], vi = bi[0];
      for (int off = width; off > 0; off >>= 1) {
        vr += __shfl_xor_sync(0xffffffffu, vr, off);
        vi += __shfl_xor_sync(0xffffffffu, vi, off);
      }
      // lane group g (of 32 / M lanes) holds source index sidx(g): the
      // split keeps the upper half's source in the upper lanes
      if ((lane & (32 / M - 1)) == 0) {
        int sidx = 0, w2 = 16;
#pragma unroll
        for (int s = 0, c2 = M; (1 << s) < M; ++s) {
          c2 >>= 1;
          if (lane & w2) sidx += c2;
          w2 >>= 1;
        }
        const int tt = t + sidx;
        if (tt < n) scr[cb + tt] = make_double2(vr, vi);
      }
    }
  }
}

// Symmetric dense-leaf near field: as k_p2p_sym (same lists, scratch layout
// and gather), with the pair loop above.  Block = 128 threads.
template <int NC, int M, bool TAB>
__device__ __forceinline__ void p2p_sym_pass(P2PShared& sh, const double2* __restrict__ tab, int tmax, int n_o_pass,
                                             double k, double cx, double cy,
                                             double cz, double qs, int64_t leaf, int ob, int64_t p0, int64_t total,
                                             const int* __restrict__ sym, int j0, int j1,
                                             const int64_t* __restrict__ sym_scr, int64_t scr_pass,
                                             const int64_t* __restrict__ leaf_start, const double* __restrict__ x,
                                             const double* __restrict__ y, const double* __restrict__ z,
                                             const double2* __restrict__ q, double2* __restrict__ pot,
                                             double2* __restrict__ scratch, double2 (*red)[32 * kSymObs]) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
  double xo[NC], yo[NC], zo[NC], qr[NC], qi[NC], ar[NC], ai[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int o = lane + 32 * c;
    const bool v = o < n_o_pass;
    // idle slots: far away but finite, zero charge -> exact-zero terms
    xo[c] = v ? k * (x[p0 + o] - cx) : 1.0e4;
    yo[c] = v ? k * (y[p0 + o] - cy) : 0.0;
    zo[c] = v ? k * (z[p0 + o] - cz) : 0.0;
    const double2 qq = v ? q[p0 + o] : make_double2(0.0, 0.0);
    qr[c] = qs * qq.x;
    qi[c] = qs * qq.y;
    ar[c] = 0.0;
    ai[c] = 0.0;
  }
  // one-sided part: small / ghost neighbours (and the self leaf under
  // HFMM_P2P_V1's lists; exact-zero separation masked, operators.cpp:118)
  for (int64_t cb = 0; cb < total; cb += kP2PChunk) {
    const int n = int(total - cb < kP2PChunk ? total - cb : kP2PChunk);
    __syncthreads();
    p2p_stage(sh, cb, n, x, y, z, q, cx, cy, cz, k, qs);
    __syncthreads();
    for (int t = warp; t < n; t += nwarp) {
      const double px = sh.sx[t], py = sh.sy[t], pz = sh.sz[t];
      const double2 qq = sh.sq[t];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double dx = xo[c] - px, dy = yo[c] - py, dz = zo[c] - pz;
        const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
        const bool self = r2 == 0.0;
        double gr, gi;
        if constexpr (TAB) green_tab(self ? 1.0 : r2, tab, tmax, gr, gi); else green_scaled(self ? 1.0 : r2, gr, gi);
        gr = self ? 0.0 : gr;
        gi = self ? 0.0 : gi;
        ar[c] = fma(gr, qq.x, fma(-gi, qq.y, ar[c]));
        ai[c] = fma(gr, qq.y, fma(gi, qq.x, ai[c]));
      }
    }
  }
  // symmetric part: dense partners B > A, and the leaf itself (self pairs
  // o < t, from this pass's first observer on); M sources per warp iteration
  for (int j = j0; j < j1; ++j) {
    const int lb = sym[j];
    double2* scr = scratch + sym_scr[j] + scr_pass;
    if (lb == leaf) {
      for (int t = threadIdx.x; t < ob; t += blockDim.x) scr[t] = make_double2(0.0, 0.0);  // earlier passes' rows
      const int64_t b0 = leaf_start[lb] + ob;
      sym_block<NC, M, true, TAB>(sh, tab, tmax, k, cx, cy, cz, qs, b0, leaf_start[lb + 1] - b0, scr + ob, x, y, z, q, xo, yo, zo, qr,
                             qi, ar, ai);
    } else {
      const int64_t b0 = leaf_start[lb];
      sym_block<NC, M, false, TAB>(sh, tab, tmax, k, cx, cy, cz, qs, b0, leaf_start[lb + 1] - b0, scr, x, y, z, q, xo, yo, zo, qr,
                              qi, ar, ai);
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) red[warp][lane + 32 * c] = make_double2(ar[c], ai[c]);
  __syncthreads();
  for (int o = threadIdx.x; o < n_o_pass; o += blockDim.x) {
    double2 sum = red[0][o];
    for (int w = 1; w < nwarp; ++w) {
      sum.x += red[w][o].x;
      sum.y += red[w][o].y;
    }
    double2 cur = pot[p0 + o];
    cur.x += sum.x;
    cur.y += sum.y;
    pot[p0 + o] = cur;
  }
  __syncthreads();
}

#ifndef HFMM_P2P_M
#define HFMM_P2P_M 4
#endif

// One CTA per work item {dense leaf index, pass}: the pass's observers
// (ob = 128 pass, NC slots per lane) against the leaf's one-sided list and
// its symmetric partners; pass p writes the scratch rows sym_scr + p rows.
#ifndef HFMM_P2P_MINB
#define HFMM_P2P_MINB 4  // CTAs per SM the register budget is sized for
#endif
template <int NC, bool TAB>
__global__ void __launch_bounds__(128, HFMM_P2P_MINB) k_p2p_sym2(const int2* __restrict__ items, const int* __restrict__ leaves,
                                                     const int64_t* __restrict__ leaf_start,
                                                     const int* __restrict__ plain_off, const int* __restrict__ plain,
                                                     const int* __restrict__ sym_off, const int* __restrict__ sym,
                                                     const int64_t* __restrict__ sym_scr,
                                                     const int64_t* __restrict__ sym_rows,
                                                     const double* __restrict__ centers, const double* __restrict__ x,
                                                     const double* __restrict__ y, const double* __restrict__ z,
                                                     const double2* __restrict__ q, double k,
                                                     double2* __restrict__ pot, double2* __restrict__ scratch,
                                                     const double2* __restrict__ ptab, int tmax) {
  __shared__ P2PShared sh;
  __shared__ double2 red[4][32 * kSymObs];
  __shared__ double2 stab[TAB ? kPhaseTabMax : 1];
  if constexpr (TAB) {
    for (int t = threadIdx.x; t <= tmax; t += blockDim.x) stab[t] = ptab[t];  // visible after the next barrier
  }
  const int2 item = items[blockIdx.x];
  const int i = item.x, pass = item.y;
  const int64_t leaf = leaves[i];
  const int64_t p0 = leaf_start[leaf], p1 = leaf_start[leaf + 1];
  const double cx = centers[3 * leaf], cy = centers[3 * leaf + 1], cz = centers[3 * leaf + 2];
  const double qs = k * 0.079577471545947667884;  // k / (4 pi)
  if (threadIdx.x == 0) {
    const int b = plain_off[i], nn = plain_off[i + 1] - b;
    int64_t run = 0;
    for (int j = 0; j < nn; ++j) {
      const int lf = plain[b + j];
      sh.pref[j] = run;
      sh.nbeg[j] = leaf_start[lf];
      run += leaf_start[lf + 1] - leaf_start[lf];
    }
    sh.pref[nn] = run;
    sh.nn = nn;
  }
  __syncthreads();
  const int64_t total = sh.pref[sh.nn];
  const int ob = pass * 32 * kSymObs;
  const int no = min(int(p1 - p0) - ob, 32 * kSymObs);
  p2p_sym_pass<NC, HFMM_P2P_M, TAB>(sh, stab, tmax, no, k, cx, cy, cz, qs, leaf, ob, p0 + ob, total, sym, sym_off[i], sym_off[i + 1],
                               sym_scr, int64_t(pass) * sym_rows[i], leaf_start, x, y, z, q, pot, scratch, red);
}

// ---------------------------------------------------------------------------
// Near field of leaves with <= 32 observers (configs 2 and 4: 4-8 particles
// per leaf), one WARP per leaf.  ncu (config 4) showed the previous kernels
// issue-bound -- ~60% of their instructions were not FP64: per-pair
// self-pair masking, table-index clamping, four shared loads, and lanes
// idled by power-of-two observer groups.  Here:
//  * G = floor(32 / n_o) lanes per observer (any G, not only powers of two),
//    reduced with a guarded shuffle tree;
//  * sources are staged as (x, y, z, q_re) + q_im: two shared loads per pair;
//  * the exact-zero self pair can only occur in the leaf itself, whose
//    sources are a contiguous range of the staged list: only that range takes
//    the masked pair; every other pair skips the mask and the index clamp
//    (all lanes that compute hold a real observer, r' stays in the table);
//  * two independent accumulators per lane (even / odd sources).
template <bool TAB>
__device__ __forceinline__ void p2p_pair_fast(double xo, double yo, double zo, const double4 s, double qim,
                                              double& ar, double& ai, const double2* __restrict__ tab, int tmax) {
  const double dx = xo - s.x, dy = yo - s.y, dz = zo - s.z;
  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
  double gr, gi;
  if constexpr (TAB) green_tab_nc(r2, tab, gr, gi); else green_scaled(r2, gr, gi);
  ar = fma(gr, s.w, fma(-gi, qim, ar));
  ai = fma(gr, qim, fma(gi, s.w, ai));
}

constexpr int kTW = 64;  // sources staged per round (per warp)
template <bool TAB>
__global__ void __launch_bounds__(128) k_p2p_leaf2(int n_leaves, const int* __restrict__ leaves,
                                                   const int64_t* __restrict__ leaf_start,
                                                   const int64_t* __restrict__ near_off, const int* __restrict__ near,
                                                   const double* __restrict__ centers, const double* __restrict__ x,
                                                   const double* __restrict__ y, const double* __restrict__ z,
                                                   const double2* __restrict__ q, double k, double2* __restrict__ pot,
                                                   const double2* __restrict__ ptab = nullptr, int tmax = 0) {
  __shared__ double4 sA[4][kTW];
  __shared__ double sQ[4][kTW];
  __shared__ int64_t spref[4][32], sbeg[4][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x * 4 + warp;
  if (i >= n_leaves) return;  // whole warp
  const int64_t leaf = leaves[i];
  const int64_t p0 = leaf_start[leaf], p1 = leaf_start[leaf + 1];
  const int n_o = int(p1 - p0);
  const double cx = centers[3 * leaf], cy = centers[3 * leaf + 1], cz = centers[3 * leaf + 2];
  const double qs = k * 0.079577471545947667884;  // k / (4 pi)
  const int64_t nb = near_off[leaf];
  const int nn = int(near_off[leaf + 1] - nb);
  int64_t cnt = 0, beg = 0;
  int self = 0;
  if (lane < nn) {
    const int lf = near[nb + lane];
    beg = leaf_start[lf];
    cnt = leaf_start[lf + 1] - beg;
    self = lf == leaf;
  }
  int64_t incl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int64_t u = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += u;
  }
  const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
  const unsigned selfmask = __ballot_sync(0xffffffffu, self);
  const int sl = selfmask ? __ffs(selfmask) - 1 : 0;
  const int64_t self_b = selfmask ? __shfl_sync(0xffffffffu, incl - cnt, sl) : total;  // self range in the list
  const int64_t self_e = selfmask ? self_b + n_o : total;
  spref[warp][lane] = incl - cnt;  // lanes >= nn: total
  sbeg[warp][lane] = beg;
  const int G = n_o > 0 ? 32 / n_o : 32;
  const int o = lane / G, sub = lane - o * G;
  const bool valid = o < n_o;
  const double xo = valid ? k * (x[p0 + o] - cx) : 0.0;
  const double yo = valid ? k * (y[p0 + o] - cy) : 0.0;
  const double zo = valid ? k * (z[p0 + o] - cz) : 0.0;
  double ar0 = 0.0, ai0 = 0.0, ar1 = 0.0, ai1 = 0.0;
  for (int64_t cb = 0; cb < total; cb += kTW) {
    const int n = int(total - cb < kTW ? total - cb : kTW);
    __syncwarp();
    for (int t = lane; t < n; t += 32) {
      const int64_t v = cb + t;
      int lo = 0, hi = nn;  // largest j with spref[j] <= v
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (spref[warp][mid] <= v) lo = mid; else hi = mid;
      }
      const int64_t src = sbeg[warp][lo] + (v - spref[warp][lo]);
      const double2 qq = q[src];
      sA[warp][t] = make_double4(k * (x[src] - cx), k * (y[src] - cy), k * (z[src] - cz), qs * qq.x);
      sQ[warp][t] = qs * qq.y;
    }
    __syncwarp();
    if (valid) {
      // [0, n) minus the self range [sb, se) of this chunk: two plain segments
      const int sb = int(min(max(self_b - cb, int64_t(0)), int64_t(n)));
      const int se = int(min(max(self_e - cb, int64_t(0)), int64_t(n)));
#pragma unroll
      for (int seg = 0; seg < 2; ++seg) {
        const int lo = seg == 0 ? 0 : se, hi = seg == 0 ? sb : n;
        int t = lo + sub;
        for (; t + G < hi; t += 2 * G) {
          p2p_pair_fast<TAB>(xo, yo, zo, sA[warp][t], sQ[warp][t], ar0, ai0, ptab, tmax);
          p2p_pair_fast<TAB>(xo, yo, zo, sA[warp][t + G], sQ[warp][t + G], ar1, ai1, ptab, tmax);
        }
        if (t < hi) p2p_pair_fast<TAB>(xo, yo, zo, sA[warp][t], sQ[warp][t], ar0, ai0, ptab, tmax);
      }
      // the leaf's own particles: the exact-zero self pair is masked (operators.cpp:118)
      for (int t = sb + sub; t < se; t += G) {
        const double4 sa = sA[warp][t];
        p2p_pair<TAB>(xo, yo, zo, sa.x, sa.y, sa.z, make_double2(sa.w, sQ[warp][t]), ar1, ai1, ptab, tmax);
      }
    }
  }
  double ar = ar0 + ar1, ai = ai0 + ai1;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {  // guarded tree over the G lanes of an observer
    const double ur = __shfl_down_sync(0xffffffffu, ar, off);
    const double ui = __shfl_down_sync(0xffffffffu, ai, off);
    if (sub + off < G) {
      ar += ur;
      ai += ui;
    }
  }
  if (valid && sub == 0) {
    double2 cur = pot[p0 + o];
    cur.x += ar;
    cur.y += ai;
    pot[p0 + o] = cur;
  }
}

}  // namespace hfmm_b200

#endif  // HFMM_B200_P2P_CUH
