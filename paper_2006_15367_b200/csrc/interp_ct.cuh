// Compile-time-shaped fused M2M / L2L (DMMA) for the level pairs of the
// BASELINE configurations.  Same algorithm as interp_tc.cuh (see its header
// for the real + rank-1 split and the row orderings); with (n_c, n_p) known
// at compile time every index map folds to constants, the k-loops unroll,
// padded 8x8 sub-tiles are skipped statically, the two real B matrices live
// in shared memory for the CTA's lifetime, and CTAs are persistent over
// parents so the B staging and the Sacc setup are amortised.
#ifndef HFMM_B200_INTERP_CT_CUH
#define HFMM_B200_INTERP_CT_CUH

#include "interp_tc.cuh"

namespace hfmm_b200 {
namespace ct {

__host__ __device__ constexpr int round4(int v) { return (v + 3) / 4 * 4; }
__host__ __device__ constexpr int round8(int v) { return (v + 7) / 8 * 8; }
__host__ __device__ constexpr int lda_for(int K) { return (K % 8 == 4) ? K : K + 4; }
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

template <int NC, int NP>
struct Shape {
  static constexpr int HALF = NP / 2, SC = NC * NC, SP = NP * NP;
  // M2M passes
  static constexpr int UPHI_K = round4(NC + 1), UPHI_N = round8(NP), UPHI_LDA = lda_for(UPHI_K);
  static constexpr int UTH_K = round4(2 * NC + 1), UTH_N = round8(2 * NP), UTH_LDA = lda_for(UTH_K);
  // L2L passes
  static constexpr int DTH_K = round4(2 * NP + 1), DTH_N = round8(2 * NC), DTH_LDA = lda_for(DTH_K);
  static constexpr int DPHI_K = round4(NP + 1), DPHI_N = round8(NC), DPHI_LDA = lda_for(DPHI_K);
  // B row strides: a multiple of 16 doubles puts the four k-rows of a DMMA
  // B fragment on the same 8 banks, so pad those by 8 (two wavefronts, ideal)
  static constexpr int ldb(int n) { return n % 16 == 0 ? n + 8 : n; }
  static constexpr int UPHI_LDB = ldb(UPHI_N), UTH_LDB = ldb(UTH_N), DTH_LDB = ldb(DTH_N), DPHI_LDB = ldb(DPHI_N);
  // shared-memory footprints in bytes
  static constexpr int m2m_bytes(int cb, int db) {
    return ((db ? 2 : 1) * cb * NC * UPHI_LDA + cb * HALF * UTH_LDA + SP) * 16 +
           (UPHI_K * UPHI_LDB + UTH_K * UTH_LDB) * 8;
  }
  static constexpr int l2l_bytes(int cb, int db) {
    return ((db ? SP : 0) + cb * HALF * DTH_LDA + cb * NC * DPHI_LDA) * 16 + (DTH_K * DTH_LDB + DPHI_K * DPHI_LDB) * 8;
  }
  // plan: children per batch and buffering, two CTAs/SM if possible
  static constexpr int kBudget2 = 113 * 1024, kBudget1 = 227 * 1024;
  static constexpr int pick(bool m2m, int budget, int which) {
    const int cbs[6] = {4, 2, 4, 2, 1, 1}, dbs[6] = {1, 1, 0, 0, 1, 0};
    for (int i = 0; i < 6; ++i) {
      const int b = m2m ? m2m_bytes(cbs[i], dbs[i]) : l2l_bytes(cbs[i], dbs[i]);
      if (b <= budget) return which == 0 ? cbs[i] : which == 1 ? dbs[i] : b;
    }
    return -1;
  }
  static constexpr int M2M_CB = pick(true, kBudget2, 0) > 0 ? pick(true, kBudget2, 0) : pick(true, kBudget1, 0);
  static constexpr int M2M_DB = pick(true, kBudget2, 0) > 0 ? pick(true, kBudget2, 1) : pick(true, kBudget1, 1);
  static constexpr int M2M_BYTES = M2M_CB > 0 ? m2m_bytes(M2M_CB, M2M_DB) : 0;
  static constexpr int L2L_CB = pick(false, kBudget2, 0) > 0 ? pick(false, kBudget2, 0) : pick(false, kBudget1, 0);
  static constexpr int L2L_DB = pick(false, kBudget2, 0) > 0 ? pick(false, kBudget2, 1) : pick(false, kBudget1, 1);
  static constexpr int L2L_BYTES = L2L_CB > 0 ? l2l_bytes(L2L_CB, L2L_DB) : 0;
  // resident CTAs per SM the plan is sized for (the register cap follows it)
  static constexpr int M2M_MINB = M2M_BYTES > 0 && M2M_BYTES <= kBudget2 ? 2 : 1;
  static constexpr int L2L_MINB = L2L_BYTES > 0 && L2L_BYTES <= kBudget2 ? 2 : 1;
};

// Warp-tiled DMMA GEMM with compile-time shape; B (K x N, row-major) in smem.
// Warp tile = up to 2 x 2 8x8 sub-tiles; padded sub-tiles are skipped.
// pre(m0, n0) runs for every live 8x8 sub-tile BEFORE the k-loop (all lanes;
// its result -- e.g. prefetched epilogue operands -- is handed to epi, so
// their latency hides behind the DMMAs); epi(m0, n0, c0, c1, pre) after it.
struct F2x2 {
  double2 v[2];
};
struct D2 {
  double v[2];
};
struct NoPre {
  __device__ __forceinline__ int operator()(int, int) const { return 0; }
};

// One warp tile's k-loop, specialised on its shape (MV x NV live 8x8
// sub-tiles) so the unrolled loop is branch-free: no per-DMMA guards, loads
// unconditional (rows past M point at row 0 and produce finite values the
// epilogues discard), and the compiler can run the loads ahead of the DMMAs.
template <int K, int N, int MV, int NV>
__device__ __forceinline__ void tile_k(const double* __restrict__ a0p, const double* __restrict__ a1p,
                                       const double* __restrict__ bp, double (&c)[2][2][2]) {
#pragma unroll
  for (int k = 0; k < K; k += 4) {
    const double a0 = a0p[2 * k];
    const double b0 = bp[k * N];  // N = B row stride here
    dmma884(c[0][0][0], c[0][0][1], a0, b0);
    if (NV == 2) {
      const double b1 = bp[k * N + 8];
      dmma884(c[0][1][0], c[0][1][1], a0, b1);
      if (MV == 2) {
        const double a1 = a1p[2 * k];
        dmma884(c[1][0][0], c[1][0][1], a1, b0);
        dmma884(c[1][1][0], c[1][1][1], a1, b1);
      }
    } else if (MV == 2) {
      const double a1 = a1p[2 * k];
      dmma884(c[1][0][0], c[1][0][1], a1, b0);
    }
  }
}

template <int M, int N, int K, int LDB = N, class RowPtr, class Epi, class Pre = NoPre>
__device__ __forceinline__ void gemm_ct(RowPtr rowp, const double* __restrict__ Bs, Epi epi, Pre pre = Pre()) {
  constexpr int MT8 = (M + 7) / 8, NT8 = N / 8;
  constexpr int MT = (MT8 + 1) / 2, NT = (NT8 + 1) / 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  for (int w = warp; w < MT * NT; w += kWarps) {
    const int mt = w / NT, nt = w - mt * NT;
    const int m0 = mt * 16, n0 = nt * 16;
    const bool vm1 = 2 * mt + 1 < MT8, vn1 = 2 * nt + 1 < NT8;
    const auto p00 = pre(m0, n0);
    const auto p01 = pre(m0, vn1 ? n0 + 8 : n0);
    const auto p10 = pre(vm1 ? m0 + 8 : m0, n0);
    const auto p11 = pre(vm1 ? m0 + 8 : m0, vn1 ? n0 + 8 : n0);
    const int r0 = m0 + g, r1 = m0 + 8 + g;
    const double* a0p = reinterpret_cast<const double*>(rowp(r0 < M ? r0 >> 1 : 0)) + (r0 < M ? r0 & 1 : 0) + 2 * tq;
    const double* a1p = reinterpret_cast<const double*>(rowp(r1 < M ? r1 >> 1 : 0)) + (r1 < M ? r1 & 1 : 0) + 2 * tq;
    const double* bp = Bs + tq * LDB + n0 + g;
    double c[2][2][2] = {};
    if (vm1 && vn1)
      tile_k<K, LDB, 2, 2>(a0p, a1p, bp, c);
    else if (vm1)
      tile_k<K, LDB, 2, 1>(a0p, a1p, bp, c);
    else if (vn1)
      tile_k<K, LDB, 1, 2>(a0p, a1p, bp, c);
    else
      tile_k<K, LDB, 1, 1>(a0p, a1p, bp, c);
    epi(m0, n0, c[0][0][0], c[0][0][1], p00);
    if (vn1) epi(m0, n0 + 8, c[0][1][0], c[0][1][1], p01);
    if (vm1) {
      epi(m0 + 8, n0, c[1][0][0], c[1][0][1], p10);
      if (vn1) epi(m0 + 8, n0 + 8, c[1][1][0], c[1][1][1], p11);
    }
  }
}

// x[KIN] = i (v . x) for ROWS complex rows (the rank-1 imaginary part of the
// resampling map, interp_tc.cuh).  Four lanes per row, eight rows per warp
// pass: two shuffle levels instead of five.
template <int ROWS, int KIN, int LD>
__device__ __forceinline__ void rank1_ct(double2* X, const double* __restrict__ v) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane & 3;
  constexpr int RUP = (ROWS + 7) / 8 * 8;  // whole warps iterate together (shuffles)
  for (int r = warp * 8 + (lane >> 2); r < RUP; r += kWarps * 8) {
    const bool live = r < ROWS;
    double sr = 0.0, si = 0.0;
    double2* x = X + (live ? r : 0) * LD;
#pragma unroll
    for (int k = sub; k < KIN; k += 4) {
      const double vk = __ldg(v + k);
      const double2 xv = x[k];
      sr = fma(vk, xv.x, sr);
      si = fma(vk, xv.y, si);
    }
    sr += __shfl_xor_sync(0xffffffffu, sr, 1);
    si += __shfl_xor_sync(0xffffffffu, si, 1);
    sr += __shfl_xor_sync(0xffffffffu, sr, 2);
    si += __shfl_xor_sync(0xffffffffu, si, 2);
    if (live && sub == 0) x[KIN] = make_double2(-si, sr);
  }
}

// K x N row-major (global) -> rows of stride ldb (shared), cp.async 16 B.
__device__ __forceinline__ void stage_rows(double* dst, const double* __restrict__ src, int K, int N, int ldb) {
  const int h = N / 2;  // N even
  for (int t = threadIdx.x; t < K * h; t += kThreads) {
    const int r = t / h, c = 2 * (t - r * h);
    cp_async16(dst + r * ldb + c, src + r * N + c, true);
  }
}

__device__ __forceinline__ void stage_doubles(double* dst, const double* __restrict__ src, int n) {
  for (int t = threadIdx.x * 2; t < n; t += kThreads * 2) {
    if (t + 1 < n)
      cp_async16(dst + t, src + t, true);
    else
      dst[t] = src[t];
  }
}

}  // namespace ct

// ---------------------------------------------------------------------------
template <int NC, int NP>
__global__ void __launch_bounds__(ct::kThreads, (ct::Shape<NC, NP>::M2M_MINB)) k_m2m_ct(int n_par, const int* __restrict__ plist,
                                                        const int* __restrict__ child_off,
                                                        const int* __restrict__ children,
                                                        const uint8_t* __restrict__ oct_c,
                                                        const double2* __restrict__ mp_c, double2* __restrict__ mp_p,
                                                        const double* __restrict__ RphiT, const double* __restrict__ vphi,
                                                        const double* __restrict__ RthT, const double* __restrict__ vth,
                                                        const double2* __restrict__ shift_up) {
  using S = ct::Shape<NC, NP>;
  constexpr int CB = S::M2M_CB, DB = S::M2M_DB, HALF = S::HALF, SP = S::SP, SC = S::SC;
  constexpr int XSZ = CB * NC * S::UPHI_LDA, R2 = 2 * CB;
  extern __shared__ double2 sm[];
  double2* Xb0 = sm;
  double2* Xb1 = DB ? sm + XSZ : sm;
  double2* Fs = sm + (DB ? 2 : 1) * XSZ;
  double2* Sacc = Fs + CB * HALF * S::UTH_LDA;
  double* Bphi = reinterpret_cast<double*>(Sacc + SP);
  double* Bth = Bphi + S::UPHI_K * S::UPHI_LDB;
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;

  ct::stage_rows(Bphi, RphiT, S::UPHI_K, S::UPHI_N, S::UPHI_LDB);
  ct::stage_rows(Bth, RthT, S::UTH_K, S::UTH_N, S::UTH_LDB);
  cp_async_commit();
  for (int t = threadIdx.x; t < CB * HALF * S::UTH_LDA; t += ct::kThreads) Fs[t] = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < SP; t += ct::kThreads) Sacc[t] = make_double2(0.0, 0.0);

  // (parent, batch) sequence of this CTA
  auto load = [&](double2* X, int par, int b0) {
    const int ce = child_off[par + 1];
    const int nb = min(CB, ce - b0);
    for (int t = threadIdx.x; t < XSZ; t += ct::kThreads) {
      const int row = t / S::UPHI_LDA, k = t - row * S::UPHI_LDA;
      const int c = row / NC, i = row - c * NC;
      const bool ok = c < nb && k < NC;
      cp_async16(X + t, ok ? mp_c + int64_t(children[b0 + c]) * SC + i * NC + k : mp_c, ok);
    }
    cp_async_commit();
  };
  int par = blockIdx.x;
  if (par >= n_par) return;
  int b0 = child_off[par];
  load(Xb0, par, b0);
  int it = 0;
  while (par < n_par) {
    const int ce = child_off[par + 1];
    const int nb = min(CB, ce - b0);
    // next (parent, batch) of this CTA
    int npar = par, nb0 = b0 + CB;
    if (nb0 >= ce) {
      npar = par + gridDim.x;
      nb0 = npar < n_par ? child_off[npar] : 0;
    }
    double2* X = (it & 1) ? Xb1 : Xb0;
    if (DB && npar < n_par) {
      load((it & 1) ? Xb0 : Xb1, npar, nb0);
      cp_async_wait<1>();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    ct::rank1_ct<CB * NC, NC, S::UPHI_LDA>(X, vphi);
    __syncthreads();
    // phi pass -> folded circles
    ct::gemm_ct<CB * NC * 2, S::UPHI_N, S::UPHI_K, S::UPHI_LDB>(
        [&](int r) { return X + r * S::UPHI_LDA; }, Bphi, [&](int m0, int n0, double v0, double v1, int) {
          const int r = m0 + g, ci = r >> 1, c = ci / NC, i = ci - c * NC;
          if (c >= CB) return;
          double2* base = Fs + c * HALF * S::UTH_LDA;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = n0 + 2 * tq + q;
            if (n < NP) {
              const int p = n < HALF ? n : n - HALF;
              const int ii = n < HALF ? i : 2 * NC - 1 - i;
              set_part(base + p * S::UTH_LDA + ii, r & 1, q ? v1 : v0);
            }
          }
        });
    __syncthreads();
    if (!DB && npar < n_par) load(Xb0, npar, nb0);  // single buffer: overlap the next load with theta
    ct::rank1_ct<CB * HALF, 2 * NC, S::UTH_LDA>(Fs, vth);
    __syncthreads();
    int octs[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) octs[c] = c < nb ? oct_c[children[b0 + c]] : 0;
    // theta pass, rows (circle, child, re/im); children reduce in-warp
    ct::gemm_ct<HALF * R2, S::UTH_N, S::UTH_K, S::UTH_LDB>(
        [&](int row) {
          const int p = row / CB, c = row - p * CB;
          return Fs + (c * HALF + p) * S::UTH_LDA;
        },
        Bth,
        [&](int m0, int n0, double v0, double v1, const ct::F2x2& f) {
          const int r = m0 + g, part = r & 1, c = (r >> 1) % CB, p = r / R2;
          const double o0 = __shfl_xor_sync(0xffffffffu, v0, 4);
          const double o1 = __shfl_xor_sync(0xffffffffu, v1, 4);
          double cr[2], cim[2];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const double re = part ? (q ? o1 : o0) : (q ? v1 : v0);
            const double im = part ? (q ? v1 : v0) : (q ? o1 : o0);
            cr[q] = re * f.v[q].x - im * f.v[q].y;
            cim[q] = re * f.v[q].y + im * f.v[q].x;
          }
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
          if (part == 0 && c == 0 && p < HALF) {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int n = n0 + 2 * tq + q;
              if (n < 2 * NP) {
                const int s = n < NP ? n * NP + p : (2 * NP - 1 - n) * NP + p + HALF;
                double2 a = Sacc[s];
                a.x += cr[q];
                a.y += cim[q];
                Sacc[s] = a;
              }
            }
          }
        },
        [&](int m0, int n0) {  // shift factors of this lane's two outputs, loaded ahead of the k-loop
          const int r = m0 + g, c = (r >> 1) % CB, p = r / R2;
          const bool live = c < nb && p < HALF;
          const double2* sh = shift_up + octs[c] * SP;
          ct::F2x2 f;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = n0 + 2 * tq + q;
            const int s = n < NP ? n * NP + p : (2 * NP - 1 - n) * NP + p + HALF;
            f.v[q] = (live && n < 2 * NP) ? __ldg(sh + s) : make_double2(0.0, 0.0);
          }
          return f;
        });
    __syncthreads();
    if (npar != par) {  // parent complete: write out and reset the accumulator
      for (int t = threadIdx.x; t < SP; t += ct::kThreads) {
        mp_p[int64_t(plist ? plist[par] : par) * SP + t] = Sacc[t];
        Sacc[t] = make_double2(0.0, 0.0);
      }
    }
    par = npar;
    b0 = nb0;
    ++it;
  }
}

// ---------------------------------------------------------------------------
template <int NC, int NP>
__global__ void __launch_bounds__(ct::kThreads, (ct::Shape<NC, NP>::L2L_MINB)) k_l2l_ct(int n_par, const int* __restrict__ plist,
                                                        const int* __restrict__ child_off,
                                                        const int* __restrict__ children,
                                                        const uint8_t* __restrict__ oct_c,
                                                        const double2* __restrict__ loc_p, double2* __restrict__ loc_c,
                                                        const double* __restrict__ RthT, const double* __restrict__ vth,
                                                        const double* __restrict__ RphiT, const double* __restrict__ vphi,
                                                        const double2* __restrict__ shift_dn) {
  using S = ct::Shape<NC, NP>;
  constexpr int CB = S::L2L_CB, DB = S::L2L_DB, HALF = S::HALF, SP = S::SP, SC = S::SC;
  extern __shared__ double2 sm[];
  double2* Lp = sm;
  double2* Fs = DB ? sm + SP : sm;
  double2* Ns = Fs + CB * HALF * S::DTH_LDA;
  double* Bth = reinterpret_cast<double*>(Ns + CB * NC * S::DPHI_LDA);
  double* Bphi = Bth + S::DTH_K * S::DTH_LDB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  double* lc = reinterpret_cast<double*>(loc_c);

  ct::stage_rows(Bth, RthT, S::DTH_K, S::DTH_N, S::DTH_LDB);
  ct::stage_rows(Bphi, RphiT, S::DPHI_K, S::DPHI_N, S::DPHI_LDB);
  cp_async_commit();
  for (int t = threadIdx.x; t < CB * HALF * S::DTH_LDA; t += ct::kThreads) Fs[t] = make_double2(0.0, 0.0);
  for (int t = threadIdx.x; t < CB * NC * S::DPHI_LDA; t += ct::kThreads) Ns[t] = make_double2(0.0, 0.0);

  for (int par = blockIdx.x; par < n_par; par += gridDim.x) {
    const int cb = child_off[par], ce = child_off[par + 1];
    const double2* lpg = loc_p + int64_t(plist ? plist[par] : par) * SP;
    __syncthreads();  // previous parent done with Lp
    if (DB) {
      for (int t = threadIdx.x; t < SP; t += ct::kThreads) cp_async16(Lp + t, lpg + t, true);
      cp_async_commit();
    }
    cp_async_wait_all();
    __syncthreads();
    const double2* L = DB ? Lp : lpg;
    for (int b0 = cb; b0 < ce; b0 += CB) {
      const int nb = min(CB, ce - b0);
      // Child pointers of the batch first (dependent loads), then the shifted
      // parent circles: flat over (child, circle, sample), FB elements per
      // thread per round with every load of the round in flight together.
      int64_t cnode[CB];
      const double2* shc[CB];
#pragma unroll
      for (int c = 0; c < CB; ++c) {
        cnode[c] = c < nb ? children[b0 + c] : 0;
        shc[c] = shift_dn + int64_t(c < nb ? oct_c[cnode[c]] : 0) * SP;
      }
      {
        constexpr int FE = CB * HALF * 2 * NP, FPT = (FE + ct::kThreads - 1) / ct::kThreads, FB = 5;
#pragma unroll
        for (int j0 = 0; j0 < FPT; j0 += FB) {
          double2 lv[FB], sv[FB];
#pragma unroll
          for (int u = 0; u < FB; ++u) {
            const int t = threadIdx.x + (j0 + u) * ct::kThreads;
            const int c = t / (HALF * 2 * NP), rem = t - c * (HALF * 2 * NP), p = rem / (2 * NP), i = rem - p * (2 * NP);
            const int s = i < NP ? i * NP + p : (2 * NP - 1 - i) * NP + p + HALF;
            const double2* sh = shc[0];
#pragma unroll
            for (int cc = 1; cc < CB; ++cc) sh = c == cc ? shc[cc] : sh;
            const bool ok = j0 + u < FPT && t < FE && c < nb;
            lv[u] = ok ? L[s] : make_double2(0.0, 0.0);
            sv[u] = ok ? __ldg(sh + s) : make_double2(0.0, 0.0);
          }
#pragma unroll
          for (int u = 0; u < FB; ++u) {
            const int t = threadIdx.x + (j0 + u) * ct::kThreads;
            const int c = t / (HALF * 2 * NP), rem = t - c * (HALF * 2 * NP), p = rem / (2 * NP), i = rem - p * (2 * NP);
            if (j0 + u < FPT && t < FE) Fs[(c * HALF + p) * S::DTH_LDA + i] = cmul(lv[u], sv[u]);
          }
        }
      }
      __syncthreads();
      ct::rank1_ct<CB * HALF, 2 * NP, S::DTH_LDA>(Fs, vth);
      __syncthreads();
      ct::gemm_ct<CB * HALF * 2, S::DTH_N, S::DTH_K, S::DTH_LDB>(
          [&](int r) { return Fs + r * S::DTH_LDA; }, Bth, [&](int m0, int n0, double v0, double v1, int) {
            const int r = m0 + g, ci = r >> 1, c = ci / HALF, p = ci - c * HALF;
            if (c >= CB) return;
            double2* base = Ns + c * NC * S::DPHI_LDA;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int n = n0 + 2 * tq + q;
              if (n < 2 * NC) {
                const int row = n < NC ? n : 2 * NC - 1 - n;
                const int col = n < NC ? p : p + HALF;
                set_part(base + row * S::DPHI_LDA + col, r & 1, q ? v1 : v0);
              }
            }
          });
      __syncthreads();
      ct::rank1_ct<CB * NC, NP, S::DPHI_LDA>(Ns, vphi);
      __syncthreads();
      ct::gemm_ct<CB * NC * 2, S::DPHI_N, S::DPHI_K, S::DPHI_LDB>(
          [&](int r) { return Ns + r * S::DPHI_LDA; }, Bphi,
          [&](int m0, int n0, double v0, double v1, const ct::D2& old) {
            const int r = m0 + g, ci = r >> 1, c = ci / NC, row = ci - c * NC;
            if (c >= nb) return;
            int64_t node = cnode[0];
#pragma unroll
            for (int cc = 1; cc < CB; ++cc) node = c == cc ? cnode[cc] : node;
            double* dst = lc + 2 * (node * SC + row * NC) + (r & 1);
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int n = n0 + 2 * tq + q;
              if (n < NC) dst[2 * n] = old.v[q] + (q ? v1 : v0);
            }
          },
          [&](int m0, int n0) {  // the child locals this lane adds to, loaded ahead of the k-loop
            const int r = m0 + g, ci = r >> 1, c = ci / NC, row = ci - c * NC;
            int64_t node = cnode[0];
#pragma unroll
            for (int cc = 1; cc < CB; ++cc) node = c == cc ? cnode[cc] : node;
            const double* dst = lc + 2 * (node * SC + row * NC) + (r & 1);
            ct::D2 o;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const int n = n0 + 2 * tq + q;
              o.v[q] = (c < nb && n < NC) ? dst[2 * n] : 0.0;
            }
            return o;
          });
      __syncthreads();
    }
  }
}

// Dispatch over the instantiated (n_c, n_p) pairs; returns false if the pair
// has no compile-time kernel (the runtime-shaped kernels then run).
#define HFMM_CT_PAIRS(X) \
  X(18, 28) X(28, 42) X(42, 68) X(22, 30) X(30, 44) X(44, 72) X(26, 34) X(34, 52) X(52, 80)

struct CtLaunch {
  int n_par;
  const int* plist;  // parent indices (nullptr: identity)
  const int* child_off;
  const int* children;
  const uint8_t* oct_c;
  cudaStream_t st;
};

template <int NC, int NP>
inline int ct_grid(int n_par, int bytes, const void* fn) {
  int per_sm = 0, sms = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, ct::kThreads, size_t(bytes));
  const int g = sms * (per_sm > 0 ? per_sm : 1) * 4;
  return n_par < g ? n_par : g;
}

template <int A, int B>
bool try_m2m_ct(const CtLaunch& L, const double2* mp_c, double2* mp_p, const double* Bphi, const double* vphi,
                const double* Bth, const double* vth, const double2* shift_up) {
  using S = ct::Shape<A, B>;
  if constexpr (S::M2M_CB > 0) {
    auto fn = k_m2m_ct<A, B>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, S::M2M_BYTES);
    const int grid = ct_grid<A, B>(L.n_par, S::M2M_BYTES, reinterpret_cast<const void*>(fn));
    fn<<<grid, ct::kThreads, S::M2M_BYTES, L.st>>>(L.n_par, L.plist, L.child_off, L.children, L.oct_c, mp_c, mp_p, Bphi,
                                                   vphi, Bth, vth, shift_up);
    return true;
  } else {
    return false;
  }
}

template <int A, int B>
bool try_l2l_ct(const CtLaunch& L, const double2* loc_p, double2* loc_c, const double* Bth, const double* vth,
                const double* Bphi, const double* vphi, const double2* shift_dn) {
  using S = ct::Shape<A, B>;
  // Measured against the two-stage kernels (interp_big.cuh) at config 2:
  // (26,34) 7.9 vs 9.9 ms; (34,52) L2L phase 12.33 vs 12.74 ms; neutral on configs 1, 3-5.
  if constexpr (S::L2L_CB > 0) {
    auto fn = k_l2l_ct<A, B>;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, S::L2L_BYTES);
    const int grid = ct_grid<A, B>(L.n_par, S::L2L_BYTES, reinterpret_cast<const void*>(fn));
    fn<<<grid, ct::kThreads, S::L2L_BYTES, L.st>>>(L.n_par, L.plist, L.child_off, L.children, L.oct_c, loc_p, loc_c, Bth,
                                                   vth, Bphi, vphi, shift_dn);
    return true;
  } else {
    return false;
  }
}

inline bool launch_m2m_ct(int nc, int np, const CtLaunch& L, const double2* mp_c, double2* mp_p, const double* Bphi,
                          const double* vphi, const double* Bth, const double* vth, const double2* shift_up) {
#define HFMM_M2M_CASE(A, B) \
  if (nc == A && np == B) return try_m2m_ct<A, B>(L, mp_c, mp_p, Bphi, vphi, Bth, vth, shift_up);
  HFMM_CT_PAIRS(HFMM_M2M_CASE)
#undef HFMM_M2M_CASE
  return false;
}

inline bool launch_l2l_ct(int nc, int np, const CtLaunch& L, const double2* loc_p, double2* loc_c, const double* Bth,
                          const double* vth, const double* Bphi, const double* vphi, const double2* shift_dn) {
#define HFMM_L2L_CASE(A, B) \
  if (nc == A && np == B) return try_l2l_ct<A, B>(L, loc_p, loc_c, Bth, vth, Bphi, vphi, shift_dn);
  HFMM_CT_PAIRS(HFMM_L2L_CASE)
#undef HFMM_L2L_CASE
  return false;
}

}  // namespace hfmm_b200

#endif
