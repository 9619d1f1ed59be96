// Streaming M2M / L2L on DMMA with complex-row warp tiles.
//
// Same algorithm as interp_ct.cuh (real matrix + rank-1 imaginary part of
// resample_circle, sphere_grid.cpp:128-155; M2M = phi pass, fold, theta pass,
// shift, child sum, traversal.cpp:322-429; L2L mirrored, :583-707), organised
// for throughput:
//  * a warp tile is 8 COMPLEX rows x N: two m8 DMMA fragments (real parts,
//    imaginary parts) that share every B fragment, so a lane holds both parts
//    of its row -- the rank-1 column i (v . x) needs no partner shuffle and the
//    epilogue sees complex values;
//  * B (the level's real interpolation matrix) is staged once per persistent
//    CTA in shared memory; A rows stream from global memory / L1 straight
//    into registers; there are no barriers after the B staging;
//  * the two passes are two kernels with the intermediate in HBM scratch
//    (M2M: folded circles F; L2L: narrow rows Nb);
//  * the M2M theta pass puts the 8 child slots of a parent in the 8 rows of a
//    tile, so the child sum is a 3-level shuffle and every parent sample is
//    written exactly once (no shared accumulator);
//  * the theta passes of the compile-time-shaped kernels run in the even / odd
//    form (interp.hpp:even_odd): the theta map of a folded great circle is
//    centrosymmetric, so it splits into two half-size products on
//    x_e = x + Jx and x_o = x - Jx -- 80 DMMA per (18, 28) circle tile instead
//    of 140.  The fold is baked into the columns of the M2M phi matrix and the
//    unfold into the rows of the L2L phi matrix (fold_columns / unfold_rows),
//    so the phi passes deliver and consume (e, o) pairs at no cost.
#ifndef HFMM_B200_INTERP_RB_CUH
#define HFMM_B200_INTERP_RB_CUH

#include "bulk.cuh"
#include "dmma.cuh"

namespace hfmm_b200 {
namespace rb {

__host__ __device__ constexpr int r4(int v) { return (v + 3) / 4 * 4; }
__host__ __device__ constexpr int r8(int v) { return (v + 7) / 8 * 8; }
// B fragment of m8n8k4: lane (g, tq) reads B[4 kk + tq][8 j + g], an 8-byte load
// served per half-warp (g in a group of 4, tq = 0..3): conflict free when the
// four tq rows land 4 doubles apart (mod 16), i.e. row stride == 4 (mod 8).
// (ncu showed the earlier stride == 8 (mod 16) at 4 wavefronts per load, 2 of
// them bank conflicts.)
__host__ __device__ constexpr int ldb(int n) { return n % 8 == 4 ? n : n + 4 + (8 - n % 8) % 8; }
constexpr int kThreads = 256;

// Parent descriptor (3 int4 per parent, built once per level by k_build_pdesc):
// {first child position, child count, parent row, octants (4 bits per child
// slot)} + the 8 child rows.  The work loops of the theta passes load it one
// item ahead; before, every item began with a chain of dependent global loads
// (child_off -> children -> octant -> shift table -> data), which ncu showed as
// the long-scoreboard stall at the top of these kernels.
__device__ __forceinline__ int pdesc_oct(const int4& d, int slot) { return (d.w >> (4 * slot)) & 7; }

// K x N row-major B (global) -> shared rows of stride LDB (persistent CTA, once).
template <int K, int N, int LDB>
__device__ __forceinline__ void stage_b(double* dst, const double* __restrict__ src) {
  for (int t = threadIdx.x; t < K * N / 2; t += blockDim.x) {
    const int r = t / (N / 2), c = 2 * (t - r * (N / 2));
    cp_async16(dst + r * LDB + c, src + r * N + c, true);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
}

// Rank-1 column: lane (g, tq) holds x_re / x_im of row g at columns 4 kk + tq
// (zeros past KIN); inject i (v . x) at column KIN.
template <int KS, int KIN, class V>
__device__ __forceinline__ void rank1_inject_f(double (&are)[KS], double (&aim)[KS], V vf) {
  const int tq = threadIdx.x & 3;
  // two partial sums per part (even / odd k-steps): the dependent DFMA chain is
  // KS / 2 deep instead of KS (FP64 latency is ~8 issue slots, tools/fp64_lat.cu)
  double sr[2] = {0.0, 0.0}, si[2] = {0.0, 0.0};
#pragma unroll
  for (int kk = 0; kk < KS; ++kk) {
    const int k = 4 * kk + tq;
    if (k < KIN) {
      const double vk = vf(k);
      sr[kk & 1] = fma(vk, are[kk], sr[kk & 1]);
      si[kk & 1] = fma(vk, aim[kk], si[kk & 1]);
    }
  }
  double tr = sr[0] + sr[1], ti = si[0] + si[1];
  tr += __shfl_xor_sync(0xffffffffu, tr, 1);
  ti += __shfl_xor_sync(0xffffffffu, ti, 1);
  tr += __shfl_xor_sync(0xffffffffu, tr, 2);
  ti += __shfl_xor_sync(0xffffffffu, ti, 2);
  constexpr int KR = KIN / 4, TR = KIN % 4;
  if (tq == TR) {
    are[KR] = -ti;  // Re(i alpha)
    aim[KR] = tr;   // Im(i alpha)
  }
}
template <int KS, int KIN>
__device__ __forceinline__ void rank1_inject(double (&are)[KS], double (&aim)[KS], const double* __restrict__ v) {
  rank1_inject_f<KS, KIN>(are, aim, [&](int k) { return __ldg(v + k); });
}

// Sum over the 8 child rows of a warp tile (lane bits 2..4 = g) of a chunk of
// 4 n8 tiles: v[(2 jc + q) 2 + part] are the lane's 16 values (tile jc,
// column 2 tq + q, re/im).  A reduce-scatter (8 + 4 + 2 shuffles instead of
// 3 x 16) leaves lane (g, tq) with column n = 8 (g >> 1) + 2 tq + (g & 1) of
// the chunk, returned as (re, im).
__device__ __forceinline__ double2 child_sum_scatter(double (&v)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int w = 16, h = 8; w >= 4; w >>= 1, h >>= 1) {
    const bool hi = lane & w;
#pragma unroll
    for (int i = 0; i < h; ++i) {
      const double send = hi ? v[i] : v[i + h], keep = hi ? v[i + h] : v[i];
      v[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
  return make_double2(v[0], v[1]);
}

// C (8 complex rows x NT n8 tiles) += A (8 x K) B (K x 8 NT): 2 NT DMMA per k-step.
template <int KS, int NT, int LDB>
__device__ __forceinline__ void tile_mma(const double (&are)[KS], const double (&aim)[KS], const double* __restrict__ Bs,
                                         double (&cre)[NT][2], double (&cim)[NT][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const double* bp = Bs + tq * LDB + g;
#pragma unroll
  for (int kk = 0; kk < KS; ++kk)
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const double b = bp[4 * kk * LDB + 8 * j];
      dmma884(cre[j][0], cre[j][1], are[kk], b);
      dmma884(cim[j][0], cim[j][1], aim[kk], b);
    }
}

// Rank-1 column of the even / odd theta passes: alpha = v_e . x_e + v_o . x_o
// (v laid out like the B rows: v_o at 4 KH), injected as i alpha at column KIN
// of both halves (the B rows there hold the symmetric / antisymmetric part of u).
template <int KH, int KIN, class V>
__device__ __forceinline__ void rank1_inject_eo_f(double (&er)[KH], double (&ei)[KH], double (&qr)[KH], double (&qi)[KH],
                                                  V vf) {
  const int tq = threadIdx.x & 3;
  // separate partial sums for the even and the odd half (and alternate k-steps):
  // dependent chains of KH / 2 DFMA instead of 2 KH
  double se[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, so[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int kk = 0; kk < KH; ++kk) {
    const int k = 4 * kk + tq;
    if (k < KIN) {
      const double ve = vf(k), vo = vf(4 * KH + k);
      se[kk & 1][0] = fma(ve, er[kk], se[kk & 1][0]);
      se[kk & 1][1] = fma(ve, ei[kk], se[kk & 1][1]);
      so[kk & 1][0] = fma(vo, qr[kk], so[kk & 1][0]);
      so[kk & 1][1] = fma(vo, qi[kk], so[kk & 1][1]);
    }
  }
  double sr = (se[0][0] + se[1][0]) + (so[0][0] + so[1][0]);
  double si = (se[0][1] + se[1][1]) + (so[0][1] + so[1][1]);
  sr += __shfl_xor_sync(0xffffffffu, sr, 1);
  si += __shfl_xor_sync(0xffffffffu, si, 1);
  sr += __shfl_xor_sync(0xffffffffu, sr, 2);
  si += __shfl_xor_sync(0xffffffffu, si, 2);
  constexpr int KR = KIN / 4, TR = KIN % 4;
  static_assert(KR < KH, "rank-1 column outside the padded K");
  if (tq == TR) {
    er[KR] = qr[KR] = -si;  // Re(i alpha)
    ei[KR] = qi[KR] = sr;   // Im(i alpha)
  }
}
template <int KH, int KIN>
__device__ __forceinline__ void rank1_inject_eo(double (&er)[KH], double (&ei)[KH], double (&qr)[KH], double (&qi)[KH],
                                                const double* __restrict__ v) {
  rank1_inject_eo_f<KH, KIN>(er, ei, qr, qi, [&](int k) { return __ldg(v + k); });
}

template <int NC, int NP>
struct Dims {
  static constexpr int HALF = NP / 2, SC = NC * NC, SP = NP * NP;
  // M2M phi: X (NC x NC) rows -> NP outputs (column 2 p + h: circle p, part e / o);
  // theta, even / odd form: x_e, x_o (NC each, + rank-1 column) -> Ye, Yo (NP each)
  static constexpr int UPHI_K = r4(NC + 1), UPHI_N = r8(NP), UPHI_LDB = ldb(UPHI_N);
  static constexpr int UTH_KH = r4(NC + 1) / 4;  // k-steps per half
  static constexpr int UTH_K = 8 * UTH_KH, UTH_N = r8(NP), UTH_LDB = ldb(UTH_N);  // B rows: [Be ; Bo]
  static constexpr int LDF = UTH_K;  // F scratch row stride (complex): x_e at 0, x_o at 4 UTH_KH
  // L2L theta, even / odd form: NP + NP -> NC + NC; phi: NP (pairs Ye, Yo) -> NC
  static constexpr int DTH_KH = r4(NP + 1) / 4;
  static constexpr int DTH_K = 8 * DTH_KH, DTH_N = r8(NC), DTH_LDB = ldb(DTH_N);
  static constexpr int DPHI_K = r4(NP + 1), DPHI_N = r8(NC), DPHI_LDB = ldb(DPHI_N);
  static constexpr int LDN = NP;  // Nb scratch row stride (complex): NP / 2 (Ye, Yo) pairs, no padding
                                  // (the phi pass never reads past column NP: 12% less scratch traffic at (18, 28))
};

// M2M theta pass of one work item (parent, circle p), even / odd form: tile
// rows = the parent's 8 child slots; ld(k) reads element k of the lane's F row
// (x_e at [0, NC), x_o at [4 KH, 4 KH + NC)).  Ye +- Yo are the circle's front
// (theta row n, column p) and back (column p + HALF) samples; both get their
// shift factor and go through one child-sum reduce-scatter per 2 n8 tiles.
// shf(n, back) -> the shift factor of the lane's child at (theta row n, column
// p + back HALF); vf(k) -> entry k of the [v_e ; v_o] vector.
template <int NC, int NP, class Ld, class Sh, class V>
__device__ __forceinline__ void m2m_theta_item_f(Ld ld, bool ok, Sh shf_, double2* __restrict__ out, int p,
                                                 const double* __restrict__ Bt, V vf) {
  using D = Dims<NC, NP>;
  constexpr int KH = D::UTH_KH, NT = D::UTH_N / 8, HALF = D::HALF, LDB = D::UTH_LDB;
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  double er[KH], ei[KH], qr[KH], qi[KH];
#pragma unroll
  for (int kk = 0; kk < KH; ++kk) {
    const int k = 4 * kk + tq;
    const bool in = ok && k < NC;
    const double2 e = in ? ld(k) : make_double2(0.0, 0.0);
    const double2 o = in ? ld(4 * KH + k) : make_double2(0.0, 0.0);
    er[kk] = e.x;
    ei[kk] = e.y;
    qr[kk] = o.x;
    qi[kk] = o.y;
  }
  rank1_inject_eo_f<KH, NC>(er, ei, qr, qi, vf);
  constexpr int NTC = 2;
#pragma unroll
  for (int j0 = 0; j0 < NT; j0 += NTC) {
    double2 shf[NTC][2], shb[NTC][2];
#pragma unroll
    for (int jc = 0; jc < NTC; ++jc)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int n = 8 * (j0 + jc) + 2 * tq + q;
        const bool live = ok && j0 + jc < NT && n < NP;
        shf[jc][q] = live ? shf_(n, 0) : make_double2(0.0, 0.0);
        shb[jc][q] = live ? shf_(n, 1) : make_double2(0.0, 0.0);
      }
    double cer[NTC][2] = {}, cei[NTC][2] = {}, cqr[NTC][2] = {}, cqi[NTC][2] = {};
    const double* bp = Bt + tq * LDB + g + 8 * j0;
#pragma unroll
    for (int kk = 0; kk < KH; ++kk)
#pragma unroll
      for (int jc = 0; jc < NTC; ++jc)
        if (j0 + jc < NT) {
          const double be = bp[4 * kk * LDB + 8 * jc];
          dmma884(cer[jc][0], cer[jc][1], er[kk], be);
          dmma884(cei[jc][0], cei[jc][1], ei[kk], be);
          const double bo = bp[4 * (KH + kk) * LDB + 8 * jc];
          dmma884(cqr[jc][0], cqr[jc][1], qr[kk], bo);
          dmma884(cqi[jc][0], cqi[jc][1], qi[kk], bo);
        }
    double v[16];  // child_sum_scatter slots: front tiles 0, 1, then back tiles 0, 1
#pragma unroll
    for (int jc = 0; jc < NTC; ++jc)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double fr = cer[jc][q] + cqr[jc][q], fi = cei[jc][q] + cqi[jc][q];
        const double br = cer[jc][q] - cqr[jc][q], bi = cei[jc][q] - cqi[jc][q];
        const double2 f = shf[jc][q], b = shb[jc][q];
        v[(2 * jc + q) * 2] = fr * f.x - fi * f.y;
        v[(2 * jc + q) * 2 + 1] = fr * f.y + fi * f.x;
        v[(2 * (NTC + jc) + q) * 2] = br * b.x - bi * b.y;
        v[(2 * (NTC + jc) + q) * 2 + 1] = br * b.y + bi * b.x;
      }
    const double2 val = child_sum_scatter(v);
    const int slot = g >> 1, back = slot >= NTC, jt = j0 + slot - back * NTC, n = 8 * jt + 2 * tq + (g & 1);
    if (jt < NT && n < NP) out[n * NP + p + back * HALF] = val;
  }
}
template <int NC, int NP, class Ld>
__device__ __forceinline__ void m2m_theta_item(Ld ld, bool ok, const double2* __restrict__ sh, double2* __restrict__ out,
                                               int p, const double* __restrict__ Bt, const double* __restrict__ vth) {
  constexpr int HALF = NP / 2;
  m2m_theta_item_f<NC, NP>(ld, ok, [&](int n, int back) { return __ldg(sh + n * NP + p + back * HALF); }, out, p, Bt,
                           [&](int k) { return __ldg(vth + k); });
}

}  // namespace rb

__global__ void k_build_pdesc(int n_par, const int* __restrict__ plist, const int* __restrict__ child_off,
                              const int* __restrict__ children, const uint8_t* __restrict__ oct_c,
                              int4* __restrict__ out) {
  const int par = blockIdx.x * blockDim.x + threadIdx.x;
  if (par >= n_par) return;
  const int cb = child_off[par], n = child_off[par + 1] - cb;
  int ch[8], octs = 0;
  for (int c = 0; c < 8; ++c) {
    ch[c] = c < n ? children[cb + c] : -1;
    if (c < n) octs |= int(oct_c[ch[c]]) << (4 * c);
  }
  out[3 * par] = make_int4(cb, n, plist ? plist[par] : par, octs);
  out[3 * par + 1] = make_int4(ch[0], ch[1], ch[2], ch[3]);
  out[3 * par + 2] = make_int4(ch[4], ch[5], ch[6], ch[7]);
}

// ---------------------------------------------------------------------------
// M2M stage 1: phi pass of every child row -> folded circles in (e, o) form,
// F[j][p][..] (j = position in the children array): x_e[i] at i, x_o[i] at
// 4 UTH_KH + i (the phi matrix's column 2 p + h carries part h of circle p).
template <int NC, int NP>
__global__ void __launch_bounds__(rb::kThreads, 2) k_m2m_phi_rb(int64_t nch, const int* __restrict__ children,
                                                                const double2* __restrict__ mp_c,
                                                                const double* __restrict__ B,
                                                                const double* __restrict__ v,
                                                                double2* __restrict__ F) {
  using D = rb::Dims<NC, NP>;
  constexpr int KS = D::UPHI_K / 4, NT = D::UPHI_N / 8, HALF = D::HALF;
  __shared__ __align__(16) double Bs[D::UPHI_K * D::UPHI_LDB];
  rb::stage_b<D::UPHI_K, D::UPHI_N, D::UPHI_LDB>(Bs, B);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int64_t rows = nch * NC, tiles = (rows + 7) / 8;
  for (int64_t t = int64_t(blockIdx.x) * (rb::kThreads / 32) + warp; t < tiles;
       t += int64_t(gridDim.x) * (rb::kThreads / 32)) {
    const int64_t R = t * 8 + g;
    const bool ok = R < rows;
    const int64_t j = ok ? R / NC : 0;
    const int i = ok ? int(R - j * NC) : 0;
    const int64_t node = children ? children[j] : j;
    const double2* x = mp_c + node * D::SC + i * NC;
    double are[KS], aim[KS];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      const int k = 4 * kk + tq;
      const double2 xv = (ok && k < NC) ? __ldg(x + k) : make_double2(0.0, 0.0);
      are[kk] = xv.x;
      aim[kk] = xv.y;
    }
    rb::rank1_inject<KS, NC>(are, aim, v);
    double cre[NT][2] = {}, cim[NT][2] = {};
    rb::tile_mma<KS, NT, D::UPHI_LDB>(are, aim, Bs, cre, cim);
    if (ok) {
      double2* Fj = F + j * HALF * D::LDF;
#pragma unroll
      for (int jn = 0; jn < NT; ++jn)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int n = 8 * jn + 2 * tq + q;
          if (n < NP) Fj[(n >> 1) * D::LDF + (n & 1) * 4 * D::UTH_KH + i] = make_double2(cre[jn][q], cim[jn][q]);
        }
    }
  }
}

// M2M stage 2: theta pass + shift + child sum.  Work item = (parent, circle p);
// tile rows = the parent's 8 child slots (absent children read as zero).
template <int NC, int NP>
__global__ void __launch_bounds__(rb::kThreads, 2) k_m2m_theta_rb(int n_par, const int4* __restrict__ pdesc,
                                                                  const double2* __restrict__ F,
                                                                  const double* __restrict__ B,
                                                                  const double* __restrict__ v,
                                                                  const double2* __restrict__ shift_up,
                                                                  double2* __restrict__ mp_p) {
  using D = rb::Dims<NC, NP>;
  constexpr int HALF = D::HALF, SP = D::SP;
  extern __shared__ __align__(16) double Bsm[];
  rb::stage_b<D::UTH_K, D::UTH_N, D::UTH_LDB>(Bsm, B);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2;
  const int64_t items = int64_t(n_par) * HALF, stride = int64_t(gridDim.x) * (rb::kThreads / 32);
  int64_t it = int64_t(blockIdx.x) * (rb::kThreads / 32) + warp;
  int4 dn = it < items ? __ldg(pdesc + 3 * (it / HALF)) : make_int4(0, 0, 0, 0);
  for (; it < items; it += stride) {
    const int4 dc = dn;  // parent descriptor, loaded one item ahead (rb::PDesc)
    if (it + stride < items) dn = __ldg(pdesc + 3 * ((it + stride) / HALF));
    const int par = int(it / HALF), p = int(it - int64_t(par) * HALF);
    const int cb = dc.x, nchp = dc.y;
    const bool ok = g < nchp;
    const double2* frow = F + (int64_t(cb + (ok ? g : 0)) * HALF + p) * D::LDF;
    const double2* sh = shift_up + int64_t(ok ? rb::pdesc_oct(dc, g) : 0) * SP;
    double2* out = mp_p + int64_t(dc.z) * SP;
    rb::m2m_theta_item<NC, NP>([&](int k) { return __ldg(frow + k); }, ok, sh, out, p, Bsm, v);
  }
}

// ---------------------------------------------------------------------------
// L2L stage 1: shifted, folded parent circles -> theta anterpolation -> narrow
// rows Nb[j][row][col] (j = position in the children array).  Work item =
// (parent, 8 rows of the (child slot, circle) space); each lane builds its A
// row on the fly, L_p[s] shift_c[s] (one complex product feeds both parts).
template <int NC, int NP>
__global__ void __launch_bounds__(rb::kThreads, 2) k_l2l_theta_rb(int n_par, const int4* __restrict__ pdesc,
                                                                  const double2* __restrict__ loc_p,
                                                                  const double* __restrict__ B,
                                                                  const double* __restrict__ v,
                                                                  const double2* __restrict__ shift_dn,
                                                                  double2* __restrict__ Nb) {
  using D = rb::Dims<NC, NP>;
  constexpr int KH = D::DTH_KH, NT = D::DTH_N / 8, HALF = D::HALF, SP = D::SP, LDB = D::DTH_LDB;
  extern __shared__ __align__(16) double Bsm[];
  rb::stage_b<D::DTH_K, D::DTH_N, D::DTH_LDB>(Bsm, B);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int64_t items = int64_t(n_par) * HALF;  // 8 HALF rows per parent = HALF tiles
  const int64_t stride = int64_t(gridDim.x) * (rb::kThreads / 32);
  int64_t it = int64_t(blockIdx.x) * (rb::kThreads / 32) + warp;
  int4 dn = it < items ? __ldg(pdesc + 3 * (it / HALF)) : make_int4(0, 0, 0, 0);
  for (; it < items; it += stride) {
    const int4 dc = dn;  // parent descriptor, loaded one item ahead (rb::PDesc)
    if (it + stride < items) dn = __ldg(pdesc + 3 * ((it + stride) / HALF));
    const int par = int(it / HALF), tile = int(it - int64_t(par) * HALF);
    const int cb = dc.x, nchp = dc.y;
    const int rho = tile * 8 + g, c = rho / HALF, p = rho - c * HALF;
    const bool ok = c < nchp;
    const double2* L = loc_p + int64_t(dc.z) * SP;
    const double2* sh = shift_dn + int64_t(ok ? rb::pdesc_oct(dc, c) : 0) * SP;
    // even / odd parts of the shifted circle: front sample (row k, column p)
    // plus / minus back sample (row k, column p + HALF)
    double er[KH], ei[KH], qr[KH], qi[KH];
#pragma unroll
    for (int kk = 0; kk < KH; ++kk) {
      const int k = 4 * kk + tq;
      double2 f = make_double2(0.0, 0.0), b = f;
      if (ok && k < NP) {
        const int s = k * NP + p;
        f = cmul(__ldg(L + s), __ldg(sh + s));
        b = cmul(__ldg(L + s + HALF), __ldg(sh + s + HALF));
      }
      er[kk] = f.x + b.x;
      ei[kk] = f.y + b.y;
      qr[kk] = f.x - b.x;
      qi[kk] = f.y - b.y;
    }
    rb::rank1_inject_eo<KH, NP>(er, ei, qr, qi, v);
    double2* Nc = Nb + int64_t(cb + (ok ? c : 0)) * NC * D::LDN;
    constexpr int NTC = 2;
#pragma unroll
    for (int j0 = 0; j0 < NT; j0 += NTC) {
      double cer[NTC][2] = {}, cei[NTC][2] = {}, cqr[NTC][2] = {}, cqi[NTC][2] = {};
      const double* bp = Bsm + tq * LDB + g + 8 * j0;
#pragma unroll
      for (int kk = 0; kk < KH; ++kk)
#pragma unroll
        for (int jc = 0; jc < NTC; ++jc)
          if (j0 + jc < NT) {
            const double be = bp[4 * kk * LDB + 8 * jc];
            dmma884(cer[jc][0], cer[jc][1], er[kk], be);
            dmma884(cei[jc][0], cei[jc][1], ei[kk], be);
            const double bo = bp[4 * (KH + kk) * LDB + 8 * jc];
            dmma884(cqr[jc][0], cqr[jc][1], qr[kk], bo);
            dmma884(cqi[jc][0], cqi[jc][1], qi[kk], bo);
          }
      if (ok) {
        // theta row n of the child: (Ye, Yo) of circle p at columns 2 p, 2 p + 1
        // (the phi matrix's rows undo the split, interp.hpp:unfold_rows)
#pragma unroll
        for (int jc = 0; jc < NTC; ++jc)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = 8 * (j0 + jc) + 2 * tq + q;
            if (j0 + jc < NT && n < NC) {
              double2* d = Nc + n * D::LDN + 2 * p;
              d[0] = make_double2(cer[jc][q], cei[jc][q]);
              d[1] = make_double2(cqr[jc][q], cqi[jc][q]);
            }
          }
      }
    }
  }
}

// L2L stage 2: phi anterpolation of every narrow row, added into the child's
// local expansion (the old values are loaded ahead of the DMMAs).
template <int NC, int NP>
__global__ void __launch_bounds__(rb::kThreads, 2) k_l2l_phi_rb(int64_t nch, const int* __restrict__ children,
                                                                const double2* __restrict__ Nb,
                                                                const double* __restrict__ B,
                                                                const double* __restrict__ v,
                                                                double2* __restrict__ loc_c) {
  using D = rb::Dims<NC, NP>;
  constexpr int KS = D::DPHI_K / 4, NT = D::DPHI_N / 8;
  __shared__ __align__(16) double Bs[D::DPHI_K * D::DPHI_LDB];
  rb::stage_b<D::DPHI_K, D::DPHI_N, D::DPHI_LDB>(Bs, B);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int64_t rows = nch * NC, tiles = (rows + 7) / 8;
  for (int64_t t = int64_t(blockIdx.x) * (rb::kThreads / 32) + warp; t < tiles;
       t += int64_t(gridDim.x) * (rb::kThreads / 32)) {
    const int64_t R = t * 8 + g;
    const bool ok = R < rows;
    const int64_t j = ok ? R / NC : 0;
    const int row = ok ? int(R - j * NC) : 0;
    const double2* a = Nb + (j * NC + row) * D::LDN;
    double2* dst = loc_c + (children ? children[j] : j) * int64_t(D::SC) + row * NC;
    double are[KS], aim[KS];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
      const int k = 4 * kk + tq;
      const double2 xv = (ok && k < NP) ? __ldg(a + k) : make_double2(0.0, 0.0);
      are[kk] = xv.x;
      aim[kk] = xv.y;
    }
    double2 old[NT][2];
#pragma unroll
    for (int jn = 0; jn < NT; ++jn)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int n = 8 * jn + 2 * tq + q;
        old[jn][q] = (ok && n < NC) ? dst[n] : make_double2(0.0, 0.0);
      }
    rb::rank1_inject<KS, NP>(are, aim, v);
    double cre[NT][2] = {}, cim[NT][2] = {};
    rb::tile_mma<KS, NT, D::DPHI_LDB>(are, aim, Bs, cre, cim);
    if (ok) {
#pragma unroll
      for (int jn = 0; jn < NT; ++jn)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int n = 8 * jn + 2 * tq + q;
          if (n < NC) dst[n] = make_double2(old[jn][q].x + cre[jn][q], old[jn][q].y + cim[jn][q]);
        }
    }
  }
}

// ---------------------------------------------------------------------------
// Runtime-shaped variants for the larger level pairs (upper levels): A values
// are re-read (L1) per chunk of kChunk n8 tiles instead of living in
// registers, the rank-1 alpha comes from a first pass over K, and B (up to
// ~350 KB) is read through L1/L2.
namespace rb {
#ifndef HFMM_RBL_CHUNK
#define HFMM_RBL_CHUNK 4
#endif
constexpr int kChunk = HFMM_RBL_CHUNK;
#ifndef HFMM_RBL_UNROLL_S
#define HFMM_RBL_UNROLL_S 8
#endif
constexpr int kRblUnrollS = HFMM_RBL_UNROLL_S;  // k-step unroll of the chunk GEMM of the phi passes

// Rows [0, K) x columns [c0, c0 + nc) of a row-major K x N matrix -> shared
// rows of stride ldb (cp.async 16 B; nc and c0 even).
__device__ __forceinline__ void stage_block(double* dst, const double* __restrict__ src, int K, int N, int c0, int nc,
                                            int ldb) {
  const int h = nc / 2;
  for (int t = threadIdx.x; t < K * h; t += blockDim.x) {
    const int r = t / h, c = 2 * (t - r * h);
    const bool ok = c0 + c < N;
    cp_async16(dst + r * ldb + c, ok ? src + r * N + c0 + c : src, ok);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
}
__host__ __device__ constexpr int blk_ldb(int cols) { return ldb(cols); }

// alpha = v . x over the K_in data columns of a complex row; fetch(k) -> double2.
template <class Fetch>
__device__ __forceinline__ double2 row_alpha(int kin, const double* __restrict__ v, Fetch fetch) {
  const int tq = threadIdx.x & 3;
  double pr[4] = {0.0, 0.0, 0.0, 0.0}, pi[4] = {0.0, 0.0, 0.0, 0.0};  // independent partial sums
  int k = tq;
  for (; k + 12 < kin; k += 16) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double vk = __ldg(v + k + 4 * u);
      const double2 x = fetch(k + 4 * u);
      pr[u] = fma(vk, x.x, pr[u]);
      pi[u] = fma(vk, x.y, pi[u]);
    }
  }
  for (int u = 0; k < kin; k += 4, ++u) {
    const double vk = __ldg(v + k);
    const double2 x = fetch(k);
    pr[u & 3] = fma(vk, x.x, pr[u & 3]);
    pi[u & 3] = fma(vk, x.y, pi[u & 3]);
  }
  double sr = (pr[0] + pr[1]) + (pr[2] + pr[3]), si = (pi[0] + pi[1]) + (pi[2] + pi[3]);
  sr += __shfl_xor_sync(0xffffffffu, sr, 1);
  si += __shfl_xor_sync(0xffffffffu, si, 1);
  sr += __shfl_xor_sync(0xffffffffu, sr, 2);
  si += __shfl_xor_sync(0xffffffffu, si, 2);
  return make_double2(-si, sr);  // i alpha
}

// C chunk (8 complex rows x kChunk n8 tiles from n8 tile j0) over K = 4 ks:
// column kin holds ia (rank-1), columns > kin are zero.
template <int CH = kChunk, class Fetch>
__device__ __forceinline__ void chunk_mma(int ks, int kin, double2 ia, Fetch fetch, const double* __restrict__ B, int N,
                                          int j0, int nt, double (&cre)[CH][2], double (&cim)[CH][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const double* bp = B + tq * N + 8 * j0 + g;
#pragma unroll(kRblUnrollS)
  for (int kk = 0; kk < ks; ++kk) {
    const int k = 4 * kk + tq;
    const double2 x = k < kin ? fetch(k) : (k == kin ? ia : make_double2(0.0, 0.0));
#pragma unroll
    for (int jc = 0; jc < CH; ++jc)
      if (j0 + jc < nt) {
        const double b = bp[4 * kk * N + 8 * jc];
        dmma884(cre[jc][0], cre[jc][1], x.x, b);
        dmma884(cim[jc][0], cim[jc][1], x.y, b);
      }
  }
}
}  // namespace rb

__global__ void __launch_bounds__(rb::kThreads) k_m2m_phi_rbl(int nc, int np, int64_t nch, const int* __restrict__ children,
                                                              const double2* __restrict__ mp_c,
                                                              const double* __restrict__ B, const double* __restrict__ v,
                                                              double2* __restrict__ F) {
  // (B = the phi matrix with the (e, o) fold in its columns: output column
  // 2 p + h is part h of circle p; F row (child, p): x_e at [0, nc), x_o at [K, K + nc))
  const int K = rb::r4(nc + 1), N = rb::r8(np), ks = K / 4, nt = N / 8, half = np / 2, ldf = 2 * K;
  const int ldb = rb::blk_ldb(N);
  extern __shared__ __align__(16) double Bsh[];
  rb::stage_block(Bsh, B, K, N, 0, N, ldb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int64_t rows = nch * nc, tiles = (rows + 7) / 8;
  for (int64_t t = int64_t(blockIdx.x) * (rb::kThreads / 32) + warp; t < tiles;
       t += int64_t(gridDim.x) * (rb::kThreads / 32)) {
    const int64_t R = t * 8 + g;
    const bool ok = R < rows;
    const int64_t j = ok ? R / nc : 0;
    const int i = ok ? int(R - j * nc) : 0;
    const double2* x = mp_c + (children ? children[j] : j) * int64_t(nc) * nc + int64_t(i) * nc;
    auto fetch = [&](int k) { return ok ? __ldg(x + k) : make_double2(0.0, 0.0); };
    const double2 ia = rb::row_alpha(nc, v, fetch);
    double2* Fj = F + j * half * ldf;
    for (int j0 = 0; j0 < nt; j0 += rb::kChunk) {
      double cre[rb::kChunk][2] = {}, cim[rb::kChunk][2] = {};
      rb::chunk_mma(ks, nc, ia, fetch, Bsh, ldb, j0, nt, cre, cim);
      if (ok) {
#pragma unroll
        for (int jc = 0; jc < rb::kChunk; ++jc)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = 8 * (j0 + jc) + 2 * tq + q;
            if (j0 + jc < nt && n < np) Fj[int64_t(n >> 1) * ldf + (n & 1) * K + i] = make_double2(cre[jc][q], cim[jc][q]);
          }
      }
    }
  }
}

// Even / odd chunk GEMM over a runtime K (interp.hpp:even_odd): rows [0, KH4) of
// the staged B block hold Be, rows [KH4, 2 KH4) hold Bo; fetch(k, e, o) delivers
// x_e[k], x_o[k] of the lane's row; column kin of both halves carries i alpha.
namespace rb {
template <int CH, class Fetch>
__device__ __forceinline__ void chunk_mma_eo(int kh, int kin, double2 ia, Fetch fetch, const double* __restrict__ Bs,
                                             int ldb, int KH4, int nt_left, double (&cer)[CH][2], double (&cei)[CH][2],
                                             double (&cqr)[CH][2], double (&cqi)[CH][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const double* bpe = Bs + tq * ldb + g;
  const double* bpo = bpe + KH4 * ldb;
#pragma unroll 4
  for (int kk = 0; kk < kh; ++kk) {
    const int k = 4 * kk + tq;
    double2 e = make_double2(0.0, 0.0), o = e;
    if (k < kin) fetch(k, e, o);
    else if (k == kin) e = o = ia;
#pragma unroll
    for (int jc = 0; jc < CH; ++jc)
      if (jc < nt_left) {
        const double be = bpe[4 * kk * ldb + 8 * jc];
        dmma884(cer[jc][0], cer[jc][1], e.x, be);
        dmma884(cei[jc][0], cei[jc][1], e.y, be);
        const double bo = bpo[4 * kk * ldb + 8 * jc];
        dmma884(cqr[jc][0], cqr[jc][1], o.x, bo);
        dmma884(cqi[jc][0], cqi[jc][1], o.y, bo);
      }
  }
}

// i alpha of the even / odd form: alpha = v_e . x_e + v_o . x_o (v_o at v + KH4).
template <class Fetch>
__device__ __forceinline__ double2 row_alpha_eo(int kin, int KH4, const double* __restrict__ v, Fetch fetch) {
  const int tq = threadIdx.x & 3;
  double pr[4] = {0.0, 0.0, 0.0, 0.0}, pi[4] = {0.0, 0.0, 0.0, 0.0};  // [2 u + half]: independent partial sums
  int k = tq;
  for (; k + 4 < kin; k += 8) {
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const double ve = __ldg(v + k + 4 * u), vo = __ldg(v + KH4 + k + 4 * u);
      double2 e, o;
      fetch(k + 4 * u, e, o);
      pr[2 * u] = fma(ve, e.x, pr[2 * u]);
      pi[2 * u] = fma(ve, e.y, pi[2 * u]);
      pr[2 * u + 1] = fma(vo, o.x, pr[2 * u + 1]);
      pi[2 * u + 1] = fma(vo, o.y, pi[2 * u + 1]);
    }
  }
  if (k < kin) {
    const double ve = __ldg(v + k), vo = __ldg(v + KH4 + k);
    double2 e, o;
    fetch(k, e, o);
    pr[0] = fma(ve, e.x, pr[0]);
    pi[0] = fma(ve, e.y, pi[0]);
    pr[1] = fma(vo, o.x, pr[1]);
    pi[1] = fma(vo, o.y, pi[1]);
  }
  double sr = (pr[0] + pr[1]) + (pr[2] + pr[3]), si = (pi[0] + pi[1]) + (pi[2] + pi[3]);
  sr += __shfl_xor_sync(0xffffffffu, sr, 1);
  si += __shfl_xor_sync(0xffffffffu, si, 1);
  sr += __shfl_xor_sync(0xffffffffu, sr, 2);
  si += __shfl_xor_sync(0xffffffffu, si, 2);
  return make_double2(-si, sr);
}
constexpr int kChunkEO = 2;  // M2M theta: n8 tiles of the half-size output per CTA column block
}  // namespace rb

// M2M theta pass, even / odd form (the runtime-shaped twin of rb::m2m_theta_item_f):
// B = [Be ; Bo] (2 KH4 x NH), this CTA's block of `chb` n8 tiles in shared memory
// (blockIdx.y; the whole matrix when it fits), walked in sub-chunks of 2 tiles:
// the lane's F row is read from L2 once (the rank-1 pass) and re-read from L1
// per sub-chunk.
__global__ void __launch_bounds__(rb::kThreads) k_m2m_theta_rbl(int nc, int np, int chb, int n_par,
                                                                const int4* __restrict__ pdesc,
                                                                const double2* __restrict__ F,
                                                                const double* __restrict__ B,
                                                                const double* __restrict__ v,
                                                                const double2* __restrict__ shift_up,
                                                                double2* __restrict__ mp_p) {
  const int KH4 = rb::r4(nc + 1), kh = KH4 / 4, NH = rb::r8(np), nt = NH / 8, half = np / 2, ldf = 2 * KH4;
  const int64_t SP = int64_t(np) * np;
  constexpr int CH = rb::kChunkEO;
  const int jb = blockIdx.y * chb, ldb = rb::blk_ldb(8 * chb);
  const int jend = jb + chb < nt ? jb + chb : nt;
  extern __shared__ __align__(16) double Bsh[];
  rb::stage_block(Bsh, B, 2 * KH4, NH, 8 * jb, 8 * chb, ldb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int64_t items = int64_t(n_par) * half, stride = int64_t(gridDim.x) * (rb::kThreads / 32);
  int64_t it = int64_t(blockIdx.x) * (rb::kThreads / 32) + warp;
  int4 dn = it < items ? __ldg(pdesc + 3 * (it / half)) : make_int4(0, 0, 0, 0);
  for (; it < items; it += stride) {
    const int4 dc = dn;  // parent descriptor, loaded one item ahead (rb::PDesc)
    if (it + stride < items) dn = __ldg(pdesc + 3 * ((it + stride) / half));
    const int par = int(it / half), p = int(it - int64_t(par) * half);
    const int cb = dc.x, nchp = dc.y;
    const bool ok = g < nchp;
    const double2* frow = F + (int64_t(cb + (ok ? g : 0)) * half + p) * ldf;
    const double2* sh = shift_up + int64_t(ok ? rb::pdesc_oct(dc, g) : 0) * SP;
    auto fetch = [&](int k, double2& e, double2& o) {
      e = ok ? __ldg(frow + k) : make_double2(0.0, 0.0);
      o = ok ? __ldg(frow + KH4 + k) : make_double2(0.0, 0.0);
    };
    const double2 ia = rb::row_alpha_eo(nc, KH4, v, fetch);
    double2* out = mp_p + int64_t(dc.z) * SP;
    for (int j0 = jb; j0 < jend; j0 += CH) {
      double2 shf[CH][2], shb[CH][2];
#pragma unroll
      for (int jc = 0; jc < CH; ++jc)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int n = 8 * (j0 + jc) + 2 * tq + q;
          const bool live = ok && j0 + jc < jend && n < np;
          shf[jc][q] = live ? __ldg(sh + int64_t(n) * np + p) : make_double2(0.0, 0.0);
          shb[jc][q] = live ? __ldg(sh + int64_t(n) * np + p + half) : make_double2(0.0, 0.0);
        }
      double cer[CH][2] = {}, cei[CH][2] = {}, cqr[CH][2] = {}, cqi[CH][2] = {};
      rb::chunk_mma_eo<CH>(kh, nc, ia, fetch, Bsh + 8 * (j0 - jb), ldb, KH4, jend - j0, cer, cei, cqr, cqi);
      static_assert(CH == 2, "child_sum_scatter takes the front and back halves of 2 n8 tiles");
      double vv[16];  // front tiles 0, 1, then back tiles 0, 1
#pragma unroll
      for (int jc = 0; jc < CH; ++jc)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double fr = cer[jc][q] + cqr[jc][q], fi = cei[jc][q] + cqi[jc][q];
          const double br = cer[jc][q] - cqr[jc][q], bi = cei[jc][q] - cqi[jc][q];
          const double2 f = shf[jc][q], b = shb[jc][q];
          vv[(2 * jc + q) * 2] = fr * f.x - fi * f.y;
          vv[(2 * jc + q) * 2 + 1] = fr * f.y + fi * f.x;
          vv[(2 * (CH + jc) + q) * 2] = br * b.x - bi * b.y;
          vv[(2 * (CH + jc) + q) * 2 + 1] = br * b.y + bi * b.x;
        }
      const double2 val = rb::child_sum_scatter(vv);
      const int slot = g >> 1, back = slot >= CH, jt = j0 + slot - back * CH, n = 8 * jt + 2 * tq + (g & 1);
      if (jt < jend && n < np) out[int64_t(n) * np + p + back * half] = val;
    }
  }
}

#ifndef HFMM_L2L_RBL_CHUNK
#define HFMM_L2L_RBL_CHUNK 3
#endif
// L2L theta pass, even / odd form: the lane's row (child c, circle p) is
// x_e / x_o[k] = L_p[k][p] shift_c[k][p] +- L_p[k][p + half] shift_c[k][p + half],
// built on the fly; B = [Be ; Bo] (2 KH4 x NH), this CTA's block of `chb` n8 tiles
// in shared memory (blockIdx.y), walked in sub-chunks of CH tiles; output row n
// of the child: (Ye, Yo) of circle p at columns 2 p, 2 p + 1 of the narrow rows.
__global__ void __launch_bounds__(rb::kThreads) k_l2l_theta_rbl(int nc, int np, int chb, int n_par,
                                                                const int4* __restrict__ pdesc,
                                                                const double2* __restrict__ loc_p,
                                                                const double* __restrict__ B,
                                                                const double* __restrict__ v,
                                                                const double2* __restrict__ shift_dn,
                                                                double2* __restrict__ Nb) {
  const int KH4 = rb::r4(np + 1), kh = KH4 / 4, NH = rb::r8(nc), nt = NH / 8, half = np / 2, ldn = rb::r4(np + 1);
  const int64_t SP = int64_t(np) * np;
  const int jb = blockIdx.y * chb, ldb = rb::blk_ldb(8 * chb);
  const int jend = jb + chb < nt ? jb + chb : nt;
  extern __shared__ __align__(16) double Bsh[];
  rb::stage_block(Bsh, B, 2 * KH4, NH, 8 * jb, 8 * chb, ldb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int64_t items = int64_t(n_par) * half, stride = int64_t(gridDim.x) * (rb::kThreads / 32);
  int64_t it = int64_t(blockIdx.x) * (rb::kThreads / 32) + warp;
  int4 dn = it < items ? __ldg(pdesc + 3 * (it / half)) : make_int4(0, 0, 0, 0);
  for (; it < items; it += stride) {
    const int4 dc = dn;  // parent descriptor, loaded one item ahead (rb::PDesc)
    if (it + stride < items) dn = __ldg(pdesc + 3 * ((it + stride) / half));
    const int par = int(it / half), tile = int(it - int64_t(par) * half);
    const int cb = dc.x, nchp = dc.y;
    const int rho = tile * 8 + g, c = rho / half, p = rho - c * half;
    const bool ok = c < nchp;
    const double2* L = loc_p + int64_t(dc.z) * SP;
    const double2* sh = shift_dn + int64_t(ok ? rb::pdesc_oct(dc, c) : 0) * SP;
    auto fetch = [&](int k, double2& e, double2& o) {
      if (!ok) {
        e = o = make_double2(0.0, 0.0);
        return;
      }
      const int64_t s = int64_t(k) * np + p;
      const double2 f = cmul(__ldg(L + s), __ldg(sh + s)), b = cmul(__ldg(L + s + half), __ldg(sh + s + half));
      e = make_double2(f.x + b.x, f.y + b.y);
      o = make_double2(f.x - b.x, f.y - b.y);
    };
    const double2 ia = rb::row_alpha_eo(np, KH4, v, fetch);
    double2* Nc = Nb + int64_t(cb + (ok ? c : 0)) * nc * ldn;
    constexpr int CH = HFMM_L2L_RBL_CHUNK;
    for (int j0 = jb; j0 < jend; j0 += CH) {
      double cer[CH][2] = {}, cei[CH][2] = {}, cqr[CH][2] = {}, cqi[CH][2] = {};
      rb::chunk_mma_eo<CH>(kh, np, ia, fetch, Bsh + 8 * (j0 - jb), ldb, KH4, jend - j0, cer, cei, cqr, cqi);
      if (ok) {
#pragma unroll
        for (int jc = 0; jc < CH; ++jc)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = 8 * (j0 + jc) + 2 * tq + q;
            if (j0 + jc < jend && n < nc) {
              double2* d = Nc + int64_t(n) * ldn + 2 * p;
              d[0] = make_double2(cer[jc][q], cei[jc][q]);
              d[1] = make_double2(cqr[jc][q], cqi[jc][q]);
            }
          }
      }
    }
  }
}

__global__ void __launch_bounds__(rb::kThreads) k_l2l_phi_rbl(int nc, int np, int64_t nch, const int* __restrict__ children,
                                                              const double2* __restrict__ Nb,
                                                              const double* __restrict__ B, const double* __restrict__ v,
                                                              double2* __restrict__ loc_c) {
  const int K = rb::r4(np + 1), N = rb::r8(nc), ks = K / 4, nt = N / 8, ldn = K;
  const int ldb = rb::blk_ldb(N);
  extern __shared__ __align__(16) double Bsh[];
  rb::stage_block(Bsh, B, K, N, 0, N, ldb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int64_t rows = nch * nc, tiles = (rows + 7) / 8;
  for (int64_t t = int64_t(blockIdx.x) * (rb::kThreads / 32) + warp; t < tiles;
       t += int64_t(gridDim.x) * (rb::kThreads / 32)) {
    const int64_t R = t * 8 + g;
    const bool ok = R < rows;
    const int64_t j = ok ? R / nc : 0;
    const int row = ok ? int(R - j * nc) : 0;
    const double2* a = Nb + (j * nc + row) * ldn;
    double2* dst = loc_c + (children ? children[j] : j) * int64_t(nc) * nc + int64_t(row) * nc;
    auto fetch = [&](int k) { return ok ? __ldg(a + k) : make_double2(0.0, 0.0); };
    const double2 ia = rb::row_alpha(np, v, fetch);
    for (int j0 = 0; j0 < nt; j0 += rb::kChunk) {
      double2 old[rb::kChunk][2];
#pragma unroll
      for (int jc = 0; jc < rb::kChunk; ++jc)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int n = 8 * (j0 + jc) + 2 * tq + q;
          old[jc][q] = (ok && j0 + jc < nt && n < nc) ? dst[n] : make_double2(0.0, 0.0);
        }
      double cre[rb::kChunk][2] = {}, cim[rb::kChunk][2] = {};
      rb::chunk_mma(ks, np, ia, fetch, Bsh, ldb, j0, nt, cre, cim);
      if (ok) {
#pragma unroll
        for (int jc = 0; jc < rb::kChunk; ++jc)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = 8 * (j0 + jc) + 2 * tq + q;
            if (j0 + jc < nt && n < nc) dst[n] = make_double2(old[jc][q].x + cre[jc][q], old[jc][q].y + cim[jc][q]);
          }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Dispatch over the level pairs with a theta-pass K <= 72 (register budget).
#define HFMM_RB_PAIRS(X) X(18, 28) X(28, 42) X(22, 30) X(30, 44) X(26, 34) X(34, 52)

inline bool rb_pair(int nc, int np) {
#define HFMM_RB_HAS(A, B) if (nc == A && np == B) return true;
  HFMM_RB_PAIRS(HFMM_RB_HAS)
#undef HFMM_RB_HAS
  return false;
}
// complex elements of the M2M F scratch / L2L Nb scratch for nch children
inline size_t rb_m2m_scratch(int64_t nch, int nc, int np) {
  return size_t(nch) * size_t(np / 2) * size_t(std::max(rb::r4(2 * nc + 1), 2 * rb::r4(nc + 1)));
}
inline size_t rb_l2l_scratch(int64_t nch, int nc, int np) { return size_t(nch) * size_t(nc) * size_t(rb::r4(np + 1)); }

struct RbLaunch {
  int n_par;
  const int* plist;
  const int* child_off;  // device CSR over parents
  const int* children;
  int64_t nch;           // total children (= child_off[n_par])
  const uint8_t* oct_c;
  const int4* pdesc;     // rb::PDesc per parent (3 int4)
  int grid;              // persistent CTAs
  cudaStream_t st;
  int phi_grid = 0;      // persistent CTAs of the (HBM-bound) phi passes; 0 = grid
};

template <int A, int B>
void m2m_rb(const RbLaunch& L, const double2* mp_c, double2* mp_p, const double* Bphi, const double* vphi,
            const double* Bth, const double* vth, const double2* shift_up, double2* F) {
  using D = rb::Dims<A, B>;
  if (L.nch > 0)
    k_m2m_phi_rb<A, B><<<L.phi_grid ? L.phi_grid : L.grid, rb::kThreads, 0, L.st>>>(L.nch, L.children, mp_c, Bphi,
                                                                                    vphi, F);
  const int smem = D::UTH_K * D::UTH_LDB * 8;
  cudaFuncSetAttribute(k_m2m_theta_rb<A, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_m2m_theta_rb<A, B><<<L.grid, rb::kThreads, smem, L.st>>>(L.n_par, L.pdesc, F,
                                                            Bth, vth, shift_up, mp_p);
}

template <int A, int B>
void l2l_rb(const RbLaunch& L, const double2* loc_p, double2* loc_c, const double* Bth, const double* vth,
            const double* Bphi, const double* vphi, const double2* shift_dn, double2* Nb) {
  using D = rb::Dims<A, B>;
  const int smem = D::DTH_K * D::DTH_LDB * 8;
  cudaFuncSetAttribute(k_l2l_theta_rb<A, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_l2l_theta_rb<A, B><<<L.grid, rb::kThreads, smem, L.st>>>(L.n_par, L.pdesc,
                                                            loc_p, Bth, vth, shift_dn, Nb);
  if (L.nch > 0)
    k_l2l_phi_rb<A, B><<<L.phi_grid ? L.phi_grid : L.grid, rb::kThreads, 0, L.st>>>(L.nch, L.children, Nb, Bphi,
                                                                                    vphi, loc_c);
}

inline bool launch_l2l_rb(int nc, int np, const RbLaunch& L, const double2* loc_p, double2* loc_c, const double* Bth,
                          const double* vth, const double* Bphi, const double* vphi, const double2* shift_dn,
                          double2* Nb) {
#define HFMM_RB_L2L(A, B) \
  if (nc == A && np == B) { l2l_rb<A, B>(L, loc_p, loc_c, Bth, vth, Bphi, vphi, shift_dn, Nb); return true; }
  HFMM_RB_PAIRS(HFMM_RB_L2L)
#undef HFMM_RB_L2L
  return false;
}

inline bool launch_m2m_rb(int nc, int np, const RbLaunch& L, const double2* mp_c, double2* mp_p, const double* Bphi,
                          const double* vphi, const double* Bth, const double* vth, const double2* shift_up,
                          double2* F) {
#define HFMM_RB_M2M(A, B) \
  if (nc == A && np == B) { m2m_rb<A, B>(L, mp_c, mp_p, Bphi, vphi, Bth, vth, shift_up, F); return true; }
  HFMM_RB_PAIRS(HFMM_RB_M2M)
#undef HFMM_RB_M2M
  return false;
}

}  // namespace hfmm_b200

#endif
