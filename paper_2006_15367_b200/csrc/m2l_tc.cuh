// M2L on dense levels as DMMA GEMMs over sibling groups (alternative to the
// DFMA stencil of m2l.cuh; same staging, same far rule).
//
// For one sample s, observer parent P and parent offset D in [-1,1]^3 \ {0},
// the translation from the 8 children c of source parent P + D to the 8
// children o of P is an 8x8 complex matrix K_D[o][c] = T[o - c - 2D][s], zero
// where the boxes are adjacent (interaction_lists.cpp:54-98: parents adjacent,
// boxes not).  Real form: rows (o, re/im), columns (c, re/im):
//     [ Tr  -Ti ]
//     [ Ti   Tr ]
// so a block's 64 observer parents would be  C(16 x 64) += K_D(16 x 16) B_D(16 x 64)
// with B_D the source children's multipoles, summed over the 26 offsets D.
// The kernel evaluates the same complex product in its 3-multiplication form
// (below), a quarter fewer DMMA.  A fragments are gathered from the staged taps
// per D (their lane pattern is fixed), B fragments straight from the staged
// source region.
#ifndef HFMM_B200_M2L_TC_CUH
#define HFMM_B200_M2L_TC_CUH

#include "dmma.cuh"
#include "m2l.cuh"

namespace hfmm_b200 {

// 3M complex product (Karatsuba): with tap t = c + i d and source x = a + i b,
//     m1 = c a,  m2 = d b,  m3 = (c + d) (a + b),
//     Re(t x) = m1 - m2,  Im(t x) = m3 - m1 - m2,
// so the complex GEMM is three real 8 x 8 GEMMs per offset instead of the four
// of the [Tr -Ti; Ti Tr] real form: 26 x 3 x 2 x 4 = 624 DMMA per warp
// (a warp = one sample x 32 parents) against 832.  The lane loads (re, im) of
// its source element and (Tr, Ti) of its tap as one 16-byte shared load each;
// the third variant of each costs one DADD.  All three products of an
// output land in the same lane, so the epilogue needs no shuffle.
//
// blist != nullptr (distributed mode): blockIdx.x indexes a list of the 8^3
// observer blocks holding this rank's held nodes.
__global__ void __launch_bounds__(128, 3) k_m2l_dmma(int G, int nb, int64_t S, int ppc,
                                                     const int* __restrict__ blist,
                                                     const int* __restrict__ lookup,
                                                     const double2* __restrict__ T,
                                                     const double2* __restrict__ mp,
                                                     double2* __restrict__ loc) {
  using namespace m2l;
  extern __shared__ double2 smem[];
  double2* Ms = smem;
  double2* Ts = smem + REGION;
  int* nodes = reinterpret_cast<int*>(Ts + TAPS * 2);
  const int blk = blist ? blist[blockIdx.x] : int(blockIdx.x);
  const int bx = (blk % nb) * MB, by = ((blk / nb) % nb) * MB, bz = (blk / (nb * nb)) * MB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  {
    const int GP = (G > MB ? G : MB) + 6;
    for (int c = threadIdx.x; c < CELLS; c += blockDim.x) {
      const int cz = c / (MR * MR), cy = (c / MR) % MR, cx = c % MR;
      nodes[c] = __ldg(lookup + (int64_t(bz + cz + 3 - HALO) * GP + (by + cy + 3 - HALO)) * GP + (bx + cx + 3 - HALO));
    }
  }
  // Warp = sample sw x parent tiles t0 .. t0 + 3 (tile t: parents pn = 8 t + n,
  // n = 0..7, with P = (n & 3, 2 (t & 1) + (n >> 2), t >> 1)).
  const int sw = warp & 1, t0 = (warp >> 1) * 4;
  // B fragment (lane holds B[k = tq][n = g]): source child c = 4 kj + tq
  // (cx = tq & 1, cy = tq >> 1, cz = kj) of parent P_g + D; its region cell is
  // 2 (P + D) + c + HALO per axis.  kj and D are compile-time offsets.
  const double2* pb4[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int tt = t0 + t;
    const int px = g & 3, py = 2 * (tt & 1) + (g >> 2), pz = tt >> 1;
    pb4[t] = Ms + (2 * pz + HALO) * ZS + (2 * py + HALO + (tq >> 1)) * ROW + 2 * (2 * px + HALO + (tq & 1)) + sw;
  }
  // A fragment (lane holds A[row = g][k = tq]): observer child o = g
  // (ox = g & 1, oy = (g >> 1) & 1, oz = g >> 2), source child as above; the
  // tap is o - c - 2 D, its lane part (ox - cx, oy - cy, oz).
  const double2* Tl = Ts + sw * TAPS + ((g & 1) - (tq & 1)) * TSX + (((g >> 1) & 1) - (tq >> 1)) * 7 + (g >> 2);
  const int64_t pairs = S / 2;
  const int64_t pb = int64_t(blockIdx.y) * ppc, pe = pb + ppc < pairs ? pb + ppc : pairs;

  for (int64_t pr = pb; pr < pe; ++pr) {
    const int64_t s0 = pr * 2;
    __syncthreads();
#ifdef HFMM_M2L_PROBE_NOSTAGE  // timing probe only (wrong results): stage the first pair, then recompute on it
    if (pr == pb)
#endif
    {
    for (int t = threadIdx.x; t < kSlots * 2; t += blockDim.x) {
      // taps of adjacent boxes (|offset| <= 1 per axis) are never far: staged
      // as zeros, so K_D needs no per-entry mask
      const int sl = t >> 1, ax = sl / 49 - 3, ay = (sl / 7) % 7 - 3, az = sl % 7 - 3;
      const bool far_tap = iabs(ax) > 1 || iabs(ay) > 1 || iabs(az) > 1;
      cp_async16(Ts + (t & 1) * TAPS + (ax + 3) * TSX + (ay + 3) * 7 + (az + 3),
                 T + (far_tap ? int64_t(sl) * S + s0 + (t & 1) : 0), far_tap);
    }
    // region: a thread keeps its (cell x, sample) entry `ent` of a 24-entry row and
    // walks the 144 (z, y) rows five at a time -- no per-copy divisions
    if (threadIdx.x < 5 * 2 * MR) {
      const int rg = threadIdx.x / (2 * MR), ent = threadIdx.x - rg * (2 * MR);
      int cy = rg, cz = 0;
#pragma unroll 4
      for (int k = 0; k < (MR * MR + 4) / 5; ++k) {
        if (cz < MR) {
          const int node = nodes[(cz * MR + cy) * MR + (ent >> 1)];
          cp_async16(Ms + cz * ZS + cy * ROW + ent,
                     mp + (node >= 0 ? uint64_t(uint32_t(node)) * uint32_t(S) + uint64_t(s0 + (ent & 1)) : 0), node >= 0);
        }
        cy += 5;
        if (cy >= MR) {
          cy -= MR;
          ++cz;
        }
      }
    }
    }
    cp_async_wait_all();
    __syncthreads();

    double acc[3][4][2];
#pragma unroll
    for (int v = 0; v < 3; ++v)
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[v][t][0] = acc[v][t][1] = 0.0;

#pragma unroll
    for (int d = 0; d < 27; ++d) {
      if (d == 13) continue;  // D = 0: siblings are always adjacent
      const int Dx = d % 3 - 1, Dy = (d / 3) % 3 - 1, Dz = d / 9 - 1;  // compile-time
      const int doff = (2 * Dz) * ZS + (2 * Dy) * ROW + 2 * (2 * Dx);
#pragma unroll
      for (int kj = 0; kj < 2; ++kj) {
        // tap = (ax + 3) TSX + (ay + 3) 7 + (az + 3) = lane part + compile-time part;
        // adjacent taps read the staged zeros
        const double2 tv = Tl[(-2 * Dx + 3) * TSX + (-2 * Dy + 3) * 7 + (-kj - 2 * Dz + 3)];
        const double a3 = tv.x + tv.y;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const double2 b = pb4[t][doff + kj * ZS];
          dmma884(acc[0][t][0], acc[0][t][1], tv.x, b.x);
          dmma884(acc[1][t][0], acc[1][t][1], tv.y, b.y);
          dmma884(acc[2][t][0], acc[2][t][1], a3, b.x + b.y);
        }
      }
    }
    // C[row = o][col = parent]: lane holds row g, cols 2 tq, 2 tq + 1 of all three products.
    const int ocx = g & 1, ocy = (g >> 1) & 1, ocz = g >> 2;  // observer child offsets
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int tt = t0 + t;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int n = 2 * tq + q;
        const int px = n & 3, py = 2 * (tt & 1) + (n >> 2), pz = tt >> 1;
        const int rx = 2 * px + ocx + HALO, ry = 2 * py + ocy + HALO, rz = 2 * pz + ocz + HALO;
        const int node = nodes[(rz * MR + ry) * MR + rx];
        if (node >= 0)
          loc[int64_t(node) * S + s0 + sw] = make_double2(acc[0][t][q] - acc[1][t][q], acc[2][t][q] - acc[0][t][q] - acc[1][t][q]);
      }
    }
  }
}

// (A warp-specialised form -- one CTA per SM, 8 compute warps in two groups plus a
// producer warp filling a ring of three staged sample pairs, mbarrier hand-off -- was
// built and measured this round: 48.8 ms against 42.5 ms at config 4.  Two compute
// warps per SM sub-partition do not keep the DMMA pipe as busy as the three of this
// kernel's 3 CTAs x 4 warps, and a 13-warp block would cap a thread at 128 registers.)

}  // namespace hfmm_b200

#endif
