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
// so a block's 64 observer parents are  C(16 x 64) += K_D(16 x 16) B_D(16 x 64)
// with B_D the source children's multipoles, summed over the 26 offsets D:
// 26 x 2 x 4 x 4 = 832 DMMA.8x8x4 per warp (a warp = one sample x 32 parents),
// about 1.1x the useful complex MACs but one fragment load per two DMMAs
// (the DFMA stencil issues 55 shared-memory wavefronts per 40 complex MACs).
// A fragments are gathered from the staged taps per D (their lane pattern is
// fixed), B fragments straight from the staged source region.
#ifndef HFMM_B200_M2L_TC_CUH
#define HFMM_B200_M2L_TC_CUH

#include "dmma.cuh"
#include "m2l.cuh"

namespace hfmm_b200 {

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
  int* nodes = reinterpret_cast<int*>(Ts + kSlots * 2);
  const double* Md = reinterpret_cast<const double*>(Ms);
  const double* Td = reinterpret_cast<const double*>(Ts);
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
  // B fragment (lane holds B[k = tq][n = g]): source child c = 2 kj + (tq >> 1),
  // part tq & 1; its region cell is 2 (P + D) + c_vec + HALO per axis.
  int pbase[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int tt = t0 + t;
    const int px = g & 3, py = 2 * (tt & 1) + (g >> 2), pz = tt >> 1;
    pbase[t] = (((2 * pz + HALO) * ZS + (2 * py + HALO) * ROW + 2 * (2 * px + HALO) + sw) << 1) + (tq & 1);
  }
  int coff[4];  // child offset for k-block kj: cx = tq >> 1, cy = kj & 1, cz = kj >> 1
#pragma unroll
  for (int kj = 0; kj < 4; ++kj) coff[kj] = ((kj >> 1) * ZS + (kj & 1) * ROW + 2 * (tq >> 1)) << 1;
  // A fragment (lane holds A[row = g][k = tq] of block (mi, kj)): observer child
  // o = 4 mi + (g >> 1) (ox = (g >> 1) & 1, oy = g >> 2, oz = mi), part g & 1;
  // source child as above.  value = +Tr, -Ti, +Ti, +Tr by (part_o, part_c).
  const int po = g & 1, pc = tq & 1;
  const int comp = po ^ pc;                        // 0: Tr, 1: Ti
  const int sgn = (po == 0 && pc == 1) ? int(0x80000000u) : 0;  // -Ti: sign bit XOR (integer pipe)
  const int bxo = ((g >> 1) & 1) - (tq >> 1);      // ox - cx
  // lane base of the tap gather: Td[4 tap + 2 sw + comp], tap's lane part bxo 49 + (g >> 2) 7
  const double* Tl = Td + (bxo * 49 + (g >> 2) * 7) * 4 + 2 * sw + comp;
  const int64_t pairs = S / 2;
  const int64_t pb = int64_t(blockIdx.y) * ppc, pe = pb + ppc < pairs ? pb + ppc : pairs;

  for (int64_t pr = pb; pr < pe; ++pr) {
    const int64_t s0 = pr * 2;
    __syncthreads();
    for (int t = threadIdx.x; t < kSlots * 2; t += blockDim.x) {
      // taps of adjacent boxes (|offset| <= 1 per axis) are never far: staged
      // as zeros, so K_D needs no per-entry mask
      const int sl = t >> 1, ax = sl / 49 - 3, ay = (sl / 7) % 7 - 3, az = sl % 7 - 3;
      const bool far_tap = iabs(ax) > 1 || iabs(ay) > 1 || iabs(az) > 1;
      cp_async16(Ts + t, T + (far_tap ? int64_t(sl) * S + s0 + (t & 1) : 0), far_tap);
    }
    for (int t = threadIdx.x; t < CELLS * 2; t += blockDim.x) {
      const int c = t >> 1, cz = c / (MR * MR), cy = (c / MR) % MR, cx = c % MR;
      const int node = nodes[c];
      cp_async16(Ms + cz * ZS + cy * ROW + 2 * cx + (t & 1), mp + (node >= 0 ? int64_t(node) * S + s0 + (t & 1) : 0),
                 node >= 0);
    }
    cp_async_wait_all();
    __syncthreads();

    double acc[2][4][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int t = 0; t < 4; ++t) acc[mi][t][0] = acc[mi][t][1] = 0.0;

#pragma unroll
    for (int d = 0; d < 27; ++d) {
      if (d == 13) continue;  // D = 0: siblings are always adjacent
      const int Dx = d % 3 - 1, Dy = (d / 3) % 3 - 1, Dz = d / 9 - 1;  // compile-time
      const int doff = ((2 * Dz) * ZS + (2 * Dy) * ROW + 2 * (2 * Dx)) << 1;
      double a[2][4];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int kj = 0; kj < 4; ++kj) {
          // tap = (ox + 3) 49 + (oy + 3) 7 + (oz + 3) = lane part + compile-time part;
          // adjacent taps read the staged zeros
          const int tofs = ((-2 * Dx + 3) * 49 + (-(kj & 1) - 2 * Dy + 3) * 7 + (mi - (kj >> 1) - 2 * Dz + 3)) * 4;
          const double v = Tl[tofs];
          a[mi][kj] = __hiloint2double(__double2hiint(v) ^ sgn, __double2loint(v));
        }
#pragma unroll
      for (int kj = 0; kj < 4; ++kj)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const double b = Md[pbase[t] + coff[kj] + doff];
          dmma884(acc[0][t][0], acc[0][t][1], a[0][kj], b);
          dmma884(acc[1][t][0], acc[1][t][1], a[1][kj], b);
        }
    }
    // C[row = (o, part)][col = parent]: lane holds rows g (+8), cols 2 tq, 2 tq + 1;
    // the partner lane (g ^ 1 -> lane ^ 4) holds the other part.
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const double o0 = __shfl_xor_sync(0xffffffffu, acc[mi][t][0], 4);
        const double o1 = __shfl_xor_sync(0xffffffffu, acc[mi][t][1], 4);
        if (po == 0) {
          const int tt = t0 + t;
          const int ocx = (g >> 1) & 1, ocy = g >> 2, ocz = mi;  // observer child offsets
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = 2 * tq + q;
            const int px = n & 3, py = 2 * (tt & 1) + (n >> 2), pz = tt >> 1;
            const int rx = 2 * px + ocx + HALO, ry = 2 * py + ocy + HALO, rz = 2 * pz + ocz + HALO;
            const int node = nodes[(rz * MR + ry) * MR + rx];
            if (node >= 0)
              loc[int64_t(node) * S + s0 + sw] = make_double2(q ? acc[mi][t][1] : acc[mi][t][0], q ? o1 : o0);
          }
        }
      }
  }
}

}  // namespace hfmm_b200

#endif
