// Staging layout of the dense-level M2L (m2l_tc.cuh, k_m2l_dmma).
//
// For one sample s the far-field translation of a level (operators.cpp:82-87,
// traversal.cpp:443-581) is a sparse convolution over the level's cell grid:
//   L_o[s] = sum_d  T[d][s] * M_{o-d}[s],   d in [-3,3]^3,
// restricted to far pairs: parents adjacent (Chebyshev <= 1) and the boxes
// themselves not adjacent (interaction_lists.cpp:54-98).
//
// Work decomposition (B200): one CTA = an 8x8x8 observer block x a chunk of
// sample pairs.  The node indices of the 12^3 source region (block + one
// parent group) are resolved once into shared memory; then, per pair, the
// region's 2 samples and the 343 T taps are staged in shared memory (~76 KB
// with the index table, 3 CTAs/SM).
#ifndef HFMM_B200_M2L_CUH
#define HFMM_B200_M2L_CUH

#include "kernels.cuh"

namespace hfmm_b200 {

namespace m2l {
constexpr int MB = 8;               // observer block edge
// Far sources have adjacent PARENTS, so the halo is exactly one parent group:
// cells [b - 2, b + MB + 2) per axis (a tap at distance 3 only reaches an
// adjacent parent from the block's interior).
constexpr int HALO = 2;
constexpr int MR = MB + 2 * HALO;   // source region edge (12)
constexpr int ROW = MR * 2 + 1;     // double2 per region row (2 samples/cell + 16 B pad, odd)
constexpr int ZS = MR * ROW + 2;    // double2 per z-slice: 2 ZS == 4 (mod 8) keeps the
                                    // 16-byte row loads of a warp bank-conflict free
constexpr int REGION = MR * ZS;     // double2 in the region
constexpr int CELLS = MR * MR * MR;  // region cells (node index table)
// Staged taps: per sample (ax + 3) TSX + (ay + 3) 7 + (az + 3); TSX == 2 (mod 8) keeps the
// 16-byte tap gathers of a warp (lane parts (ox - cx) TSX + (oy - cy) 7 + oz) conflict free.
constexpr int TSX = 50;
constexpr int TAPS = 7 * TSX;       // double2 per sample
constexpr int SMEM_BYTES = (REGION + TAPS * 2) * 16 + CELLS * 4;

__host__ __device__ constexpr int fdiv2(int v) { return v >= 0 ? v / 2 : -((1 - v) / 2); }
__host__ __device__ constexpr int iabs(int v) { return v < 0 ? -v : v; }
// parent of (2a + p) vs parent of (2a + p - d) are adjacent
__host__ __device__ constexpr bool parent_near(int p, int d) { return iabs(fdiv2(p - d)) <= 1; }

}  // namespace m2l

// Sample pairs per CTA: enough CTAs for ~6 waves at 3 CTAs/SM, at most 16.
inline int m2l_pairs_per_cta(int nblocks, int64_t S, int sms) {
  const int64_t target = int64_t(sms) * 3 * 6;
  int64_t ppc = int64_t(nblocks) * (S / 2) / (target > 0 ? target : 1);
  return int(ppc < 1 ? 1 : ppc > 16 ? 16 : ppc);
}

}  // namespace hfmm_b200

#endif
