// M2L on densely populated levels as a per-sample 3-D stencil.
//
// For one sample s the far-field translation of a level (operators.cpp:82-87,
// traversal.cpp:443-581) is a sparse convolution over the level's cell grid:
//   L_o[s] = sum_d  T[d][s] * M_{o-d}[s],   d in [-3,3]^3,
// restricted to far pairs: parents adjacent (Chebyshev <= 1) and the boxes
// themselves not adjacent (interaction_lists.cpp:54-98).  Whether a pair is
// far depends only on d and on the parities of o, so the mask is resolved at
// compile time along x and is warp-uniform along y, z.
//
// Work decomposition (B200): one CTA = an 8x8x8 observer block x a chunk of
// sample pairs.  The node indices of the 12^3 source region (block + one
// parent group) are resolved once into shared memory; then, per pair, the
// region's 2 samples and the 343 T taps are staged in shared memory (~76 KB
// with the index table, 3 CTAs/SM).  Each thread owns
// an x-row of 8 observers for one sample; for every (dy, dz) tap row it loads
// the 12 source values of its row once and the 7 taps (a warp broadcast) and
// issues up to 48 complex FMAs from registers.  A warp holds 16 rows of one
// (y, z) parity class x 2 samples, so every mask branch is warp-uniform and
// the padded row stride makes the 16-byte loads bank-conflict free.
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
constexpr int SMEM_BYTES = (REGION + kSlots * 2) * 16 + CELLS * 4;

__host__ __device__ constexpr int fdiv2(int v) { return v >= 0 ? v / 2 : -((1 - v) / 2); }
__host__ __device__ constexpr int iabs(int v) { return v < 0 ? -v : v; }
// parent of (2a + p) vs parent of (2a + p - d) are adjacent
__host__ __device__ constexpr bool parent_near(int p, int d) { return iabs(fdiv2(p - d)) <= 1; }

template <bool INNER>
__device__ __forceinline__ void tap_row(double2 (&acc)[MB], const double2 (&m)[MR], const double2 (&t)[7]) {
#pragma unroll
  for (int k = 0; k < MB; ++k) {
#pragma unroll
    for (int dx = -3; dx <= 3; ++dx) {
      // observer x = 8 bx + k: parent-adjacency along x depends on k and dx only
      const bool xnear = iabs(fdiv2(k) - fdiv2(k - dx)) <= 1;
      const bool adjacent = INNER && iabs(dx) <= 1;
      if (xnear && !adjacent) cmac(acc[k], t[dx + 3], m[k - dx + HALO]);
    }
  }
}
}  // namespace m2l

__global__ void __launch_bounds__(128, 3) k_m2l_dense(int G, int nb, int64_t S, int ppc,
                                                      const int* __restrict__ lookup,
                                                      const double2* __restrict__ T,
                                                      const double2* __restrict__ mp,
                                                      double2* __restrict__ loc) {
  using namespace m2l;
  extern __shared__ double2 smem[];
  double2* Ms = smem;
  double2* Ts = smem + REGION;
  int* nodes = reinterpret_cast<int*>(Ts + kSlots * 2);  // region cell -> node (-1: empty)
  const int blk = blockIdx.x;
  const int bx = (blk % nb) * MB, by = ((blk / nb) % nb) * MB, bz = (blk / (nb * nb)) * MB;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // Node indices of the region, once per CTA.  The lookup is halo-padded by 3
  // cells (entries -1), so every region cell has an entry.
  {
    const int GP = (G > MB ? G : MB) + 6;  // padded edge (host: same formula, halo 3)
    for (int c = threadIdx.x; c < CELLS; c += blockDim.x) {
      const int cz = c / (MR * MR), cy = (c / MR) % MR, cx = c % MR;
      nodes[c] = __ldg(lookup + (int64_t(bz + cz + 3 - HALO) * GP + (by + cy + 3 - HALO)) * GP + (bx + cx + 3 - HALO));
    }
  }
  const int py = warp & 1, pz = warp >> 1;
  const int sw = lane & 1, r = lane >> 1;
  const int oy = 2 * (r & 3) + py, oz = 2 * (r >> 2) + pz;
  const int64_t pairs = S / 2;
  const int64_t pb = int64_t(blockIdx.y) * ppc, pe = pb + ppc < pairs ? pb + ppc : pairs;

  for (int64_t pr = pb; pr < pe; ++pr) {
    const int64_t s0 = pr * 2;
    __syncthreads();  // node table ready / previous pair done with the buffers
    // Stage the T taps and the region's two samples with cp.async (LDGSTS):
    // every load in flight at once; empty cells are zero-filled by the copy.
    for (int t = threadIdx.x; t < kSlots * 2; t += blockDim.x)
      cp_async16(Ts + t, T + int64_t(t >> 1) * S + s0 + (t & 1), true);
    for (int t = threadIdx.x; t < CELLS * 2; t += blockDim.x) {
      const int c = t >> 1, cz = c / (MR * MR), cy = (c / MR) % MR, cx = c % MR;
      const int node = nodes[c];
      cp_async16(Ms + cz * ZS + cy * ROW + 2 * cx + (t & 1), mp + (node >= 0 ? int64_t(node) * S + s0 + (t & 1) : 0),
                 node >= 0);
    }
    cp_async_wait_all();
    __syncthreads();

    double2 acc[MB];
#pragma unroll
    for (int k = 0; k < MB; ++k) acc[k] = make_double2(0.0, 0.0);

    for (int dz = -3; dz <= 3; ++dz) {
      if (!parent_near(pz, dz)) continue;
      for (int dy = -3; dy <= 3; ++dy) {
        if (!parent_near(py, dy)) continue;
        const double2* row = Ms + (oz - dz + HALO) * ZS + (oy - dy + HALO) * ROW + sw;
        double2 m[MR];
#pragma unroll
        for (int i = 0; i < MR; ++i) m[i] = row[2 * i];
        const double2* trow = Ts + ((dy + 3) * 7 + (dz + 3)) * 2 + sw;
        double2 t[7];
#pragma unroll
        for (int j = 0; j < 7; ++j) t[j] = trow[j * 49 * 2];
        if (iabs(dy) <= 1 && iabs(dz) <= 1)
          tap_row<true>(acc, m, t);
        else
          tap_row<false>(acc, m, t);
      }
    }

    // observers are region cells (k + HALO, oy + HALO, oz + HALO)
    const int* orow = nodes + ((oz + HALO) * MR + (oy + HALO)) * MR + HALO;
#pragma unroll
    for (int k = 0; k < MB; ++k) {
      const int node = orow[k];
      if (node >= 0) loc[int64_t(node) * S + s0 + sw] = acc[k];
    }
  }
}

// Sample pairs per CTA: enough CTAs for ~6 waves at 3 CTAs/SM, at most 16.
inline int m2l_pairs_per_cta(int nblocks, int64_t S, int sms) {
  const int64_t target = int64_t(sms) * 3 * 6;
  int64_t ppc = int64_t(nblocks) * (S / 2) / (target > 0 ? target : 1);
  return int(ppc < 1 ? 1 : ppc > 16 ? 16 : ppc);
}

}  // namespace hfmm_b200

#endif
