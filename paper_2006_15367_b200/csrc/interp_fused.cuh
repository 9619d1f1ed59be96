// Fused single-kernel M2M for the leaf-side level pair (18, 28) of the
// BASELINE cubes (configs 1, 3, 4 leaf level): one CTA per SM, persistent over
// parents, both passes of the separable resampling in one kernel with the
// intermediate (folded circles F) in SHARED memory -- it never touches HBM (the
// two-kernel streaming form, interp_rb.cuh, writes and re-reads it: 27.8 GB +
// 25.9 GB per evaluation at config 4; fused, the kernel moves the compulsory
// 14.2 GB).  (The mirrored fused L2L -- parent local by bulk copy, narrow rows in
// shared memory -- was built twice this round and measured 1.3 and 2.8 ms slower
// than the two-kernel form at config 4; it is not kept.)  Same algebra and the same device helpers as
// interp_rb.cuh (real + rank-1 matrices on DMMA, even / odd theta passes,
// complex-row warp tiles, child sum as a reduce-scatter); traversal.cpp:322-429,
// sphere_grid.cpp:183-192.  Per-parent inputs arrive through the Blackwell
// bulk-copy engine (cp.async.bulk + mbarrier, bulk.cuh), one parent ahead.
#ifndef HFMM_B200_INTERP_FUSED_CUH
#define HFMM_B200_INTERP_FUSED_CUH

#include "bulk.cuh"
#include "interp_rb.cuh"

namespace hfmm_b200 {
namespace fz {
__host__ __device__ constexpr int pad4mod8(int x) { return x + ((4 - x % 8) + 8) % 8; }  // stride == 4 (mod 8) double2
}  // namespace fz

// Pairs served by the fused kernels.
inline bool fz_pair(int nc, int np) { return nc == 18 && np == 28; }

// ---------------------------------------------------------------------------
// Fused (18, 28) M2M: one CTA per SM, 14 warps, and NO global load inside the two
// passes.  The children of a parent arrive as bulk
// asynchronous copies (cp.async.bulk, mbarrier completion) into a
// double-buffered shared-memory block, issued a whole parent ahead; the shift
// factors come from a quarter table in shared memory (the sphere grid's
// symmetries theta -> pi - theta and phi -> phi + pi map a sample of octant o
// to the mirrored sample of octant o ^ 4 / o ^ 3, so rows < NP / 2 and columns
// < NP / 2 of the 8 octant tables suffice: 25 KB instead of 100 KB); the rank-1
// vectors sit in shared memory as well, and the parent descriptors (rb::PDesc)
// travel one parent ahead in registers.  (ncu on the first version -- 2 CTAs of
// 7 warps, children and shifts read through L1 -- showed long-scoreboard stalls
// on those loads at 43% tensor pipe.)
namespace fz2 {

constexpr int kWarps = 14, kThreads = 32 * kWarps;

template <int NC, int NP>
struct Lay {
  using D = rb::Dims<NC, NP>;
  static constexpr int H = NP / 2, SC = NC * NC;
  // folded circles: x_e at [0, NC), x_o at [4 KH, 4 KH + NC) of a row of LDF
  // complex; LDF == 2 (mod 8) spreads the phi pass's 16-byte stores over the banks
  static constexpr int LDF = D::UTH_K + 2;
  static constexpr int CSF = fz::pad4mod8(H * LDF);
  static constexpr int BPHI = D::UPHI_K * D::UPHI_LDB, BTH = D::UTH_K * D::UTH_LDB;  // doubles
  static constexpr int VPHI = D::UPHI_K, VTH = D::UTH_K;                               // doubles
  static constexpr int SHROW = H + 1, SHOCT = H * SHROW + 1;                           // double2 (padded)
  static constexpr int OFF_SH = (BPHI + BTH + VPHI + VTH) * 8;
  static constexpr int OFF_F = OFF_SH + 8 * SHOCT * 16;
  static constexpr int OFF_CH = OFF_F + 8 * CSF * 16;
  static constexpr int OFF_BAR = OFF_CH + 2 * 8 * SC * 16;
  static constexpr int SMEM = OFF_BAR + 16;
  static_assert(OFF_SH % 16 == 0 && H % 2 == 0, "layout");
};

}  // namespace fz2

template <int NC, int NP>
__global__ void __launch_bounds__(fz2::kThreads, 1) k_m2m_fz2(int n_par, const int4* __restrict__ pdesc,
                                                              const double2* __restrict__ mp_c,
                                                              const double* __restrict__ Bphi,
                                                              const double* __restrict__ vphi,
                                                              const double* __restrict__ Bth,
                                                              const double* __restrict__ vth,
                                                              const double2* __restrict__ shift_up,
                                                              double2* __restrict__ mp_p) {
  using D = rb::Dims<NC, NP>;
  using Y = fz2::Lay<NC, NP>;
  constexpr int KSP = D::UPHI_K / 4, HALF = D::HALF, SP = D::SP, SC = D::SC, H = Y::H;
  constexpr int NW = fz2::kWarps, WI = NW - 1;  // WI: the issuing warp (one with fewer phi items)
  extern __shared__ __align__(16) unsigned char fz2_smem[];
  double* Bp = reinterpret_cast<double*>(fz2_smem);
  double* Bt = Bp + Y::BPHI;
  double* vp = Bt + Y::BTH;
  double* vt = vp + Y::VPHI;
  double2* shq = reinterpret_cast<double2*>(fz2_smem + Y::OFF_SH);
  double2* Fs = reinterpret_cast<double2*>(fz2_smem + Y::OFF_F);
  double2* Ch = reinterpret_cast<double2*>(fz2_smem + Y::OFF_CH);
  uint64_t* bar = reinterpret_cast<uint64_t*>(fz2_smem + Y::OFF_BAR);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int G = gridDim.x;
  const int* pdi = reinterpret_cast<const int*>(pdesc);

  // Parent descriptors (rb::PDesc) travel one parent ahead in registers: dn for
  // every thread, and the child row of slot (lane & 7) for the issuing warp --
  // no global load sits between a parent's barrier and its work.
  auto desc = [&](int par) { return par < n_par ? __ldg(pdesc + 3 * par) : make_int4(0, 0, 0, 0); };
  auto crow = [&](int par) { return par < n_par ? __ldg(pdi + 12 * par + 4 + (lane & 7)) : -1; };
  // the issuing warp: children of a parent -> buffer b (one bulk copy per child)
  auto issue = [&](const int4& d, int cr, int b) {
    if (lane == 0) bulk::mbar_expect_tx(bar + b, uint32_t(d.y) * uint32_t(SC) * 16u);
    __syncwarp();
    if (lane < d.y) bulk::copy_g2s(Ch + (b * 8 + lane) * SC, mp_c + int64_t(cr) * SC, uint32_t(SC) * 16u, bar + b);
  };
  if (threadIdx.x == 0) {
    bulk::mbar_init(bar, 1);
    bulk::mbar_init(bar + 1, 1);
    bulk::fence_mbar_init();
  }
  __syncthreads();
  int par = blockIdx.x;
  int4 dc = desc(par), dn = desc(par + G);
  int cn = warp == WI ? crow(par + G) : -1;
  if (warp == WI && par < n_par) issue(dc, crow(par), 0);
  for (int t = threadIdx.x; t < Y::VPHI; t += blockDim.x) vp[t] = t < NC ? vphi[t] : 0.0;
  for (int t = threadIdx.x; t < Y::VTH; t += blockDim.x) vt[t] = vth[t];
  for (int t = threadIdx.x; t < 8 * H * H; t += blockDim.x) {
    const int o = t / (H * H), r = t - o * H * H, n = r / H, pc = r - n * H;
    shq[o * Y::SHOCT + n * Y::SHROW + pc] = shift_up[int64_t(o) * SP + n * NP + pc];
  }
  rb::stage_b<D::UPHI_K, D::UPHI_N, D::UPHI_LDB>(Bp, Bphi);
  rb::stage_b<D::UTH_K, D::UTH_N, D::UTH_LDB>(Bt, Bth);  // (ends with a CTA barrier)

  for (int it = 0; par < n_par; par += G, ++it) {
    const int b = it & 1;
    const int nch = dc.y;
    // buffer b ^ 1 was last read by the phi pass of the previous parent, which
    // every warp left before that parent's theta pass
    if (warp == WI && par + G < n_par) issue(dn, cn, b ^ 1);
    const int4 d2 = desc(par + 2 * G);  // consumed at the bottom of this iteration
    const int c2 = warp == WI ? crow(par + 2 * G) : -1;
    bulk::mbar_wait(bar + b, uint32_t(it >> 1) & 1u);
    const double2* ch = Ch + b * 8 * SC;
    // phi pass: item = (row tile, half of the output columns) -> folded circles
    const int rows = nch * NC, tiles = (rows + 7) / 8;
    for (int item = warp; item < 2 * tiles; item += NW) {
      const int t = item >> 1, hh = item & 1;
      const int R = t * 8 + g;
      const bool ok = R < rows;
      const int c = ok ? R / NC : 0, i = ok ? R - c * NC : 0;
      const double2* x = ch + c * SC + i * NC;
      double are[KSP], aim[KSP];
#pragma unroll
      for (int kk = 0; kk < KSP; ++kk) {
        const int k = 4 * kk + tq;
        const double2 xv = (ok && k < NC) ? x[k] : make_double2(0.0, 0.0);
        are[kk] = xv.x;
        aim[kk] = xv.y;
      }
      rb::rank1_inject_f<KSP, NC>(are, aim, [&](int k) { return vp[k]; });
      constexpr int NTH = D::UPHI_N / 16;  // n8 tiles per half
      static_assert(D::UPHI_N % 16 == 0, "phi output tiles split in two halves");
      double cre[NTH][2] = {}, cim[NTH][2] = {};
      rb::tile_mma<KSP, NTH, D::UPHI_LDB>(are, aim, Bp + 8 * NTH * hh, cre, cim);
      if (ok) {
        double2* Fc = Fs + c * Y::CSF;
#pragma unroll
        for (int jn = 0; jn < NTH; ++jn)
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int n = 8 * (NTH * hh + jn) + 2 * tq + q;  // column 2 p + h: circle p, part e / o
            if (n < NP) Fc[(n >> 1) * Y::LDF + (n & 1) * 4 * D::UTH_KH + i] = make_double2(cre[jn][q], cim[jn][q]);
          }
      }
    }
    __syncthreads();
    // theta pass + shift + child sum: item = circle p, tile rows = child slots
    const bool ok = g < nch;
    const int oct = ok ? rb::pdesc_oct(dc, g) : 0;
    double2* out = mp_p + int64_t(dc.z) * SP;
    for (int p = warp; p < HALF; p += NW) {
      const double2* frow = Fs + (ok ? g : 0) * Y::CSF + p * Y::LDF;
      rb::m2m_theta_item_f<NC, NP>(
          [&](int k) { return frow[k]; }, ok,
          [&](int n, int back) {
            const int up = n >= H;  // mirrored theta row: octant with z flipped
            const int o = oct ^ (up ? 4 : 0) ^ (back ? 3 : 0);
            return shq[o * Y::SHOCT + (up ? NP - 1 - n : n) * Y::SHROW + p];
          },
          out, p, Bt, [&](int k) { return vt[k]; });
    }
    __syncthreads();
    dc = dn;
    dn = d2;
    cn = c2;
  }
}

inline void launch_m2m_fz2(const RbLaunch& L, int sms, const double2* mp_c, double2* mp_p, const double* Bphi,
                           const double* vphi, const double* Bth, const double* vth, const double2* shift_up) {
  constexpr int smem = fz2::Lay<18, 28>::SMEM;
  static_assert(smem <= 227 * 1024, "fused M2M v2 shared memory");
  cudaFuncSetAttribute(k_m2m_fz2<18, 28>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = std::min(L.n_par, sms);
  k_m2m_fz2<18, 28><<<grid, fz2::kThreads, smem, L.st>>>(L.n_par, L.pdesc, mp_c, Bphi, vphi, Bth, vth, shift_up, mp_p);
}

}  // namespace hfmm_b200

#endif
