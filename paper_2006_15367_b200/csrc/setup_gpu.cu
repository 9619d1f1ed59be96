// Setup on the device, bit-exact with the host build in
// setup.cpp and therefore with the reference's build_setup:
//
//  * Morton keys of every particle (morton.cpp:29-49; same FP64 expression
//    as the host: (p - corner) * inv truncated, clamped to cells - 1) and
//    the stable sort by key (traversal.cpp:100-110) as a CUB LSD radix sort
//    of (key, input index) pairs over the 3 (L - 1) code bits -- a stable
//    sort's permutation is unique, so it equals the host's; the sorted
//    particles are gathered on the device;
//  * far lists of levels max(top, 2)..L (interaction_lists.cpp:54-98) and
//    near lists of the leaves (:62-80): one thread per node, count pass ->
//    offsets -> fill pass.  A node's present neighbours are enumerated in
//    ascending code order and the children of a present parent are the
//    contiguous run [pn << 3, pn << 3 | 7] of the level's sorted codes, so
//    the lists come out in the host's (sorted) order without a sort.
//
// Selected by hfmm_run_config.setup_device = 1.  The rest of the setup
// (partition, levels, slices, plans) is O(nodes) host work.
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "setup.hpp"

namespace hfmm_b200 {
namespace {

void cu(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("setup_device: ") + what + ": " + cudaGetErrorString(e));
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  explicit DevBuf(size_t n) { cu(cudaMalloc(&p, (n ? n : 1) * sizeof(T)), "cudaMalloc"); }
  ~DevBuf() { cudaFree(p); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
};

template <class T>
void to_dev(T* d, const T* h, size_t n) {
  if (n) cu(cudaMemcpy(d, h, n * sizeof(T), cudaMemcpyHostToDevice), "H2D");
}
template <class T>
void to_host(T* h, const T* d, size_t n) {
  if (n) cu(cudaMemcpy(h, d, n * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
}

__device__ __forceinline__ uint64_t d_interleave(uint32_t x, uint32_t y, uint32_t z, int level) {
  uint64_t code = 0;  // x bit lowest, then y, then z (morton.cpp:43-47)
  for (int t = 0; t < level - 1; ++t) {
    code |= uint64_t((x >> t) & 1) << (3 * t);
    code |= uint64_t((y >> t) & 1) << (3 * t + 1);
    code |= uint64_t((z >> t) & 1) << (3 * t + 2);
  }
  return code;
}

__device__ __forceinline__ uint32_t d_cell(uint64_t code, int level, int axis) {
  uint32_t v = 0;  // MortonKey::deinterleave, morton.hpp:34-39
  for (int t = 0; t < level - 1; ++t) v |= uint32_t((code >> (3 * t + axis)) & 1) << t;
  return v;
}

__device__ __forceinline__ int64_t d_lower_bound(const uint64_t* __restrict__ a, int64_t n, uint64_t v) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Present same-level boxes within Chebyshev distance one (self included),
// ascending codes; returns the count and their indices.
__device__ int d_neighbors(const uint64_t* __restrict__ codes, int64_t n, uint64_t code, int level,
                           uint64_t (&out)[27], int64_t (&idx)[27]) {
  const int64_t cells = int64_t(1) << (level - 1);
  const int64_t x = d_cell(code, level, 0), y = d_cell(code, level, 1), z = d_cell(code, level, 2);
  int nf = 0;
  for (int64_t dx = -1; dx <= 1; ++dx)
    for (int64_t dy = -1; dy <= 1; ++dy)
      for (int64_t dz = -1; dz <= 1; ++dz) {
        const int64_t nx = x + dx, ny = y + dy, nz = z + dz;
        if (nx < 0 || ny < 0 || nz < 0 || nx >= cells || ny >= cells || nz >= cells) continue;
        const uint64_t c = d_interleave(uint32_t(nx), uint32_t(ny), uint32_t(nz), level);
        const int64_t k = d_lower_bound(codes, n, c);
        if (k < n && codes[k] == c) {
          int j = nf++;  // insertion into ascending order
          while (j > 0 && out[j - 1] > c) {
            out[j] = out[j - 1];
            idx[j] = idx[j - 1];
            --j;
          }
          out[j] = c;
          idx[j] = k;
        }
      }
  return nf;
}

__device__ __forceinline__ bool d_boxes_near(uint64_t a, uint64_t b, int l) {
  for (int ax = 0; ax < 3; ++ax) {  // interaction_lists.cpp:11-19
    const uint32_t u = d_cell(a, l, ax), v = d_cell(b, l, ax);
    if ((u > v ? u - v : v - u) > 1) return false;
  }
  return true;
}

__global__ void k_keys(int64_t n, const double* __restrict__ xyz, double c0, double c1, double c2, double root_side,
                       double inv, uint32_t cells, int L, uint64_t* __restrict__ keys, uint64_t* __restrict__ idx,
                       int* __restrict__ bad) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double corner[3] = {c0, c1, c2};
  uint32_t c3[3];
  for (int a = 0; a < 3; ++a) {
    const double v = __dsub_rn(xyz[3 * i + a], corner[a]);
    if (v < 0.0 || v > root_side) {
      atomicExch(bad, 1);
      c3[a] = 0;
    } else {
      const uint32_t c = uint32_t(__dmul_rn(v, inv));
      c3[a] = c < cells - 1 ? c : cells - 1;
    }
  }
  keys[i] = d_interleave(c3[0], c3[1], c3[2], L);
  idx[i] = uint64_t(i);
}

__global__ void k_gather_particles(int64_t n, const uint64_t* __restrict__ order, const double* __restrict__ xyz,
                                   const double* __restrict__ q, double* __restrict__ xyz_s,
                                   double* __restrict__ q_s) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t j = int64_t(order[i]);
  xyz_s[3 * i] = xyz[3 * j];
  xyz_s[3 * i + 1] = xyz[3 * j + 1];
  xyz_s[3 * i + 2] = xyz[3 * j + 2];
  q_s[2 * i] = q[2 * j];
  q_s[2 * i + 1] = q[2 * j + 1];
}

// FILL = false: counts[i] = far list length; FILL = true: writes the list at off[i].
template <bool FILL>
__global__ void k_far(int l, const uint64_t* __restrict__ codes, int64_t n, const uint64_t* __restrict__ pcodes,
                      int64_t np, const uint64_t* __restrict__ off, uint32_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t c = codes[i];
  uint64_t nb[27];
  int64_t ni[27];
  const int m = d_neighbors(pcodes, np, c >> 3, l - 1, nb, ni);
  uint32_t cnt = 0;
  uint64_t w = FILL ? off[i] : 0;
  for (int j = 0; j < m; ++j) {
    const uint64_t base = nb[j] << 3;
    for (int64_t k = d_lower_bound(codes, n, base); k < n && codes[k] <= (base | 7); ++k) {
      if (d_boxes_near(c, codes[k], l)) continue;
      if (FILL) out[w++] = uint32_t(k); else ++cnt;
    }
  }
  if (!FILL) out[i] = cnt;
}

template <bool FILL>
__global__ void k_near(int L, const uint64_t* __restrict__ codes, int64_t n, const uint64_t* __restrict__ off,
                       uint32_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t nb[27];
  int64_t ni[27];
  const int m = d_neighbors(codes, n, codes[i], L, nb, ni);
  if (!FILL) {
    out[i] = uint32_t(m);
    return;
  }
  const uint64_t w = off[i];
  for (int j = 0; j < m; ++j) out[w + j] = uint32_t(ni[j]);
}

unsigned blocks(int64_t n, int t) { return unsigned((n + t - 1) / t); }

// counts -> CSR offsets (n + 1) on the host
std::vector<uint64_t> scan(const std::vector<uint32_t>& cnt) {
  std::vector<uint64_t> off(cnt.size() + 1, 0);
  for (size_t i = 0; i < cnt.size(); ++i) off[i + 1] = off[i] + cnt[i];
  return off;
}

}  // namespace

void device_keys_sort(const double* xyz, const double* q, size_t n, const double corner[3], double root_side,
                      double inv, uint32_t cells, int L, std::vector<uint64_t>& sorted_keys,
                      std::vector<uint64_t>& order, std::vector<double>& xyz_s, std::vector<double>& q_s) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw std::runtime_error("setup_device: no CUDA device (use setup_device = 0 for the host build)");
  DevBuf<double> dxyz(3 * n), dq(2 * n), dxyz_s(3 * n), dq_s(2 * n);
  DevBuf<uint64_t> keys(n), keys_s(n), idx(n), idx_s(n);
  DevBuf<int> bad(1);
  to_dev(dxyz.p, xyz, 3 * n);
  to_dev(dq.p, q, 2 * n);
  cu(cudaMemset(bad.p, 0, sizeof(int)), "memset");
  k_keys<<<blocks(int64_t(n), 256), 256>>>(int64_t(n), dxyz.p, corner[0], corner[1], corner[2], root_side, inv,
                                           cells, L, keys.p, idx.p, bad.p);
  cu(cudaGetLastError(), "k_keys");
  int hbad = 0;
  to_host(&hbad, bad.p, 1);
  if (hbad) throw std::out_of_range("morton_key: position outside root box");
  const int bits = 3 * (L - 1);
  if (bits > 0) {
    size_t tmp_bytes = 0;
    cu(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, keys_s.p, idx.p, idx_s.p, int64_t(n), 0, bits),
       "radix sort size");
    DevBuf<unsigned char> tmp(tmp_bytes);
    cu(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, keys_s.p, idx.p, idx_s.p, int64_t(n), 0, bits),
       "radix sort");
  } else {
    cu(cudaMemcpy(keys_s.p, keys.p, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice), "copy");
    cu(cudaMemcpy(idx_s.p, idx.p, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice), "copy");
  }
  k_gather_particles<<<blocks(int64_t(n), 256), 256>>>(int64_t(n), idx_s.p, dxyz.p, dq.p, dxyz_s.p, dq_s.p);
  cu(cudaGetLastError(), "k_gather_particles");
  sorted_keys.resize(n);
  order.resize(n);
  xyz_s.resize(3 * n);
  q_s.resize(2 * n);
  to_host(sorted_keys.data(), keys_s.p, n);
  to_host(order.data(), idx_s.p, n);
  to_host(xyz_s.data(), dxyz_s.p, 3 * n);
  to_host(q_s.data(), dq_s.p, 2 * n);
}

void device_lists(Setup& s) {
  const int L = s.L;
  std::vector<LevelData>& lv = s.levels;
  const int lo = std::max(s.top, 2) - 1;
  std::vector<DevBuf<uint64_t>*> dcodes(size_t(L + 1), nullptr);
  try {
    for (int l = lo; l <= L; ++l) {
      dcodes[size_t(l)] = new DevBuf<uint64_t>(lv[size_t(l)].codes.size());
      to_dev(dcodes[size_t(l)]->p, lv[size_t(l)].codes.data(), lv[size_t(l)].codes.size());
    }
    for (int l = s.top; l <= L; ++l) {
      LevelData& t = lv[size_t(l)];
      const int64_t n = int64_t(t.codes.size());
      if (l < std::max(s.top, 2)) {
        t.far_off.assign(size_t(n) + 1, 0);
        t.far.clear();
        continue;
      }
      const int64_t np = int64_t(lv[size_t(l - 1)].codes.size());
      DevBuf<uint32_t> cnt(static_cast<size_t>(n));
      k_far<false><<<blocks(n, 128), 128>>>(l, dcodes[size_t(l)]->p, n, dcodes[size_t(l - 1)]->p, np, nullptr,
                                            cnt.p);
      cu(cudaGetLastError(), "k_far count");
      std::vector<uint32_t> hc(static_cast<size_t>(n));
      to_host(hc.data(), cnt.p, size_t(n));
      t.far_off = scan(hc);
      DevBuf<uint64_t> off(size_t(n) + 1);
      to_dev(off.p, t.far_off.data(), size_t(n) + 1);
      DevBuf<uint32_t> far(size_t(t.far_off.back()));
      k_far<true><<<blocks(n, 128), 128>>>(l, dcodes[size_t(l)]->p, n, dcodes[size_t(l - 1)]->p, np, off.p, far.p);
      cu(cudaGetLastError(), "k_far fill");
      t.far.resize(size_t(t.far_off.back()));
      to_host(t.far.data(), far.p, t.far.size());
    }
    {
      const int64_t n = int64_t(lv[size_t(L)].codes.size());
      DevBuf<uint32_t> cnt(static_cast<size_t>(n));
      k_near<false><<<blocks(n, 128), 128>>>(L, dcodes[size_t(L)]->p, n, nullptr, cnt.p);
      cu(cudaGetLastError(), "k_near count");
      std::vector<uint32_t> hc(static_cast<size_t>(n));
      to_host(hc.data(), cnt.p, size_t(n));
      s.near_off = scan(hc);
      DevBuf<uint64_t> off(size_t(n) + 1);
      to_dev(off.p, s.near_off.data(), size_t(n) + 1);
      DevBuf<uint32_t> nr(size_t(s.near_off.back()));
      k_near<true><<<blocks(n, 128), 128>>>(L, dcodes[size_t(L)]->p, n, off.p, nr.p);
      cu(cudaGetLastError(), "k_near fill");
      s.near.resize(size_t(s.near_off.back()));
      to_host(s.near.data(), nr.p, s.near.size());
    }
  } catch (...) {
    for (auto* p : dcodes) delete p;
    throw;
  }
  for (auto* p : dcodes) delete p;
}

}  // namespace hfmm_b200
