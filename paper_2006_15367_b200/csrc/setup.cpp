// Host setup, bit-exact with the reference build_setup.  Each step cites the
// reference lines whose floating-point expression order it reproduces.
#include "setup.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <numeric>
#include <set>
#include <unordered_map>

namespace hfmm_b200 {

namespace {

// HFMM_SETUP_TIMING=1: per-section wall time of build_setup on stderr.
struct SectionTimer {
  bool on = std::getenv("HFMM_SETUP_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[setup] %-22s %8.3f s\n", what, std::chrono::duration<double>(now - t).count());
    t = now;
  }
};

constexpr uint64_t kCodeMask = (uint64_t(1) << 58) - 1;

inline uint64_t interleave(uint32_t x, uint32_t y, uint32_t z, int level) {
  // x bit lowest, then y, then z (morton.cpp:43-47, interaction_lists.cpp:41-50)
  uint64_t code = 0;
  for (int t = 0; t < level - 1; ++t) {
    code |= uint64_t((x >> t) & 1) << (3 * t);
    code |= uint64_t((y >> t) & 1) << (3 * t + 1);
    code |= uint64_t((z >> t) & 1) << (3 * t + 2);
  }
  return code;
}

inline uint32_t cell_of_code(uint64_t code, int level, int axis) {
  uint32_t v = 0;  // MortonKey::deinterleave, morton.hpp:34-39
  for (int t = 0; t < level - 1; ++t) v |= uint32_t((code >> (3 * t + axis)) & 1) << t;
  return v;
}

// compute_num_levels, morton.cpp:19-27
int num_levels(double root_diameter, double leaf_diameter) {
  if (!(leaf_diameter > 0.0) || root_diameter < leaf_diameter)
    throw std::invalid_argument("compute_num_levels: need D0 >= leaf > 0");
  double lv = std::log2(root_diameter / leaf_diameter) + 1.0;
  int L = int(std::ceil(lv));
  if (L > 1 && double(L - 1) >= lv) --L;
  return std::max(L, 1);
}

}  // namespace

int truncation_order(double diameter, double k, double digits) {
  // sphere_grid.cpp:13-23
  if (k == 0.0)
    throw std::invalid_argument("truncation_order: Laplace limit (k == 0) unsupported");
  if (!(diameter > 0.0) || !(digits > 0.0))
    throw std::invalid_argument("truncation_order: need diameter, digits > 0");
  double kd = k * diameter;
  double L = std::ceil(kd + 1.8 * std::pow(digits, 2.0 / 3.0) * std::cbrt(kd));
  return std::max(4, int(L));
}

void fejer_weights(int64_t nt, std::vector<double>& w) {
  // make_quadrature, sphere_grid.cpp:52-70 (same expression order)
  w.resize(size_t(nt));
  for (size_t i = 0; i < size_t(nt); ++i) {
    double th = (double(i) + 0.5) * M_PI / double(nt);
    double s = 0.0;
    for (size_t m = 1; m <= size_t(nt) / 2; ++m)
      s += std::cos(2.0 * double(m) * th) / double(4 * m * m - 1);
    w[i] = (2.0 / double(nt)) * (1.0 - 2.0 * s);
  }
}

int64_t LevelData::find(uint64_t code) const {
  if (!dense_lookup.empty()) return code < dense_lookup.size() ? dense_lookup[code] : -1;
  auto it = std::lower_bound(codes.begin(), codes.end(), code);
  if (it == codes.end() || *it != code) return -1;
  return int64_t(it - codes.begin());
}

int Setup::rank_of_leaf(uint64_t li) const {
  // Partition::rank_of_leaf, tree.cpp:12-17 (ranges are contiguous and sorted)
  auto it = std::upper_bound(rank_begin.begin(), rank_begin.end(), li);
  if (it == rank_begin.begin()) throw std::out_of_range("rank_of_leaf: index outside partition");
  int r = int(it - rank_begin.begin()) - 1;
  if (li >= rank_end[size_t(r)]) throw std::out_of_range("rank_of_leaf: index outside partition");
  return r;
}

namespace {

// partition_leaves, tree.cpp:19-75
void partition(Setup& s, const std::vector<uint64_t>& weights) {
  const int P = s.cfg.num_ranks;
  const size_t nl = weights.size();
  if (P < 1) throw std::invalid_argument("partition_leaves: num_ranks < 1");
  if (nl == 0) throw std::invalid_argument("partition_leaves: no nonempty leaves");
  if (size_t(P) > nl)
    throw std::invalid_argument("partition_leaves: more ranks than nonempty leaves");
  size_t total = 0;
  for (uint64_t w : weights) total += w;
  std::vector<int> rank_of(nl);
  size_t prefix = 0;
  for (size_t i = 0; i < nl; ++i) {
    double mid = double(prefix) + 0.5 * double(weights[i]);
    rank_of[i] = std::min(P - 1, int(mid * double(P) / double(total)));
    prefix += weights[i];
  }
  for (size_t i = 1; i < nl; ++i)
    if (rank_of[i] < rank_of[i - 1]) rank_of[i] = rank_of[i - 1];
  for (int r = 1; r < P; ++r) {
    if (std::find(rank_of.begin(), rank_of.end(), r) == rank_of.end()) {
      auto pos = std::find_if(rank_of.rbegin(), rank_of.rend(), [&](int v) { return v < r; });
      *pos = r;
    }
  }
  std::sort(rank_of.begin(), rank_of.end());
  s.P = P;
  s.rank_begin.assign(size_t(P), 0);
  s.rank_end.assign(size_t(P), 0);
  size_t idx = 0;
  for (int r = 0; r < P; ++r) {
    size_t b = idx;
    while (idx < nl && rank_of[idx] == r) ++idx;
    s.rank_begin[size_t(r)] = b;
    s.rank_end[size_t(r)] = idx;
    if (b == idx) throw std::logic_error("partition_leaves: produced an empty rank");
  }
  s.splitters.clear();
  for (int r = 1; r < P; ++r)
    s.splitters.push_back((uint64_t(s.L) << 58) | s.leaf_codes[s.rank_begin[size_t(r)]]);
}

struct Stake {
  double lowest = 2.0;
  size_t samples = 0;
};

// assign_sample_slices, tree.cpp:180-239
std::vector<SliceRec> assign_slices(size_t nt, size_t np, const std::vector<int>& users,
                                    const std::vector<Stake>& stakes, int policy) {
  if (users.empty()) throw std::invalid_argument("assign_sample_slices: empty user set");
  std::vector<size_t> order(users.size());
  std::iota(order.begin(), order.end(), 0);
  const bool aligned = policy == HFMM_POLICY_ALIGNED;
  if (aligned) {
    std::sort(order.begin(), order.end(), [&](size_t a, size_t b) {
      if (stakes[a].lowest != stakes[b].lowest) return stakes[a].lowest < stakes[b].lowest;
      if (stakes[a].samples != stakes[b].samples) return stakes[a].samples < stakes[b].samples;
      return users[a] < users[b];
    });
  }
  std::vector<size_t> cols(users.size(), 0);
  auto equal_split = [&] {
    size_t base = nt / users.size(), rem = nt % users.size();
    for (size_t i = 0; i < users.size(); ++i) cols[i] = base + (i < rem ? 1 : 0);
  };
  if (!aligned) {
    equal_split();
  } else {
    size_t total = 0;
    for (auto& st : stakes) total += st.samples;
    if (total == 0) {
      equal_split();
    } else {
      size_t assigned = 0;
      for (size_t i = 0; i < order.size(); ++i) {
        cols[i] = nt * stakes[order[i]].samples / total;
        assigned += cols[i];
      }
      for (size_t i = 0; assigned < nt; i = (i + 1) % cols.size()) {
        ++cols[i];
        ++assigned;
      }
    }
  }
  std::vector<SliceRec> out;
  size_t begin = 0;
  for (size_t i = 0; i < order.size(); ++i) {
    size_t len = cols[i] * np;
    out.push_back({users[order[i]], int64_t(begin), int64_t(begin + len)});
    begin += len;
  }
  if (begin != nt * np) throw std::logic_error("assign_sample_slices: cover mismatch");
  return out;
}

void build_lookup(LevelData& t) {
  const int l = t.level;
  if (3 * (l - 1) <= 27) {
    t.dense_lookup.assign(size_t(1) << (3 * (l - 1)), -1);
    for (size_t i = 0; i < t.codes.size(); ++i) t.dense_lookup[t.codes[i]] = int64_t(i);
  }
}

// Same-level present boxes within Chebyshev distance one, self included,
// Morton-sorted (interaction_lists.cpp:62-80).
template <class F>
void for_neighbors(const LevelData& t, uint64_t code, F&& f) {
  const int l = t.level;
  const long cells = long(1) << (l - 1);
  const long x = cell_of_code(code, l, 0), y = cell_of_code(code, l, 1), z = cell_of_code(code, l, 2);
  uint64_t found[27];
  int nf = 0;
  for (long dx = -1; dx <= 1; ++dx)
    for (long dy = -1; dy <= 1; ++dy)
      for (long dz = -1; dz <= 1; ++dz) {
        long nx = x + dx, ny = y + dy, nz = z + dz;
        if (nx < 0 || ny < 0 || nz < 0 || nx >= cells || ny >= cells || nz >= cells) continue;
        uint64_t c = interleave(uint32_t(nx), uint32_t(ny), uint32_t(nz), l);
        if (t.find(c) >= 0) found[nf++] = c;
      }
  std::sort(found, found + nf);
  for (int i = 0; i < nf; ++i) f(found[i]);
}

inline bool boxes_near(uint64_t a, uint64_t b, int l) {
  // interaction_lists.cpp:11-19
  for (int ax = 0; ax < 3; ++ax) {
    uint32_t u = cell_of_code(a, l, ax), v = cell_of_code(b, l, ax);
    if ((u > v ? u - v : v - u) > 1) return false;
  }
  return true;
}

}  // namespace

Setup build_setup(const double* xyz, const double* q, size_t n,
                  const hfmm_run_config& cfg) {
  // RunConfig::validate, traversal.cpp:42-46
  if (!(cfg.lambda > 0) || !(cfg.digits > 0) || !(cfg.leaf_lambda > 0) || cfg.num_ranks < 1 ||
      cfg.buffer_limit == 0 || cfg.top_level < 1)
    throw std::invalid_argument("RunConfig: invalid fields");
  if (n == 0) throw std::invalid_argument("build_setup: no particles");

  SectionTimer timer;
  Setup s;
  s.cfg = cfg;
  s.k = 2.0 * M_PI / cfg.lambda;  // Wavenumber::from_lambda, geometry.cpp:17-20
  const double leaf = cfg.leaf_lambda * cfg.lambda;

  double lo[3] = {xyz[0], xyz[1], xyz[2]}, hi[3] = {xyz[0], xyz[1], xyz[2]};
  for (size_t i = 0; i < n; ++i) {
    const double* p = xyz + 3 * i;
    if (!(std::isfinite(p[0]) && std::isfinite(p[1]) && std::isfinite(p[2])))
      throw std::invalid_argument("build_setup: non-finite position");
    for (int a = 0; a < 3; ++a) {
      lo[a] = std::min(lo[a], p[a]);
      hi[a] = std::max(hi[a], p[a]);
    }
  }
  timer.mark("bbox");
  // traversal.cpp:85-98
  for (int a = 0; a < 3; ++a) s.corner[a] = std::floor(lo[a] / leaf) * leaf;
  double span = std::max({hi[0] - s.corner[0], hi[1] - s.corner[1], hi[2] - s.corner[2]});
  const int L = num_levels(std::max(span, leaf), leaf);
  s.L = L;
  s.root_side = std::ldexp(leaf, L - 1);
  s.leaf_side = leaf;
  s.d_class = cfg.d_override ? cfg.d_override : ((hi[2] - lo[2]) < 0.5 * leaf ? 2 : 3);
  s.top = std::clamp(cfg.top_level, 1, L);

  // Morton keys at the leaf level (morton.cpp:29-49) and a stable sort
  // (traversal.cpp:100-110).  A stable LSD radix sort over the code bits is
  // order-identical to std::stable_sort with the packed-key comparator.
  const uint32_t cells = uint32_t(1) << (L - 1);
  const double inv = double(cells) / s.root_side;
  s.n = n;
  std::vector<uint64_t> skeys;  // keys in sorted order
  if (cfg.setup_device == 1) {
    device_keys_sort(xyz, q, n, s.corner, s.root_side, inv, cells, L, skeys, s.original_index, s.xyz, s.q);
  } else if (cfg.setup_device != 0) {
    throw std::invalid_argument("build_setup: setup_device must be 0 (host) or 1 (device)");
  } else {
    std::vector<uint64_t> keys(n);
    for (size_t i = 0; i < n; ++i) {
      uint32_t c3[3];
      for (int a = 0; a < 3; ++a) {
        double v = xyz[3 * i + a] - s.corner[a];
        if (v < 0.0 || v > s.root_side)
          throw std::out_of_range("morton_key: position outside root box");
        c3[a] = std::min(uint32_t(v * inv), cells - 1);
      }
      keys[i] = interleave(c3[0], c3[1], c3[2], L);
    }
    std::vector<uint64_t> order(n), tmp(n);
    std::iota(order.begin(), order.end(), 0);
    {
      const int bits = 3 * (L - 1);
      std::vector<size_t> count(1 << 16);
      for (int shift = 0; shift < bits; shift += 16) {
        std::fill(count.begin(), count.end(), 0);
        for (size_t i = 0; i < n; ++i) ++count[(keys[order[i]] >> shift) & 0xffff];
        size_t run = 0;
        for (auto& c : count) {
          size_t v = c;
          c = run;
          run += v;
        }
        for (size_t i = 0; i < n; ++i) tmp[count[(keys[order[i]] >> shift) & 0xffff]++] = order[i];
        order.swap(tmp);
      }
    }
    skeys.resize(n);
    for (size_t i = 0; i < n; ++i) skeys[i] = keys[order[i]];
    s.original_index = order;
    s.xyz.resize(3 * n);
    s.q.resize(2 * n);
    for (size_t i = 0; i < n; ++i) {
      const size_t jj = order[i];
      std::memcpy(&s.xyz[3 * i], xyz + 3 * jj, 3 * sizeof(double));
      std::memcpy(&s.q[2 * i], q + 2 * jj, 2 * sizeof(double));
    }
  }
  timer.mark("keys+sort+gather");
  // Leaves and particle ranges (traversal.cpp:112-126)
  for (size_t i = 0; i < n; ++i) {
    const uint64_t pk = skeys[i];
    if (s.leaf_codes.empty() || s.leaf_codes.back() != pk) {
      s.leaf_codes.push_back(pk);
      s.leaf_start.push_back(i);
    }
  }
  s.leaf_start.push_back(n);
  const size_t nl = s.leaf_codes.size();
  if (cfg.one_particle_per_leaf)
    for (size_t i = 0; i < nl; ++i)
      if (s.leaf_start[i + 1] - s.leaf_start[i] != 1)
        throw std::invalid_argument(
            "build_setup: one_particle_per_leaf set but a leaf holds " +
            std::to_string(s.leaf_start[i + 1] - s.leaf_start[i]) + " particles");

  std::vector<uint64_t> weights(nl);
  for (size_t i = 0; i < nl; ++i) weights[i] = s.leaf_start[i + 1] - s.leaf_start[i];
  if (cfg.partition_weight == 1) {
    // near-field pairs per leaf: n_i * sum over its near leaves (self included)
    LevelData t;
    t.level = L;
    t.codes = s.leaf_codes;
    std::vector<uint64_t> pairs(nl, 0);
    for (size_t i = 0; i < nl; ++i) {
      uint64_t srcs = 0;
      for_neighbors(t, t.codes[i], [&](uint64_t nc) {
        const int64_t j = t.find(nc);
        srcs += s.leaf_start[size_t(j) + 1] - s.leaf_start[size_t(j)];
      });
      pairs[i] = weights[i] * srcs;
    }
    weights.swap(pairs);
  } else if (cfg.partition_weight != 0) {
    throw std::invalid_argument("build_setup: partition_weight must be 0 (particles) or 1 (near pairs)");
  }
  partition(s, weights);

  timer.mark("leaves+partition");
  // Per-level node sets for every level 1..L (collect_level_nodes,
  // interaction_lists.cpp:21-37); tables are kept for top..L.
  s.levels.assign(size_t(L + 1), LevelData{});
  std::vector<LevelData>& lv = s.levels;
  for (int l = 1; l <= L; ++l) lv[size_t(l)].level = l;
  lv[size_t(L)].codes = s.leaf_codes;
  for (int l = L; l > 1; --l) {
    auto& up = lv[size_t(l - 1)].codes;
    for (uint64_t c : lv[size_t(l)].codes) {
      uint64_t p = c >> 3;
      if (up.empty() || up.back() != p) up.push_back(p);
    }
  }
  for (int l = 1; l <= L; ++l) build_lookup(lv[size_t(l)]);

  for (int l = s.top; l <= L; ++l) {
    LevelData& t = lv[size_t(l)];
    t.side = s.box_side(l);
    // make_level_sampling, sphere_grid.cpp:39-50
    t.trunc = truncation_order(t.side * std::sqrt(3.0), s.k, cfg.digits);
    t.nt = t.np = 2 * t.trunc + 2;
    fejer_weights(t.nt, t.theta_w);
    t.phi_w = 2.0 * M_PI / double(t.np);
    const size_t nn = t.codes.size();
    t.centers.resize(3 * nn);
    t.first_user.resize(nn);
    t.last_user.resize(nn);
    t.plural.resize(nn);
    const int shift = 3 * (L - l);
    for (size_t i = 0; i < nn; ++i) {
      const uint64_t c = t.codes[i];
      for (int a = 0; a < 3; ++a)  // TreeConfig::box_center, morton.cpp:12-17
        t.centers[3 * i + a] = s.corner[a] + (double(cell_of_code(c, l, a)) + 0.5) * t.side;
      uint64_t lo_leaf = c << shift, hi_leaf = (c + 1) << shift;
      size_t fl = size_t(std::lower_bound(s.leaf_codes.begin(), s.leaf_codes.end(), lo_leaf) -
                         s.leaf_codes.begin());
      size_t ll = size_t(std::lower_bound(s.leaf_codes.begin(), s.leaf_codes.end(), hi_leaf) -
                         s.leaf_codes.begin());
      t.first_user[i] = s.rank_of_leaf(fl);
      t.last_user[i] = s.rank_of_leaf(ll - 1);
      t.plural[i] = t.first_user[i] != t.last_user[i];
    }
  }
  timer.mark("levels+centers");
  // Child links (traversal.cpp:165-173): children in ascending index order.
  for (int l = s.top; l < L; ++l) {
    LevelData& t = lv[size_t(l)];
    const LevelData& ct = lv[size_t(l + 1)];
    std::vector<std::vector<uint64_t>> ch(t.codes.size());
    for (size_t ci = 0; ci < ct.codes.size(); ++ci) {
      int64_t pi = t.find(ct.codes[ci] >> 3);
      if (pi >= 0) ch[size_t(pi)].push_back(ci);
    }
    t.child_off.assign(1, 0);
    for (auto& v : ch) {
      t.children.insert(t.children.end(), v.begin(), v.end());
      t.child_off.push_back(t.children.size());
    }
  }
  lv[size_t(L)].child_off.assign(lv[size_t(L)].codes.size() + 1, 0);

  timer.mark("child links");
  // Sample slices bottom-up (traversal.cpp:174-195)
  for (int l = L; l >= s.top; --l) {
    LevelData& t = lv[size_t(l)];
    const size_t nn = t.codes.size();
    t.slice_off.assign(1, 0);
    for (size_t i = 0; i < nn; ++i) {
      if (!t.plural[i]) {
        t.slices.push_back({t.first_user[i], 0, t.samples()});
      } else {
        std::vector<int> users;
        for (int r = t.first_user[i]; r <= t.last_user[i]; ++r) users.push_back(r);
        // compute_child_stakes, tree.cpp:163-178
        std::vector<Stake> stakes(users.size());
        const LevelData& ct = lv[size_t(l + 1)];
        const double total = double(ct.samples());
        for (size_t u = 0; u < users.size(); ++u)
          for (uint64_t k = t.child_off[i]; k < t.child_off[i + 1]; ++k) {
            const uint64_t ci = t.children[k];
            for (uint64_t z = ct.slice_off[ci]; z < ct.slice_off[ci + 1]; ++z) {
              const SliceRec& sl = ct.slices[z];
              if (sl.rank != users[u] || sl.size() == 0) continue;
              stakes[u].samples += size_t(sl.size());
              stakes[u].lowest = std::min(stakes[u].lowest, double(sl.begin) / total);
            }
          }
        auto m = assign_slices(size_t(t.nt), size_t(t.np), users, stakes, cfg.policy);
        t.slices.insert(t.slices.end(), m.begin(), m.end());
      }
      t.slice_off.push_back(t.slices.size());
    }
  }
  // Interpolation layouts of plural nodes (traversal.cpp:196-224)
  for (int l = s.top; l <= L; ++l) {
    LevelData& t = lv[size_t(l)];
    t.interp_off.assign(1, 0);
    for (size_t i = 0; i < t.codes.size(); ++i) {
      if (l > s.top && t.plural[i]) {
        const uint64_t nt_parent = uint64_t(lv[size_t(l - 1)].nt);
        const uint64_t np_parent = uint64_t(lv[size_t(l - 1)].np);
        const uint64_t nt_child = uint64_t(t.nt);
        const size_t parts = t.slice_off[i + 1] - t.slice_off[i];
        std::vector<uint64_t> cols(parts);
        uint64_t assigned = 0;
        for (size_t u = 0; u < parts; ++u) {
          uint64_t src_cols = uint64_t(t.slices[t.slice_off[i] + u].size()) / uint64_t(t.np);
          cols[u] = nt_parent * src_cols / nt_child;
          assigned += cols[u];
        }
        for (size_t u = 0; assigned < nt_parent; u = (u + 1) % parts) {
          ++cols[u];
          ++assigned;
        }
        t.interp.push_back(nt_parent);
        t.interp.push_back(np_parent);
        uint64_t run = 0;
        t.interp.push_back(0);
        for (size_t u = 0; u < parts; ++u) {
          run += cols[u];
          t.interp.push_back(run);
        }
      }
      t.interp_off.push_back(t.interp.size());
    }
  }

  timer.mark("slices+interp");
  if (cfg.setup_device == 1) {
    device_lists(s);  // far + near lists on the device (setup_gpu.cu)
  } else {
    // Far lists, levels max(top, 2)..L (interaction_lists.cpp:54-98)
    for (int l = s.top; l <= L; ++l) {
      LevelData& t = lv[size_t(l)];
      t.far_off.assign(1, 0);
      const bool has_far = l >= std::max(s.top, 2);
      std::vector<uint64_t> far;
      for (size_t i = 0; i < t.codes.size(); ++i) {
        if (has_far) {
          far.clear();
          const uint64_t c = t.codes[i];
          for_neighbors(lv[size_t(l - 1)], c >> 3, [&](uint64_t pn) {
            for (uint64_t oct = 0; oct < 8; ++oct) {
              uint64_t cand = (pn << 3) | oct;
              if (t.find(cand) < 0) continue;
              if (!boxes_near(c, cand, l)) far.push_back(cand);
            }
          });
          std::sort(far.begin(), far.end());
          for (uint64_t fc : far) t.far.push_back(uint32_t(t.find(fc)));
        }
        t.far_off.push_back(t.far.size());
      }
    }
    timer.mark("far lists");
    // Near lists per leaf
    {
      const LevelData& t = lv[size_t(L)];
      s.near_off.assign(1, 0);
      for (size_t i = 0; i < nl; ++i) {
        for_neighbors(t, t.codes[i], [&](uint64_t nc) { s.near.push_back(uint32_t(t.find(nc))); });
        s.near_off.push_back(s.near.size());
      }
    }
  }
  timer.mark("near lists");
  // M2L exchange plan (comm_plan.cpp:31-82)
  {
    const int P = s.P;
    std::map<std::pair<int, int>, std::map<uint64_t, std::vector<std::pair<int64_t, int64_t>>>> raw;
    for (int l = s.top; l <= L && P > 1; ++l) {  // one rank: every slice is its own, no items
      const LevelData& t = lv[size_t(l)];
      for (size_t o = 0; o < t.codes.size(); ++o)
        for (uint64_t f = t.far_off[o]; f < t.far_off[o + 1]; ++f) {
          const size_t src = t.far[f];
          const uint64_t packed = (uint64_t(l) << 58) | t.codes[src];
          for (uint64_t a = t.slice_off[o]; a < t.slice_off[o + 1]; ++a) {
            const SliceRec& ro = t.slices[a];
            if (ro.size() == 0) continue;
            for (uint64_t b = t.slice_off[src]; b < t.slice_off[src + 1]; ++b) {
              const SliceRec& ss = t.slices[b];
              if (ss.size() == 0 || ss.rank == ro.rank) continue;
              int64_t lo2 = std::max(ro.begin, ss.begin), hi2 = std::min(ro.end, ss.end);
              if (lo2 >= hi2) continue;
              raw[{int(ss.rank), int(ro.rank)}][packed].emplace_back(lo2, hi2);
            }
          }
        }
    }
    (void)P;
    for (auto& [pair, per_node] : raw) {
      PairPlanRec pp;
      pp.src = pair.first;
      pp.dst = pair.second;
      for (auto& [packed, ranges] : per_node) {
        std::sort(ranges.begin(), ranges.end());
        std::vector<std::pair<int64_t, int64_t>> merged;
        for (auto& r : ranges) {
          if (!merged.empty() && r.first <= merged.back().second)
            merged.back().second = std::max(merged.back().second, r.second);
          else
            merged.push_back(r);
        }
        const int l = int(packed >> 58);
        const uint64_t idx = uint64_t(lv[size_t(l)].find(packed & kCodeMask));
        for (auto& r : merged) pp.items.push_back({l, idx, r.first, r.second});
      }
      s.m2l_plan.push_back(std::move(pp));
    }
  }
  timer.mark("m2l plan");
  // Near ghost plan (comm_plan.cpp:84-109)
  {
    const int P = s.P;
    std::vector<std::set<uint64_t>> needed(size_t(P) * size_t(P));
    for (int w = 0; w < P; ++w)
      for (uint64_t li = s.rank_begin[size_t(w)]; li < s.rank_end[size_t(w)]; ++li)
        for (uint64_t z = s.near_off[li]; z < s.near_off[li + 1]; ++z) {
          uint64_t ni = s.near[z];
          int qq = s.rank_of_leaf(ni);
          if (qq != w) needed[size_t(qq * P + w)].insert(ni);
        }
    s.near_send.resize(size_t(P) * size_t(P));
    for (size_t i = 0; i < needed.size(); ++i)
      s.near_send[i].assign(needed[i].begin(), needed[i].end());
  }
  timer.mark("near plan");
  return s;
}

RankPlan build_rank_plan(const Setup& s, int r) {
  if (r < 0 || r >= s.P) throw std::out_of_range("build_rank_plan: bad rank");
  const int L = s.L, P = s.P;
  RankPlan rp;
  rp.rank = r;
  rp.held.assign(size_t(L + 1), {});
  rp.child_off.assign(size_t(L + 1), {});
  rp.children.assign(size_t(L + 1), {});
  rp.halo.assign(size_t(L + 1), {});
  for (int k = 0; k < 4; ++k) {
    rp.send[k].assign(size_t(P), {});
    rp.recv[k].assign(size_t(P), {});
  }
  std::vector<std::vector<uint8_t>> is_held(size_t(L + 1));
  for (int l = s.top; l <= L; ++l) {
    const LevelData& t = s.levels[size_t(l)];
    is_held[size_t(l)].assign(t.num_nodes(), 0);
    for (size_t i = 0; i < t.num_nodes(); ++i)
      if (t.first_user[i] <= r && r <= t.last_user[i]) {
        rp.held[size_t(l)].push_back(int(i));
        is_held[size_t(l)][i] = 1;
      }
  }
  for (int l = s.top; l < L; ++l) {
    const LevelData& t = s.levels[size_t(l)];
    auto& co = rp.child_off[size_t(l)];
    auto& ch = rp.children[size_t(l)];
    co.assign(1, 0);
    for (int p : rp.held[size_t(l)]) {
      for (uint64_t z = t.child_off[size_t(p)]; z < t.child_off[size_t(p) + 1]; ++z)
        if (is_held[size_t(l + 1)][t.children[z]]) ch.push_back(int(t.children[z]));
      co.push_back(int(ch.size()));
    }
  }
  rp.child_off[size_t(L)].assign(rp.held[size_t(L)].size() + 1, 0);
  // kinds 2 and 3: plural nodes r holds, against each other user's slice
  for (int l = s.top; l <= L; ++l) {
    const LevelData& t = s.levels[size_t(l)];
    for (int n : rp.held[size_t(l)]) {
      if (!t.plural[size_t(n)]) continue;
      const SliceRec* mine = nullptr;
      for (uint64_t z = t.slice_off[size_t(n)]; z < t.slice_off[size_t(n) + 1]; ++z)
        if (t.slices[z].rank == r && t.slices[z].size() > 0) mine = &t.slices[z];
      for (uint64_t z = t.slice_off[size_t(n)]; z < t.slice_off[size_t(n) + 1]; ++z) {
        const SliceRec& sl = t.slices[z];
        if (sl.rank == r || sl.size() == 0) continue;
        rp.send[kXReduce][size_t(sl.rank)].push_back({l, n, sl.begin, sl.end});  // my partial of q's rows
        rp.recv[kXGather][size_t(sl.rank)].push_back({l, n, sl.begin, sl.end});  // q's final rows
      }
      if (mine)
        for (int q = t.first_user[size_t(n)]; q <= t.last_user[size_t(n)]; ++q) {
          if (q == r) continue;
          rp.recv[kXReduce][size_t(q)].push_back({l, n, mine->begin, mine->end});
          rp.send[kXGather][size_t(q)].push_back({l, n, mine->begin, mine->end});
        }
    }
  }
  // kind 0: the reference's M2L CommPlan (comm_plan.cpp:31-82), items in
  // (level, Morton, begin) order
  std::vector<std::vector<uint8_t>> in_halo(size_t(L + 1));
  for (int l = s.top; l <= L; ++l) in_halo[size_t(l)].assign(s.levels[size_t(l)].num_nodes(), 0);
  for (const PairPlanRec& pp : s.m2l_plan) {
    if (pp.src != r && pp.dst != r) continue;
    auto& dst = pp.src == r ? rp.send[kXHalo][size_t(pp.dst)] : rp.recv[kXHalo][size_t(pp.src)];
    for (const PlanItemRec& it : pp.items) {
      dst.push_back({it.level, int(it.node), it.begin, it.end});
      if (pp.dst == r && !is_held[size_t(it.level)][it.node]) in_halo[size_t(it.level)][it.node] = 1;
    }
  }
  for (int l = s.top; l <= L; ++l)
    for (size_t i = 0; i < in_halo[size_t(l)].size(); ++i)
      if (in_halo[size_t(l)][i]) rp.halo[size_t(l)].push_back(int(i));
  return rp;
}

namespace {
template <class T>
std::vector<unsigned char> bytes_of(const std::vector<T>& v) {
  std::vector<unsigned char> b(v.size() * sizeof(T));
  if (!v.empty()) std::memcpy(b.data(), v.data(), b.size());
  return b;
}
}  // namespace

std::vector<unsigned char> setup_array(const Setup& s, const std::string& name) {
  const int L = s.L;
  if (name == "meta_i64")
    return bytes_of(std::vector<int64_t>{L, s.top, s.d_class, int64_t(s.n),
                                         int64_t(s.num_leaves()), s.P});
  if (name == "meta_f64")
    return bytes_of(std::vector<double>{s.root_side, s.leaf_side, s.corner[0], s.corner[1],
                                        s.corner[2], s.k});
  if (name == "particles") {
    std::vector<double> p(5 * s.n);
    for (size_t i = 0; i < s.n; ++i) {
      p[5 * i] = s.xyz[3 * i];
      p[5 * i + 1] = s.xyz[3 * i + 1];
      p[5 * i + 2] = s.xyz[3 * i + 2];
      p[5 * i + 3] = s.q[2 * i];
      p[5 * i + 4] = s.q[2 * i + 1];
    }
    return bytes_of(p);
  }
  if (name == "original_index") return bytes_of(s.original_index);
  if (name == "leaf_codes") return bytes_of(s.leaf_codes);
  if (name == "leaf_start") return bytes_of(s.leaf_start);
  if (name == "rank_ranges") {
    std::vector<uint64_t> rr;
    for (int r = 0; r < s.P; ++r) {
      rr.push_back(s.rank_begin[size_t(r)]);
      rr.push_back(s.rank_end[size_t(r)]);
    }
    return bytes_of(rr);
  }
  if (name == "splitters") return bytes_of(s.splitters);
  if (name == "near_off") return bytes_of(s.near_off);
  if (name == "near") {
    std::vector<uint64_t> c;
    for (uint32_t i : s.near) c.push_back(s.leaf_codes[i]);
    return bytes_of(c);
  }
  if (name == "m2l_plan") {
    std::vector<int64_t> v;
    for (const auto& pp : s.m2l_plan) {
      v.push_back(pp.src);
      v.push_back(pp.dst);
      v.push_back(int64_t(pp.items.size()));
      for (const auto& it : pp.items) {
        v.push_back(it.level);
        v.push_back(int64_t(s.levels[size_t(it.level)].codes[it.node]));
        v.push_back(it.begin);
        v.push_back(it.end);
      }
    }
    return bytes_of(v);
  }
  if (name == "near_plan") {
    std::vector<int64_t> v;
    for (const auto& lst : s.near_send) {
      v.push_back(int64_t(lst.size()));
      for (uint64_t li : lst) v.push_back(int64_t(li));
    }
    return bytes_of(v);
  }
  if (name.size() > 2 && name[0] == 'R') {
    // R<r>.<field>[.L<l> | .<peer>]: per-rank plans (build_rank_plan)
    const size_t d1 = name.find('.');
    if (d1 != std::string::npos) {
      const int r = std::atoi(name.substr(1, d1 - 1).c_str());
      std::string rest = name.substr(d1 + 1);
      const size_t d2 = rest.find('.');
      const std::string field = rest.substr(0, d2);
      const std::string arg = d2 == std::string::npos ? "" : rest.substr(d2 + 1);
      RankPlan rp = build_rank_plan(s, r);
      auto level_of = [&](const std::string& a) {
        if (a.size() < 2 || a[0] != 'L') throw std::invalid_argument("hfmm_setup_get: bad level in " + name);
        const int l = std::atoi(a.substr(1).c_str());
        if (l < s.top || l > L) throw std::out_of_range("hfmm_setup_get: level not computed");
        return size_t(l);
      };
      auto rows = [&](const std::vector<RowItem>& v) {
        std::vector<int64_t> o;
        for (const RowItem& it : v) {
          o.push_back(it.level);
          o.push_back(it.node);
          o.push_back(it.begin);
          o.push_back(it.end);
        }
        return bytes_of(o);
      };
      if (field == "held") return bytes_of(rp.held[level_of(arg)]);
      if (field == "child_off") return bytes_of(rp.child_off[level_of(arg)]);
      if (field == "children") return bytes_of(rp.children[level_of(arg)]);
      if (field == "halo") return bytes_of(rp.halo[level_of(arg)]);
      // send<k>.<q> / recv<k>.<q>: exchange kind k items with peer q, int64
      // quadruples (level, node, begin, end)
      if ((field.rfind("send", 0) == 0 || field.rfind("recv", 0) == 0) && field.size() == 5) {
        const int kind = field[4] - '0';
        const int q = std::atoi(arg.c_str());
        if (kind != kXHalo && kind != kXReduce && kind != kXGather)
          throw std::invalid_argument("hfmm_setup_get: bad exchange kind in " + name);
        if (q < 0 || q >= s.P) throw std::out_of_range("hfmm_setup_get: bad peer");
        return rows(field[0] == 's' ? rp.send[kind][size_t(q)] : rp.recv[kind][size_t(q)]);
      }
    }
  }
  if (name.size() > 2 && name[0] == 'L') {
    size_t dot = name.find('.');
    if (dot != std::string::npos) {
      int l = std::atoi(name.substr(1, dot - 1).c_str());
      std::string f = name.substr(dot + 1);
      if (l >= s.top && l <= L) {
        const LevelData& t = s.levels[size_t(l)];
        if (f == "sampling") return bytes_of(std::vector<int64_t>{t.trunc, t.nt, t.np});
        if (f == "theta_weight") return bytes_of(t.theta_w);
        if (f == "phi_weight") return bytes_of(std::vector<double>{t.phi_w});
        if (f == "codes") return bytes_of(t.codes);
        if (f == "centers") return bytes_of(t.centers);
        if (f == "users") {
          std::vector<int64_t> u;
          for (size_t i = 0; i < t.codes.size(); ++i) {
            u.push_back(t.first_user[i]);
            u.push_back(t.last_user[i]);
            u.push_back(t.plural[i]);
          }
          return bytes_of(u);
        }
        if (f == "slices_off") return bytes_of(t.slice_off);
        if (f == "slices") {
          std::vector<int64_t> v;
          for (auto& sl : t.slices) {
            v.push_back(sl.rank);
            v.push_back(sl.begin);
            v.push_back(sl.end);
          }
          return bytes_of(v);
        }
        if (f == "child_off") return bytes_of(t.child_off);
        if (f == "children") return bytes_of(t.children);
        if (f == "interp_off") return bytes_of(t.interp_off);
        if (f == "interp") return bytes_of(t.interp);
        if (f == "far_off") return bytes_of(t.far_off);
        if (f == "far") {
          std::vector<uint64_t> c;
          for (uint32_t i : t.far) c.push_back(t.codes[i]);
          return bytes_of(c);
        }
      }
    }
  }
  throw std::invalid_argument("hfmm_setup_get: unknown array " + name);
}

}  // namespace hfmm_b200
