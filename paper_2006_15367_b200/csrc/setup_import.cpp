// Setup import: builds the engine's Setup from a caller's existing
// GlobalSetup (traversal.hpp:93-118) instead of re-running build_setup.
//
// The caller hands over the same named flat arrays hfmm_setup_get() returns
// (one put per array, any order), so a reference-side binding flattens its
// GlobalSetup once and the engine never re-sorts or rebuilds lists
// (INTEGRATION.md).  import_end() validates every size, offset table and
// index, resolves Morton codes to node indices and builds the lookups; any
// inconsistency throws std::invalid_argument / std::out_of_range, as
// build_setup does for bad inputs.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "setup.hpp"

namespace hfmm_b200 {

namespace {

template <class T>
std::vector<T> as_vec(const void* data, size_t nbytes, const std::string& name) {
  if (nbytes % sizeof(T) != 0) throw std::invalid_argument("hfmm_setup_import: bad byte size for " + name);
  std::vector<T> v(nbytes / sizeof(T));
  if (nbytes) std::memcpy(v.data(), data, nbytes);
  return v;
}

void need_size(size_t have, size_t want, const std::string& name) {
  if (have != want)
    throw std::invalid_argument("hfmm_setup_import: " + name + " has " + std::to_string(have) + " entries, expected " +
                                std::to_string(want));
}

void check_csr(const std::vector<uint64_t>& off, size_t rows, size_t total, const std::string& name) {
  need_size(off.size(), rows + 1, name);
  if (off.front() != 0 || off.back() != total) throw std::invalid_argument("hfmm_setup_import: " + name + " ends");
  for (size_t i = 0; i + 1 < off.size(); ++i)
    if (off[i] > off[i + 1]) throw std::invalid_argument("hfmm_setup_import: " + name + " not monotone");
}

}  // namespace

struct SetupImport {
  Setup s;
  std::map<std::string, std::vector<unsigned char>> raw;
};

SetupImport* setup_import_begin(const hfmm_run_config& cfg) {
  auto* im = new SetupImport;
  im->s.cfg = cfg;
  return im;
}

void setup_import_put(SetupImport* im, const std::string& name, const void* data, size_t nbytes) {
  if (nbytes && !data) throw std::invalid_argument("hfmm_setup_import_put: null data for " + name);
  auto& dst = im->raw[name];
  dst.resize(nbytes);
  if (nbytes) std::memcpy(dst.data(), data, nbytes);
}

Setup setup_import_end(SetupImport* im) {
  Setup& s = im->s;
  auto get = [&](const std::string& name) -> const std::vector<unsigned char>& {
    auto it = im->raw.find(name);
    if (it == im->raw.end()) throw std::invalid_argument("hfmm_setup_import: missing array " + name);
    return it->second;
  };
  auto vec = [&](const std::string& name, auto tag) {
    using T = decltype(tag);
    const auto& b = get(name);
    return as_vec<T>(b.data(), b.size(), name);
  };
  const auto mi = vec("meta_i64", int64_t{});
  need_size(mi.size(), 6, "meta_i64");
  s.L = int(mi[0]);
  s.top = int(mi[1]);
  s.d_class = int(mi[2]);
  s.n = size_t(mi[3]);
  const size_t nleaves = size_t(mi[4]);
  s.P = int(mi[5]);
  if (s.L < 1 || s.L > 21 || s.top < 1 || s.top > s.L || s.n == 0 || nleaves == 0 || s.P < 1)
    throw std::invalid_argument("hfmm_setup_import: bad meta_i64");
  if (s.P != s.cfg.num_ranks) throw std::invalid_argument("hfmm_setup_import: num_ranks differs from the partition");
  const auto mf = vec("meta_f64", double{});
  need_size(mf.size(), 6, "meta_f64");
  s.root_side = mf[0];
  s.leaf_side = mf[1];
  s.corner[0] = mf[2];
  s.corner[1] = mf[3];
  s.corner[2] = mf[4];
  s.k = mf[5];
  if (!(s.root_side > 0) || !(s.leaf_side > 0) || !(s.k > 0)) throw std::invalid_argument("hfmm_setup_import: bad meta_f64");

  const auto parts = vec("particles", double{});
  need_size(parts.size(), 5 * s.n, "particles");
  s.xyz.resize(3 * s.n);
  s.q.resize(2 * s.n);
  for (size_t i = 0; i < s.n; ++i) {
    for (int a = 0; a < 3; ++a) s.xyz[3 * i + size_t(a)] = parts[5 * i + size_t(a)];
    s.q[2 * i] = parts[5 * i + 3];
    s.q[2 * i + 1] = parts[5 * i + 4];
  }
  s.original_index = vec("original_index", uint64_t{});
  need_size(s.original_index.size(), s.n, "original_index");
  {
    std::vector<uint8_t> seen(s.n, 0);
    for (uint64_t v : s.original_index) {
      if (v >= s.n || seen[v]) throw std::invalid_argument("hfmm_setup_import: original_index is not a permutation");
      seen[v] = 1;
    }
  }
  s.leaf_codes = vec("leaf_codes", uint64_t{});
  need_size(s.leaf_codes.size(), nleaves, "leaf_codes");
  for (size_t i = 1; i < nleaves; ++i)
    if (s.leaf_codes[i - 1] >= s.leaf_codes[i]) throw std::invalid_argument("hfmm_setup_import: leaves not Morton-sorted");
  s.leaf_start = vec("leaf_start", uint64_t{});
  check_csr(s.leaf_start, nleaves, s.n, "leaf_start");
  const auto rr = vec("rank_ranges", uint64_t{});
  need_size(rr.size(), 2 * size_t(s.P), "rank_ranges");
  s.rank_begin.resize(size_t(s.P));
  s.rank_end.resize(size_t(s.P));
  for (int r = 0; r < s.P; ++r) {
    s.rank_begin[size_t(r)] = rr[2 * size_t(r)];
    s.rank_end[size_t(r)] = rr[2 * size_t(r) + 1];
    if (s.rank_begin[size_t(r)] > s.rank_end[size_t(r)] || s.rank_end[size_t(r)] > nleaves ||
        (r > 0 && s.rank_begin[size_t(r)] != s.rank_end[size_t(r) - 1]))
      throw std::invalid_argument("hfmm_setup_import: rank_ranges do not tile the leaves");
  }
  if (s.rank_begin.front() != 0 || s.rank_end.back() != nleaves)
    throw std::invalid_argument("hfmm_setup_import: rank_ranges do not tile the leaves");
  s.splitters = vec("splitters", uint64_t{});

  // Levels top..L.
  s.levels.assign(size_t(s.L + 1), LevelData{});
  for (int l = s.top; l <= s.L; ++l) {
    LevelData& t = s.levels[size_t(l)];
    const std::string p = "L" + std::to_string(l) + ".";
    t.level = l;
    t.side = s.box_side(l);
    const auto smp = vec(p + "sampling", int64_t{});
    need_size(smp.size(), 3, p + "sampling");
    t.trunc = int(smp[0]);
    t.nt = smp[1];
    t.np = smp[2];
    if (t.trunc < 0 || t.nt < 2 || t.np < 2) throw std::invalid_argument("hfmm_setup_import: bad " + p + "sampling");
    t.theta_w = vec(p + "theta_weight", double{});
    need_size(t.theta_w.size(), size_t(t.nt), p + "theta_weight");
    const auto pw = vec(p + "phi_weight", double{});
    need_size(pw.size(), 1, p + "phi_weight");
    t.phi_w = pw[0];
    t.codes = vec(p + "codes", uint64_t{});
    const size_t nn = t.codes.size();
    if (nn == 0) throw std::invalid_argument("hfmm_setup_import: empty level " + std::to_string(l));
    for (size_t i = 1; i < nn; ++i)
      if (t.codes[i - 1] >= t.codes[i]) throw std::invalid_argument("hfmm_setup_import: " + p + "codes not sorted");
    if (3 * (l - 1) <= 27) {
      t.dense_lookup.assign(size_t(1) << (3 * (l - 1)), -1);
      for (size_t i = 0; i < nn; ++i) {
        if (t.codes[i] >= t.dense_lookup.size()) throw std::out_of_range("hfmm_setup_import: code outside level");
        t.dense_lookup[t.codes[i]] = int64_t(i);
      }
    }
    t.centers = vec(p + "centers", double{});
    need_size(t.centers.size(), 3 * nn, p + "centers");
    const auto users = vec(p + "users", int64_t{});
    need_size(users.size(), 3 * nn, p + "users");
    t.first_user.resize(nn);
    t.last_user.resize(nn);
    t.plural.resize(nn);
    for (size_t i = 0; i < nn; ++i) {
      t.first_user[i] = int32_t(users[3 * i]);
      t.last_user[i] = int32_t(users[3 * i + 1]);
      t.plural[i] = uint8_t(users[3 * i + 2] != 0);
      if (t.first_user[i] < 0 || t.last_user[i] >= s.P || t.first_user[i] > t.last_user[i] ||
          bool(t.plural[i]) != (t.first_user[i] != t.last_user[i]))
        throw std::invalid_argument("hfmm_setup_import: bad " + p + "users");
    }
    const auto sl = vec(p + "slices", int64_t{});
    if (sl.size() % 3) throw std::invalid_argument("hfmm_setup_import: bad " + p + "slices");
    t.slices.resize(sl.size() / 3);
    for (size_t i = 0; i < t.slices.size(); ++i) {
      t.slices[i] = {sl[3 * i], sl[3 * i + 1], sl[3 * i + 2]};
      if (t.slices[i].begin < 0 || t.slices[i].begin > t.slices[i].end || t.slices[i].end > t.samples() ||
          t.slices[i].rank < 0 || t.slices[i].rank >= s.P)
        throw std::invalid_argument("hfmm_setup_import: bad " + p + "slices");
    }
    t.slice_off = vec(p + "slices_off", uint64_t{});
    check_csr(t.slice_off, nn, t.slices.size(), p + "slices_off");
    t.children = vec(p + "children", uint64_t{});
    t.child_off = vec(p + "child_off", uint64_t{});
    if (l < s.L) check_csr(t.child_off, nn, t.children.size(), p + "child_off");
    t.interp = vec(p + "interp", uint64_t{});
    t.interp_off = vec(p + "interp_off", uint64_t{});
    check_csr(t.interp_off, nn, t.interp.size(), p + "interp_off");
    t.far_off = vec(p + "far_off", uint64_t{});
    const auto far_codes = vec(p + "far", uint64_t{});
    check_csr(t.far_off, nn, far_codes.size(), p + "far_off");
    t.far.resize(far_codes.size());
    for (size_t i = 0; i < far_codes.size(); ++i) {
      const int64_t j = t.find(far_codes[i]);
      if (j < 0) throw std::out_of_range("hfmm_setup_import: far source not in level " + std::to_string(l));
      t.far[i] = uint32_t(j);
    }
  }
  for (int l = s.top; l < s.L; ++l)
    for (uint64_t c : s.levels[size_t(l)].children)
      if (c >= s.levels[size_t(l) + 1].num_nodes()) throw std::out_of_range("hfmm_setup_import: child index");
  need_size(s.levels[size_t(s.L)].num_nodes(), nleaves, "leaf level nodes");

  // Near lists (leaf codes -> leaf indices).
  s.near_off = vec("near_off", uint64_t{});
  const auto near_codes = vec("near", uint64_t{});
  check_csr(s.near_off, nleaves, near_codes.size(), "near_off");
  s.near.resize(near_codes.size());
  for (size_t i = 0; i < near_codes.size(); ++i) {
    auto it = std::lower_bound(s.leaf_codes.begin(), s.leaf_codes.end(), near_codes[i]);
    if (it == s.leaf_codes.end() || *it != near_codes[i]) throw std::out_of_range("hfmm_setup_import: near leaf");
    s.near[i] = uint32_t(it - s.leaf_codes.begin());
  }
  // Plans.
  {
    const auto v = vec("m2l_plan", int64_t{});
    size_t i = 0;
    while (i < v.size()) {
      if (i + 3 > v.size()) throw std::invalid_argument("hfmm_setup_import: truncated m2l_plan");
      PairPlanRec pp;
      pp.src = int(v[i]);
      pp.dst = int(v[i + 1]);
      const size_t cnt = size_t(v[i + 2]);
      i += 3;
      if (pp.src < 0 || pp.src >= s.P || pp.dst < 0 || pp.dst >= s.P || i + 4 * cnt > v.size())
        throw std::invalid_argument("hfmm_setup_import: bad m2l_plan pair");
      for (size_t c = 0; c < cnt; ++c, i += 4) {
        const int l = int(v[i]);
        if (l < s.top || l > s.L) throw std::out_of_range("hfmm_setup_import: m2l_plan level");
        const int64_t node = s.levels[size_t(l)].find(uint64_t(v[i + 1]));
        if (node < 0 || v[i + 2] < 0 || v[i + 2] > v[i + 3] || v[i + 3] > s.levels[size_t(l)].samples())
          throw std::out_of_range("hfmm_setup_import: m2l_plan item");
        pp.items.push_back({l, uint64_t(node), v[i + 2], v[i + 3]});
      }
      s.m2l_plan.push_back(std::move(pp));
    }
  }
  {
    const auto v = vec("near_plan", int64_t{});
    s.near_send.assign(size_t(s.P) * size_t(s.P), {});
    size_t i = 0;
    for (size_t e = 0; e < s.near_send.size(); ++e) {
      if (i >= v.size()) throw std::invalid_argument("hfmm_setup_import: truncated near_plan");
      const size_t cnt = size_t(v[i++]);
      if (i + cnt > v.size()) throw std::invalid_argument("hfmm_setup_import: truncated near_plan");
      for (size_t c = 0; c < cnt; ++c) {
        if (v[i] < 0 || size_t(v[i]) >= nleaves) throw std::out_of_range("hfmm_setup_import: near_plan leaf");
        s.near_send[e].push_back(uint64_t(v[i++]));
      }
    }
    if (i != v.size()) throw std::invalid_argument("hfmm_setup_import: trailing near_plan entries");
  }
  im->raw.clear();
  return std::move(s);
}

void setup_import_abort(SetupImport* im) { delete im; }

}  // namespace hfmm_b200
