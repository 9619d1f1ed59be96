// setup_flat.hpp -- flattens a reference GlobalSetup (traversal.hpp:93-118)
// into the named flat arrays of the B200 C ABI (hfmm_setup_get /
// hfmm_setup_import_put, include/hfmm_gpu.h).  Part of the reference-side
// binding (gpu_eval.cpp); the oracle driver (ref_driver.cpp) uses the same
// code for its setup dumps.  put(name, const std::vector<T>&) receives every
// array once.
#ifndef HFMM_SETUP_FLAT_HPP
#define HFMM_SETUP_FLAT_HPP

#include <cstdint>
#include <string>
#include <vector>

#include "hfmm/traversal.hpp"

namespace hfmm {

template <class Put>
void flatten_setup(const GlobalSetup& s, Put&& put) {
  const int L = s.tree.levels;
  const int P = s.partition.num_ranks;
  put("meta_i64", std::vector<int64_t>{L, s.top_level, s.d_class,
                                         int64_t(s.particles.size()),
                                         int64_t(s.leaves.size()), P});
  put("meta_f64", std::vector<double>{s.tree.root_side, s.tree.leaf_side,
                                        s.tree.root_corner.x, s.tree.root_corner.y,
                                        s.tree.root_corner.z, s.k.k});
  std::vector<double> parts;
  parts.reserve(s.particles.size() * 5);
  for (const Particle& p : s.particles) {
    parts.push_back(p.position.x);
    parts.push_back(p.position.y);
    parts.push_back(p.position.z);
    parts.push_back(p.intensity.real());
    parts.push_back(p.intensity.imag());
  }
  put("particles", parts);
  std::vector<uint64_t> oi(s.original_index.begin(), s.original_index.end());
  put("original_index", oi);
  std::vector<uint64_t> lc, ls;
  for (const MortonKey& k : s.leaves) lc.push_back(k.code);
  for (auto& [b, e] : s.leaf_particles) ls.push_back(b);
  ls.push_back(s.leaf_particles.empty() ? 0 : s.leaf_particles.back().second);
  put("leaf_codes", lc);
  put("leaf_start", ls);
  std::vector<uint64_t> rr, sp;
  for (auto& [b, e] : s.partition.rank_ranges) {
    rr.push_back(b);
    rr.push_back(e);
  }
  for (const MortonKey& k : s.partition.splitters) sp.push_back(k.packed());
  put("rank_ranges", rr);
  put("splitters", sp);

  for (int l = s.top_level; l <= L; ++l) {
    std::string p = "L" + std::to_string(l) + ".";
    const LevelSampling& sm = s.samplings[l];
    put(p + "sampling", std::vector<int64_t>{sm.trunc_order, int64_t(sm.n_theta),
                                               int64_t(sm.n_phi)});
    put(p + "theta_weight", s.quads[l].theta_weight);
    put(p + "phi_weight", std::vector<double>{s.quads[l].phi_weight});
    const LevelTable& t = s.levels[l];
    std::vector<uint64_t> codes, soff{0}, coff{0}, ioff{0}, foff{0}, children, interp, far;
    std::vector<double> centers;
    std::vector<int64_t> users, slices;
    for (const NodeInfo& n : t.nodes) {
      codes.push_back(n.key.code);
      centers.push_back(n.center.x);
      centers.push_back(n.center.y);
      centers.push_back(n.center.z);
      users.push_back(n.first_user);
      users.push_back(n.last_user);
      users.push_back(n.plural ? 1 : 0);
      for (const Slice& sl : n.slices) {
        slices.push_back(sl.rank);
        slices.push_back(int64_t(sl.begin));
        slices.push_back(int64_t(sl.end));
      }
      soff.push_back(slices.size() / 3);
      for (size_t c : n.children) children.push_back(c);
      coff.push_back(children.size());
      if (!n.interp_layout.splits.empty()) {
        interp.push_back(n.interp_layout.n_theta);
        interp.push_back(n.interp_layout.n_phi);
        for (size_t v : n.interp_layout.splits) interp.push_back(v);
      }
      ioff.push_back(interp.size());
      auto it = s.lists.far.find(n.key.packed());
      if (it != s.lists.far.end())
        for (const MortonKey& k : it->second) far.push_back(k.code);
      foff.push_back(far.size());
    }
    put(p + "codes", codes);
    put(p + "centers", centers);
    put(p + "users", users);
    put(p + "slices_off", soff);
    put(p + "slices", slices);
    put(p + "child_off", coff);
    put(p + "children", children);
    put(p + "interp_off", ioff);
    put(p + "interp", interp);
    put(p + "far_off", foff);
    put(p + "far", far);
  }
  std::vector<uint64_t> noff{0}, near;
  for (const MortonKey& k : s.leaves) {
    for (const MortonKey& nk : s.lists.near.at(k.packed())) near.push_back(nk.code);
    noff.push_back(near.size());
  }
  put("near_off", noff);
  put("near", near);
  std::vector<int64_t> plan;
  for (const PairPlan& pp : s.m2l_plan.pairs) {
    plan.push_back(pp.src);
    plan.push_back(pp.dst);
    plan.push_back(int64_t(pp.items.size()));
    for (const PlanItem& it : pp.items) {
      plan.push_back(it.node.level);
      plan.push_back(int64_t(it.node.code));
      plan.push_back(int64_t(it.begin));
      plan.push_back(int64_t(it.end));
    }
  }
  put("m2l_plan", plan);
  std::vector<int64_t> np;
  for (int q = 0; q < P; ++q)
    for (int w = 0; w < P; ++w) {
      const auto& lst = s.near_plan.send_leaves[q][w];
      np.push_back(int64_t(lst.size()));
      for (size_t li : lst) np.push_back(int64_t(li));
    }
  put("near_plan", np);
}

}  // namespace hfmm

#endif
