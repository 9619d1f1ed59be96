// Host-side MLFMA setup: Morton keys, octree levels, partition, sample
// slices, interaction lists and exchange plans -- a from-scratch flat-array
// rewrite of the reference's build_setup (/root/reference/proj/src/traversal.cpp:66-238)
// whose outputs are bit-exact with it (tests/test_setup_parity.py).
//
// Layout choices (B200-first): every per-node table is a dense array in
// Morton order per level; lists are CSR over node indices, not hash maps
// of keys, so the device upload is a straight memcpy.
#ifndef HFMM_B200_SETUP_HPP
#define HFMM_B200_SETUP_HPP

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "hfmm_gpu.h"

namespace hfmm_b200 {

struct SliceRec {
  int64_t rank, begin, end;  // samples [begin, end) of the node, held by rank
  int64_t size() const { return end - begin; }
};

// One computed tree level (top_level .. L), nodes in Morton order.
struct LevelData {
  int level = 0;
  int trunc = 0;               // L_t, sphere_grid.cpp:13-23
  int64_t nt = 0, np = 0;      // n_theta = n_phi = 2 L_t + 2
  std::vector<double> theta_w; // Fejer weights, sphere_grid.cpp:52-70
  double phi_w = 0.0;
  double side = 0.0;

  std::vector<uint64_t> codes;
  std::vector<double> centers;  // 3 per node
  std::vector<int32_t> first_user, last_user;
  std::vector<uint8_t> plural;
  std::vector<uint64_t> slice_off;  // CSR into slices
  std::vector<SliceRec> slices;
  std::vector<uint64_t> child_off;  // CSR into children (indices at level+1)
  std::vector<uint64_t> children;
  std::vector<uint64_t> interp_off;  // CSR: per plural node {nt, np, splits...}
  std::vector<uint64_t> interp;
  std::vector<uint64_t> far_off;  // CSR: far list as same-level node indices
  std::vector<uint32_t> far;

  int64_t samples() const { return nt * np; }
  size_t num_nodes() const { return codes.size(); }
  // Index of the node with this code, or -1.
  int64_t find(uint64_t code) const;
  std::vector<int64_t> dense_lookup;  // code -> index (levels with <= 2^27 cells)
};

struct PlanItemRec {
  int level;
  uint64_t node;  // node index at `level`
  int64_t begin, end;
};
struct PairPlanRec {
  int src = 0, dst = 0;
  std::vector<PlanItemRec> items;
};

struct Setup {
  hfmm_run_config cfg{};
  double k = 0.0;  // 2 pi / lambda
  int L = 1, top = 1, d_class = 3;
  double root_side = 1.0, leaf_side = 1.0;
  double corner[3] = {0, 0, 0};

  size_t n = 0;
  std::vector<double> xyz;  // sorted, 3 per particle
  std::vector<double> q;    // sorted, 2 per particle
  std::vector<uint64_t> original_index;  // sorted position -> input position

  std::vector<uint64_t> leaf_codes;
  std::vector<uint64_t> leaf_start;  // n_leaves + 1
  int P = 1;
  std::vector<uint64_t> rank_begin, rank_end;  // leaf index ranges per rank
  std::vector<uint64_t> splitters;             // packed keys

  std::vector<LevelData> levels;  // index = level; valid top..L
  std::vector<uint64_t> near_off;  // per leaf, CSR
  std::vector<uint32_t> near;      // leaf indices

  std::vector<PairPlanRec> m2l_plan;
  std::vector<std::vector<uint64_t>> near_send;  // [q*P + w] leaf indices q sends w

  size_t num_leaves() const { return leaf_codes.size(); }
  int rank_of_leaf(uint64_t li) const;
  double box_side(int level) const {
    return root_side / double(uint64_t(1) << (level - 1));
  }
};

// Per-rank evaluation plan for one process per GPU.
// Rank r "holds" every node whose leaf range meets its Morton leaf range
// (first_user <= r <= last_user).  The upward pass runs on held nodes and
// yields PARTIAL multipoles (M2M is linear); plural (shared) nodes are then
// SLICED: every user keeps the full multipole on its own theta-row slice
// (assign_sample_slices, tree.cpp:180-239) after a reduce-scatter among the
// node's users.  M2L runs per observer slice and receives the missing source
// rows through the reference's M2L CommPlan (comm_plan.cpp:31-82); the
// downward pass gathers the plural parents' local slices among their users
// before anterpolating.  Ghost particles follow the reference's near plan
// (comm_plan.cpp:84-109).
//
// Exchange kinds (rows = flat sample ranges [begin, end) of one node):
//   0  M2L halo: the reference CommPlan items, overwrite (per level)
//   1  ghost particles (x, y, z, re, im)
//   2  plural multipole reduce-scatter: partial rows of the peer's slice, add
//   3  plural local all-gather: own slice rows to the other users, overwrite
struct RowItem {
  int level;
  int node;
  int64_t begin, end;
};
enum ExchangeKind { kXHalo = 0, kXGhost = 1, kXReduce = 2, kXGather = 3 };
struct RankPlan {
  int rank = 0;
  std::vector<std::vector<int>> held;       // [level] held node indices, sorted
  std::vector<std::vector<int>> child_off;  // [level] CSR over held[level] (held children only)
  std::vector<std::vector<int>> children;   // [level] indices at level + 1
  std::vector<std::vector<int>> halo;       // [level] nodes received through kind 0 that r does not hold
  // per kind (0, 2, 3) and peer q: items r sends q / receives from q, (level, node, begin) order
  std::vector<std::vector<RowItem>> send[4], recv[4];
};
RankPlan build_rank_plan(const struct Setup& s, int r);

// Replicates build_setup; throws the same std exception types.
Setup build_setup(const double* xyz, const double* q, size_t n,
                  const hfmm_run_config& cfg);

// Device parts of the setup (setup_gpu.cu), used when cfg.setup_device = 1.
void device_keys_sort(const double* xyz, const double* q, size_t n, const double corner[3], double root_side,
                      double inv, uint32_t cells, int L, std::vector<uint64_t>& sorted_keys,
                      std::vector<uint64_t>& order, std::vector<double>& xyz_s, std::vector<double>& q_s);
void device_lists(Setup& s);

// Import of an existing setup from the named flat arrays of setup_array()
// (setup_import.cpp): begin, put every array, end (validates; consumes).
struct SetupImport;
SetupImport* setup_import_begin(const hfmm_run_config& cfg);
void setup_import_put(SetupImport* im, const std::string& name, const void* data, size_t nbytes);
Setup setup_import_end(SetupImport* im);
void setup_import_abort(SetupImport* im);

// Flat dump under the names used by oracle/ref_driver.cpp.
std::vector<unsigned char> setup_array(const Setup& s, const std::string& name);

// Host numerics shared with the device upload.
int truncation_order(double diameter, double k, double digits);
void fejer_weights(int64_t nt, std::vector<double>& w);

}  // namespace hfmm_b200

#endif
