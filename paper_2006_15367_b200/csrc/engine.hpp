// Device engine: one logical rank of the MLFMA evaluation on one B200.
// Replaces RankEngine (/root/reference/proj/include/hfmm/traversal.hpp:125-156).
#ifndef HFMM_B200_ENGINE_HPP
#define HFMM_B200_ENGINE_HPP

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

#include "setup.hpp"

namespace hfmm_b200 {

// Per-level device tables.  Expansions are dense [node][theta][phi]
// complex128 in Morton order (the reference keeps one std::vector per node
// in a hash map, traversal.hpp:151-152).
struct DevLevel {
  int level = 0, nt = 0, np = 0, trunc = 0;
  int64_t S = 0;
  int n_nodes = 0;
  int n_rows = 0;             // expansion rows allocated (one logical rank: n_nodes; see Engine::rows_)
  double side = 0.0;
  double* dir = nullptr;      // S*3 sample directions (sphere_grid.cpp:31-37)
  double* wq = nullptr;       // S quadrature weights theta_w[i]*phi_w
  double* centers = nullptr;  // 3*n_nodes
  double2* mp = nullptr;      // n_nodes*S multipole samples
  double2* loc = nullptr;     // n_nodes*S local samples
  int64_t* far_off = nullptr; // n_nodes+1
  int2* far = nullptr;        // (source node, offset slot)
  int64_t n_far = 0;
  double2* T = nullptr;       // 343*S translation operator samples
  double2* tcoef = nullptr;   // 343*(trunc+1) Legendre-series coefficients
  uint8_t* slot_used = nullptr;
  int G = 0;                  // cells per axis = 2^(level-1)
  int* lookup = nullptr;      // dense row-major cell -> node index (-1 empty), dense levels only
  bool dense = false;         // M2L as a stencil over the cell grid (m2l.cuh)
  int* m2l_blk = nullptr;     // distributed mode: observer blocks holding held nodes (dense levels)
  int m2l_nblk = 0;
  int* child_off = nullptr;   // n_nodes+1 (children at level+1)
  int* children = nullptr;
  int* parent = nullptr;      // n_nodes, parent index at level-1 (or -1)
  // As a parent level of level+1:
  double2* shift_up = nullptr;  // 8*S: exp(+i k khat.(c_child - c_parent)) on this grid
  double2* shift_dn = nullptr;  // 8*S: exp(+i k khat.(c_parent - c_child))
  // DMMA M2M / L2L (dmma.cuh): real matrices + rank-1 vectors.  Two-stage large-grid kernels (interp_big.cuh): circles per CTA and smem bytes.
  int big_m2m_cp = 1, big_l2l_cp = 1;
  size_t big_smem[4] = {0, 0, 0, 0};  // m2m phi, m2m theta, l2l theta, l2l phi
  int big_ldn = 0;                    // narrow-row stride of the L2L temp
  int big_rc[2] = {1, 1};             // rows per CTA: m2m phi, l2l phi
  int up_phi[4] = {0, 0, 0, 0}, up_th[4] = {0, 0, 0, 0};  // PassDims {K, N, lda, ldo}
  int dn_th[4] = {0, 0, 0, 0}, dn_phi[4] = {0, 0, 0, 0};
  double* up_phi_B = nullptr;
  double* up_phi_v = nullptr;
  double* up_th_B = nullptr;
  double* up_th_v = nullptr;
  double* dn_th_B = nullptr;
  double* dn_th_v = nullptr;
  double* dn_phi_B = nullptr;
  double* dn_phi_v = nullptr;
  // even / odd theta passes (fused and compile-time-shaped kernels; interp.hpp)
  double* up_phi_Bf = nullptr;  // phi matrix with the (e, o) fold in its columns
  double* up_th_Be = nullptr;   // [Be ; Bo]
  double* up_th_ve = nullptr;
  double* dn_th_Be = nullptr;
  double* dn_th_ve = nullptr;
  double* dn_phi_Bu = nullptr;  // phi matrix with the (e, o) unfold in its rows
  double* dn_phi_vu = nullptr;
};

// Per-rank lists for one level acting as parent (distributed mode).
struct RankLevel {
  int n_par = 0;
  int* plist = nullptr;      // held parents (global node indices)
  int* child_off = nullptr;  // CSR over plist
  int* children = nullptr;   // held children (global indices at level + 1)
  int64_t n_children = 0;    // entries of children
};

// One direction of a row exchange (kinds 0, 2, 3 of setup.hpp) with one
// peer: per level, device items {node, begin, length, offset} with offsets
// in double2 from the level's start in the buffer; levels are laid out
// level-major in the peer buffer.
struct RowXfer {
  std::vector<int64_t*> items;  // [level]
  std::vector<int> cnt;         // [level]
  std::vector<int64_t> len;     // [level] double2 elements
  std::vector<int64_t> maxlen;  // [level] longest item (grid sizing)
  int64_t total = 0;            // double2 elements over all levels
};

// Static exchange plan with one peer (distributed mode).
struct PeerPlan {
  RowXfer send[4], recv[4];  // by exchange kind (index 1 = ghosts: below)
  // ghost particles (x, y, z, re, im) by sorted particle index
  int64_t* gh_send_idx = nullptr;
  int64_t* gh_recv_idx = nullptr;
  int64_t n_gh_send = 0, n_gh_recv = 0;
};

class Engine {
 public:
  // The engine shares ownership of the setup, so a C caller may destroy its
  // hfmm_setup handle before the engine (include/hfmm_gpu.h).
  Engine(std::shared_ptr<const Setup> s, int device, int rank);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  // charges in input order (n*2) -> device sorted order
  void set_charges(const double* q_input_order);
  void run_phase(int phase);
  // Full evaluation from the current device charges; fills ms[8].
  void evaluate(double* ms);
  // Device-resident: sorted charges in, sorted potentials out.
  void evaluate_device(const double* d_q_sorted, double* d_pot_sorted, cudaStream_t st);
  // e2e: host charges (input order) -> host potentials (input order).
  void evaluate_host(const double* q_in, double* pot_out, double* ms);

  void get_expansion(int kind, int level, double* out, size_t cap_doubles);
  // Distributed mode (P > 1): exchange buffers are driven by the caller
  // (torch.distributed over NCCL); kinds as in setup.hpp (0 M2L halo,
  // 1 ghosts, 2 plural multipole reduce-scatter, 3 plural local gather).
  // level -1 = all levels, laid out level-major (kinds 0, 2, 3).
  void exchange_sizes(int kind, int peer, int level, int64_t* send_doubles, int64_t* recv_doubles) const;
  void pack(int kind, int peer, int level, double* d_buf);
  void unpack(int kind, int peer, int level, const double* d_buf);
  // One level of M2L (observer level) or L2L (parent level) after the T build.
  void run_level(int phase, int level);
  void set_stream(cudaStream_t st);
  void synchronize();
  void load_charges_device(const double* d_q_sorted);
  void store_potentials_device(double* d_pot_sorted);
  int64_t launch_count() const { return launches_; }
  void set_overlap(bool on) { overlap_ = on; }
  int64_t particle_begin() const { return part_b_; }
  int64_t particle_end() const { return part_e_; }
  void get_potentials_sorted(double* out, size_t cap_doubles);
  // This rank's particle range of the sorted potentials into a host array of
  // n*2 doubles (same offsets; synchronous).
  void store_potentials_host(double* host_sorted);
  cudaStream_t stream() const { return st_; }
  int device() const { return dev_; }
  int64_t launches() const { return launches_; }
  // Per-phase ms of the last evaluation (events on its stream), [0] T build .. [7] total.
  void last_timing(double* ms, int64_t* launches);

 private:
  void upload();
  void setup_interp(DevLevel& P, const DevLevel& C, const LevelData& tp, const LevelData& tc);
  void build_T();
  void phase_c2m();
  void phase_m2m();
  void phase_m2l(int lo = -1, int hi = -1);  // levels lo..hi (default all)
  void phase_l2l(int lo = -1, int hi = -1);  // parent levels lo..hi (default all)
  void phase_l2t();
  void phase_near();
  template <class T>
  T* alloc(size_t count);
  template <class T>
  T* upload_vec(const std::vector<T>& v);

  std::shared_ptr<const Setup> keep_;
  const Setup& s_;
  int dev_ = 0, rank_ = 0;
  int sms_ = 148;  // multiprocessors of dev_
  cudaStream_t st_ = nullptr;
  bool owns_stream_ = true;
  std::vector<DevLevel> lv_;
  std::vector<uint8_t*> oct_;  // per level: child octant (code & 7) of each node
  std::vector<const int4*> pdesc_;  // per parent level: parent descriptors (interp_rb.cuh:PDesc)
  std::vector<void*> allocs_;
  int64_t launches_ = 0;
  // test hooks (HFMM_NO_RB, HFMM_NO_RBL, HFMM_NO_QUAD; tests/test_gpu_paths.py)
  bool hook_no_rb_ = false, hook_no_rbl_ = false, hook_no_quad_ = false;
  static constexpr int kBigThreads = 256;  // block size of the two-stage large-grid kernels
  static constexpr int kPhiCtas = 2;       // persistent CTAs per SM of the streaming phi passes
  size_t tmp_need_ = 0;    // temp elements required by the large-level kernels
  // particles (sorted)
  double* d_x = nullptr;
  double* d_y = nullptr;
  double* d_z = nullptr;
  double2* d_q = nullptr;
  double2* d_pot = nullptr;      // sorted potentials
  double2* d_q_in = nullptr;     // input-order staging
  double2* d_pot_in = nullptr;   // input-order staging
  int64_t* d_orig = nullptr;     // sorted -> input index
  int64_t* d_leaf_start = nullptr;
  int64_t* d_near_off = nullptr;
  int* d_near = nullptr;
  int* d_tiny_leaves_ = nullptr;   // own leaves with <= 8 particles (warp per leaf)
  int* d_small_leaves_ = nullptr;  // own leaves with 9..32 particles
  int* d_dense_leaves_ = nullptr;
  int n_small_ = 0, n_dense_ = 0, n_tiny_ = 0;
  int* d_plain_off_ = nullptr;  // symmetric P2P lists over dense own leaves
  int* d_plain_ = nullptr;
  int* d_sym_off_ = nullptr;
  int* d_sym_ = nullptr;
  int64_t* d_sym_scr_ = nullptr;
  int* d_in_off_ = nullptr;
  int64_t* d_in_scr_ = nullptr;
  double2* d_p2p_scratch_ = nullptr;
  int2* d_p2p_items_ = nullptr;  // k_p2p_sym2 work items {dense leaf idx, pass}, grouped by slots per lane
  int64_t* d_sym_rows_ = nullptr;
  int p2p_items_b_[4] = {0, 0, 0, 0}, p2p_items_n_[4] = {0, 0, 0, 0};
  int* d_sparse_leaves_ = nullptr;  // own leaves with <= 32 particles (L2T)
  int n_sparse_ = 0;
  bool m2l_seq_ = false;                     // leaf M2L inside the chain (autotuned choice)
  bool tune_done_ = false;                   // leaf-M2L placement autotune (evaluate_device)
  int tune_evals_ = 0;
  float tune_ms_[2] = {0.f, 0.f};
  double2* d_ptab_ = nullptr;  // near-field phase table (green_tab), nullptr: sincos polynomials
  int ptab_max_ = 0;
  double2* d_ltab_ = nullptr;  // leaf phase table (sincos_l), centred; nullptr: polynomials
  int ltab_half_ = 0;
  double2* d_tmp = nullptr;  // interpolation temporaries
  size_t tmp_elems_ = 0;
  int64_t leaf_b_ = 0, leaf_e_ = 0;  // owned leaf range
  int64_t part_b_ = 0, part_e_ = 0;  // owned particle range
  cudaEvent_t ev_[8] = {};
  // near field on a side stream, overlapped with the far-field chain
  cudaStream_t st2_ = nullptr;
  cudaStream_t st_cp_ = nullptr;  // host charges in (evaluate_host), beside the T build
  cudaEvent_t ev_q_ = nullptr;
  cudaEvent_t ev_cp_order_ = nullptr;  // st_ -> st_cp_: the host-charge copy waits for queued work
  bool q_pending_ = false;
  // evaluate_device overlap: far chain (high priority) + leaf M2L (low priority)
  cudaStream_t st_hi_ = nullptr, st_lo_ = nullptr;
  cudaEvent_t ev_ofork_ = nullptr, ev_ojoin_ = nullptr, ev_c2m_ = nullptr, ev_m2l_leaf_ = nullptr;
  bool overlap_ = true, overlapped_ = false;
  cudaEvent_t ev_lf0_ = nullptr, ev_lf1_ = nullptr, ev_la_ = nullptr, ev_lb_ = nullptr;  // timing in overlap mode
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr, ev_near0_ = nullptr, ev_near1_ = nullptr;
  double2* d_pot_near = nullptr;
  bool near_started_ = false;
  void near_start();
  // distributed mode
  bool dist_ = false;
  std::vector<RankLevel> rl_;               // [level as parent]
  std::vector<int*> held_;                  // [level] held nodes (distributed mode)
  std::vector<int> held_cnt_;
  std::vector<PeerPlan> peers_;             // [peer]
  void upload_rank_plan();
  // Compact per-rank storage (distributed mode): the expansions of level l
  // are rows [held nodes (sorted) | halo nodes received through the M2L plan
  // | one zero row]; rows_[l][node] = row or -1.  One logical rank: rows =
  // nodes (rows_ empty).
  std::unique_ptr<RankPlan> rp_;
  std::vector<std::vector<int>> rows_;
  int row(int l, int node) const { return rows_.empty() ? node : rows_[size_t(l)][size_t(node)]; }
  int64_t last_launches_ = 0;
  bool timed_ = false;
};

// Device O(N M) direct sum (kernel.cpp:16-41) for the accuracy checks.
void direct_sum(const double* positions, const double* charges, size_t n, const int64_t* obs,
                size_t m, double k, int device, double* pot_out);

}  // namespace hfmm_b200

#endif
