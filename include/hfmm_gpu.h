/* hfmm_gpu.h -- C ABI of the B200-native MLFMA evaluation engine.
 *
 * Drop-in boundary for the evaluation phase of the reference (hfmm, arXiv
 * 2006.15367).  The reference has no FFI: callers use its C++ API,
 *
 *   GlobalSetup build_setup(const std::vector<Particle>&, const RunConfig&)
 *       /root/reference/proj/include/hfmm/traversal.hpp:120
 *   EvalResult  evaluate_with_setup(const GlobalSetup&)
 *       /root/reference/proj/include/hfmm/traversal.hpp:166
 *   EvalResult  evaluate_potential(const std::vector<Particle>&, const RunConfig&)
 *       /root/reference/proj/include/hfmm/traversal.hpp:163
 *   RankEngine::{c2m_phase,m2m_pass,m2l_pass,l2l_pass,l2o_near_phase},
 *   RankEngine::{multipole,local_expansion}
 *       /root/reference/proj/include/hfmm/traversal.hpp:129-143
 *
 * Every entry point below replaces one of those (cited per function).  Plain
 * pointers and sizes only; the caller owns host arrays (copied in), handles
 * own device buffers, outputs are written into caller buffers.  Every call
 * returns an hfmm_status; the message of the last failure on the calling
 * thread is available from hfmm_last_error().  Status codes mirror the
 * exception types the reference throws (traversal.cpp:42-46, operators.cpp:43-50,
 * kernel.cpp:11, operators.cpp:160), so a C++ wrapper can rethrow the same type.
 *
 * Handles are not thread-safe; use one handle per host thread / device.
 */
#ifndef HFMM_GPU_H
#define HFMM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum hfmm_status {
  HFMM_OK = 0,
  HFMM_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  HFMM_ERR_OUT_OF_RANGE = 2,     /* std::out_of_range     */
  HFMM_ERR_DOMAIN = 3,           /* std::domain_error     */
  HFMM_ERR_LOGIC = 4,            /* std::logic_error      */
  HFMM_ERR_LENGTH = 5,           /* std::length_error     */
  HFMM_ERR_CUDA = 6,             /* device / driver failure */
  HFMM_ERR_NO_DEVICE = 7,        /* no CUDA device: there is no CPU fallback */
  HFMM_ERR_INTERNAL = 8
} hfmm_status;

typedef enum hfmm_policy { HFMM_POLICY_RANK_ORDERED = 0, HFMM_POLICY_ALIGNED = 1 } hfmm_policy;

/* Mirrors hfmm::RunConfig (traversal.hpp:21-38) field for field.  The
 * scheduler field has no device meaning (one logical rank per GPU) and is
 * kept only so configs round-trip. */
typedef struct hfmm_run_config {
  double lambda;        /* wavelength, meters (default 1)      */
  double digits;        /* truncation accuracy knob (default 3) */
  double leaf_lambda;   /* leaf side in wavelengths (0.25)      */
  int32_t num_ranks;    /* logical ranks = GPUs (1)             */
  int32_t policy;       /* hfmm_policy (Aligned)                */
  uint64_t buffer_limit;/* M_S bytes (UINT64_MAX = unlimited)    */
  int32_t one_particle_per_leaf;
  int32_t top_level;    /* highest level carrying expansions (3) */
  int32_t d_override;   /* 0 = classify from geometry            */
  int32_t scheduler;    /* 0 deterministic, 1 adversarial, 2 threaded */
  uint64_t seed;
  /* Leaf weights of the Morton partition (partition_leaves, tree.cpp:19-75):
   * 0 = particles per leaf, the reference's rule (traversal.cpp:128-131; the
   * setup is bit-exact with the reference only in this mode); 1 = near-field
   * pairs per leaf, n_leaf * sum of its near leaves' populations (opt-in load
   * balance for P2P-dominated geometries). */
  int32_t partition_weight;
  /* 1 = build the Morton keys / sort and the far and near lists on the CUDA
   * device (bit-exact with the host build); 0 = host only. */
  int32_t setup_device;
} hfmm_run_config;

/* Fills the reference defaults (RunConfig{} in traversal.hpp:21-35). */
void hfmm_run_config_default(hfmm_run_config* cfg);

/* Thread-local message of the last failed call ("" if none). */
const char* hfmm_last_error(void);

/* ---------------- host setup (bit-exact with build_setup) ---------------- */

typedef struct hfmm_setup hfmm_setup;

/* Replaces build_setup (traversal.cpp:66-238).  positions: n*3 doubles (x,y,z
 * per particle), charges: n*2 doubles (re,im), input order. */
hfmm_status hfmm_setup_build(const double* positions, const double* charges,
                             size_t n, const hfmm_run_config* cfg,
                             hfmm_setup** out);
void hfmm_setup_destroy(hfmm_setup* s);

/* Named flat views of the setup (Morton keys, tree, lists, slices, plans)
 * used by the bit-exactness tests; see DESIGN.md "setup arrays".  Copies at
 * most cap bytes into dst (dst may be NULL) and returns the full byte size in
 * *nbytes.  Unknown names give HFMM_ERR_INVALID_ARGUMENT. */
hfmm_status hfmm_setup_get(const hfmm_setup* s, const char* name, void* dst,
                           size_t cap, size_t* nbytes);

/* Import of an EXISTING setup (the caller's GlobalSetup, traversal.hpp:93-118)
 * without re-running build_setup: put every array under the names and
 * layouts hfmm_setup_get() returns ("meta_i64", "meta_f64", "particles",
 * "original_index", "leaf_codes", "leaf_start", "rank_ranges", "splitters",
 * "near_off", "near", "m2l_plan", "near_plan" and per computed level l
 * "L<l>.sampling|theta_weight|phi_weight|codes|centers|users|slices_off|
 * slices|child_off|children|interp_off|interp|far_off|far"), then end.
 * end validates sizes, offsets and indices (HFMM_ERR_INVALID_ARGUMENT /
 * HFMM_ERR_OUT_OF_RANGE) and always consumes the import handle.  A setup
 * imported from the reference's build_setup equals hfmm_setup_build's byte
 * for byte (tests/test_setup_import.py, oracle/adapter). */
typedef struct hfmm_setup_import hfmm_setup_import;
hfmm_status hfmm_setup_import_begin(const hfmm_run_config* cfg, hfmm_setup_import** out);
hfmm_status hfmm_setup_import_put(hfmm_setup_import* im, const char* name, const void* data,
                                  size_t nbytes);
hfmm_status hfmm_setup_import_end(hfmm_setup_import* im, hfmm_setup** out);
void hfmm_setup_import_abort(hfmm_setup_import* im);

/* ---------------- device engine (one logical rank per GPU) ---------------- */

typedef struct hfmm_gpu hfmm_gpu;

typedef enum hfmm_phase {
  HFMM_PHASE_C2M = 1, /* RankEngine::c2m_phase   traversal.cpp:306 */
  HFMM_PHASE_M2M = 2, /* RankEngine::m2m_pass    traversal.cpp:322 */
  HFMM_PHASE_M2L = 3, /* RankEngine::m2l_pass    traversal.cpp:443 */
  HFMM_PHASE_L2L = 4, /* RankEngine::l2l_pass    traversal.cpp:583 */
  HFMM_PHASE_L2T = 5, /* l2o part of l2o_near_phase traversal.cpp:717-728 */
  HFMM_PHASE_NEAR = 6, /* near part of l2o_near_phase traversal.cpp:768-786: joins it into
                          the potentials (launching it first if not started) */
  HFMM_PHASE_NEAR_START = 7, /* launches the near field on the engine's side stream
                               (overlaps the far-field phases; needs charges/ghosts) */
  HFMM_PHASE_T_BUILD = 8 /* translation operators of every level (OperatorCache::build,
                            operators.cpp:124-176); HFMM_PHASE_M2L includes it, the
                            level-wise hfmm_gpu_run_level(M2L) needs it first */
} hfmm_phase;

/* Per-phase device milliseconds of the last hfmm_gpu_evaluate (CUDA events
 * on the engine stream), indexed by hfmm_phase; [0] = T-operator build,
 * [6] = near field (side stream, overlapped), [7] = whole evaluation. */
typedef struct hfmm_gpu_timing {
  double ms[8];
  int64_t kernel_launches;
} hfmm_gpu_timing;

/* Creates an engine on CUDA device `device` for logical rank `rank` of the
 * setup's partition.  Uploads the setup (sorted particles, level tables,
 * lists, samplings, interpolation matrices, translation coefficients).
 * Replaces RankEngine's constructor (traversal.cpp:242-288).  The engine
 * shares ownership of the setup: the caller may hfmm_setup_destroy() the
 * setup handle at any time; the data stays alive until the last engine made
 * from it is destroyed. */
hfmm_status hfmm_gpu_create(const hfmm_setup* s, int device, int rank,
                            hfmm_gpu** out);
void hfmm_gpu_destroy(hfmm_gpu* g);

/* Replaces evaluate_with_setup (traversal.cpp:790-817) for one rank:
 * charges (n*2, input order, may be NULL to keep the uploaded ones) are
 * copied in, all phases run, and this rank's potentials are scattered to
 * pot_out (n*2 doubles, input order; entries of other ranks untouched).
 * timing may be NULL. */
hfmm_status hfmm_gpu_evaluate(hfmm_gpu* g, const double* charges,
                              double* pot_out, hfmm_gpu_timing* timing);

/* Device-resident variant used by the benchmark: charges already on the
 * device in sorted order (n*2), potentials left on the device in sorted
 * order (n*2).  `stream` is a cudaStream_t (NULL = the engine stream). */
hfmm_status hfmm_gpu_evaluate_device(hfmm_gpu* g, const double* d_charges_sorted,
                                     double* d_pot_sorted, void* stream);

/* Per-phase device ms and kernel count of the last evaluation on this handle
 * (either entry point); events are recorded on the stream it ran on. */
hfmm_status hfmm_gpu_last_timing(hfmm_gpu* g, hfmm_gpu_timing* timing);

/* Runs a single phase (hfmm_phase) on the engine's current state, for
 * per-phase parity (RankEngine phase drivers, traversal.hpp:129-140).
 * HFMM_PHASE_C2M resets the state and uploads `charges` if given via
 * hfmm_gpu_set_charges. */
hfmm_status hfmm_gpu_set_charges(hfmm_gpu* g, const double* charges);
hfmm_status hfmm_gpu_run_phase(hfmm_gpu* g, int phase);

/* Copies this rank's multipole (kind 0) or local (kind 1) expansions of all
 * nodes of `level` it holds, as n_nodes * n_samples complex (re,im) in node
 * (Morton) order; nodes/samples this rank does not hold are zero.  Mirrors
 * RankEngine::multipole / local_expansion (traversal.hpp:142-143). */
hfmm_status hfmm_gpu_get_expansion(hfmm_gpu* g, int kind, int level, double* out,
                                   size_t cap_doubles);

/* Sorted-order potentials of this rank after HFMM_PHASE_NEAR/L2T (n*2). */
hfmm_status hfmm_gpu_get_potentials_sorted(hfmm_gpu* g, double* out,
                                           size_t cap_doubles);

/* ---------------- distributed mode (num_ranks > 1, one process per GPU) ----
 * Rank r holds the nodes whose leaf range meets its Morton leaf range.  The
 * upward pass (C2M, M2M) yields partial multipoles of held nodes; plural
 * (shared) nodes are SLICED by theta rows (assign_sample_slices,
 * tree.cpp:180-239): after the upward pass each user holds the full
 * multipole on its own slice.  Exchange kinds (static plans, rows = flat
 * sample ranges of a node):
 *   0  M2L halo: the reference's M2L CommPlan (comm_plan.cpp:31-82), the
 *      source rows (sender slice) x (receiver observer slice); per level;
 *   1  ghost particles (x, y, z, re, im) of the reference near plan
 *      (comm_plan.cpp:84-109);
 *   2  plural multipole reduce-scatter among a node's users (partials of the
 *      receiver's slice, added in the order unpack is called: call it in
 *      ascending peer rank);
 *   3  plural local all-gather among a node's users (each user's final slice
 *      rows), per level, before the L2L from that level.
 * The caller moves the buffers (e.g. NCCL); the engine packs / unpacks them on
 * its stream.  `level` = -1 selects all levels laid out level-major (kinds 0,
 * 2, 3; ignored for kind 1).  Sequence per evaluation (distributed.py):
 *   set_charges | load_charges_device; kind 1; run_phase(NEAR_START, C2M, M2M);
 *   kind 2 (all levels); run_phase(T_BUILD); for l = top..L: kind 0 (level l),
 *   run_level(M2L, l); for l = top..L-1: kind 3 (level l), run_level(L2L, l);
 *   run_phase(L2T), run_phase(NEAR).
 * In distributed mode hfmm_gpu_set_charges takes the full input-order array
 * and keeps this rank's particles only. */
hfmm_status hfmm_gpu_exchange_sizes(hfmm_gpu* g, int kind, int peer, int level,
                                    int64_t* send_doubles, int64_t* recv_doubles);
hfmm_status hfmm_gpu_pack(hfmm_gpu* g, int kind, int peer, int level, double* d_send);
hfmm_status hfmm_gpu_unpack(hfmm_gpu* g, int kind, int peer, int level, const double* d_recv);
/* One level of a phase: HFMM_PHASE_M2L (observer level, after HFMM_PHASE_T_BUILD)
 * or HFMM_PHASE_L2L (parent level l -> children at l + 1). */
hfmm_status hfmm_gpu_run_level(hfmm_gpu* g, int phase, int level);
/* All engine work goes to `stream` (cudaStream_t; NULL = a private stream). */
hfmm_status hfmm_gpu_set_stream(hfmm_gpu* g, void* stream);
hfmm_status hfmm_gpu_synchronize(hfmm_gpu* g);
/* Copies this rank's particles' charges (sorted order, device pointer). */
hfmm_status hfmm_gpu_load_charges_device(hfmm_gpu* g, const double* d_charges_sorted);
/* This rank's sorted particle range [*begin, *end). */
hfmm_status hfmm_gpu_particle_range(hfmm_gpu* g, int64_t* begin, int64_t* end);
/* Copies this rank's potentials (sorted order, its particle range) into the
 * device array d_pot_sorted at the same offsets, asynchronously on the
 * engine's stream (the per-rank output of l2o_near_phase, traversal.cpp:717-788). */
hfmm_status hfmm_gpu_store_potentials_device(hfmm_gpu* g, double* d_pot_sorted);
/* Kernels this handle has launched so far (cumulative; a bench counts its
 * timed region by difference). */
hfmm_status hfmm_gpu_launch_count(hfmm_gpu* g, int64_t* launches);
/* Phase overlap inside hfmm_gpu_evaluate / _evaluate_device (default on):
 * the leaf-level M2L runs on a low-priority stream beside the high-priority
 * far-field chain.  Off: strictly sequential phases, so hfmm_gpu_last_timing
 * reports each phase's own kernel time.  Results are identical either way. */
hfmm_status hfmm_gpu_set_overlap(hfmm_gpu* g, int on);

/* ---------------- world: every logical rank in one process ----------------
 * The counterpart of the reference's run_world + evaluate_with_setup
 * (runtime.cpp:274-290, traversal.cpp:790-817), which simulate all MPI ranks
 * in one process: one engine per logical rank of the setup's partition, rank
 * r on devices[r % ndev], the exchanges of the distributed schedule done by
 * device (peer) copies inside the library.  Works for any num_ranks >= 1. */
typedef struct hfmm_world hfmm_world;
hfmm_status hfmm_world_create(const hfmm_setup* s, const int* devices, int ndev, hfmm_world** out);
void hfmm_world_destroy(hfmm_world* w);
/* Input-order charges (n*2) to every rank. */
hfmm_status hfmm_world_set_charges(hfmm_world* w, const double* charges);
/* One reference RankEngine phase on every rank (traversal.hpp:129-140), with
 * the exchanges it owns: HFMM_PHASE_C2M, _M2M (+ plural reduce-scatter),
 * _M2L (T build + sliced halo per level), _L2L (plural gather per level),
 * _L2T (= l2o_near_phase: ghosts, L2T, near field). */
hfmm_status hfmm_world_run_phase(hfmm_world* w, int phase);
/* Full evaluation (charges may be NULL: keep); potentials in input order
 * (n*2).  rank_ms (may be NULL) receives num_ranks * 7 device milliseconds in
 * the reference ledger's phase order (ledger.hpp: Setup = T build, C2M, M2M,
 * M2L, L2L, L2O, Near). */
hfmm_status hfmm_world_evaluate(hfmm_world* w, const double* charges, double* pot_out,
                                double* rank_ms);
/* Potentials of all ranks in input order after hfmm_world_run_phase(L2T). */
hfmm_status hfmm_world_potentials(hfmm_world* w, double* pot_out);
/* Expansions of `level` as held by `rank` (n_nodes * S complex); the rows of
 * the rank's own slice of every node it holds are valid (RankEngine::multipole /
 * local_expansion, traversal.hpp:142-143). */
hfmm_status hfmm_world_get_expansion(hfmm_world* w, int rank, int kind, int level, double* out,
                                     size_t cap_doubles);

/* One-shot: build_setup + evaluate on one device (evaluate_potential,
 * traversal.cpp:819-823).  Requires cfg->num_ranks == 1. */
hfmm_status hfmm_evaluate_potential(const double* positions, const double* charges,
                                    size_t n, const hfmm_run_config* cfg, int device,
                                    double* pot_out);

/* O(N*M) direct sum on the device (direct_potential, kernel.cpp:16-41):
 * observers are given as particle indices into the source set; the first
 * exact coincidence per observer is skipped as the self term. */
hfmm_status hfmm_gpu_direct(const double* positions, const double* charges, size_t n,
                            const int64_t* observer_index, size_t m, double k,
                            int device, double* pot_out);

/* Dense complex matrix (n_out x n_in, row-major, re/im interleaved) of the
 * linear map resample_circle(n_in, s_in -> n_out, s_out)
 * (/root/reference/proj/src/sphere_grid.cpp:128-155) that the device M2M/L2L
 * kernels apply per theta row (shift 0) and per folded great circle
 * (shift 0.5).  out must hold 2*n_out*n_in doubles. */
hfmm_status hfmm_resample_matrix(int64_t n_in, double s_in, int64_t n_out, double s_out,
                                 double* out);

/* Packed operands of the device M2M passes of a level pair (child grid nc, parent
 * grid np, both even): what engine.cu uploads for fft_interpolate
 * (sphere_grid.cpp:183-192).  Host logic only (csrc/interp.hpp), no device needed.
 *   bphi: Kp x Np row-major, the phi map n_c -> n_p as real matrix + rank-1 row, with
 *         the (e, o) fold in its columns (column 2 p + h: circle p, part h);
 *   vphi: nc entries (rank-1 input vector);
 *   bth:  2 KH x NH row-major, [Be ; Bo] of the even / odd theta map 2 n_c -> 2 n_p;
 *   vth:  2 KH entries, laid out like the rows of bth;
 *   dims: {Kp, Np, KH, NH}.  Pass null pointers to query dims only. */
hfmm_status hfmm_m2m_operands(int nc, int np, double* bphi, double* vphi, double* bth, double* vth,
                              int dims[4]);

/* Same for the L2L passes (fft_anterpolate_adjoint, sphere_grid.cpp:194-214): theta map
 * 2 n_p -> 2 n_c with row_scale (2 nc entries) and col_scale (2 np entries) applied, in
 * even / odd form; phi map n_p -> n_c reading (Ye, Yo) pairs (unfold in its rows).
 *   bth: 2 KH x NH, vth: 2 KH;  bphi: Kp x Np, vphi: np;  dims: {KH, NH, Kp, Np}. */
hfmm_status hfmm_l2l_operands(int nc, int np, const double* row_scale, const double* col_scale,
                              double* bth, double* vth, double* bphi, double* vphi, int dims[4]);

/* Frozen seeded generator of the BASELINE inputs:
 * shape 0 = uniform cube of side `extent`, 1 = sphere surface of radius `extent`. */
void hfmm_generate_inputs(int shape, size_t n, double extent, uint64_t seed,
                          double* positions, double* charges);

#ifdef __cplusplus
}
#endif

#endif /* HFMM_GPU_H */
