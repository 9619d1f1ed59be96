// World: every logical rank of a distributed evaluation in ONE process, on
// one or several CUDA devices -- the B200 counterpart of the reference's
// run_world + evaluate_with_setup (runtime.cpp:274-290, traversal.cpp:790-817),
// which simulates its MPI ranks as threads in one process.
//
// Each rank is an Engine (rank r on devices[r % ndev]); the exchanges of the
// distributed schedule (setup.hpp: ghosts, plural reduce-scatter, sliced M2L
// halo from the reference CommPlan, plural local gather) are packed on the
// sender's stream, copied device to device (peer copies across devices) and
// unpacked on the receiver's stream after an event wait, receivers taking
// senders in ascending rank order.  No kernel waits on another rank's kernel.
// The one-process-per-GPU NCCL driver (paper_2006_15367_b200/distributed.py)
// runs the same schedule over the same engine entry points.
#ifndef HFMM_B200_WORLD_HPP
#define HFMM_B200_WORLD_HPP

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include "engine.hpp"

namespace hfmm_b200 {

// Ledger phases of the reference (ledger.hpp: Setup, C2M, M2M, M2L, L2L, L2O, Near).
constexpr int kLedgerPhases = 7;

class World {
 public:
  World(std::shared_ptr<const Setup> s, const std::vector<int>& devices);
  ~World();
  World(const World&) = delete;
  World& operator=(const World&) = delete;

  int ranks() const { return int(eng_.size()); }
  Engine& engine(int r) { return *eng_.at(size_t(r)); }

  // Input-order charges (n*2) to every rank (each keeps its own particles).
  void set_charges(const double* q_in);
  // One RankEngine phase of the reference on every rank, with the exchanges
  // that phase owns: C2M; M2M (+ plural reduce-scatter); M2L (T build, sliced
  // halo per level); L2L (plural gather per level); L2T = l2o_near_phase
  // (ghosts, L2T, near field).
  void run_phase(int phase);
  // Full evaluation: charges (may be NULL: keep) -> potentials in input order.
  void evaluate(const double* q_in, double* pot_out);
  // Potentials of every rank's particles in input order (after L2T).
  void potentials(double* pot_out);
  // Device ms per ledger phase of `rank` in the last evaluate().
  void rank_ms(int rank, double* ms) const;

 private:
  void exchange(int kind, int level);
  void sync_all();
  struct Buf {
    double* p = nullptr;
    int64_t n = 0;
    int dev = 0;
  };
  double* buffer(std::map<std::tuple<int, int, int, int>, Buf>& m, std::tuple<int, int, int, int> key, int64_t n,
                 int dev);

  std::shared_ptr<const Setup> s_;
  std::vector<int> dev_;  // per rank
  std::vector<std::unique_ptr<Engine>> eng_;
  std::vector<cudaEvent_t> sent_;  // per rank: its copies of the current exchange are done
  std::map<std::tuple<int, int, int, int>, Buf> send_, recv_;  // (kind, from, to, level)
  std::vector<std::vector<cudaEvent_t>> marks_;  // per rank: kLedgerPhases + 1 timing events
  bool timed_ = false;
};

}  // namespace hfmm_b200

#endif
