// World: all logical ranks of a distributed evaluation in one process (world.hpp).
#include "world.hpp"

#include <stdexcept>
#include <string>

#include "hfmm_gpu.h"

namespace hfmm_b200 {

namespace {
void wck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  }
}
}  // namespace

World::World(std::shared_ptr<const Setup> s, const std::vector<int>& devices) : s_(std::move(s)) {
  if (devices.empty()) throw std::invalid_argument("hfmm_world_create: no devices");
  const int P = s_->P;
  for (int r = 0; r < P; ++r) dev_.push_back(devices[size_t(r) % devices.size()]);
  // Peer access between the devices in use (copies work without it, through
  // the host; with it they go over NVLink).
  for (int a : devices)
    for (int b : devices)
      if (a != b) {
        int ok = 0;
        if (cudaDeviceCanAccessPeer(&ok, a, b) == cudaSuccess && ok) {
          cudaSetDevice(a);
          if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();  // already enabled
        }
      }
  for (int r = 0; r < P; ++r) eng_.push_back(std::make_unique<Engine>(s_, dev_[size_t(r)], r));
  sent_.assign(size_t(P), nullptr);
  marks_.assign(size_t(P), std::vector<cudaEvent_t>(size_t(kLedgerPhases + 1), nullptr));
  for (int r = 0; r < P; ++r) {
    wck(cudaSetDevice(dev_[size_t(r)]), "cudaSetDevice");
    wck(cudaEventCreateWithFlags(&sent_[size_t(r)], cudaEventDisableTiming), "event");
    for (auto& e : marks_[size_t(r)]) wck(cudaEventCreate(&e), "event");
  }
}

World::~World() {
  for (int r = 0; r < ranks(); ++r) {
    cudaSetDevice(dev_[size_t(r)]);
    eng_[size_t(r)]->synchronize();
  }
  for (auto* m : {&send_, &recv_})
    for (auto& kv : *m) {
      cudaSetDevice(kv.second.dev);
      cudaFree(kv.second.p);
    }
  for (int r = 0; r < int(sent_.size()); ++r) {
    cudaSetDevice(dev_[size_t(r)]);
    if (sent_[size_t(r)]) cudaEventDestroy(sent_[size_t(r)]);
    for (auto e : marks_[size_t(r)])
      if (e) cudaEventDestroy(e);
  }
  eng_.clear();
}

double* World::buffer(std::map<std::tuple<int, int, int, int>, Buf>& m, std::tuple<int, int, int, int> key, int64_t n,
                      int dev) {
  Buf& b = m[key];
  if (b.n < n) {
    wck(cudaSetDevice(dev), "cudaSetDevice");
    if (b.p) cudaFree(b.p);
    wck(cudaMalloc(&b.p, size_t(n) * sizeof(double)), "cudaMalloc exchange");
    b.n = n;
    b.dev = dev;
  }
  return b.p;
}

void World::sync_all() {
  for (auto& e : eng_) e->synchronize();
}

// One exchange of the distributed schedule among all ranks: every sender
// packs and copies on its own stream, then every receiver waits for its
// senders' copies and unpacks them in ascending sender rank.
void World::exchange(int kind, int level) {
  const int P = ranks();
  if (P == 1) return;
  for (int r = 0; r < P; ++r) {
    Engine& e = *eng_[size_t(r)];
    for (int q = 0; q < P; ++q) {
      if (q == r) continue;
      int64_t sd = 0, rd = 0;
      e.exchange_sizes(kind, q, level, &sd, &rd);
      if (sd == 0) continue;
      double* src = buffer(send_, {kind, r, q, level}, sd, dev_[size_t(r)]);
      double* dst = buffer(recv_, {kind, r, q, level}, sd, dev_[size_t(q)]);
      e.pack(kind, q, level, src);
      wck(cudaSetDevice(dev_[size_t(r)]), "cudaSetDevice");
      if (dev_[size_t(r)] == dev_[size_t(q)])
        wck(cudaMemcpyAsync(dst, src, size_t(sd) * sizeof(double), cudaMemcpyDeviceToDevice, e.stream()), "copy");
      else
        wck(cudaMemcpyPeerAsync(dst, dev_[size_t(q)], src, dev_[size_t(r)], size_t(sd) * sizeof(double), e.stream()),
            "peer copy");
    }
    wck(cudaSetDevice(dev_[size_t(r)]), "cudaSetDevice");
    wck(cudaEventRecord(sent_[size_t(r)], e.stream()), "sent");
  }
  for (int q = 0; q < P; ++q) {
    Engine& e = *eng_[size_t(q)];
    for (int r = 0; r < P; ++r) {
      if (r == q) continue;
      int64_t sd = 0, rd = 0;
      e.exchange_sizes(kind, r, level, &sd, &rd);
      if (rd == 0) continue;
      auto it = recv_.find({kind, r, q, level});
      if (it == recv_.end() || it->second.n < rd) throw std::logic_error("world exchange: plan mismatch");
      wck(cudaSetDevice(dev_[size_t(q)]), "cudaSetDevice");
      wck(cudaStreamWaitEvent(e.stream(), sent_[size_t(r)], 0), "wait sent");
      e.unpack(kind, r, level, it->second.p);
    }
  }
}

void World::set_charges(const double* q_in) {
  for (auto& e : eng_) e->set_charges(q_in);
}

void World::run_phase(int phase) {
  const int top = s_->top, L = s_->L;
  switch (phase) {
    case HFMM_PHASE_C2M:
      for (auto& e : eng_) e->run_phase(HFMM_PHASE_C2M);
      break;
    case HFMM_PHASE_M2M:
      for (auto& e : eng_) e->run_phase(HFMM_PHASE_M2M);
      exchange(kXReduce, -1);
      break;
    case HFMM_PHASE_M2L:
      for (auto& e : eng_) e->run_phase(HFMM_PHASE_T_BUILD);
      for (int l = top; l <= L; ++l) {
        exchange(kXHalo, l);
        for (auto& e : eng_) e->run_level(HFMM_PHASE_M2L, l);
      }
      break;
    case HFMM_PHASE_L2L:
      for (int l = top; l < L; ++l) {
        exchange(kXGather, l);
        for (auto& e : eng_) e->run_level(HFMM_PHASE_L2L, l);
      }
      break;
    case HFMM_PHASE_L2T:  // l2o_near_phase (traversal.cpp:709-788): ghosts, L2T, near field
      exchange(kXGhost, -1);
      for (auto& e : eng_) {
        e->run_phase(HFMM_PHASE_L2T);
        e->run_phase(HFMM_PHASE_NEAR);
      }
      break;
    default:
      throw std::invalid_argument("hfmm_world_run_phase: phase must be C2M, M2M, M2L, L2L or L2T");
  }
}

void World::evaluate(const double* q_in, double* pot_out) {
  const int top = s_->top, L = s_->L, P = ranks();
  if (q_in) set_charges(q_in);
  auto mark = [&](int i) {
    for (int r = 0; r < P; ++r) {
      wck(cudaSetDevice(dev_[size_t(r)]), "cudaSetDevice");
      wck(cudaEventRecord(marks_[size_t(r)][size_t(i)], eng_[size_t(r)]->stream()), "mark");
    }
  };
  // ghosts first: the near field then runs on each engine's side stream
  // beside the far-field chain
  exchange(kXGhost, -1);
  for (auto& e : eng_) e->run_phase(HFMM_PHASE_NEAR_START);
  mark(0);
  for (auto& e : eng_) e->run_phase(HFMM_PHASE_C2M);
  mark(1);
  for (auto& e : eng_) e->run_phase(HFMM_PHASE_M2M);
  exchange(kXReduce, -1);
  mark(2);
  for (auto& e : eng_) e->run_phase(HFMM_PHASE_T_BUILD);
  mark(3);
  for (int l = top; l <= L; ++l) {
    exchange(kXHalo, l);
    for (auto& e : eng_) e->run_level(HFMM_PHASE_M2L, l);
  }
  mark(4);
  for (int l = top; l < L; ++l) {
    exchange(kXGather, l);
    for (auto& e : eng_) e->run_level(HFMM_PHASE_L2L, l);
  }
  mark(5);
  for (auto& e : eng_) e->run_phase(HFMM_PHASE_L2T);
  mark(6);
  for (auto& e : eng_) e->run_phase(HFMM_PHASE_NEAR);
  mark(7);
  timed_ = true;
  if (pot_out) potentials(pot_out);
}

void World::potentials(double* pot_out) {
  const size_t n = s_->n;
  std::vector<double> sorted(2 * n);
  for (auto& e : eng_) e->store_potentials_host(sorted.data());  // own particle range, synchronous
  for (size_t i = 0; i < n; ++i) {
    const uint64_t j = s_->original_index[i];
    pot_out[2 * j] = sorted[2 * i];
    pot_out[2 * j + 1] = sorted[2 * i + 1];
  }
}

void World::rank_ms(int rank, double* ms) const {
  if (!timed_) throw std::logic_error("hfmm_world: no evaluation recorded");
  if (rank < 0 || rank >= int(eng_.size())) throw std::out_of_range("hfmm_world: bad rank");
  const auto& m = marks_[size_t(rank)];
  wck(cudaSetDevice(dev_[size_t(rank)]), "cudaSetDevice");
  wck(cudaEventSynchronize(m[7]), "event sync");
  auto el = [&](int a, int b) {
    float f = 0.f;
    wck(cudaEventElapsedTime(&f, m[size_t(a)], m[size_t(b)]), "elapsed");
    return double(f);
  };
  // ledger.hpp order: Setup (T build), C2M, M2M, M2L, L2L, L2O, Near
  ms[0] = el(2, 3);
  ms[1] = el(0, 1);
  ms[2] = el(1, 2);
  ms[3] = el(3, 4);
  ms[4] = el(4, 5);
  ms[5] = el(5, 6);
  ms[6] = el(6, 7);
}

}  // namespace hfmm_b200
