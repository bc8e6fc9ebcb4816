// Lightweight in-library phase timer: CUDA events recorded on the launching
// stream around each phase while enabled, resolved lazily on read. Used by
// bench.py for the per-kernel roofline (launch duration from events on the
// kernel's own stream, never from a profiler).
//
// NVTX: with GDSW_NVTX=1 every phase is also an NVTX range named after its
// kernel (header-only nvtx3; ranges appear in Nsight Systems / ncu
// --nvtx-include filters; eager launches only -- a replayed CUDA graph has no
// host-side ranges).
#pragma once
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

namespace gdsw {

struct Prof {
  struct Phase {
    std::string name;
    double ms = 0.0;
    int64_t launches = 0;
    double bytes = 0.0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
  };
  std::mutex mu;
  bool on = false;
  std::vector<Phase> phases;
  std::vector<cudaEvent_t> pool;

  int id(const char* name) {
    for (size_t k = 0; k < phases.size(); ++k)
      if (phases[k].name == name) return (int)k;
    phases.push_back(Phase{name});
    return (int)phases.size() - 1;
  }
  cudaEvent_t take() {
    if (pool.empty()) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      return e;
    }
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  void resolve(Phase& p) {
    for (auto& pr : p.pending) {
      float ms = 0.f;
      CK(cudaEventSynchronize(pr.second));
      CK(cudaEventElapsedTime(&ms, pr.first, pr.second));
      p.ms += ms;
      pool.push_back(pr.first);
      pool.push_back(pr.second);
    }
    p.pending.clear();
  }
};

inline Prof& prof() {
  static Prof p;
  return p;
}

// RAII scope: records start/stop events on `stream` when profiling is on
inline bool nvtx_on() {
  static const bool on = [] {
    const char* e = std::getenv("GDSW_NVTX");
    return e && e[0] == '1';
  }();
  return on;
}

struct ProfScope {
  int k = -1;
  cudaStream_t s;
  cudaEvent_t e0 = nullptr;
  double bytes;
  bool nvtx = false;
  ProfScope(const char* name, cudaStream_t stream, double algorithmic_bytes)
      : s(stream), bytes(algorithmic_bytes) {
    if (nvtx_on()) {
      nvtxRangePushA(name);
      nvtx = true;
    }
    Prof& P = prof();
    if (!P.on) return;
    std::lock_guard<std::mutex> g(P.mu);
    k = P.id(name);
    e0 = P.take();
    CK(cudaEventRecord(e0, s));
  }
  ~ProfScope() {
    if (nvtx) nvtxRangePop();
    if (k < 0) return;
    Prof& P = prof();
    std::lock_guard<std::mutex> g(P.mu);
    cudaEvent_t e1 = P.take();
    cudaEventRecord(e1, s);
    auto& ph = P.phases[k];
    ph.pending.emplace_back(e0, e1);
    ph.launches += 1;
    ph.bytes += bytes;
  }
};

}  // namespace gdsw
