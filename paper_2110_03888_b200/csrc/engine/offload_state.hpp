// Private: state of the granular offload engine (csrc/engine/offload.cpp).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "p2r/engine.hpp"

namespace p2r {

struct OffloadSlot {
  DevBuf p32, g32, m, v, p16;
  int layer = -1;
  cudaEvent_t loaded = nullptr, free_ev = nullptr;
  bool free_recorded = false;
  bool grads_loaded = false;  // Bn staging brought the layer's parked partial gradients
  bool p16_loaded = false;    // staged as bf16 shadow + fp32 vectors (no master)
};

struct OffloadState {
  int ring = 2;
  std::vector<OffloadSlot> slots;
  std::vector<int> slot_of;    // owned layer -> slot used by the phase being computed
  std::vector<int> slot_fwd, slot_bwd;  // owned layer -> slot staged for that phase or -1
  // step schedule of SLOW granule uses: forward ascending, then backward descending
  std::vector<std::pair<int, bool>> sched;
  std::size_t next_issue = 0;
  int in_flight = 0;
  int next_slot_rr = 0;
  std::vector<int> host_idx;   // owned layer -> index in host arrays or -1
  std::vector<int> slow_list;  // SLOW owned layers, ascending
  std::vector<char> hgrad_valid;  // owned layer -> host holds its partial gradients (accumulation)
  std::vector<cudaEvent_t> wb_ev;     // owned layer -> its last write-back complete
  std::vector<cudaEvent_t> wb_fn_ev;  // ... its bf16 shadow written back (what a forward reloads)
  std::vector<char> wb_recorded;
  float* hp32 = nullptr;
  std::uint16_t* hp16 = nullptr;
  float* hm = nullptr;
  float* hv = nullptr;
  float* hg = nullptr;
  long long stride = 0;  // elements per granule
  cudaStream_t h2d = nullptr, d2h = nullptr;
  int next_slot = 0;
  bool training = false;
  bool skip = false;
  // Master form (P2R_OFFLOAD_FN_MASTER=1): Fn loads the fp32 master and re-derives the
  // bf16 operand on the device, so the write-back drops the bf16 shadow (H2D 16, D2H
  // 12 B/param per step). Default shadow form: Fn (and accumulating Bn) load the bf16
  // shadow + fp32 vectors, the write-back includes the shadow (14 / 14 B/param).
  bool fwd_master = false;
  OffloadStats stats;
  struct CopyRec {
    cudaEvent_t a, b;
    bool h2d;
  };
  std::vector<CopyRec> copies;
  std::vector<cudaEvent_t> pool;
  std::size_t pool_used = 0;

  cudaEvent_t ev() {
    if (pool_used == pool.size()) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "event");
      pool.push_back(e);
    }
    return pool[pool_used++];
  }
  ~OffloadState() {
    if (h2d) cudaStreamSynchronize(h2d);
    if (d2h) cudaStreamSynchronize(d2h);
    for (auto& s : slots) {
      if (s.loaded) cudaEventDestroy(s.loaded);
      if (s.free_ev) cudaEventDestroy(s.free_ev);
    }
    for (cudaEvent_t e : wb_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : wb_fn_ev) cudaEventDestroy(e);
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
    for (void* p : {static_cast<void*>(hp32), static_cast<void*>(hp16), static_cast<void*>(hm),
                    static_cast<void*>(hv), static_cast<void*>(hg)})
      if (p) cudaFreeHost(p);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
  }
};

}  // namespace p2r
