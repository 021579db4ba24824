// Private: state of the two parallel dimensions (csrc/engine/comm.cpp).
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <mutex>
#include <vector>

#include "p2r/engine.hpp"

namespace p2r {

// W expert-parallel / data-parallel shards driven by W host threads of ONE
// process on one device (SURVEY §4's single-GPU loopback comm): the EP exchange
// runs the same peer-store kernels and stream flag operations as on a multi-GPU
// node, with the shards' arenas as the "peer" memory; the DP all-reduce sums the
// shards' buffers in rank order through a staging area.
struct LoopbackGroup {
  explicit LoopbackGroup(int w);
  ~LoopbackGroup();
  void barrier();  // host barrier of the W shard threads
  int world;
  std::vector<char*> bases;  // EP arena base of every shard
  std::vector<cudaEvent_t> ev_in, ev_out;
  DevBuf stage;  // all-reduce staging [W][n] fp32
  std::size_t stage_floats = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  std::uint64_t gen = 0;
};

// Peer-memory arena of an expert-parallel shard: every buffer a peer writes into
// (identical layout on every rank, so a peer address is base + offset).
struct EpState {
  DevBuf arena;
  std::size_t off_flags = 0, off_cnt = 0, off_slot = 0, off_ye = 0, ye_bytes = 0, off_dxe = 0;
  std::vector<char*> peer;      // [W] arena bases (this rank's own at ep_rank)
  std::vector<void*> ipc_open;  // peer arenas mapped with cudaIpcOpenMemHandle (multi-process)
  std::uint32_t epoch[2] = {0, 0};
  ~EpState();
};

}  // namespace p2r
