// The two parallel dimensions of the step:
//   * expert parallelism: expert e lives on rank e / (E / W) (the contiguous map
//     of Engine::expert_shard, model.cpp:334-340). Dispatch / combine (and their
//     transposes in the backward) are peer-store kernels (csrc/ep.cu) that write
//     the routed rows straight into the other ranks' arenas; completion is a flag
//     per (channel, source) in the receiver's arena, written with a stream memory
//     operation after the kernel (release) and awaited with another (no spinning
//     kernel). On a multi-GPU node the arenas are exchanged as CUDA IPC handles
//     over NCCL; in a loopback group (W shards, one device, one thread each) they
//     are the shards' own buffers.
//   * data parallelism: the replicated granule parts (embeddings, attention,
//     norms, gate, dense FFN) are summed with ncclAllReduce after backward, or in
//     rank order through a staging area in a loopback group.
// libnccl.so.2 is dlopen'ed on first use so the library never pins an NCCL
// version at link time (torch may already have loaded its own).
#include <cuda.h>
#include <dlfcn.h>

#include <chrono>
#include <cstring>
#include <mutex>

#include "comm_state.hpp"
#include "offload_state.hpp"
#include "p2r_cuda.h"

namespace p2r {

namespace {
using ncclComm_t = void*;
using ncclResult_t = int;
constexpr int kNcclInt8 = 0, kNcclFloat32 = 7, kNcclSum = 0;
struct NcclUid {
  char b[128];
};

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(NcclUid*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, NcclUid, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.h = h;
    api.getUniqueId = reinterpret_cast<decltype(api.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.commInitRank = reinterpret_cast<decltype(api.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.commDestroy = reinterpret_cast<decltype(api.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.groupStart = reinterpret_cast<decltype(api.groupStart)>(dlsym(h, "ncclGroupStart"));
    api.groupEnd = reinterpret_cast<decltype(api.groupEnd)>(dlsym(h, "ncclGroupEnd"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.allGather = reinterpret_cast<decltype(api.allGather)>(dlsym(h, "ncclAllGather"));
    api.errStr = reinterpret_cast<decltype(api.errStr)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.h || !api.getUniqueId || !api.allReduce || !api.allGather)
    throw std::runtime_error("nccl: libnccl.so.2 not available");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* s = nccl().errStr ? nccl().errStr(r) : "error";
    throw std::runtime_error(std::string("nccl ") + what + ": " + s);
  }
}

// Stream memory operations (driver API, resolved through the runtime).
struct StreamMemOps {
  CUresult (*write32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  CUresult (*wait32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
};

StreamMemOps& memops() {
  static StreamMemOps ops;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q{};
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      ops.write32 = reinterpret_cast<decltype(ops.write32)>(f);
    f = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      ops.wait32 = reinterpret_cast<decltype(ops.wait32)>(f);
  });
  if (!ops.write32 || !ops.wait32) throw std::runtime_error("expert parallel: stream memory operations unavailable");
  return ops;
}

std::size_t align256(std::size_t x) { return (x + 255) / 256 * 256; }
}  // namespace

// ---------------------------------------------------------------- loopback group
LoopbackGroup::LoopbackGroup(int w) : world(w), bases(static_cast<std::size_t>(w), nullptr) {
  if (w < 1) throw std::invalid_argument("loopback group: world must be >= 1");
  ev_in.resize(static_cast<std::size_t>(w));
  ev_out.resize(static_cast<std::size_t>(w));
  for (int i = 0; i < w; ++i) {
    cuda_check(cudaEventCreateWithFlags(&ev_in[static_cast<std::size_t>(i)], cudaEventDisableTiming), "event");
    cuda_check(cudaEventCreateWithFlags(&ev_out[static_cast<std::size_t>(i)], cudaEventDisableTiming), "event");
  }
}

LoopbackGroup::~LoopbackGroup() {
  cudaDeviceSynchronize();
  for (cudaEvent_t e : ev_in) cudaEventDestroy(e);
  for (cudaEvent_t e : ev_out) cudaEventDestroy(e);
}

void LoopbackGroup::barrier() {
  std::unique_lock<std::mutex> lk(mu);
  const std::uint64_t g = gen;
  if (++arrived == world) {
    arrived = 0;
    ++gen;
    cv.notify_all();
    return;
  }
  // a shard that threw (or was never driven) must not hang the others forever
  if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g; }))
    throw std::runtime_error("loopback group: a shard did not reach the exchange (300 s)");
}

EpState::~EpState() {
  for (void* p : ipc_open)
    if (p) cudaIpcCloseMemHandle(p);
}

// ---------------------------------------------------------------- init
void comm_unique_id(char* out128) {
  NcclUid u{};
  nccl_check(nccl().getUniqueId(&u), "get unique id");
  std::memcpy(out128, u.b, 128);
}

void Engine::comm_init(const char* id128) {
  if (comm_ || loop_) return;
  NcclUid u{};
  std::memcpy(u.b, id128, 128);
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  ncclComm_t c = nullptr;
  nccl_check(nccl().commInitRank(&c, ep_world_, u, ep_rank_), "comm init");
  comm_ = c;
}

void Engine::comm_init_loopback(LoopbackGroup* group) {
  if (comm_ || loop_) throw std::logic_error("comm_init: communicator already initialised");
  if (group == nullptr || group->world != ep_world_)
    throw std::invalid_argument("loopback group: world size does not match the model's");
  loop_ = group;
  // the all-reduce staging area is sized here, before any shard's step runs: growing it
  // later (device sync + reallocation) could race another shard's step-graph capture
  const std::size_t n = static_cast<std::size_t>(std::max<long long>(emb_.numel, layer_.numel));
  std::lock_guard<std::mutex> lk(group->mu);
  if (group->stage_floats < n) {
    cuda_check(cudaDeviceSynchronize(), "sync");
    group->stage = DevBuf(static_cast<std::size_t>(group->world) * n * 4);
    group->stage_floats = n;
  }
}

void Engine::comm_destroy() {
  if (comm_ && nccl().commDestroy) nccl().commDestroy(comm_);
  comm_ = nullptr;
  loop_ = nullptr;
}

// ---------------------------------------------------------------- expert parallel arena
// Called from ensure_acts on every rank (collective: same shapes everywhere).
void Engine::ep_connect(int seg, int n_ye) {
  const int W = ep_world_, E = cfg_.moe.n_experts, El = E / W, d = cfg_.d_model;
  if (W > 1 && comm_ == nullptr && loop_ == nullptr)
    throw std::logic_error("expert parallel: call comm_init before the first step");
  ep_.reset();  // closes the previous peer mappings
  auto st = std::make_unique<EpState>();
  std::size_t off = 0;
  st->off_flags = off;
  off = align256(off + 2 * static_cast<std::size_t>(W) * 4);
  st->off_cnt = off;
  off = align256(off + static_cast<std::size_t>(El) * W * 4);
  st->off_slot = off;
  off = align256(off + static_cast<std::size_t>(El) * W * seg * d * 2);
  st->ye_bytes = align256(static_cast<std::size_t>(E) * seg * d * 2);
  st->off_ye = off;
  off += st->ye_bytes * static_cast<std::size_t>(n_ye);
  st->off_dxe = off;
  off += st->ye_bytes;
  st->arena = DevBuf(off);
  cuda_check(cudaMemsetAsync(st->arena.p, 0, st->off_cnt, stream_), "zero flags");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  char* base = st->arena.as<char>();
  st->peer.assign(static_cast<std::size_t>(W), nullptr);
  st->peer[static_cast<std::size_t>(ep_rank_)] = base;
  if (loop_) {
    loop_->bases[static_cast<std::size_t>(ep_rank_)] = base;
    loop_->barrier();  // every shard has published its arena
    st->peer = loop_->bases;
    loop_->barrier();  // ... and read every other one
  } else if (W > 1) {
    // multi-process: all-gather the CUDA IPC handles of the arenas over NCCL
    cudaIpcMemHandle_t mine{};
    cuda_check(cudaIpcGetMemHandle(&mine, base), "ipc handle");
    DevBuf hd(sizeof(cudaIpcMemHandle_t) * static_cast<std::size_t>(W));
    cuda_check(cudaMemcpyAsync(hd.as<char>() + sizeof(mine) * static_cast<std::size_t>(ep_rank_), &mine, sizeof(mine),
                               cudaMemcpyHostToDevice, stream_),
               "h2d handle");
    nccl_check(nccl().allGather(hd.as<char>() + sizeof(mine) * static_cast<std::size_t>(ep_rank_), hd.p, sizeof(mine),
                                kNcclInt8, comm_, stream_),
               "allgather ipc handles");
    std::vector<cudaIpcMemHandle_t> all(static_cast<std::size_t>(W));
    cuda_check(cudaMemcpyAsync(all.data(), hd.p, hd.bytes, cudaMemcpyDeviceToHost, stream_), "d2h handles");
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    for (int q = 0; q < W; ++q) {
      if (q == ep_rank_) continue;
      void* p = nullptr;
      cuda_check(cudaIpcOpenMemHandle(&p, all[static_cast<std::size_t>(q)], cudaIpcMemLazyEnablePeerAccess),
                 "ipc open");
      st->ipc_open.push_back(p);
      st->peer[static_cast<std::size_t>(q)] = static_cast<char*>(p);
    }
  }
  ep_ = std::move(st);
}

void* Engine::ep_peer(int q, std::size_t off) const { return ep_->peer[static_cast<std::size_t>(q)] + off; }
void* Engine::ep_local(std::size_t off) const { return ep_->arena.as<char>() + off; }

// Completion of this rank's stores for channel ch (0 = rows to the owners,
// 1 = rows back to the sources): flag[ch][my rank] = epoch in every peer's arena,
// ordered after the preceding kernels by the write's memory barrier.
void Engine::ep_signal(int ch) {
  const std::uint32_t epoch = ++ep_->epoch[ch];
  const int W = ep_world_;
  for (int q = 0; q < W; ++q) {
    auto* flag = static_cast<char*>(ep_peer(q, ep_->off_flags)) + (static_cast<std::size_t>(ch) * W + ep_rank_) * 4;
    if (memops().write32(stream_, reinterpret_cast<CUdeviceptr>(flag), epoch, CU_STREAM_WRITE_VALUE_DEFAULT) !=
        CUDA_SUCCESS)
      throw std::runtime_error("expert parallel: stream write value failed");
  }
  // loopback: every shard's stores and flag writes are enqueued before any shard
  // enqueues its waits, so no stream can wait ahead of the work it depends on
  if (loop_) loop_->barrier();
}

// Wait (on the model stream, no kernel) until every rank signalled channel ch.
void Engine::ep_wait(int ch) {
  const std::uint32_t epoch = ep_->epoch[ch];
  const int W = ep_world_;
  for (int w = 0; w < W; ++w) {
    auto* flag = static_cast<char*>(ep_local(ep_->off_flags)) + (static_cast<std::size_t>(ch) * W + w) * 4;
    if (memops().wait32(stream_, reinterpret_cast<CUdeviceptr>(flag), epoch, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      throw std::runtime_error("expert parallel: stream wait value failed");
  }
}

// ---------------------------------------------------------------- data parallel
void Engine::allreduce_f32(float* buf, std::size_t n) {
  if (loop_) {
    LoopbackGroup& G = *loop_;
    const int W = G.world, r = ep_rank_;
    {
      std::lock_guard<std::mutex> lk(G.mu);
      if (G.stage_floats < n) {  // grown by the first arriving shard; nobody is using it yet
        cuda_check(cudaDeviceSynchronize(), "sync");
        G.stage = DevBuf(static_cast<std::size_t>(W) * n * 4);
        G.stage_floats = n;
      }
    }
    G.barrier();
    float* st = G.stage.as<float>();
    cuda_check(cudaMemcpyAsync(st + static_cast<std::size_t>(r) * n, buf, n * 4, cudaMemcpyDeviceToDevice, stream_),
               "stage");
    cuda_check(cudaEventRecord(G.ev_in[static_cast<std::size_t>(r)], stream_), "event");
    G.barrier();
    for (int w = 0; w < W; ++w) cuda_check(cudaStreamWaitEvent(stream_, G.ev_in[static_cast<std::size_t>(w)], 0), "wait");
    p2r_check(p2r_sum_ranks(st, W, static_cast<long long>(n), buf, stream_), "allreduce sum");
    cuda_check(cudaEventRecord(G.ev_out[static_cast<std::size_t>(r)], stream_), "event");
    G.barrier();
    for (int w = 0; w < W; ++w) cuda_check(cudaStreamWaitEvent(stream_, G.ev_out[static_cast<std::size_t>(w)], 0), "wait");
    G.barrier();  // nobody records ev_in/ev_out again before every shard enqueued its waits
    return;
  }
  if (!comm_) throw std::logic_error("allreduce_grads: communicator not initialised");
  nccl_check(nccl().allReduce(buf, buf, n, kNcclFloat32, kNcclSum, comm_, stream_), "allreduce");
}

// DP: sum the replicated gradient parts over ranks, in place, on the model stream.
// SLOW (offloaded) granules are summed inside their backward, before the fused AdamW.
void Engine::allreduce_grads() {
  if (!comm_ && !loop_) throw std::logic_error("allreduce_grads: communicator not initialised");
  // MoE layers: everything before the expert block (norms, attention, gate) is
  // replicated; experts are sharded. Dense layers are replicated entirely.
  const long long repl = cfg_.moe.enabled() ? layer_.w1 : layer_.numel;
  if (comm_) nccl_check(nccl().groupStart(), "group start");
  allreduce_f32(emb_g_.as<float>(), static_cast<std::size_t>(emb_.numel));
  for (int o = 0; o < n_owned_; ++o) {
    if (res_idx_[static_cast<std::size_t>(o)] < 0) continue;  // SLOW: reduced in offload_release
    allreduce_f32(lg(o, 0), static_cast<std::size_t>(repl));
  }
  if (comm_) nccl_check(nccl().groupEnd(), "group end");
}

}  // namespace p2r
