// NCCL plumbing for the two parallel dimensions of the step:
//   * expert parallelism: expert e lives on rank e / (E / W) (the contiguous
//     map of Model::expert_shard, model.cpp:334-340); MoE dispatch / combine
//     (and their transposes in the backward) are stream-ordered grouped
//     ncclSend / ncclRecv of fixed-capacity expert segments (no count exchange);
//   * data parallelism: the replicated granule parts (embeddings, attention,
//     norms, gate, dense FFN) are summed with ncclAllReduce after backward.
// libnccl.so.2 is dlopen'ed on first use so the library never pins an NCCL
// version at link time (torch may already have loaded its own).
#include <dlfcn.h>

#include <cstring>
#include <mutex>

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
  ncclResult_t (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
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
    api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
    api.allReduce = reinterpret_cast<decltype(api.allReduce)>(dlsym(h, "ncclAllReduce"));
    api.errStr = reinterpret_cast<decltype(api.errStr)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!api.h || !api.getUniqueId || !api.send || !api.recv || !api.allReduce)
    throw std::runtime_error("nccl: libnccl.so.2 not available");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* s = nccl().errStr ? nccl().errStr(r) : "error";
    throw std::runtime_error(std::string("nccl ") + what + ": " + s);
  }
}
}  // namespace

void comm_unique_id(char* out128) {
  NcclUid u{};
  nccl_check(nccl().getUniqueId(&u), "get unique id");
  std::memcpy(out128, u.b, 128);
}

void Model::comm_init(const char* id128) {
  if (comm_) return;
  NcclUid u{};
  std::memcpy(u.b, id128, 128);
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  ncclComm_t c = nullptr;
  nccl_check(nccl().commInitRank(&c, ep_world_, u, ep_rank_), "comm init");
  comm_ = c;
}

void Model::comm_destroy() {
  if (comm_ && nccl().commDestroy) nccl().commDestroy(comm_);
  comm_ = nullptr;
}

// Expert segments between the local expert-major layout [E][seg] (E = W*El,
// rows of expert e at e*seg) and the owner-side layout [El][W][seg] (rows from
// source rank q for local expert e at (e*W + q)*seg). to_experts = dispatch
// direction; otherwise the combine direction.
void Model::ep_exchange(const void* src, void* dst, std::size_t row_bytes, int seg, bool to_experts) {
  NcclApi& api = nccl();
  const int W = ep_world_, El = cfg_.moe.n_experts / W;
  const std::size_t blk = row_bytes * static_cast<std::size_t>(seg);
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  nccl_check(api.groupStart(), "group start");
  for (int q = 0; q < W; ++q) {
    for (int e = 0; e < El; ++e) {
      const std::size_t local = static_cast<std::size_t>(q * El + e) * blk;  // [E][seg] side
      const std::size_t owner = static_cast<std::size_t>(e * W + q) * blk;   // [El][W][seg] side
      if (to_experts) {
        nccl_check(api.send(s + local, blk, kNcclInt8, q, comm_, stream_), "send");
        nccl_check(api.recv(d + owner, blk, kNcclInt8, q, comm_, stream_), "recv");
      } else {
        nccl_check(api.send(s + owner, blk, kNcclInt8, q, comm_, stream_), "send");
        nccl_check(api.recv(d + local, blk, kNcclInt8, q, comm_, stream_), "recv");
      }
    }
  }
  nccl_check(api.groupEnd(), "group end");
}

void Model::allreduce_f32(float* buf, std::size_t n) {
  if (!comm_) throw std::logic_error("allreduce_grads: communicator not initialised");
  nccl_check(nccl().allReduce(buf, buf, n, kNcclFloat32, kNcclSum, comm_, stream_), "allreduce");
}

// DP: sum the replicated gradient parts over ranks, in place, on the model stream.
// SLOW (offloaded) granules are summed inside their backward, before the fused AdamW.
void Model::allreduce_grads() {
  if (!comm_) throw std::logic_error("allreduce_grads: communicator not initialised");
  NcclApi& api = nccl();
  nccl_check(api.groupStart(), "group start");
  nccl_check(api.allReduce(emb_g_.p, emb_g_.p, static_cast<std::size_t>(emb_.numel), kNcclFloat32, kNcclSum, comm_,
                           stream_),
             "allreduce embeddings");
  // MoE layers: everything before the expert block (norms, attention, gate) is
  // replicated; experts are sharded. Dense layers are replicated entirely.
  const long long repl = cfg_.moe.enabled() ? layer_.w1 : layer_.numel;
  for (int o = 0; o < n_owned_; ++o) {
    if (res_idx_[static_cast<std::size_t>(o)] < 0) continue;  // SLOW: reduced in offload_release
    nccl_check(api.allReduce(lg(o, 0), lg(o, 0), static_cast<std::size_t>(repl), kNcclFloat32, kNcclSum, comm_,
                             stream_),
               "allreduce layer");
  }
  nccl_check(api.groupEnd(), "group end");
}

}  // namespace p2r
