// C++ host engine of the B200 build: parameters in device granules, the
// reference's layer/step semantics (model.hpp, optim.hpp, tensor.hpp of
// /root/reference/proj/core) as fused sm_100a kernel sequences (p2r_cuda.h),
// granular offload, expert / data parallelism, checkpoints. The drop-in classes
// with the reference's exact declarations (p2r/model.hpp, optim.hpp, tensor.hpp)
// are handles on this engine; the C-ABI (p2r_engine.h) exposes it to C / ctypes.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "p2r/model.hpp"

namespace p2r {

// Reference-compatible per-tensor init (model.cpp:11-36).
std::uint64_t init_mix_seed(std::uint64_t seed, const std::string& name);
void init_normal_host(float* out, std::size_t n, std::uint64_t seed, const std::string& name,
                      float stddev = 0.02f);

// ---------------------------------------------------------------- device memory
struct DevBuf {
  void* p = nullptr;
  std::size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(std::size_t n);
  ~DevBuf();
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept;
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// Device activation handle (fp32, row-major [rows, cols]); `grad` is the
// gradient buffer the backward closures read/write.
struct DevTensor {
  int rows = 0, cols = 0;
  float* data = nullptr;
  float* grad = nullptr;
  void* grad16 = nullptr;  // bf16 shadow of grad (GEMM operand)
  bool defined() const { return data != nullptr; }
};

// One parameter as the reference names it, viewed inside a granule buffer.
// Stage bookkeeping carried by a checkpoint (SPEC.md:250-254 StageState).
struct StageState {
  int stage = 0;  // 0 = PSEUDO, 1 = REAL
  std::int64_t global_step = 0;
  std::int64_t samples_consumed = 0;
  double wall_time_s = 0.0;
  std::uint64_t rng_state = 0;
  std::int64_t last_eval_step = -1;
};

struct ParamView {
  std::string name;
  int granule;        // -1 = embeddings granule, else owned layer index
  long long off;      // element offset in the granule
  int rows, cols, ld; // 2-D view (vectors: rows = 1)
  std::vector<int> shape;
};

// Element layout of one granule (a layer, or the embeddings) — all of its
// parameters contiguous so delink / offload / AdamW move it as one block.
struct GranuleLayout {
  struct Seg {
    long long off, len;
    bool decay;
  };
  std::vector<Seg> segs;
  long long numel = 0;
  // layer roles
  long long ln1_g = 0, ln1_b = 0, wqkv = 0, wo = 0, ln2_g = 0, ln2_b = 0;
  long long w1 = 0, b1 = 0, w2 = 0, b2 = 0, gate = 0;
  // embedding roles
  long long tok = 0, pos = 0, fin_g = 0, fin_b = 0;
  long long add(long long n, bool decay);
};

struct Acts;  // per-shape activation / workspace buffers
struct OffloadState;
struct EpState;
struct LoopbackGroup;
struct LayerActs;

// Per-step movement accounting of the granular offload engine:
// bytes moved per phase plus measured copy-engine time.
struct OffloadStats {
  double fn_load = 0;       // H2D of SLOW granules for the forward (Fn)
  double bn_load = 0;       // H2D of SLOW granules for the backward (Bn)
  double opt_load = 0;      // H2D of AdamW moments of SLOW granules (An)
  double writeback = 0;     // D2H of updated params + moments (An)
  double grad_offload = 0;  // D2H of SLOW-granule grads (no fused optimizer, or a non-final micro-step)
  double grad_load = 0;     // H2D of parked partial grads (accumulation micro-steps after the first)
  double h2d_ms = 0, d2h_ms = 0;
  std::int64_t copies = 0;
};

// plan_offload: minimise predicted step time subject to the
// FAST-tier budget; exhaustive for n <= 12, lowest-index prefix otherwise (the
// optimum for uniform layers). Returns 1 = SLOW per layer.
std::vector<int> plan_offload(const std::vector<std::int64_t>& layer_bytes, std::int64_t budget,
                              double bandwidth, double compute_s, double latency_s);
double predict_step_time(const std::vector<std::int64_t>& layer_bytes, const std::vector<int>& slow,
                         double bandwidth, double compute_s, double latency_s);

// B200 overlap model of this engine's offload. Per SLOW layer
// of P parameters the copy engines move, per step: forward H2D 2P (bf16 shadow) +
// fp32 vectors; backward H2D 12P (fp32 master, m, v); D2H 14P (p, m, v, bf16).
// Copies overlap compute on their own streams, so
//   step = max(C_fwd, H2D_fwd/h2d) + max(C_bwd, H2D_bwd/h2d, D2H/d2h),
// and at least (H2D_fwd + H2D_bwd)/h2d + the first SLOW layer's Fn load + its
// write-back (the ring prefetches backward granules during the forward).
// with C_* = per-layer compute x L (calibrated from a resident step).
struct OffloadCost {
  double h2d_bw = 50e9, d2h_bw = 50e9;  // pinned PCIe bytes/s per direction
  double fwd_s = 0, bwd_s = 0;          // compute per layer
  bool fn_master = false;               // Fn loads the fp32 master (4P), write-back drops the bf16 (12P)
  int ring_slots = 3;                   // HBM staging slots (planner budget: resident + ring x largest granule)
  int micro_steps = 1;                  // accumulation window: per micro-step Fn + Bn loads; partial grads
                                        // parked (D2H 4P) / reloaded (H2D 4P) between micro-steps; moments +
                                        // write-back once per window
  bool recompute = false;               // activation checkpointing of SLOW layers: +1 forward in the backward
};
double predict_step_time_overlap(const std::vector<std::int64_t>& layer_params,
                                 const std::vector<std::int64_t>& vector_params, const std::vector<int>& slow,
                                 const OffloadCost& c);
// fewest SLOW layers whose granules (18 B/param) bring the resident set plus the
// ring_slots staging slots under `budget`, spread evenly over the stack; minimises
// predict_step_time_overlap among placements with that count for uniform layers.
std::vector<int> plan_offload_overlap(const std::vector<std::int64_t>& layer_params, std::int64_t budget,
                                      const OffloadCost& c);
// staged device pointer of a SLOW granule: kind 0 p32, 1 grad, 2 m, 3 v, 4 bf16
float* offload_slot_ptr(const OffloadState& st, int owned, int kind);
// host fp32 -> bf16 (round to nearest even), the device __float2bfloat16_rn
void host_cast_bf16(const float* src, std::uint16_t* dst, long long n);
// wait for the offload engine's copy streams (before touching host granules)
void offload_sync(const OffloadState& st);

// Live per-kernel-class timing with CUDA events on the model stream.
struct Profiler {
  struct Rec {
    int cls;
    cudaEvent_t a, b;
    double flops, bytes;
  };
  bool on = false;
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  std::size_t used = 0;
  cudaEvent_t get();
  ~Profiler();
};

// Switch detector decision logic (csrc/engine/switch.cpp).
struct SwitchPolicy {
  int eval_interval_steps = 500;  // SPEC design decision defaults
  int trial_budget_steps = 50;
  int slope_window = 50;
  void validate() const;
};
struct SwitchDecision {
  bool fire = false;
  double pseudo_slope = 0, real_slope = 0;  // d loss / d wall-time
};
// least-squares slope of loss against time over the last `window` points (all if <= 0)
double loss_slope(const std::vector<double>& time_s, const std::vector<double>& loss, int window);
// fire when the Real trial decreases loss faster per unit time than the Pseudo continuation
SwitchDecision switch_criterion(const std::vector<double>& pseudo_t, const std::vector<double>& pseudo_loss,
                                const std::vector<double>& real_t, const std::vector<double>& real_loss,
                                const SwitchPolicy& policy);
bool switch_evaluation_due(const SwitchPolicy& policy, std::int64_t step);

class Engine;
// SPEC delink(pseudo_checkpoint) -> Checkpoint: load a PSEUDO
// checkpoint, delink (weights + moments copied into every layer), save it as REAL.
StageState delink_checkpoint(const std::string& in_path, const std::string& out_path);
// SPEC redistribute_experts(model, new_n_shards) across GPU counts (SURVEY §8(f)
// row 2; model.cpp:334-356): re-shard W1 expert-parallel shard checkpoints into
// W2 (rank r2 gets experts [r2*E/W2, (r2+1)*E/W2), weights and AdamW moments;
// replicated buffers from shard 0; config n_shards = W2). Host file I/O only.
void redistribute_checkpoints(const std::vector<std::string>& in_paths, const std::vector<std::string>& out_paths);

class Engine {
 public:
  Engine(ModelConfig config, std::uint64_t seed);
  // Real model with granular CPU offload: slow[i] = 1 keeps owned layer i in
  // pinned host DRAM and streams it through `ring_slots` HBM staging slots.
  Engine(ModelConfig config, std::uint64_t seed, const std::vector<int>& slow, int ring_slots);
  // Expert-parallel shard `ep_rank` of `ep_world`: holds experts
  // [ep_rank*E/W, (ep_rank+1)*E/W) (model.cpp:334-340) + the replicated rest.
  Engine(ModelConfig config, std::uint64_t seed, int ep_world, int ep_rank);
  // Both: an expert-parallel shard whose SLOW layer granules (replicated part +
  // local experts) live in pinned host DRAM (C5: 96-layer MoE over 8 GPUs).
  Engine(ModelConfig config, std::uint64_t seed, const std::vector<int>& slow, int ring_slots, int ep_world,
        int ep_rank);
  ~Engine();

  // NCCL (one communicator per model over all ranks; csrc/engine/comm.cpp)
  void comm_init(const char* unique_id128);
  // W shards of one process on one device, one host thread each (loopback group)
  void comm_init_loopback(LoopbackGroup* group);
  void comm_destroy();
  void allreduce_grads();  // DP: sum replicated grads (embeddings, attention, norms, gate, dense FFN)
  int ep_world() const { return ep_world_; }
  int ep_rank() const { return ep_rank_; }
  bool ep_active() const { return ep_world_ > 1 || force_ep_; }
  // Dense layers take db2 from the column sums staged by the LayerNorm backward that
  // produced their output gradient (wider rows would spill its extra accumulators).
  bool db2_fused() const { return !cfg_.moe.enabled() && cfg_.d_model <= 13 * 128; }
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const ModelConfig& config() const { return cfg_; }
  int n_graph_layers() const { return cfg_.n_layers_graph; }
  int n_owned_layers() const { return n_owned_; }
  int owned_index_of_graph_layer(int g) const { return cfg_.shared() || n_owned_ == 1 ? 0 : g; }

  // segmented API (model.hpp:101-106); token / target / mask pointers are device arrays
  DevTensor embed_forward(GradTape* tape, const int* d_tokens, int batch, int seq);
  DevTensor block_forward(GradTape* tape, int graph_layer, const DevTensor& x, int batch,
                       AttentionMode mode);
  DevTensor head_forward(GradTape* tape, const DevTensor& x);
  // fused softmax_cross_entropy(mask, denom) (tensor.cpp:670-723); returns a
  // 1-element device tensor
  DevTensor softmax_cross_entropy(GradTape* tape, const DevTensor& logits, const int* d_targets,
                               const std::uint8_t* d_mask, double denom);

  // whole micro-step (controller CS-1)
  void train_step_device(const int* d_tokens, const int* d_targets, const std::uint8_t* d_mask,
                         int batch, int seq, double denom, AttentionMode mode, bool zero,
                         float* loss_dev);
  float train_step_host(const int* tokens, const int* targets, const std::uint8_t* mask,
                        int batch, int seq, double denom, AttentionMode mode, bool zero);
  // pipelined host step: the inputs are staged in one of two pinned slots, the step and
  // the loss read-back are enqueued, and a ticket is returned at once (the next step,
  // the optimizer, ... can be enqueued before the loss is read). loss_wait(ticket)
  // returns that step's loss; a slot is reused two steps later, so only the last two
  // tickets can be waited on (older ones throw std::logic_error).
  std::uint64_t train_step_host_async(const int* tokens, const int* targets, const std::uint8_t* mask,
                                      int batch, int seq, double denom, AttentionMode mode, bool zero);
  float loss_wait(std::uint64_t ticket);
  void forward_host(const int* tokens, int batch, int seq, AttentionMode mode, float* logits_out);

  void zero_grads();
  void flush_shared_layer_grads() {}  // accumulated in place by the dW epilogues
  std::int64_t scratch_grad_bytes() const { return 0; }
  std::int64_t grad_bytes() const;

  // parameters (for_each_param order)
  const std::vector<ParamView>& params() const { return views_; }
  void get_param(int i, float* host) const;
  void set_param(int i, const float* host);
  void get_grad(int i, float* host) const;
  void get_moment(int i, int which, float* host) const;
  void set_moment(int i, int which, const float* host);

  // optimizer state (AdamW moments live beside the parameters, same layout)
  void adamw_attach(float b1, float b2, float eps, float wd);
  void adamw_step(float lr);
  std::int64_t step_count() const { return step_count_; }
  void set_step_count(std::int64_t t) { step_count_ = t; }
  std::int64_t state_bytes() const;
  bool has_optimizer() const { return has_opt_; }

  std::unique_ptr<Engine> delinked() const;

  // expert sharding bookkeeping (model.cpp:334-356): expert e lives on shard
  // e / (E / n_shards). In one process re-sharding is bookkeeping (outputs are
  // unchanged); expert-parallel runs re-shard weights and moments across GPU
  // counts with redistribute_checkpoints.
  int expert_shard(int expert) const;
  std::vector<std::vector<int>> shard_layout() const;
  void redistribute_experts(int new_n_shards);

  // Checkpoint container (csrc/engine/checkpoint.cpp):
  // version tag, ModelConfig, named layer-indexed parameter buffers, AdamW
  // moments + step count, StageState; little-endian ints, IEEE fp32 payload,
  // manifest of names / shapes / byte offsets. save -> load -> train k steps is
  // bit-identical to training k steps uninterrupted.
  void save_checkpoint(const std::string& path, const StageState& st) const;
  // Load into this model (config and EP shard must match); attaches AdamW if the
  // file carries moments and the optimizer is not attached yet.
  StageState load_checkpoint(const std::string& path);
  static std::unique_ptr<Engine> from_checkpoint(const std::string& path, StageState* st);

  cudaStream_t stream() const { return stream_; }
  // train_step_device replayed as one CUDA graph (captured on the first call,
  // re-captured when any argument changes): resident models on one rank's experts
  // (dense, or MoE without the expert-parallel exchange; the data-parallel
  // all-reduce stays outside); the launches (and their PDL edges) are those of
  // train_step_device, so results are bit-identical to it.
  void train_step_device_graph(const int* d_tokens, const int* d_targets, const std::uint8_t* d_mask, int batch,
                               int seq, double denom, AttentionMode mode, bool zero, float* loss_dev);
  void set_profiling(bool on) { prof_.on = on; }
  void profile(int cls, std::int64_t* launches, double* ms, double* flops, double* bytes);
  void profile_reset();
  void buffer(int which, void** ptr, std::size_t* bytes) const;

  // drop-in API support (p2r/model.hpp): a counter bumped by every call that may
  // change device state (host copies of device tensors are cached per version), and
  // device staging of the segmented API's token ids / targets / mask (validated)
  std::uint64_t version() const { return version_; }
  const int* stage_tokens(const int* host, int batch, int seq);
  void stage_targets(const int* targets, const std::uint8_t* mask, int n, const int** d_targets,
                     const std::uint8_t** d_mask);
  // copy a host activation [T, d] into the embedding output buffer (block_forward on a host tensor)
  float* stage_activation(const float* host, int rows);
  int vocab_ld() const;  // leading dimension of the device logits

  // granular offload
  bool offloaded() const { return off_ != nullptr; }
  const std::vector<int>& slow_layers() const { return slow_; }
  // lr of the optimizer step whose last backward runs the fused AdamW of the SLOW
  // granules; must be set (and equal the adamw_step lr) before that backward
  void set_offload_lr(float lr) { offload_lr_ = lr; }
  // gradient accumulation over n micro-steps (train_step(zero=true) then n-1 x
  // zero=false): SLOW granules park their partial gradients in pinned host memory
  // between micro-steps and run the fused AdamW in the n-th backward only
  void set_grad_accumulation(int n);
  int grad_accumulation() const { return accum_n_; }
  // activation checkpointing of offloaded models: 0 off, 1 SLOW
  // layers (default), 2 every layer; a checkpointed layer keeps only its output and
  // recomputes the rest in its backward
  void set_activation_checkpointing(int policy);
  int activation_checkpointing() const { return ckpt_policy_; }
  OffloadStats offload_stats();
  void offload_stats_reset();
  void set_offload_skip_copies(bool skip);  // timing aid: same schedule, no PCIe traffic
  std::int64_t layer_granule_bytes() const { return layer_.numel * 18; }
  std::int64_t device_param_bytes() const;
  void routing_host(int g, int* selected, std::uint8_t* survived, int* raw_load, int* capacity,
                    int* dropped) const;
  // fp32 gate logits [T, E] of graph layer g from the last forward (MoE)
  void gate_logits_host(int g, float* out) const;

 private:
  struct NoInit {};
  Engine(ModelConfig config, NoInit, int ep_world = 1, int ep_rank = 0, bool force_ep = false);
  // offload plumbing (csrc/engine/offload.cpp)
  void offload_setup(const std::vector<int>& slow, int ring_slots);
  void offload_begin_forward(bool training);
  void offload_alloc_moments();
  void offload_acquire(int owned, bool backward);
  void offload_release(int owned, bool backward);
  void offload_prefetch_next(int after_owned, bool backward);
  void offload_finish_step();
  const float* view_base(const ParamView& v, int kind) const;
  void copy_view(const ParamView& v, int kind, float* host, bool to_host) const;
  float* slow_host_grad(int owned) const;
  float* slow_host_p32(int owned) const;
  float* slow_host_m(int owned, int which) const;
  std::uint16_t* slow_host_p16(int owned) const;
  void adamw_granule(float* p, float* g, float* m, float* v, void* p16, float lr, float bc1, float bc2);
  void build_layout();
  void allocate();
  void init_params(std::uint64_t seed);
  void refresh_bf16();
  void ensure_acts(int batch, int seq);
  float* lp(int owned, long long off) const;
  float* lg(int owned, long long off) const;
  void* lp16(int owned, long long off) const;
  const float* ep(long long off) const { return emb_p_.as<float>() + off; }
  float* eg(long long off) const { return emb_g_.as<float>() + off; }
  void* ep16(long long off) const { return emb_p16_.as<std::uint16_t>() + off; }
  void block_backward(int g, AttentionMode mode);
  void block_compute(int g, const float* x, AttentionMode mode);
  bool checkpointed(int g) const;
  void offload_check_micro(int next_micro) const;
  // bracket one kernel launch with profiling events (no-op when profiling is off)
  template <typename F>
  void prof(int cls, double flops, double bytes, F&& launch) {
    if (!prof_.on) {
      launch();
      return;
    }
    cudaEvent_t a = prof_.get(), b = prof_.get();
    cudaEventRecord(a, stream_);
    launch();
    cudaEventRecord(b, stream_);
    prof_.recs.push_back({cls, a, b, flops, bytes});
  }
  void gemm(int m, int n, int k, const void* a, int lda, bool a_mn, const void* b, int ldb,
            bool b_mn, int epi, void* c, int ldc, void* c2 = nullptr, int ldc2 = 0,
            const float* bias = nullptr, const void* aux = nullptr, int ldaux = 0,
            int group_mode = 0, int groups = 0, int seg_rows = 0, const int* counts = nullptr,
            int split_k = 1, float* bias_grad = nullptr);

  ModelConfig cfg_;
  int n_owned_ = 0;
  GranuleLayout layer_, emb_;
  long long layer_stride_ = 0;  // elements between owned layer granules (aligned)
  std::vector<ParamView> views_;
  DevBuf emb_p_, emb_g_, emb_p16_, emb_m_, emb_v_;
  DevBuf lay_p_, lay_g_, lay_p16_, lay_m_, lay_v_;
  bool has_opt_ = false;
  float b1_ = 0.9f, b2_ = 0.999f, eps_ = 1e-8f, wd_ = 0.01f;
  std::int64_t step_count_ = 0;
  cudaStream_t stream_ = nullptr;
  std::unique_ptr<Acts> acts_;
  DevBuf splitk_ws_;
  DevBuf dev_in_;   // tokens / targets / mask staging
  void* pinned_ = nullptr;      // two staging slots of pin_slot_ bytes (inputs + loss word)
  std::size_t pinned_bytes_ = 0;
  std::size_t pin_slot_ = 0;
  cudaEvent_t pin_ev_[2] = {nullptr, nullptr};  // the slot's step + loss read-back completed
  std::uint64_t pin_ticket_[2] = {0, 0};        // ticket whose loss the slot holds
  std::uint64_t async_seq_ = 0;
  Profiler prof_;
  // offload: res_idx_[owned] = resident slot in lay_* or -1 (SLOW)
  std::vector<int> res_idx_;
  std::vector<int> slow_;
  int n_res_ = 0;
  std::unique_ptr<OffloadState> off_;
  struct StepGraph {
    cudaGraphExec_t exec = nullptr;
    const void *tok = nullptr, *tgt = nullptr, *mask = nullptr, *loss = nullptr;
    int batch = 0, seq = 0, mode = 0;
    double denom = 0.0;
    bool zero = false;
    std::uint64_t kernels = 0;  // kernel launches the graph replays (p2r_launch_count)
    // buffers the graph baked in: any reallocation (another batch shape through any
    // entry point, a grown GEMM workspace) forces a re-capture
    std::uint64_t acts_gen = 0;
    const void* ws = nullptr;
  } step_graph_;
  std::uint64_t acts_gen_ = 0;  // bumped whenever ensure_acts reallocates the activation buffers
  std::uint64_t version_ = 1;
  float offload_lr_ = std::numeric_limits<float>::quiet_NaN();  // set_offload_lr() before use
  int accum_n_ = 1;            // micro-steps per optimizer step (offload)
  int micro_ = 0;              // micro-steps since zero_grads
  bool slow_applied_ = false;  // SLOW granules already took this step's fused AdamW
  int ckpt_policy_ = 1;
  void init_model(std::uint64_t seed, const std::vector<int>* slow, int ring_slots, int ep_world, int ep_rank,
                  bool ep_ctor);
  void allreduce_f32(float* buf, std::size_t n);  // DP sum over ranks on the model stream
  // expert / data parallelism
  int ep_world_ = 1, ep_rank_ = 0;
  bool force_ep_ = false;  // P2R_FORCE_EP=1: run the exchange path even at W = 1 (tests)
  void* comm_ = nullptr;   // ncclComm_t
  LoopbackGroup* loop_ = nullptr;
  std::unique_ptr<EpState> ep_;
  void ep_connect(int seg, int n_ye);
  void* ep_peer(int q, std::size_t off) const;
  void* ep_local(std::size_t off) const;
  void ep_signal(int ch);
  void ep_wait(int ch);
  std::size_t ep_ye_offset(int set) const;
  std::size_t ep_dxe_offset() const;
  // dispatch side of one exchange: rows of L's routing -> owners' slots, then signal + wait
  void ep_send(const void* src, int src_dtype, LayerActs& L, const float* w);
  void ep_pack_rows(void* compact, LayerActs& L);
  // return side: compact rows -> the sources' [E][seg] buffers at arena offset dst_off
  void ep_return(const void* compact, LayerActs& L, std::size_t dst_off);
};

// ncclGetUniqueId (dlopen'ed libnccl.so.2)
void comm_unique_id(char* out128);

// moe_dispatch on host logits via the routing kernel (bit-exact, model.cpp:294-332)
struct HostRouting {
  std::vector<int> selected;
  std::vector<std::uint8_t> survived;
  std::vector<int> raw_load, offsets, rows, slots;
  int capacity = 0, dropped = 0;
};
HostRouting moe_dispatch_host(const float* logits, int T, const MoEConfig& moe);

float lr_at(float peak, double warmup_ratio, std::int64_t total, std::int64_t step);

void cuda_check(cudaError_t e, const char* what);
void p2r_check(int status, const char* what);

}  // namespace p2r
