// Host engine: Engine / GradTape / AdamW / delink over the sm_100a kernel layer.
//
// Mirrors /root/reference/proj/core/src/model.cpp and optim.cpp (and the
// absent controller's per-micro-batch step) with identical
// names, parameter naming/order, init RNG and error messages. Differences are
// the B200 design: parameters of a layer live in one contiguous granule
// (fp32 master + grad + AdamW m/v + a bf16 shadow for the tensor cores),
// Q/K/V are stored fused as one [d, 3d] matrix (views keep the reference
// names), shared-layer gradients are accumulated in place by the dW GEMM
// epilogues (no scratch buffer + flush), and the forward/backward of a block
// is a handful of fused kernels instead of ~40 primitive closures.
#include "p2r/engine.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>

#include "comm_state.hpp"
#include "offload_state.hpp"

namespace p2r {
void count_launches(std::uint64_t n);  // status.cu: graph replays add their kernels to p2r_launch_count
}
#include "p2r_cuda.h"
#include "p2r_engine.h"

namespace p2r {

// ---------------------------------------------------------------- errors
void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

void p2r_check(int st, const char* what) {
  if (st == P2R_OK) return;
  const std::string msg = p2r_last_error();
  switch (st) {
    case P2R_EINVAL: throw std::invalid_argument(msg);
    case P2R_ERANGE: throw std::out_of_range(msg);
    case P2R_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(std::string(what) + ": " + msg);
  }
}

// ---------------------------------------------------------------- DevBuf
DevBuf::DevBuf(std::size_t n) : bytes(n) {
  if (n) cuda_check(cudaMalloc(&p, n), "cudaMalloc");
}
DevBuf::~DevBuf() {
  if (p) cudaFree(p);
}
DevBuf& DevBuf::operator=(DevBuf&& o) noexcept {
  if (this != &o) {
    if (p) cudaFree(p);
    p = o.p;
    bytes = o.bytes;
    o.p = nullptr;
    o.bytes = 0;
  }
  return *this;
}

// ---------------------------------------------------------------- configs (model.cpp:40-89)
void MoEConfig::validate() const {
  if (!enabled()) return;
  if (n_prototypes <= 0 || n_experts % n_prototypes != 0)
    throw std::invalid_argument("moe config: n_experts must be divisible by n_prototypes");
  if (n_shards <= 0 || n_experts % n_shards != 0)
    throw std::invalid_argument("moe config: n_experts must be divisible by n_shards");
  if (!(capacity_factor > 0.0f))
    throw std::invalid_argument("moe config: capacity_factor must be positive");
}

void ModelConfig::validate() const {
  if (d_model <= 0 || d_ff <= 0 || n_layers_graph <= 0 || n_heads <= 0 || vocab_size <= 0 ||
      seq_len <= 0)
    throw std::invalid_argument("model config: dimensions must be positive");
  if (d_model % n_heads != 0)
    throw std::invalid_argument("model config: d_model must be divisible by n_heads");
  if (n_layers_params != 1 && n_layers_params != n_layers_graph)
    throw std::invalid_argument("model config: n_layers_params must be 1 or n_layers_graph");
  moe.validate();
}

ModelConfig ModelConfig::as_shared() const {
  ModelConfig c = *this;
  c.n_layers_params = 1;
  return c;
}
ModelConfig ModelConfig::as_unshared() const {
  ModelConfig c = *this;
  c.n_layers_params = c.n_layers_graph;
  return c;
}

ParamCounts count_params(const ModelConfig& config) {
  config.validate();
  const std::int64_t d = config.d_model, dff = config.d_ff;
  ParamCounts out;
  out.embedding_params = static_cast<std::int64_t>(config.vocab_size) * d +
                         static_cast<std::int64_t>(config.seq_len) * d + 2 * d;
  std::int64_t layer = 4 * d * d + 4 * d;
  const std::int64_t ffn = d * dff + dff + dff * d + d;
  if (config.moe.enabled())
    layer += d * config.moe.n_experts + static_cast<std::int64_t>(config.moe.n_experts) * ffn;
  else
    layer += ffn;
  out.per_layer_params = layer;
  out.total_params = out.embedding_params + config.n_layers_params * layer;
  return out;
}

// ---------------------------------------------------------------- init (model.cpp:11-36)
namespace {
std::uint64_t fnv1a(const std::string& s) {
  std::uint64_t h = 1469598103934665603ull;
  for (char c : s) {
    h ^= static_cast<unsigned char>(c);
    h *= 1099511628211ull;
  }
  return h;
}
}  // namespace

std::uint64_t init_mix_seed(std::uint64_t seed, const std::string& name) {
  std::uint64_t z = seed ^ fnv1a(name);
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

void init_normal_host(float* out, std::size_t n, std::uint64_t seed, const std::string& name,
                      float stddev) {
  std::mt19937_64 rng(init_mix_seed(seed, name));
  std::normal_distribution<float> dist(0.0f, stddev);
  for (std::size_t i = 0; i < n; ++i) out[i] = dist(rng);
}

float lr_at(float peak, double warmup_ratio, std::int64_t total, std::int64_t step) {
  // LrSchedule::cosine + at (optim.cpp:8-24)
  if (total <= 0) throw std::invalid_argument("lr schedule: total_steps must be positive");
  const std::int64_t warm = std::max<std::int64_t>(
      1, static_cast<std::int64_t>(std::llround(warmup_ratio * static_cast<double>(total))));
  if (step < warm) return peak * static_cast<float>(step) / static_cast<float>(warm);
  const double span = static_cast<double>(std::max<std::int64_t>(1, total - warm));
  const double t = std::min(1.0, static_cast<double>(step - warm) / span);
  return static_cast<float>(peak * 0.5 * (1.0 + std::cos(t * 3.14159265358979323846)));
}

// ---------------------------------------------------------------- layout
long long GranuleLayout::add(long long n, bool decay) {
  const long long off = numel;
  segs.push_back({off, n, decay});
  numel += (n + 63) / 64 * 64;  // 256-byte aligned segments (TMA needs 16 B)
  return off;
}

// ---------------------------------------------------------------- activations
struct LayerActs {
  DevBuf xout, a16, mean1, rstd1, qkv16, o16, lse, x1, b16, mean2, rstd2;
  DevBuf hpre16, g16;  // dense FFN: GELU derivative (stored by the FFN1 epilogue for the backward), GELU output
  DevBuf b32, logits, sel, surv, pos, w, raw, counts, rows_pad, slots_pad, dropped;  // MoE
  DevBuf xe16, hpre_e16, ge16;
  // expert outputs in this rank's expert-major layout [E][seg] (bf16): a local
  // buffer, or a region of the expert-parallel arena the owners write into
  DevBuf ye16_own;
  void* ye16 = nullptr;
  DevBuf ccount, cprefix;  // expert parallel, owner side: compact rows per local expert / per source
  int ye_set = 0;          // index of ye16 among the arena's return buffers
  int capacity = 0;
};

struct Acts {
  int B = 0, S = 0, T = 0, seg = 0, cap = 0, vld = 0;
  DevBuf x0;
  std::vector<LayerActs> L;
  // activation checkpointing: layers with ckpt[g] keep only their output
  // L[g].xout; the rest of their activations live in the shared set `ck` and are
  // recomputed from the layer input in the backward
  std::vector<char> ckpt;
  LayerActs ck;
  DevBuf h16, meanf, rstdf, logits32, dlogits16, loss, loss_sum, ce_ws;
  DevBuf dres, dres16, tmp32, dx1, dx1_16, do16, dqkv16, dh16, dye16, dw, glogits, dsum;
  DevBuf dxe16_own;
  void* dxe16 = nullptr;  // expert-input gradients [E][seg] bf16 (local, or the arena's return buffer)
  DevBuf ln_ws, colsum_ws, embed_ws;
  // Dense FFN2 bias gradient: the LayerNorm backward that produces dres also writes
  // its per-block column sums here; the consuming layer's LN2 backward finishes them
  // into db2. db2_for = the graph layer they belong to (-1: none staged).
  DevBuf db2_stage;
  int db2_blocks = 0, db2_for = -1;
  DevBuf tokens, targets, mask;
  DevBuf yc16, dxc16;  // expert parallel, owner side: compact expert outputs / input gradients
};

// ---------------------------------------------------------------- expert-parallel exchange
std::size_t Engine::ep_ye_offset(int set) const { return ep_->off_ye + ep_->ye_bytes * static_cast<std::size_t>(set); }
std::size_t Engine::ep_dxe_offset() const { return ep_->off_dxe; }

void Engine::ep_send(const void* src, int src_dtype, LayerActs& L, const float* w) {
  const int W = ep_world_, E = cfg_.moe.n_experts;
  std::vector<void*> slots(static_cast<std::size_t>(W));
  std::vector<int*> cnts(static_cast<std::size_t>(W));
  for (int q = 0; q < W; ++q) {
    slots[static_cast<std::size_t>(q)] = ep_peer(q, ep_->off_slot);
    cnts[static_cast<std::size_t>(q)] = static_cast<int*>(ep_peer(q, ep_->off_cnt));
  }
  p2r_check(p2r_ep_send_rows(src, src_dtype, cfg_.d_model, E, acts_->seg, L.rows_pad.as<int>(), L.slots_pad.as<int>(),
                             L.counts.as<int>(), w, cfg_.moe.n_prototypes, W, ep_rank_, slots.data(), cnts.data(),
                             stream_),
            "ep send");
  ep_signal(0);
  ep_wait(0);
}

void Engine::ep_pack_rows(void* compact, LayerActs& L) {
  const int W = ep_world_, El = cfg_.moe.n_experts / W;
  p2r_check(p2r_ep_pack(ep_local(ep_->off_slot), static_cast<const int*>(ep_local(ep_->off_cnt)), cfg_.d_model,
                        acts_->seg, El, W, compact, L.ccount.as<int>(), L.cprefix.as<int>(), stream_),
            "ep pack");
}

void Engine::ep_return(const void* compact, LayerActs& L, std::size_t dst_off) {
  const int W = ep_world_, El = cfg_.moe.n_experts / W;
  std::vector<void*> dst(static_cast<std::size_t>(W));
  for (int q = 0; q < W; ++q) dst[static_cast<std::size_t>(q)] = ep_peer(q, dst_off);
  p2r_check(p2r_ep_return_rows(compact, L.cprefix.as<int>(), cfg_.d_model, acts_->seg, El, W, ep_rank_, dst.data(),
                               stream_),
            "ep return");
  ep_signal(1);
  ep_wait(1);
}

// ---------------------------------------------------------------- Engine
Engine::Engine(ModelConfig config, std::uint64_t seed) : cfg_(std::move(config)) {
  init_model(seed, nullptr, 0, 1, 0, false);
}

Engine::Engine(ModelConfig config, std::uint64_t seed, const std::vector<int>& slow, int ring_slots)
    : cfg_(std::move(config)) {
  init_model(seed, &slow, ring_slots, 1, 0, false);
}

Engine::Engine(ModelConfig config, std::uint64_t seed, int ep_world, int ep_rank) : cfg_(std::move(config)) {
  init_model(seed, nullptr, 0, ep_world, ep_rank, true);
}

Engine::Engine(ModelConfig config, std::uint64_t seed, const std::vector<int>& slow, int ring_slots, int ep_world,
             int ep_rank)
    : cfg_(std::move(config)) {
  init_model(seed, &slow, ring_slots, ep_world, ep_rank, true);
}

void Engine::init_model(std::uint64_t seed, const std::vector<int>* slow, int ring_slots, int ep_world, int ep_rank,
                       bool ep_ctor) {
  cfg_.validate();
  if (ep_world < 1 || ep_rank < 0 || ep_rank >= ep_world)
    throw std::invalid_argument("expert parallel: rank must be in [0, world)");
  ep_world_ = ep_world;
  ep_rank_ = ep_rank;
  if (ep_ctor) {  // P2R_FORCE_EP=1: run the exchange path even at world size 1 (tests)
    const char* f = std::getenv("P2R_FORCE_EP");
    force_ep_ = f != nullptr && f[0] == '1';
  }
  build_layout();
  if (slow) offload_setup(*slow, ring_slots);
  allocate();
  init_params(seed);
}

void Engine::set_grad_accumulation(int n) {
  if (n < 1) throw std::invalid_argument("offload: accumulation window must be >= 1 micro-step");
  accum_n_ = n;
}

void Engine::set_activation_checkpointing(int policy) {
  if (policy < 0 || policy > 2) throw std::invalid_argument("checkpointing: policy must be 0, 1 or 2");
  if (policy != ckpt_policy_) {
    ckpt_policy_ = policy;
    acts_.reset();  // the activation sets are laid out per policy
  }
}

Engine::Engine(ModelConfig config, NoInit, int ep_world, int ep_rank, bool force_ep) : cfg_(std::move(config)) {
  cfg_.validate();
  ep_world_ = ep_world;
  ep_rank_ = ep_rank;
  force_ep_ = force_ep;
  build_layout();
  allocate();
}

Engine::~Engine() {
  if (stream_) cudaStreamSynchronize(stream_);
  if (step_graph_.exec) cudaGraphExecDestroy(step_graph_.exec);
  comm_destroy();
  off_.reset();
  if (pinned_) cudaFreeHost(pinned_);
  for (cudaEvent_t e : pin_ev_)
    if (e) cudaEventDestroy(e);
  if (stream_) cudaStreamDestroy(stream_);
}

void Engine::build_layout() {
  const int d = cfg_.d_model, dff = cfg_.d_ff, V = cfg_.vocab_size, S = cfg_.seq_len;
  const int Eg = cfg_.moe.n_experts;
  if (Eg > 0 && Eg % ep_world_ != 0)
    throw std::invalid_argument("moe config: n_experts must be divisible by the expert-parallel world size");
  const int E = Eg > 0 ? Eg / ep_world_ : 0;  // experts held by this rank
  n_owned_ = cfg_.n_layers_params;
  n_res_ = n_owned_;
  res_idx_.resize(static_cast<std::size_t>(n_owned_));
  slow_.assign(static_cast<std::size_t>(n_owned_), 0);
  for (int i = 0; i < n_owned_; ++i) res_idx_[static_cast<std::size_t>(i)] = i;
  // embeddings granule (for_each_param order: tok, pos, final gain, final bias)
  emb_ = GranuleLayout{};
  emb_.tok = emb_.add(1LL * V * d, true);
  emb_.pos = emb_.add(1LL * S * d, true);
  emb_.fin_g = emb_.add(d, false);
  emb_.fin_b = emb_.add(d, false);
  // layer granule
  layer_ = GranuleLayout{};
  layer_.ln1_g = layer_.add(d, false);
  layer_.ln1_b = layer_.add(d, false);
  layer_.wqkv = layer_.add(3LL * d * d, true);  // [d, 3d] = wq | wk | wv
  layer_.wo = layer_.add(1LL * d * d, true);
  layer_.ln2_g = layer_.add(d, false);
  layer_.ln2_b = layer_.add(d, false);
  if (cfg_.moe.enabled()) {
    layer_.gate = layer_.add(1LL * d * Eg, true);  // replicated, routes over all experts
    layer_.w1 = layer_.add(1LL * E * d * dff, true);  // [E, d, dff]
    layer_.b1 = layer_.add(1LL * E * dff, false);     // [E, dff]
    layer_.w2 = layer_.add(1LL * E * dff * d, true);  // [E, dff, d]
    layer_.b2 = layer_.add(1LL * E * d, false);       // [E, d]
  } else {
    layer_.w1 = layer_.add(1LL * d * dff, true);
    layer_.b1 = layer_.add(dff, false);
    layer_.w2 = layer_.add(1LL * dff * d, true);
    layer_.b2 = layer_.add(d, false);
  }
  layer_stride_ = (layer_.numel + 63) / 64 * 64;

  // reference-named views, Engine::for_each_param order (model.cpp:188-198)
  views_.clear();
  views_.push_back({"embed.tok", -1, emb_.tok, V, d, d, {V, d}});
  views_.push_back({"embed.pos", -1, emb_.pos, S, d, d, {S, d}});
  views_.push_back({"final_norm.gain", -1, emb_.fin_g, 1, d, d, {d}});
  views_.push_back({"final_norm.bias", -1, emb_.fin_b, 1, d, d, {d}});
  for (int i = 0; i < n_owned_; ++i) {
    const std::string pre = "layer." + std::to_string(i) + ".";
    views_.push_back({pre + "ln1.gain", i, layer_.ln1_g, 1, d, d, {d}});
    views_.push_back({pre + "ln1.bias", i, layer_.ln1_b, 1, d, d, {d}});
    views_.push_back({pre + "attn.wq", i, layer_.wqkv, d, d, 3 * d, {d, d}});
    views_.push_back({pre + "attn.wk", i, layer_.wqkv + d, d, d, 3 * d, {d, d}});
    views_.push_back({pre + "attn.wv", i, layer_.wqkv + 2LL * d, d, d, 3 * d, {d, d}});
    views_.push_back({pre + "attn.wo", i, layer_.wo, d, d, d, {d, d}});
    views_.push_back({pre + "ln2.gain", i, layer_.ln2_g, 1, d, d, {d}});
    views_.push_back({pre + "ln2.bias", i, layer_.ln2_b, 1, d, d, {d}});
    if (!cfg_.moe.enabled()) {
      views_.push_back({pre + "ffn.w1", i, layer_.w1, d, dff, dff, {d, dff}});
      views_.push_back({pre + "ffn.b1", i, layer_.b1, 1, dff, dff, {dff}});
      views_.push_back({pre + "ffn.w2", i, layer_.w2, dff, d, d, {dff, d}});
      views_.push_back({pre + "ffn.b2", i, layer_.b2, 1, d, d, {d}});
    } else {
      views_.push_back({pre + "moe.gate", i, layer_.gate, d, Eg, Eg, {d, Eg}});
      for (int e = 0; e < E; ++e) {
        // global expert index: rank r owns experts [r*E, (r+1)*E) (model.cpp:334-340)
        const std::string ep = pre + "moe.expert." + std::to_string(ep_rank_ * E + e) + ".";
        views_.push_back({ep + "w1", i, layer_.w1 + 1LL * e * d * dff, d, dff, dff, {d, dff}});
        views_.push_back({ep + "b1", i, layer_.b1 + 1LL * e * dff, 1, dff, dff, {dff}});
        views_.push_back({ep + "w2", i, layer_.w2 + 1LL * e * dff * d, dff, d, d, {dff, d}});
        views_.push_back({ep + "b2", i, layer_.b2 + 1LL * e * d, 1, d, d, {d}});
      }
    }
  }
}

void Engine::allocate() {
  cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
  const std::size_t eb = static_cast<std::size_t>(emb_.numel);
  const std::size_t lb = static_cast<std::size_t>(layer_stride_) * std::max(n_res_, 1);
  emb_p_ = DevBuf(eb * 4);
  emb_g_ = DevBuf(eb * 4);
  emb_p16_ = DevBuf(eb * 2);
  lay_p_ = DevBuf(lb * 4);
  lay_g_ = DevBuf(lb * 4);
  lay_p16_ = DevBuf(lb * 2);
  cuda_check(cudaMemsetAsync(emb_p_.p, 0, eb * 4, stream_), "memset");
  cuda_check(cudaMemsetAsync(emb_g_.p, 0, eb * 4, stream_), "memset");
  cuda_check(cudaMemsetAsync(lay_p_.p, 0, lb * 4, stream_), "memset");
  cuda_check(cudaMemsetAsync(lay_g_.p, 0, lb * 4, stream_), "memset");
}

float* Engine::lp(int o, long long off) const {
  const int r = res_idx_[static_cast<std::size_t>(o)];
  if (r < 0) return offload_slot_ptr(*off_, o, 0) + off;
  return lay_p_.as<float>() + r * layer_stride_ + off;
}
float* Engine::lg(int o, long long off) const {
  const int r = res_idx_[static_cast<std::size_t>(o)];
  if (r < 0) return offload_slot_ptr(*off_, o, 1) + off;
  return lay_g_.as<float>() + r * layer_stride_ + off;
}
void* Engine::lp16(int o, long long off) const {
  const int r = res_idx_[static_cast<std::size_t>(o)];
  if (r < 0) return reinterpret_cast<std::uint16_t*>(offload_slot_ptr(*off_, o, 4)) + off;
  return lay_p16_.as<std::uint16_t>() + r * layer_stride_ + off;
}

void Engine::init_params(std::uint64_t seed) {
  // model.cpp:128-164: gains 1, biases 0, matrices N(0, 0.02) per named tensor. Every
  // tensor draws from its own generator (seed mixed with its name), so tensors are
  // filled in parallel host threads (same values) and uploaded in order, in batches
  // of about 1 GiB of host memory.
  const bool trace = std::getenv("P2R_TRACE") != nullptr;
  const int nv = static_cast<int>(views_.size());
  const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  int i0 = 0;
  while (i0 < nv) {
    int i1 = i0;
    std::size_t batch = 0;
    while (i1 < nv && (i1 == i0 || batch < (std::size_t{1} << 28))) {
      batch += static_cast<std::size_t>(views_[static_cast<std::size_t>(i1)].rows) * views_[static_cast<std::size_t>(i1)].cols;
      ++i1;
    }
    std::vector<std::vector<float>> host(static_cast<std::size_t>(i1 - i0));
    std::atomic<int> next{i0};
    auto work = [&] {
      for (int i = next++; i < i1; i = next++) {
        const ParamView& v = views_[static_cast<std::size_t>(i)];
        std::vector<float>& h = host[static_cast<std::size_t>(i - i0)];
        const std::size_t n = static_cast<std::size_t>(v.rows) * v.cols;
        h.assign(n, 0.0f);
        const std::string& nm = v.name;
        auto ends_with = [&](const char* suf) {
          const std::size_t L = std::strlen(suf);
          return nm.size() >= L && nm.compare(nm.size() - L, L, suf) == 0;
        };
        if (ends_with(".gain")) {
          std::fill(h.begin(), h.end(), 1.0f);
        } else if (ends_with(".bias") || ends_with(".b1") || ends_with(".b2")) {
          // zeros
        } else {
          init_normal_host(h.data(), n, seed, nm);
        }
      }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < hw; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    for (int i = i0; i < i1; ++i) {
      const ParamView& v = views_[static_cast<std::size_t>(i)];
      if (trace)
        std::fprintf(stderr, "init %s granule %d off %lld rows %d cols %d ld %d\n", v.name.c_str(), v.granule, v.off,
                     v.rows, v.cols, v.ld);
      set_param(i, host[static_cast<std::size_t>(i - i0)].data());
    }
    i0 = i1;
  }
  refresh_bf16();
}

void Engine::refresh_bf16() {
  p2r_check(p2r_cast_bf16(emb_p_.as<float>(), emb_p16_.p, emb_.numel, stream_), "cast");
  if (n_res_ > 0)
    p2r_check(p2r_cast_bf16(lay_p_.as<float>(), lay_p16_.p, layer_stride_ * n_res_, stream_), "cast");
  for (int o = 0; o < n_owned_; ++o)
    if (res_idx_[static_cast<std::size_t>(o)] < 0) host_cast_bf16(slow_host_p32(o), slow_host_p16(o), layer_stride_);
}

const float* Engine::view_base(const ParamView& v, int kind) const {
  // kind: 0 param, 1 grad, 2 m, 3 v
  if (v.granule < 0) {
    const DevBuf* b = kind == 0 ? &emb_p_ : kind == 1 ? &emb_g_ : kind == 2 ? &emb_m_ : &emb_v_;
    return b->as<float>() + v.off;
  }
  const int r = res_idx_[static_cast<std::size_t>(v.granule)];
  if (r >= 0) {
    const DevBuf* b = kind == 0 ? &lay_p_ : kind == 1 ? &lay_g_ : kind == 2 ? &lay_m_ : &lay_v_;
    return b->as<float>() + r * layer_stride_ + v.off;
  }
  if (kind == 0) return slow_host_p32(v.granule) + v.off;
  if (kind == 1) {
    float* g = slow_host_grad(v.granule);
    if (g == nullptr)
      throw std::logic_error("offload: gradients of SLOW granules are consumed on device by the fused AdamW");
    return g + v.off;
  }
  return slow_host_m(v.granule, kind - 2) + v.off;
}

void Engine::copy_view(const ParamView& v, int kind, float* host, bool to_host) const {
  if (off_) offload_sync(*off_);
  float* base = const_cast<float*>(view_base(v, kind));
  const std::size_t w = static_cast<std::size_t>(v.cols) * 4, ld = static_cast<std::size_t>(v.ld) * 4;
  if (to_host)
    cuda_check(cudaMemcpy2DAsync(host, w, base, ld, w, v.rows, cudaMemcpyDefault, stream_), "copy view");
  else
    cuda_check(cudaMemcpy2DAsync(base, ld, host, w, w, v.rows, cudaMemcpyDefault, stream_), "copy view");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
}

void Engine::get_param(int i, float* host) const { copy_view(views_.at(static_cast<std::size_t>(i)), 0, host, true); }

void Engine::set_param(int i, const float* host) {
  ++version_;
  const ParamView& v = views_.at(static_cast<std::size_t>(i));
  copy_view(v, 0, const_cast<float*>(host), false);
  // keep the bf16 shadow in step with the master copy (linear span of the view)
  const long long span = static_cast<long long>(v.rows - 1) * v.ld + v.cols;
  if (v.granule >= 0 && res_idx_[static_cast<std::size_t>(v.granule)] < 0) {
    host_cast_bf16(slow_host_p32(v.granule) + v.off, slow_host_p16(v.granule) + v.off, span);
  } else {
    const float* src = v.granule < 0 ? ep(v.off) : lp(v.granule, v.off);
    void* dst = v.granule < 0 ? ep16(v.off) : lp16(v.granule, v.off);
    p2r_check(p2r_cast_bf16(src, dst, span, stream_), "cast");
  }
}

void Engine::get_grad(int i, float* host) const { copy_view(views_.at(static_cast<std::size_t>(i)), 1, host, true); }

void Engine::get_moment(int i, int which, float* host) const {
  if (!has_opt_) throw std::logic_error("adamw: optimizer not attached");
  copy_view(views_.at(static_cast<std::size_t>(i)), 2 + which, host, true);
}

void Engine::set_moment(int i, int which, const float* host) {
  ++version_;
  if (!has_opt_) throw std::logic_error("adamw: optimizer not attached");
  if (which != 0 && which != 1) throw std::invalid_argument("adamw: moment index must be 0 (m) or 1 (v)");
  copy_view(views_.at(static_cast<std::size_t>(i)), 2 + which, const_cast<float*>(host), false);
}

std::int64_t Engine::grad_bytes() const {
  return (emb_.numel + layer_stride_ * n_res_) * 4;
}

void Engine::zero_grads() {
  ++version_;
  cuda_check(cudaMemsetAsync(emb_g_.p, 0, emb_g_.bytes, stream_), "zero grads");
  cuda_check(cudaMemsetAsync(lay_g_.p, 0, lay_g_.bytes, stream_), "zero grads");
  if (off_) {  // SLOW granules: drop the parked partial gradients, restart the window
    std::fill(off_->hgrad_valid.begin(), off_->hgrad_valid.end(), 0);
    micro_ = 0;
  }
}

// ---------------------------------------------------------------- activations
void Engine::ensure_acts(int B, int S) {
  const int T = B * S;
  if (acts_ && acts_->B == B && acts_->S == S) return;
  acts_.reset();
  auto A = std::make_unique<Acts>();
  const int d = cfg_.d_model, dff = cfg_.d_ff, H = cfg_.n_heads, V = cfg_.vocab_size;
  const int E = cfg_.moe.n_experts, k = cfg_.moe.n_prototypes;
  A->B = B;
  A->S = S;
  A->T = T;
  A->vld = (V + 7) / 8 * 8;
  const std::size_t Td = static_cast<std::size_t>(T) * d;
  if (cfg_.moe.enabled()) {
    A->cap = p2r_moe_capacity(cfg_.moe.capacity_factor, T, E, k);
    const int rows = std::min(A->cap, T);
    A->seg = std::max(128, (rows + 127) / 128 * 128);
  }
  const std::size_t ES = static_cast<std::size_t>(E) * A->seg;
  A->x0 = DevBuf(Td * 4);
  A->L.resize(static_cast<std::size_t>(cfg_.n_layers_graph));
  A->ckpt.assign(static_cast<std::size_t>(cfg_.n_layers_graph), 0);
  bool any_ckpt = false;
  for (int g = 0; g < cfg_.n_layers_graph; ++g) {
    const bool c = checkpointed(g);
    A->ckpt[static_cast<std::size_t>(g)] = c ? 1 : 0;
    any_ckpt = any_ckpt || c;
  }
  std::vector<LayerActs*> full;
  for (int g = 0; g < cfg_.n_layers_graph; ++g) {
    A->L[static_cast<std::size_t>(g)].xout = DevBuf(Td * 4);
    if (!A->ckpt[static_cast<std::size_t>(g)]) full.push_back(&A->L[static_cast<std::size_t>(g)]);
  }
  if (any_ckpt) full.push_back(&A->ck);
  for (LayerActs* lp_ : full) {
    LayerActs& l = *lp_;
    l.a16 = DevBuf(Td * 2);
    l.mean1 = DevBuf(T * 4);
    l.rstd1 = DevBuf(T * 4);
    l.qkv16 = DevBuf(Td * 3 * 2);
    l.o16 = DevBuf(Td * 2);
    l.lse = DevBuf(static_cast<std::size_t>(T) * H * 4);
    l.x1 = DevBuf(Td * 4);
    l.b16 = DevBuf(Td * 2);
    l.mean2 = DevBuf(T * 4);
    l.rstd2 = DevBuf(T * 4);
    if (!cfg_.moe.enabled()) {
      l.hpre16 = DevBuf(static_cast<std::size_t>(T) * dff * 2);
      l.g16 = DevBuf(static_cast<std::size_t>(T) * dff * 2);
    } else {
      l.capacity = A->cap;
      l.b32 = DevBuf(Td * 4);
      l.logits = DevBuf(static_cast<std::size_t>(T) * E * 4);
      l.sel = DevBuf(static_cast<std::size_t>(T) * k * 4);
      l.surv = DevBuf(static_cast<std::size_t>(T) * k);
      l.pos = DevBuf(static_cast<std::size_t>(T) * k * 4);
      l.w = DevBuf(static_cast<std::size_t>(T) * k * 4);
      l.raw = DevBuf(static_cast<std::size_t>(E) * 4);
      l.counts = DevBuf(static_cast<std::size_t>(E) * 4);
      l.rows_pad = DevBuf(ES * 4);
      l.slots_pad = DevBuf(ES * 4);
      l.dropped = DevBuf(4);
      l.xe16 = DevBuf(ES * d * 2);
      l.hpre_e16 = DevBuf(ES * dff * 2);
      l.ge16 = DevBuf(ES * dff * 2);
      if (!ep_active()) {
        l.ye16_own = DevBuf(ES * d * 2);
        l.ye16 = l.ye16_own.p;
      } else {
        const int El = E / ep_world_;
        l.ccount = DevBuf(static_cast<std::size_t>(El) * 4);
        l.cprefix = DevBuf(static_cast<std::size_t>(El) * (ep_world_ + 1) * 4);
      }
    }
  }
  A->h16 = DevBuf(Td * 2);
  A->meanf = DevBuf(T * 4);
  A->rstdf = DevBuf(T * 4);
  A->logits32 = DevBuf(static_cast<std::size_t>(T) * A->vld * 4);
  A->dlogits16 = DevBuf(static_cast<std::size_t>(T) * A->vld * 2);
  A->loss = DevBuf(4);
  A->loss_sum = DevBuf(8);
  A->ce_ws = DevBuf(p2r_cross_entropy_workspace(T));
  A->dres = DevBuf(Td * 4);
  A->dres16 = DevBuf(Td * 2);
  A->dx1 = DevBuf(Td * 4);
  A->dx1_16 = DevBuf(Td * 2);
  A->do16 = DevBuf(Td * 2);
  A->dqkv16 = DevBuf(Td * 3 * 2);
  A->dsum = DevBuf(static_cast<std::size_t>(T) * H * 4);
  if (!cfg_.moe.enabled()) {
    A->dh16 = DevBuf(static_cast<std::size_t>(T) * dff * 2);
  } else {
    A->dh16 = DevBuf(ES * dff * 2);
    A->tmp32 = DevBuf(Td * 4);  // fp32 sum of the dispatch backward (LN2's dy)
    A->dye16 = DevBuf(ES * d * 2);
    A->dw = DevBuf(static_cast<std::size_t>(T) * k * 4);
    if (!ep_active()) {
      A->dxe16_own = DevBuf(ES * d * 2);
      A->dxe16 = A->dxe16_own.p;
    } else {
      A->yc16 = DevBuf(ES * d * 2);
      A->dxc16 = DevBuf(ES * d * 2);
    }
    A->glogits = DevBuf(static_cast<std::size_t>(T) * E * 4);
  }
  A->ln_ws = DevBuf(p2r_layernorm_bwd_workspace(T, d));
  if (db2_fused()) {
    int nblk = 0;
    for (int f = 0; f < 4; ++f) nblk = std::max(nblk, p2r_layernorm_bwd_blocks(T, d, f));
    A->db2_stage = DevBuf(static_cast<std::size_t>(nblk) * d * 4);
  }
  const int bias_n = std::max(dff, d);
  A->colsum_ws = DevBuf(p2r_colsum_workspace(std::max(T, A->seg), bias_n, std::max(1, E)));
  A->embed_ws = DevBuf(p2r_embed_bwd_workspace(T, cfg_.vocab_size));
  A->tokens = DevBuf(static_cast<std::size_t>(T) * 4);
  A->targets = DevBuf(static_cast<std::size_t>(T) * 4);
  A->mask = DevBuf(static_cast<std::size_t>(T));
  if (cfg_.moe.enabled() && ep_active()) {
    // expert-parallel arena: the expert-output return buffer of every activation set
    // (one per stored layer + the shared checkpoint set) and the gradient return buffer
    std::vector<LayerActs*> sets;
    for (int g = 0; g < cfg_.n_layers_graph; ++g)
      if (!A->ckpt[static_cast<std::size_t>(g)]) sets.push_back(&A->L[static_cast<std::size_t>(g)]);
    if (any_ckpt) sets.push_back(&A->ck);
    ep_connect(A->seg, static_cast<int>(sets.size()));
    for (std::size_t i = 0; i < sets.size(); ++i) {
      sets[i]->ye16 = ep_local(ep_ye_offset(static_cast<int>(i)));
      sets[i]->ye_set = static_cast<int>(i);
    }
    A->dxe16 = ep_local(ep_dxe_offset());
  }
  acts_ = std::move(A);
  ++acts_gen_;
  const std::size_t slot = (static_cast<std::size_t>(T) * 9 + 63) / 64 * 64 + 64;  // inputs | loss word
  if (pin_slot_ < slot) {
    cuda_check(cudaStreamSynchronize(stream_), "pinned staging");  // no step reads the old slots
    if (pinned_) cudaFreeHost(pinned_);
    cuda_check(cudaMallocHost(&pinned_, 2 * slot), "pinned staging");
    pinned_bytes_ = 2 * slot;
    pin_slot_ = slot;
    pin_ticket_[0] = pin_ticket_[1] = 0;
  }
}

void Engine::gemm(int m, int n, int k, const void* a, int lda, bool a_mn, const void* b, int ldb,
                 bool b_mn, int epi, void* c, int ldc, void* c2, int ldc2, const float* bias,
                 const void* aux, int ldaux, int group_mode, int groups, int seg_rows,
                 const int* counts, int split_k, float* bias_grad) {
  p2r_gemm_args g{};
  g.m = m;
  g.n = n;
  g.k = k;
  g.a = a;
  g.lda = lda;
  g.a_mn_major = a_mn;
  g.b = b;
  g.ldb = ldb;
  g.b_mn_major = b_mn;
  g.epi = epi;
  g.c = c;
  g.ldc = ldc;
  g.c2 = c2;
  g.ldc2 = ldc2;
  g.bias = bias;
  g.aux = aux;
  g.ldaux = ldaux;
  g.group_mode = group_mode;
  g.groups = groups;
  g.seg_rows = seg_rows;
  g.counts = counts;
  g.split_k = split_k;
  g.bias_grad = bias_grad;
  if (split_k != 1 || bias_grad != nullptr) {
    const std::size_t need = p2r_gemm_workspace_bytes(&g);
    if (splitk_ws_.bytes < need) splitk_ws_ = DevBuf(need);
    p2r_set_workspace(splitk_ws_.p, splitk_ws_.bytes);
  }
  // algorithmic FLOPs: grouped GEMMs count the routed rows (T * k), not padding
  double rows_m = m, inner_k = k;
  if (group_mode == P2R_GROUP_M && acts_) rows_m = static_cast<double>(acts_->T) * cfg_.moe.n_prototypes;
  if (group_mode == P2R_GROUP_K && acts_) inner_k = static_cast<double>(acts_->T) * cfg_.moe.n_prototypes;
  const double flops = 2.0 * rows_m * n * inner_k;
  const double bytes = 2.0 * (rows_m * inner_k + static_cast<double>(n) * inner_k) +
                       (epi == P2R_EPI_BF16 || epi == P2R_EPI_BIAS_GELU || epi == P2R_EPI_DGELU ? 2.0 : 4.0) *
                           rows_m * n * (epi == P2R_EPI_ACC_F32 ? 2.0 : 1.0);
  prof(0, flops, bytes, [&] { p2r_check(p2r_gemm(&g, stream_), "gemm"); });
}

// ---------------------------------------------------------------- profiling
cudaEvent_t Profiler::get() {
  if (used == pool.size()) {
    cudaEvent_t e;
    cuda_check(cudaEventCreate(&e), "event");
    pool.push_back(e);
  }
  return pool[used++];
}

Profiler::~Profiler() {
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
}

void Engine::profile(int cls, std::int64_t* launches, double* ms, double* flops, double* bytes) {
  cuda_check(cudaStreamSynchronize(stream_), "profile sync");
  std::int64_t n = 0;
  double t = 0, f = 0, b = 0;
  for (const auto& r : prof_.recs) {
    if (r.cls != cls) continue;
    float e = 0;
    cuda_check(cudaEventElapsedTime(&e, r.a, r.b), "event time");
    ++n;
    t += e;
    f += r.flops;
    b += r.bytes;
  }
  *launches = n;
  *ms = t;
  *flops = f;
  *bytes = b;
}

void Engine::profile_reset() {
  cuda_check(cudaStreamSynchronize(stream_), "profile sync");
  prof_.recs.clear();
  prof_.used = 0;
}

void Engine::buffer(int which, void** ptr, std::size_t* bytes) const {
  if (which == 0) {
    *ptr = emb_g_.p;
    *bytes = emb_g_.bytes;
  } else if (which == 1) {
    *ptr = lay_g_.p;
    *bytes = lay_g_.bytes;
  } else {
    throw std::out_of_range("model buffer: unknown buffer id");
  }
}

// ---------------------------------------------------------------- forward pieces
DevTensor Engine::embed_forward(GradTape* tape, const int* d_tokens, int batch, int seq) {
  ++version_;
  if (batch <= 0) throw std::invalid_argument("forward: token count must be a multiple of batch");
  if (seq > cfg_.seq_len) throw std::invalid_argument("forward: sequence longer than configured seq_len");
  if (off_ && tape != nullptr && !off_->slow_list.empty()) {
    offload_check_micro(micro_ + 1);
    ++micro_;
  }
  ensure_acts(batch, seq);
  if (off_) offload_begin_forward(tape != nullptr);
  Acts& A = *acts_;
  const int d = cfg_.d_model;
  prof(P2R_PROF_EMBED, 0, 12.0 * A.T * d, [&] {
    p2r_check(p2r_embed_fwd(d_tokens, ep(emb_.tok), ep(emb_.pos), A.T, seq, d, A.x0.as<float>(), stream_), "embed");
  });
  if (tape) {
    tape->record([this, d_tokens, batch, seq]() {
      Acts& A2 = *acts_;
      A2.db2_for = -1;
      prof(P2R_PROF_EMBED, 0, 8.0 * A2.T * cfg_.d_model, [&] {
        p2r_check(p2r_embed_bwd(d_tokens, A2.dres.as<float>(), batch, seq, cfg_.d_model, cfg_.vocab_size,
                                eg(emb_.tok), eg(emb_.pos), A2.embed_ws.p, A2.embed_ws.bytes, stream_),
                  "embed bwd");
      });
    });
  }
  return DevTensor{A.T, d, A.x0.as<float>(), A.dres.as<float>(), A.dres16.p};
}

DevTensor Engine::block_forward(GradTape* tape, int g, const DevTensor& x, int batch, AttentionMode mode) {
  if (g < 0 || g >= cfg_.n_layers_graph) throw std::out_of_range("model: graph layer index out of range");
  Acts& A = *acts_;
  if (x.rows != A.T || batch != A.B) throw std::invalid_argument("block_forward: batch does not match embed_forward");
  const int o = owned_index_of_graph_layer(g);
  if (off_) offload_acquire(o, false);
  block_compute(g, x.data, mode);
  if (off_) offload_release(o, false);
  if (tape) tape->record([this, g, mode]() { block_backward(g, mode); });
  return DevTensor{A.T, cfg_.d_model, A.L[static_cast<std::size_t>(g)].xout.as<float>(), A.dres.as<float>(), A.dres16.p};
}

bool Engine::checkpointed(int g) const {
  if (!off_ || ckpt_policy_ == 0) return false;
  return ckpt_policy_ == 2 || slow_[static_cast<std::size_t>(owned_index_of_graph_layer(g))] != 0;
}

// The forward of graph layer g from input x (fp32 [T, d]) into its activation set
// (the shared checkpoint set for checkpointed layers) and its output L[g].xout. Run
// by block_forward, and again by block_backward to recompute a checkpointed layer.
void Engine::block_compute(int g, const float* xin_data, AttentionMode mode) {
  Acts& A = *acts_;
  LayerActs& L = A.ckpt[static_cast<std::size_t>(g)] ? A.ck : A.L[static_cast<std::size_t>(g)];
  float* xout = A.L[static_cast<std::size_t>(g)].xout.as<float>();
  const DevTensor x{A.T, cfg_.d_model, const_cast<float*>(xin_data), nullptr, nullptr};
  const int o = owned_index_of_graph_layer(g);
  const int T = A.T, d = cfg_.d_model, dff = cfg_.d_ff, H = cfg_.n_heads;
  const int causal = mode == AttentionMode::Causal ? 1 : 0;
  const double Td = static_cast<double>(T) * d;
  const double attn_flops = 2.0 * A.B * H * static_cast<double>(A.S) * A.S * (d / H) * (causal ? 1.0 : 2.0);
  // a = LN1(x)
  prof(P2R_PROF_LAYERNORM, 0, Td * 6 + 8.0 * T, [&] {
    p2r_check(p2r_layernorm_fwd(x.data, lp(o, layer_.ln1_g), lp(o, layer_.ln1_b), T, d, 1e-5f, L.a16.p, nullptr,
                                L.mean1.as<float>(), L.rstd1.as<float>(), stream_),
              "ln1");
  });
  // qkv = a . [wq|wk|wv]  (B = fused [d, 3d] bf16, N-major)
  gemm(T, 3 * d, d, L.a16.p, d, false, lp16(o, layer_.wqkv), 3 * d, true, P2R_EPI_BF16, L.qkv16.p, 3 * d);
  prof(P2R_PROF_ATTN_FWD, attn_flops, Td * 8, [&] {
    p2r_check(p2r_attention_fwd(L.qkv16.p, L.o16.p, L.lse.as<float>(), A.B, H, A.S, d, causal, stream_), "attn");
  });
  // x1 = x + o . wo
  gemm(T, d, d, L.o16.p, d, false, lp16(o, layer_.wo), d, true, P2R_EPI_F32, L.x1.p, d, nullptr, 0, nullptr,
       x.data, d);
  // b = LN2(x1)
  const bool moe = cfg_.moe.enabled();
  prof(P2R_PROF_LAYERNORM, 0, Td * (moe ? 10 : 6) + 8.0 * T, [&] {
    p2r_check(p2r_layernorm_fwd(L.x1.as<float>(), lp(o, layer_.ln2_g), lp(o, layer_.ln2_b), T, d, 1e-5f, L.b16.p,
                                moe ? L.b32.as<float>() : nullptr, L.mean2.as<float>(), L.rstd2.as<float>(), stream_),
              "ln2");
  });
  if (!moe) {
    gemm(T, dff, d, L.b16.p, d, false, lp16(o, layer_.w1), dff, true, P2R_EPI_BIAS_GELU, L.g16.p, dff, L.hpre16.p,
         dff, lp(o, layer_.b1));
    gemm(T, d, dff, L.g16.p, dff, false, lp16(o, layer_.w2), d, true, P2R_EPI_F32, xout, d, nullptr, 0,
         lp(o, layer_.b2), L.x1.p, d);
  } else {
    const int E = cfg_.moe.n_experts, k = cfg_.moe.n_prototypes, seg = A.seg;
    p2r_check(p2r_moe_gate_logits(L.b32.as<float>(), lp(o, layer_.gate), T, d, E, L.logits.as<float>(), stream_),
              "gate");
    p2r_check(p2r_moe_route(L.logits.as<float>(), T, E, k, A.cap, seg, L.sel.as<int>(), L.surv.as<std::uint8_t>(),
                            L.pos.as<int>(), L.raw.as<int>(), L.counts.as<int>(), L.rows_pad.as<int>(),
                            L.slots_pad.as<int>(), L.dropped.as<int>(), stream_),
              "route");
    p2r_check(p2r_moe_combine_weights(L.logits.as<float>(), T, E, k, L.sel.as<int>(), L.surv.as<std::uint8_t>(),
                                      L.w.as<float>(), stream_),
              "combine weights");
    const bool ep = ep_active();
    if (!ep) {
      // local experts: expert-major rows [E][seg] zero-padded to 128, grouped GEMMs over E groups
      prof(P2R_PROF_MOE, 0, 4.0 * T * d, [&] {
        p2r_check(p2r_moe_dispatch(L.b16.p, 1, d, E, seg, L.rows_pad.as<int>(), L.slots_pad.as<int>(),
                                   L.counts.as<int>(), nullptr, k, L.xe16.p, 0, stream_),
                  "dispatch");
      });
      gemm(E * seg, dff, d, L.xe16.p, d, false, lp16(o, layer_.w1), dff, true, P2R_EPI_BIAS_GELU, L.ge16.p, dff,
           L.hpre_e16.p, dff, lp(o, layer_.b1), nullptr, 0, P2R_GROUP_M, E, seg, L.counts.as<int>());
      gemm(E * seg, d, dff, L.ge16.p, dff, false, lp16(o, layer_.w2), d, true, P2R_EPI_BF16, L.ye16, d, nullptr, 0,
           lp(o, layer_.b2), nullptr, 0, P2R_GROUP_M, E, seg, L.counts.as<int>());
    } else {
      // expert parallel (csrc/ep.cu): the routed rows go straight into their owners'
      // slots; each owner packs them per local expert (exact counts, W*seg rows per
      // group), runs the grouped GEMMs, and returns the outputs into the sources'
      // expert-major layout (L.ye16 is this rank's arena region the owners write)
      const int El = E / ep_world_, gseg = ep_world_ * seg;
      prof(P2R_PROF_MOE, 0, 4.0 * T * d, [&] { ep_send(L.b16.p, 1, L, nullptr); });
      ep_pack_rows(L.xe16.p, L);
      gemm(El * gseg, dff, d, L.xe16.p, d, false, lp16(o, layer_.w1), dff, true, P2R_EPI_BIAS_GELU, L.ge16.p, dff,
           L.hpre_e16.p, dff, lp(o, layer_.b1), nullptr, 0, P2R_GROUP_M, El, gseg, L.ccount.as<int>());
      gemm(El * gseg, d, dff, L.ge16.p, dff, false, lp16(o, layer_.w2), d, true, P2R_EPI_BF16, A.yc16.p, d, nullptr, 0,
           lp(o, layer_.b2), nullptr, 0, P2R_GROUP_M, El, gseg, L.ccount.as<int>());
      ep_return(A.yc16.p, L, ep_ye_offset(L.ye_set));
    }
    p2r_check(p2r_moe_combine(L.ye16, T, d, k, seg, L.sel.as<int>(), L.pos.as<int>(), L.w.as<float>(),
                              L.x1.as<float>(), xout, stream_),
              "combine");
  }
}

// Backward of graph layer g. On entry A.dres/dres16 hold dL/d(block output);
// on exit they hold dL/d(block input). Parameter grads of the owned layer are
// accumulated in place (beta = 1), so in Pseudo mode the L graph layers sum
// into one buffer in reverse layer order exactly like the reference's
// per-layer flush (model.cpp:210-221).
void Engine::block_backward(int g, AttentionMode mode) {
  ++version_;
  Acts& A = *acts_;
  LayerActs& L = A.ckpt[static_cast<std::size_t>(g)] ? A.ck : A.L[static_cast<std::size_t>(g)];
  const int o = owned_index_of_graph_layer(g);
  if (off_) offload_acquire(o, true);
  const int T = A.T, d = cfg_.d_model, dff = cfg_.d_ff, H = cfg_.n_heads;
  const int causal = mode == AttentionMode::Causal ? 1 : 0;
  const float* xin = g == 0 ? A.x0.as<float>() : A.L[static_cast<std::size_t>(g - 1)].xout.as<float>();
  // activation checkpointing: recompute this layer's activations from its input
  // (the same kernels on the same operands, so bit-identical to the stored ones)
  if (A.ckpt[static_cast<std::size_t>(g)]) block_compute(g, xin, mode);
  float* dy = A.dres.as<float>();
  void* dy16 = A.dres16.p;
  if (!cfg_.moe.enabled()) {
    // FFN2: dW2 += g^T dy ; db2 += colsum(dy) ; dh = (dy W2^T) * gelu'(hpre)
    gemm(dff, d, T, L.g16.p, dff, true, dy16, d, true, P2R_EPI_ACC_F32, lg(o, layer_.w2), d, nullptr, 0, nullptr,
         nullptr, 0, 0, 0, 0, nullptr, 0 /* library picks the split */);
    if (A.db2_for != g) {  // dres was not produced by a staging LayerNorm backward
      prof(P2R_PROF_BIAS, 0, 4.0 * T * d, [&] {
        p2r_check(p2r_bias_grad(dy, 0, d, T, d, 1, 0, nullptr, lg(o, layer_.b2), 0, A.colsum_ws.as<float>(), stream_),
                  "db2");
      });
    }
    // db1 += colsum(dh) is folded into the GELU' epilogue (column partials of the bf16 dh)
    gemm(T, dff, d, dy16, d, false, lp16(o, layer_.w2), d, false, P2R_EPI_DGELU, A.dh16.p, dff, nullptr, 0, nullptr,
         L.hpre16.p, dff, 0, 0, 0, nullptr, 1, lg(o, layer_.b1));
    // FFN1: dW1 += b^T dh ; db = dh W1^T (bf16: the LN2 backward stages half the bytes;
    // do16 is free until the O-projection backward below)
    gemm(d, dff, T, L.b16.p, d, true, A.dh16.p, dff, true, P2R_EPI_ACC_F32, lg(o, layer_.w1), dff, nullptr, 0,
         nullptr, nullptr, 0, 0, 0, 0, nullptr, 0 /* library picks the split */);
    gemm(T, d, dff, A.dh16.p, dff, false, lp16(o, layer_.w1), dff, false, P2R_EPI_BF16, A.do16.p, d);
  } else {
    const int E = cfg_.moe.n_experts, k = cfg_.moe.n_prototypes, seg = A.seg;
    const int* cnt = L.counts.as<int>();
    const bool ep = ep_active();
    const int El = E / ep_world_;
    const int gseg = ep ? ep_world_ * seg : seg;
    const int* gcnt = ep ? L.ccount.as<int>() : cnt;
    const int G = ep ? El : E;
    // combine backward: dw = <dy, ye> (feeds the gate gradient, k > 1 only), dye = w * dy
    if (k > 1)
      p2r_check(p2r_moe_combine_bwd_weights(dy, L.ye16, T, d, k, seg, L.sel.as<int>(), L.pos.as<int>(),
                                            A.dw.as<float>(), stream_),
                "combine bwd");
    if (!ep) {
      p2r_check(p2r_moe_dispatch(dy, 0, d, E, seg, L.rows_pad.as<int>(), L.slots_pad.as<int>(), cnt, L.w.as<float>(),
                                 k, A.dye16.p, 0, stream_),
                "dispatch dy");
    } else {  // the scaled dy rows go to their owners, packed like the forward's rows
      ep_send(dy, 0, L, L.w.as<float>());
      ep_pack_rows(A.dye16.p, L);
    }
    gemm(dff, d, gseg, L.ge16.p, dff, true, A.dye16.p, d, true, P2R_EPI_ACC_F32, lg(o, layer_.w2), d, nullptr, 0,
         nullptr, nullptr, 0, P2R_GROUP_K, G, gseg, gcnt);
    p2r_check(p2r_bias_grad(A.dye16.p, 1, d, G * gseg, d, G, gseg, gcnt, lg(o, layer_.b2), d,
                            A.colsum_ws.as<float>(), stream_),
              "db2");
    gemm(G * gseg, dff, d, A.dye16.p, d, false, lp16(o, layer_.w2), d, false, P2R_EPI_DGELU, A.dh16.p, dff, nullptr,
         0, nullptr, L.hpre_e16.p, dff, P2R_GROUP_M, G, gseg, gcnt);
    gemm(d, dff, gseg, L.xe16.p, d, true, A.dh16.p, dff, true, P2R_EPI_ACC_F32, lg(o, layer_.w1), dff, nullptr, 0,
         nullptr, nullptr, 0, P2R_GROUP_K, G, gseg, gcnt);
    p2r_check(p2r_bias_grad(A.dh16.p, 1, dff, G * gseg, dff, G, gseg, gcnt, lg(o, layer_.b1), dff,
                            A.colsum_ws.as<float>(), stream_),
              "db1");
    // expert-input gradients in bf16 (local layout, or compact on the owner then returned)
    gemm(G * gseg, d, dff, A.dh16.p, dff, false, lp16(o, layer_.w1), dff, false, P2R_EPI_BF16,
         ep ? A.dxc16.p : A.dxe16, d, nullptr, 0, nullptr, nullptr, 0, P2R_GROUP_M, G, gseg, gcnt);
    if (ep) ep_return(A.dxc16.p, L, ep_dxe_offset());
    const float* glog = nullptr;
    if (k > 1) {  // top-1 => combine weights are exactly 1 and the gate gradient is exactly 0
      p2r_check(p2r_moe_gate_bwd(L.b32.as<float>(), L.w.as<float>(), A.dw.as<float>(), T, d, E, k, L.sel.as<int>(),
                                 L.surv.as<std::uint8_t>(), A.glogits.as<float>(), lg(o, layer_.gate), stream_),
                "gate bwd");
      glog = A.glogits.as<float>();
    }
    p2r_check(p2r_moe_dispatch_bwd(A.dxe16, T, d, k, seg, L.sel.as<int>(), L.pos.as<int>(), glog,
                                   lp(o, layer_.gate), E, A.tmp32.as<float>(), 0, stream_),
              "dispatch bwd");
  }
  const double Td = static_cast<double>(T) * d;
  const double attn_flops = 4.0 * A.B * H * static_cast<double>(A.S) * A.S * (d / H) * (causal ? 1.0 : 2.0);
  // LN2 backward: dx1 = dy + LN2'(db); its finish kernel also adds the staged
  // column sums of dy into db2 (dense layers whose dres came from a LayerNorm backward)
  const bool db2_staged = db2_fused() && A.db2_for == g;
  A.db2_for = -1;
  const bool moe = cfg_.moe.enabled();  // MoE: db is the fp32 sum of the dispatch backward
  prof(P2R_PROF_LAYERNORM, 0, moe ? Td * 18 : Td * 16, [&] {
    if (moe)
      p2r_check(p2r_layernorm_bwd_fused(A.tmp32.as<float>(), L.x1.as<float>(), L.mean2.as<float>(),
                                        L.rstd2.as<float>(), lp(o, layer_.ln2_g), dy, T, d, A.dx1.as<float>(),
                                        A.dx1_16.p, lg(o, layer_.ln2_g), lg(o, layer_.ln2_b), A.ln_ws.as<float>(),
                                        nullptr, nullptr, 0, nullptr, stream_),
                "ln2 bwd");
    else
      p2r_check(p2r_layernorm_bwd_fused_bf16(A.do16.p, L.x1.as<float>(), L.mean2.as<float>(), L.rstd2.as<float>(),
                                             lp(o, layer_.ln2_g), dy, T, d, A.dx1.as<float>(), A.dx1_16.p,
                                             lg(o, layer_.ln2_g), lg(o, layer_.ln2_b), A.ln_ws.as<float>(), nullptr,
                                             db2_staged ? A.db2_stage.as<float>() : nullptr,
                                             db2_staged ? A.db2_blocks : 0,
                                             db2_staged ? lg(o, layer_.b2) : nullptr, stream_),
                "ln2 bwd");
  });
  // O projection: dWo += o^T dx1 ; do = dx1 Wo^T
  gemm(d, d, T, L.o16.p, d, true, A.dx1_16.p, d, true, P2R_EPI_ACC_F32, lg(o, layer_.wo), d, nullptr, 0, nullptr,
       nullptr, 0, 0, 0, 0, nullptr, 0 /* library picks the split */);
  gemm(T, d, d, A.dx1_16.p, d, false, lp16(o, layer_.wo), d, false, P2R_EPI_BF16, A.do16.p, d);
  prof(P2R_PROF_ATTN_BWD, attn_flops, Td * 16, [&] {
    p2r_check(p2r_attention_bwd(L.qkv16.p, L.o16.p, L.lse.as<float>(), A.do16.p, A.dsum.as<float>(), A.dqkv16.p,
                                A.B, H, A.S, d, causal, stream_),
              "attn bwd");
  });
  // QKV: dWqkv += a^T dqkv ; da = dqkv Wqkv^T
  gemm(d, 3 * d, T, L.a16.p, d, true, A.dqkv16.p, 3 * d, true, P2R_EPI_ACC_F32, lg(o, layer_.wqkv), 3 * d, nullptr,
       0, nullptr, nullptr, 0, 0, 0, 0, nullptr, 0 /* library picks the split */);
  gemm(T, d, 3 * d, A.dqkv16.p, 3 * d, false, lp16(o, layer_.wqkv), 3 * d, false, P2R_EPI_BF16, A.do16.p, d);
  // LN1 backward: dx = dx1 + LN1'(da); for a dense layer below, also stage dx's column sums (its db2)
  const bool stage = db2_fused() && g > 0;
  prof(P2R_PROF_LAYERNORM, 0, Td * 16, [&] {
    p2r_check(p2r_layernorm_bwd_fused_bf16(A.do16.p, xin, L.mean1.as<float>(), L.rstd1.as<float>(),
                                           lp(o, layer_.ln1_g), A.dx1.as<float>(), T, d, dy, dy16,
                                           lg(o, layer_.ln1_g), lg(o, layer_.ln1_b), A.ln_ws.as<float>(),
                                           stage ? A.db2_stage.as<float>() : nullptr, nullptr, 0, nullptr, stream_),
              "ln1 bwd");
  });
  if (stage) {
    A.db2_blocks = p2r_layernorm_bwd_blocks(T, d, P2R_LN_RESID | P2R_LN_DY_BF16);
    A.db2_for = g - 1;
  }
  if (off_) offload_release(o, true);
}

DevTensor Engine::head_forward(GradTape* tape, const DevTensor& x) {
  Acts& A = *acts_;
  const int T = A.T, d = cfg_.d_model, V = cfg_.vocab_size;
  prof(P2R_PROF_LAYERNORM, 0, 6.0 * T * d + 8.0 * T, [&] {
    p2r_check(p2r_layernorm_fwd(x.data, ep(emb_.fin_g), ep(emb_.fin_b), T, d, 1e-5f, A.h16.p, nullptr,
                                A.meanf.as<float>(), A.rstdf.as<float>(), stream_),
              "final ln");
  });
  // logits = h . tok^T  (tied head, matmul_nt)
  gemm(T, V, d, A.h16.p, d, false, ep16(emb_.tok), d, false, P2R_EPI_F32, A.logits32.p, A.vld);
  if (tape) {
    const float* xin = x.data;
    tape->record([this, xin]() {
      ++version_;
      Acts& A2 = *acts_;
      const int T2 = A2.T, d2 = cfg_.d_model, V2 = cfg_.vocab_size;
      // dtok += dlogits^T h ; dh = dlogits . tok
      gemm(V2, d2, T2, A2.dlogits16.p, A2.vld, true, A2.h16.p, d2, true, P2R_EPI_ACC_F32, eg(emb_.tok), d2, nullptr,
           0, nullptr, nullptr, 0, 0, 0, 0, nullptr, 0 /* library picks the split */);
      gemm(T2, d2, V2, A2.dlogits16.p, A2.vld, false, ep16(emb_.tok), d2, true, P2R_EPI_BF16, A2.do16.p, d2);
      const bool stage = db2_fused();  // the last layer's db2 = column sums of this dres
      prof(P2R_PROF_LAYERNORM, 0, 12.0 * T2 * d2, [&] {
        p2r_check(p2r_layernorm_bwd_fused_bf16(A2.do16.p, xin, A2.meanf.as<float>(), A2.rstdf.as<float>(),
                                               ep(emb_.fin_g), nullptr, T2, d2, A2.dres.as<float>(), A2.dres16.p,
                                               eg(emb_.fin_g), eg(emb_.fin_b), A2.ln_ws.as<float>(),
                                               stage ? A2.db2_stage.as<float>() : nullptr, nullptr, 0, nullptr,
                                               stream_),
                  "final ln bwd");
      });
      if (stage) {
        A2.db2_blocks = p2r_layernorm_bwd_blocks(T2, d2, P2R_LN_DY_BF16);
        A2.db2_for = cfg_.n_layers_graph - 1;
      }
    });
  }
  return DevTensor{T, V, A.logits32.as<float>(), nullptr, nullptr};
}

DevTensor Engine::softmax_cross_entropy(GradTape* /*tape*/, const DevTensor& logits, const int* d_targets,
                                    const std::uint8_t* d_mask, double denom) {
  if (denom <= 0.0) throw std::invalid_argument("softmax_cross_entropy: denominator must be > 0");
  Acts& A = *acts_;
  prof(P2R_PROF_CE, 0, 6.0 * A.T * A.vld, [&] {
    p2r_check(p2r_cross_entropy(logits.data, A.T, cfg_.vocab_size, A.vld, d_targets, d_mask, denom, 1.0f,
                                A.dlogits16.p, A.vld, A.loss.as<float>(), A.loss_sum.as<double>(),
                                A.ce_ws.as<double>(), stream_),
              "cross entropy");
  });
  return DevTensor{1, 1, A.loss.as<float>(), nullptr, nullptr};
}

// A training micro-step of an offloaded model: the SLOW granules' fused AdamW runs in
// the backward of the accumulation window's last micro-step (set_grad_accumulation).
// Checked before anything is zeroed or launched, so a misuse leaves the state intact.
void Engine::offload_check_micro(int next_micro) const {
  if (!off_ || off_->slow_list.empty()) return;
  if (next_micro > accum_n_)
    throw std::logic_error(
        "offload: gradient accumulation past the window; call set_grad_accumulation(n) or start with zero=true");
  if (slow_applied_)
    throw std::logic_error("offload: adamw_step(lr) was not called after the last optimizer step's backward");
  if (has_opt_ && next_micro == accum_n_ && std::isnan(offload_lr_))
    throw std::logic_error("offload: call set_offload_lr(lr) before the backward that applies AdamW");
}

void Engine::train_step_device(const int* d_tokens, const int* d_targets, const std::uint8_t* d_mask, int batch,
                              int seq, double denom, AttentionMode mode, bool zero, float* loss_dev) {
  if (off_) offload_check_micro(zero ? 1 : micro_ + 1);
  if (zero) zero_grads();
  GradTape tape;
  DevTensor x = embed_forward(&tape, d_tokens, batch, seq);
  for (int g = 0; g < cfg_.n_layers_graph; ++g) x = block_forward(&tape, g, x, batch, mode);
  DevTensor logits = head_forward(&tape, x);
  DevTensor loss = softmax_cross_entropy(&tape, logits, d_targets, d_mask, denom);
  tape.backward();  // the fused cross-entropy already seeded dlogits for d loss = 1
  flush_shared_layer_grads();
  if (loss_dev && loss_dev != loss.data)
    cuda_check(cudaMemcpyAsync(loss_dev, loss.data, 4, cudaMemcpyDeviceToDevice, stream_), "loss copy");
}

void Engine::train_step_device_graph(const int* d_tokens, const int* d_targets, const std::uint8_t* d_mask, int batch,
                                    int seq, double denom, AttentionMode mode, bool zero, float* loss_dev) {
  // (a dense model's communicator is only used by allreduce_grads, outside the step)
  // (single-rank MoE qualifies: routing, counts and the grouped GEMMs' tile lists stay on
  // the device; the expert-parallel exchange's stream flag operations are kept eager)
  if (off_ || (cfg_.moe.enabled() && ep_active()) || prof_.on)
    throw std::logic_error("train_step_device_graph: needs a resident, single-rank, unprofiled model");
  StepGraph& G = step_graph_;
  ensure_acts(batch, seq);  // (a no-op unless the shape changed: then the generation moves on)
  const bool same = G.exec && G.tok == d_tokens && G.tgt == d_targets && G.mask == d_mask && G.loss == loss_dev &&
                    G.batch == batch && G.seq == seq && G.denom == denom && G.mode == static_cast<int>(mode) &&
                    G.zero == zero && G.acts_gen == acts_gen_ && G.ws == splitk_ws_.p;
  if (same) {
    cuda_check(cudaGraphLaunch(G.exec, stream_), "step graph launch");
    p2r::count_launches(G.kernels);
    return;
  }
  if (G.exec) {
    cuda_check(cudaGraphExecDestroy(G.exec), "step graph destroy");
    G.exec = nullptr;
  }
  // this call's step runs eagerly (lazy allocations, kernel attributes, split-K
  // counters all happen outside the capture), then the same launches are captured
  train_step_device(d_tokens, d_targets, d_mask, batch, seq, denom, mode, zero, loss_dev);
  cudaGraph_t graph = nullptr;
  const std::uint64_t k0 = p2r_launch_count();
  cuda_check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "step graph capture");
  try {
    train_step_device(d_tokens, d_targets, d_mask, batch, seq, denom, mode, zero, loss_dev);
  } catch (...) {
    cudaStreamEndCapture(stream_, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  cuda_check(cudaStreamEndCapture(stream_, &graph), "step graph capture end");
  G.kernels = p2r_launch_count() - k0;
  // the captured launches did not run: only the eager step above counts
  p2r::count_launches(static_cast<std::uint64_t>(0) - G.kernels);
  const cudaError_t e = cudaGraphInstantiate(&G.exec, graph, 0);
  cudaGraphDestroy(graph);
  cuda_check(e, "step graph instantiate");
  cuda_check(cudaGraphUpload(G.exec, stream_), "step graph upload");  // device-side copy made once, not per launch
  G.tok = d_tokens;
  G.tgt = d_targets;
  G.mask = d_mask;
  G.loss = loss_dev;
  G.batch = batch;
  G.seq = seq;
  G.denom = denom;
  G.mode = static_cast<int>(mode);
  G.zero = zero;
  G.acts_gen = acts_gen_;
  G.ws = splitk_ws_.p;
}

namespace {
void validate_ids(const int* ids, std::size_t n, int V, const char* msg) {
  for (std::size_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= V) throw std::out_of_range(msg);
}
}  // namespace

float Engine::train_step_host(const int* tokens, const int* targets, const std::uint8_t* mask, int batch, int seq,
                             double denom, AttentionMode mode, bool zero) {
  return loss_wait(train_step_host_async(tokens, targets, mask, batch, seq, denom, mode, zero));
}

std::uint64_t Engine::train_step_host_async(const int* tokens, const int* targets, const std::uint8_t* mask,
                                            int batch, int seq, double denom, AttentionMode mode, bool zero) {
  if (batch <= 0 || seq <= 0) throw std::invalid_argument("forward: token count must be a multiple of batch");
  if (seq > cfg_.seq_len) throw std::invalid_argument("forward: sequence longer than configured seq_len");
  if (denom <= 0.0) throw std::invalid_argument("softmax_cross_entropy: denominator must be > 0");
  const std::size_t T = static_cast<std::size_t>(batch) * seq;
  validate_ids(tokens, T, cfg_.vocab_size, "embedding_lookup: id out of range");
  for (std::size_t i = 0; i < T; ++i)
    if ((mask == nullptr || mask[i] != 0) && (targets[i] < 0 || targets[i] >= cfg_.vocab_size))
      throw std::out_of_range("softmax_cross_entropy: target out of range");
  ensure_acts(batch, seq);
  Acts& A = *acts_;
  const int sl = static_cast<int>(async_seq_ & 1);
  if (!pin_ev_[sl]) cuda_check(cudaEventCreateWithFlags(&pin_ev_[sl], cudaEventDisableTiming), "staging event");
  if (pin_ticket_[sl] != 0) cuda_check(cudaEventSynchronize(pin_ev_[sl]), "staging slot");  // step - 2 is done
  char* pin = static_cast<char*>(pinned_) + sl * pin_slot_;
  std::memcpy(pin, tokens, T * 4);
  std::memcpy(pin + T * 4, targets, T * 4);
  if (mask) std::memcpy(pin + T * 8, mask, T);
  cuda_check(cudaMemcpyAsync(A.tokens.p, pin, T * 4, cudaMemcpyHostToDevice, stream_), "h2d");
  cuda_check(cudaMemcpyAsync(A.targets.p, pin + T * 4, T * 4, cudaMemcpyHostToDevice, stream_), "h2d");
  if (mask) cuda_check(cudaMemcpyAsync(A.mask.p, pin + T * 8, T, cudaMemcpyHostToDevice, stream_), "h2d");
  // resident, MoE-free, single-rank steps replay one CUDA graph (P2R_STEP_GRAPH=0: eager launches)
  static const bool graph_on = [] {
    const char* e = std::getenv("P2R_STEP_GRAPH");
    return e == nullptr || std::atoi(e) != 0;
  }();
  if (graph_on && !off_ && !(cfg_.moe.enabled() && ep_active()) && !prof_.on)
    train_step_device_graph(A.tokens.as<int>(), A.targets.as<int>(), mask ? A.mask.as<std::uint8_t>() : nullptr, batch,
                            seq, denom, mode, zero, nullptr);
  else
    train_step_device(A.tokens.as<int>(), A.targets.as<int>(), mask ? A.mask.as<std::uint8_t>() : nullptr, batch, seq,
                      denom, mode, zero, nullptr);
  float* lh = reinterpret_cast<float*>(pin + pin_slot_ - 64);
  cuda_check(cudaMemcpyAsync(lh, A.loss.p, 4, cudaMemcpyDeviceToHost, stream_), "d2h loss");
  cuda_check(cudaEventRecord(pin_ev_[sl], stream_), "staging event");
  pin_ticket_[sl] = ++async_seq_;
  return pin_ticket_[sl];
}

float Engine::loss_wait(std::uint64_t ticket) {
  const int sl = static_cast<int>((ticket - 1) & 1);
  if (ticket == 0 || pin_ticket_[sl] != ticket)
    throw std::logic_error("loss_wait: ticket is not one of the last two host steps");
  cuda_check(cudaEventSynchronize(pin_ev_[sl]), "step sync");
  return *reinterpret_cast<const float*>(static_cast<const char*>(pinned_) + sl * pin_slot_ + pin_slot_ - 64);
}

void Engine::forward_host(const int* tokens, int batch, int seq, AttentionMode mode, float* logits_out) {
  if (batch <= 0 || seq <= 0) throw std::invalid_argument("forward: token count must be a multiple of batch");
  if (seq > cfg_.seq_len) throw std::invalid_argument("forward: sequence longer than configured seq_len");
  const std::size_t T = static_cast<std::size_t>(batch) * seq;
  validate_ids(tokens, T, cfg_.vocab_size, "embedding_lookup: id out of range");
  ensure_acts(batch, seq);
  Acts& A = *acts_;
  cuda_check(cudaMemcpyAsync(A.tokens.p, tokens, T * 4, cudaMemcpyHostToDevice, stream_), "h2d");
  DevTensor x = embed_forward(nullptr, A.tokens.as<int>(), batch, seq);
  for (int g = 0; g < cfg_.n_layers_graph; ++g) x = block_forward(nullptr, g, x, batch, mode);
  DevTensor logits = head_forward(nullptr, x);
  cuda_check(cudaMemcpy2DAsync(logits_out, static_cast<std::size_t>(cfg_.vocab_size) * 4, logits.data,
                               static_cast<std::size_t>(A.vld) * 4, static_cast<std::size_t>(cfg_.vocab_size) * 4, T,
                               cudaMemcpyDeviceToHost, stream_),
             "d2h logits");
  cuda_check(cudaStreamSynchronize(stream_), "forward sync");
}

void Engine::routing_host(int g, int* selected, std::uint8_t* survived, int* raw_load, int* capacity,
                         int* dropped) const {
  if (!cfg_.moe.enabled()) throw std::logic_error("routing: dense model");
  if (!acts_) throw std::logic_error("routing: no forward pass yet");
  const LayerActs& L = acts_->ckpt.at(static_cast<std::size_t>(g)) ? acts_->ck : acts_->L.at(static_cast<std::size_t>(g));
  const std::size_t Tk = static_cast<std::size_t>(acts_->T) * cfg_.moe.n_prototypes;
  cuda_check(cudaMemcpyAsync(selected, L.sel.p, Tk * 4, cudaMemcpyDeviceToHost, stream_), "d2h");
  cuda_check(cudaMemcpyAsync(survived, L.surv.p, Tk, cudaMemcpyDeviceToHost, stream_), "d2h");
  cuda_check(cudaMemcpyAsync(raw_load, L.raw.p, cfg_.moe.n_experts * 4, cudaMemcpyDeviceToHost, stream_), "d2h");
  cuda_check(cudaMemcpyAsync(dropped, L.dropped.p, 4, cudaMemcpyDeviceToHost, stream_), "d2h");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  *capacity = L.capacity;
}

void Engine::gate_logits_host(int g, float* out) const {
  if (!cfg_.moe.enabled()) throw std::logic_error("routing: dense model");
  if (!acts_) throw std::logic_error("routing: no forward pass yet");
  const LayerActs& L = acts_->ckpt.at(static_cast<std::size_t>(g)) ? acts_->ck : acts_->L.at(static_cast<std::size_t>(g));
  cuda_check(cudaMemcpyAsync(out, L.logits.p, static_cast<std::size_t>(acts_->T) * cfg_.moe.n_experts * 4,
                             cudaMemcpyDeviceToHost, stream_),
             "d2h");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
}

// ---------------------------------------------------------------- AdamW (optim.cpp:28-70)
void Engine::adamw_attach(float b1, float b2, float eps, float wd) {
  b1_ = b1;
  b2_ = b2;
  eps_ = eps;
  wd_ = wd;
  if (!has_opt_) {
    emb_m_ = DevBuf(emb_p_.bytes);
    emb_v_ = DevBuf(emb_p_.bytes);
    lay_m_ = DevBuf(lay_p_.bytes);
    lay_v_ = DevBuf(lay_p_.bytes);
    cuda_check(cudaMemsetAsync(emb_m_.p, 0, emb_m_.bytes, stream_), "memset");
    cuda_check(cudaMemsetAsync(emb_v_.p, 0, emb_v_.bytes, stream_), "memset");
    cuda_check(cudaMemsetAsync(lay_m_.p, 0, lay_m_.bytes, stream_), "memset");
    cuda_check(cudaMemsetAsync(lay_v_.p, 0, lay_v_.bytes, stream_), "memset");
    has_opt_ = true;
    if (off_) offload_alloc_moments();
  }
}

void Engine::adamw_step(float lr) {
  ++version_;
  if (!has_opt_) throw std::logic_error("adamw: unregistered parameter embed.tok");
  // checks first: a throw must leave the step count and every moment untouched
  if (off_ && !off_->slow_list.empty()) {
    if (!slow_applied_)
      throw std::logic_error(
          "offload: adamw_step before the accumulation window's last backward (SLOW granules not updated)");
    if (lr != offload_lr_)
      throw std::invalid_argument("adamw: offloaded granules were updated with set_offload_lr(); pass the same lr");
  }
  ++step_count_;
  slow_applied_ = false;
  const float bc1 = 1.0f - std::pow(b1_, static_cast<float>(step_count_));
  const float bc2 = 1.0f - std::pow(b2_, static_cast<float>(step_count_));
  auto run = [&](const GranuleLayout& lay, float* p, float* g, float* m, float* v, void* p16) {
    std::vector<long long> off, len;
    std::vector<int> dec;
    for (const auto& s : lay.segs) {
      off.push_back(s.off);
      len.push_back(s.len);
      dec.push_back(s.decay ? 1 : 0);
    }
    prof(P2R_PROF_ADAMW, 0, 30.0 * lay.numel, [&] {
      p2r_check(p2r_adamw_step(p, g, m, v, p16, off.data(), len.data(), dec.data(), static_cast<int>(off.size()),
                               b1_, b2_, eps_, wd_, lr, bc1, bc2, stream_),
                "adamw");
    });
  };
  run(emb_, emb_p_.as<float>(), emb_g_.as<float>(), emb_m_.as<float>(), emb_v_.as<float>(), emb_p16_.p);
  // resident granules here; SLOW granules were updated by the fused AdamW in their backward
  for (int i = 0; i < n_owned_; ++i) {
    const int r = res_idx_[static_cast<std::size_t>(i)];
    if (r < 0) continue;
    run(layer_, lp(i, 0), lg(i, 0), lay_m_.as<float>() + r * layer_stride_, lay_v_.as<float>() + r * layer_stride_,
        lp16(i, 0));
  }
}

void Engine::adamw_granule(float* p, float* g, float* m, float* v, void* p16, float lr, float bc1, float bc2) {
  std::vector<long long> off, len;
  std::vector<int> dec;
  for (const auto& s : layer_.segs) {
    off.push_back(s.off);
    len.push_back(s.len);
    dec.push_back(s.decay ? 1 : 0);
  }
  prof(P2R_PROF_ADAMW, 0, 30.0 * layer_.numel, [&] {
    p2r_check(p2r_adamw_step(p, g, m, v, p16, off.data(), len.data(), dec.data(), static_cast<int>(off.size()), b1_,
                             b2_, eps_, wd_, lr, bc1, bc2, stream_),
              "adamw");
  });
}

std::int64_t Engine::state_bytes() const {
  if (!has_opt_) return 0;
  // two fp32 moments per parameter element (optim.cpp:65-70)
  return 2 * 4 * (count_params(cfg_).total_params);
}

// ---------------------------------------------------------------- delink (model.cpp:358-377)
std::unique_ptr<Engine> Engine::delinked() const {
  if (cfg_.n_layers_params != 1) throw std::logic_error("delinked: model is not in shared-parameter mode");
  if (off_) throw std::logic_error("delinked: offloaded models are Real already");
  // each expert-parallel rank delinks its own shard (no communication); the Real
  // model needs its own communicator (comm_init) before an expert-parallel step
  std::unique_ptr<Engine> real(new Engine(cfg_.as_unshared(), NoInit{}, ep_world_, ep_rank_, force_ep_));
  cudaStream_t s = real->stream_;
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  // embeddings + final norm: direct copies
  cuda_check(cudaMemcpyAsync(real->emb_p_.p, emb_p_.p, emb_p_.bytes, cudaMemcpyDeviceToDevice, s), "delink emb");
  cuda_check(cudaMemcpyAsync(real->emb_p16_.p, emb_p16_.p, emb_p16_.bytes, cudaMemcpyDeviceToDevice, s), "delink emb");
  const int L = real->n_owned_;
  const std::size_t g4 = static_cast<std::size_t>(layer_stride_) * 4, g2 = static_cast<std::size_t>(layer_stride_) * 2;
  // shared layer -> L layers: master + bf16 shadow (+ moments), one read, L writes
  p2r_check(p2r_delink_broadcast(lay_p_.p, real->lay_p_.p, g4, g4, L, s), "delink");
  p2r_check(p2r_delink_broadcast(lay_p16_.p, real->lay_p16_.p, g2, g2, L, s), "delink");
  if (has_opt_) {
    real->adamw_attach(b1_, b2_, eps_, wd_);
    real->step_count_ = step_count_;
    cuda_check(cudaMemcpyAsync(real->emb_m_.p, emb_m_.p, emb_m_.bytes, cudaMemcpyDeviceToDevice, s), "delink m");
    cuda_check(cudaMemcpyAsync(real->emb_v_.p, emb_v_.p, emb_v_.bytes, cudaMemcpyDeviceToDevice, s), "delink v");
    p2r_check(p2r_delink_broadcast(lay_m_.p, real->lay_m_.p, g4, g4, L, s), "delink m");
    p2r_check(p2r_delink_broadcast(lay_v_.p, real->lay_v_.p, g4, g4, L, s), "delink v");
  }
  cuda_check(cudaStreamSynchronize(s), "delink sync");
  return real;
}

// ---------------------------------------------------------------- drop-in API staging
const int* Engine::stage_tokens(const int* host, int batch, int seq) {
  if (batch <= 0 || seq <= 0) throw std::invalid_argument("forward: token count must be a multiple of batch");
  if (seq > cfg_.seq_len) throw std::invalid_argument("forward: sequence longer than configured seq_len");
  const std::size_t T = static_cast<std::size_t>(batch) * seq;
  validate_ids(host, T, cfg_.vocab_size, "embedding_lookup: id out of range");
  ensure_acts(batch, seq);
  cuda_check(cudaMemcpyAsync(acts_->tokens.p, host, T * 4, cudaMemcpyHostToDevice, stream_), "h2d tokens");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  return acts_->tokens.as<int>();
}

void Engine::stage_targets(const int* targets, const std::uint8_t* mask, int n, const int** d_targets,
                           const std::uint8_t** d_mask) {
  if (!acts_ || acts_->T != n) throw std::invalid_argument("softmax_cross_entropy: one target per row required");
  for (int i = 0; i < n; ++i)
    if ((mask == nullptr || mask[i] != 0) && (targets[i] < 0 || targets[i] >= cfg_.vocab_size))
      throw std::out_of_range("softmax_cross_entropy: target out of range");
  cuda_check(cudaMemcpyAsync(acts_->targets.p, targets, static_cast<std::size_t>(n) * 4, cudaMemcpyHostToDevice,
                             stream_),
             "h2d targets");
  if (mask)
    cuda_check(cudaMemcpyAsync(acts_->mask.p, mask, static_cast<std::size_t>(n), cudaMemcpyHostToDevice, stream_),
               "h2d mask");
  cuda_check(cudaStreamSynchronize(stream_), "sync");
  *d_targets = acts_->targets.as<int>();
  *d_mask = mask ? acts_->mask.as<std::uint8_t>() : nullptr;
}

float* Engine::stage_activation(const float* host, int rows) {
  if (!acts_ || acts_->T != rows) throw std::invalid_argument("block_forward: batch does not match embed_forward");
  cuda_check(cudaMemcpyAsync(acts_->x0.p, host, static_cast<std::size_t>(rows) * cfg_.d_model * 4,
                             cudaMemcpyHostToDevice, stream_),
             "h2d activation");
  return acts_->x0.as<float>();
}

int Engine::vocab_ld() const { return acts_ ? acts_->vld : (cfg_.vocab_size + 7) / 8 * 8; }

// ---------------------------------------------------------------- host routing
HostRouting moe_dispatch_host(const float* logits, int T, const MoEConfig& moe) {
  moe.validate();
  if (!moe.enabled()) throw std::invalid_argument("moe_dispatch: moe disabled");
  const int E = moe.n_experts, k = moe.n_prototypes;
  HostRouting r;
  r.capacity = p2r_moe_capacity(moe.capacity_factor, T, E, k);
  const int seg = std::max(1, std::min(std::max(r.capacity, 0), T));
  cudaStream_t s = nullptr;
  const std::size_t Tk = static_cast<std::size_t>(T) * k;
  DevBuf dl(static_cast<std::size_t>(T) * E * 4 + 4), dsel(Tk * 4 + 4), dsur(Tk + 4), dpos(Tk * 4 + 4), draw(E * 4),
      dcnt(E * 4), drows(static_cast<std::size_t>(E) * seg * 4), dslots(static_cast<std::size_t>(E) * seg * 4),
      ddrop(4);
  if (T > 0) cuda_check(cudaMemcpy(dl.p, logits, static_cast<std::size_t>(T) * E * 4, cudaMemcpyHostToDevice), "h2d");
  p2r_check(p2r_moe_route(dl.as<float>(), T, E, k, r.capacity, seg, dsel.as<int>(), dsur.as<std::uint8_t>(),
                          dpos.as<int>(), draw.as<int>(), dcnt.as<int>(), drows.as<int>(), dslots.as<int>(),
                          ddrop.as<int>(), s),
            "route");
  cuda_check(cudaDeviceSynchronize(), "route sync");
  r.selected.resize(Tk);
  r.survived.resize(Tk);
  r.raw_load.resize(static_cast<std::size_t>(E));
  std::vector<int> cnt(static_cast<std::size_t>(E)), rows(static_cast<std::size_t>(E) * seg),
      slots(static_cast<std::size_t>(E) * seg);
  cuda_check(cudaMemcpy(r.selected.data(), dsel.p, Tk * 4, cudaMemcpyDeviceToHost), "d2h");
  cuda_check(cudaMemcpy(r.survived.data(), dsur.p, Tk, cudaMemcpyDeviceToHost), "d2h");
  cuda_check(cudaMemcpy(r.raw_load.data(), draw.p, E * 4, cudaMemcpyDeviceToHost), "d2h");
  cuda_check(cudaMemcpy(cnt.data(), dcnt.p, E * 4, cudaMemcpyDeviceToHost), "d2h");
  cuda_check(cudaMemcpy(rows.data(), drows.p, rows.size() * 4, cudaMemcpyDeviceToHost), "d2h");
  cuda_check(cudaMemcpy(slots.data(), dslots.p, slots.size() * 4, cudaMemcpyDeviceToHost), "d2h");
  cuda_check(cudaMemcpy(&r.dropped, ddrop.p, 4, cudaMemcpyDeviceToHost), "d2h");
  r.offsets.assign(static_cast<std::size_t>(E) + 1, 0);
  for (int e = 0; e < E; ++e) {
    r.offsets[static_cast<std::size_t>(e) + 1] = r.offsets[static_cast<std::size_t>(e)] + cnt[static_cast<std::size_t>(e)];
    for (int i = 0; i < cnt[static_cast<std::size_t>(e)]; ++i) {
      r.rows.push_back(rows[static_cast<std::size_t>(e) * seg + i]);
      r.slots.push_back(slots[static_cast<std::size_t>(e) * seg + i]);
    }
  }
  return r;
}

}  // namespace p2r
