// ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A C API over the UNMODIFIED reference C++ library (/root/reference/proj/core,
// compiled by oracle/build_ref.sh into oracle/_ref/libp2r_ref.so) so Python
// tests and bench.py's CPU-baseline leg can drive it through ctypes.
//
// Also hosts the step driver that the reference leaves absent
// (controller.cpp): zero_grads -> embed_forward ->
// block_forward x L -> head_forward -> softmax_cross_entropy(mask, denom) ->
// backward -> flush_shared_layer_grads -> (optional) AdamW::step.
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "p2r/model.hpp"
#include "p2r/optim.hpp"
#include "p2r/tensor.hpp"

using namespace p2r;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::out_of_range*>(&e)) return 2;
  if (dynamic_cast<const std::logic_error*>(&e)) return 3;
  return 4;
}

struct RefModel {
  std::unique_ptr<Model> model;
  std::unique_ptr<AdamW> opt;
  std::vector<std::pair<std::string, Tensor*>> params;  // for_each_param order
  void index() {
    params.clear();
    model->for_each_param([this](const std::string& n, Tensor& t) { params.emplace_back(n, &t); });
  }
};

}  // namespace

extern "C" {

struct ref_config {
  int d_model, d_ff, n_layers_graph, n_layers_params, n_heads, vocab_size, seq_len;
  int n_experts, n_prototypes, n_shards;
  float capacity_factor;
};

static ModelConfig to_cfg(const ref_config* c) {
  ModelConfig m;
  m.d_model = c->d_model;
  m.d_ff = c->d_ff;
  m.n_layers_graph = c->n_layers_graph;
  m.n_layers_params = c->n_layers_params;
  m.n_heads = c->n_heads;
  m.vocab_size = c->vocab_size;
  m.seq_len = c->seq_len;
  m.moe.n_experts = c->n_experts;
  m.moe.n_prototypes = c->n_prototypes;
  m.moe.n_shards = c->n_shards;
  m.moe.capacity_factor = c->capacity_factor;
  return m;
}

const char* ref_last_error() { return g_err.c_str(); }

int ref_count_params(const ref_config* c, int64_t* out3) {
  try {
    ParamCounts p = count_params(to_cfg(c));
    out3[0] = p.embedding_params;
    out3[1] = p.per_layer_params;
    out3[2] = p.total_params;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

void* ref_model_create(const ref_config* c, uint64_t seed) {
  try {
    auto* r = new RefModel;
    r->model = std::make_unique<Model>(to_cfg(c), seed);
    r->index();
    return r;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

void ref_model_destroy(void* h) { delete static_cast<RefModel*>(h); }

int ref_model_num_params(void* h) { return static_cast<int>(static_cast<RefModel*>(h)->params.size()); }

// name (NUL-terminated, <=127 chars), ndim, shape[0..3], numel
int ref_model_param_info(void* h, int i, char* name, int* ndim, int* shape, int64_t* numel) {
  auto* r = static_cast<RefModel*>(h);
  const auto& [n, t] = r->params.at(static_cast<size_t>(i));
  std::strncpy(name, n.c_str(), 127);
  name[127] = 0;
  *ndim = t->ndim();
  for (int d = 0; d < t->ndim() && d < 4; ++d) shape[d] = t->dim(d);
  *numel = static_cast<int64_t>(t->numel());
  return 0;
}

int ref_model_get_param(void* h, int i, float* out) {
  auto* r = static_cast<RefModel*>(h);
  Tensor* t = r->params.at(static_cast<size_t>(i)).second;
  std::memcpy(out, t->data(), t->nbytes());
  return 0;
}

int ref_model_set_param(void* h, int i, const float* in) {
  auto* r = static_cast<RefModel*>(h);
  Tensor* t = r->params.at(static_cast<size_t>(i)).second;
  std::memcpy(t->data(), in, t->nbytes());
  return 0;
}

int ref_model_get_grad(void* h, int i, float* out) {
  auto* r = static_cast<RefModel*>(h);
  Tensor* t = r->params.at(static_cast<size_t>(i)).second;
  if (!t->has_grad()) {
    std::memset(out, 0, t->nbytes());
    return 0;
  }
  std::memcpy(out, t->grad(), t->nbytes());
  return 0;
}

int ref_forward_logits(void* h, const int* tokens, int batch, int seq, int causal, float* out) {
  try {
    auto* r = static_cast<RefModel*>(h);
    Tensor logits = r->model->forward(std::span<const int>(tokens, static_cast<size_t>(batch) * seq),
                                      batch, causal ? AttentionMode::Causal : AttentionMode::Full);
    std::memcpy(out, logits.data(), logits.nbytes());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// One training micro-step (CS-1): returns loss via *loss_out. Gradients are
// left in the model's grad buffers (accumulated across calls unless zero=1).
// segmented=1 runs the per-layer recompute backward with a flush after every
// layer (model.hpp:101-106); segmented=0 records one tape and flushes once.
int ref_train_step(void* h, const int* tokens, const int* targets, const uint8_t* mask, int batch,
                   int seq, double denom, int causal, int zero, int segmented, float* loss_out) {
  try {
    auto* r = static_cast<RefModel*>(h);
    Model& m = *r->model;
    const size_t T = static_cast<size_t>(batch) * seq;
    std::span<const int> tok(tokens, T), tgt(targets, T);
    std::span<const uint8_t> msk;
    if (mask) msk = std::span<const uint8_t>(mask, T);
    const AttentionMode mode = causal ? AttentionMode::Causal : AttentionMode::Full;
    if (zero) m.zero_grads();
    if (!segmented) {
      GradTape tape;
      Tensor x = m.embed_forward(&tape, tok, batch);
      for (int g = 0; g < m.n_graph_layers(); ++g) x = m.block_forward(&tape, g, x, batch, mode);
      Tensor logits = m.head_forward(&tape, x);
      Tensor loss = softmax_cross_entropy(&tape, logits, tgt, msk, denom);
      tape.backward_scalar(loss);
      m.flush_shared_layer_grads();
      *loss_out = loss.at(0);
    } else {
      // forward without tape, keeping each layer input
      GradTape embed_tape;
      Tensor x0 = m.embed_forward(&embed_tape, tok, batch);
      std::vector<Tensor> xs{x0};
      for (int g = 0; g < m.n_graph_layers(); ++g)
        xs.push_back(m.block_forward(nullptr, g, xs.back(), batch, mode));
      GradTape head_tape;
      Tensor xl = xs.back().fork_for_grad();
      Tensor logits = m.head_forward(&head_tape, xl);
      Tensor loss = softmax_cross_entropy(&head_tape, logits, tgt, msk, denom);
      head_tape.backward_scalar(loss);
      *loss_out = loss.at(0);
      std::shared_ptr<std::vector<float>> gy = xl.grad_ptr();
      for (int g = m.n_graph_layers() - 1; g >= 0; --g) {
        GradTape t;
        Tensor xin = (g == 0) ? xs[0].fork_for_grad() : xs[static_cast<size_t>(g)].fork_for_grad();
        Tensor y = m.block_forward(&t, g, xin, batch, mode);
        float* yg = y.grad();
        for (size_t i = 0; i < y.numel(); ++i) yg[i] += (*gy)[i];
        t.backward();
        m.flush_shared_layer_grads();
        gy = xin.grad_ptr();
      }
      // embeddings: seed x0's grad and replay the embedding tape
      float* g0 = x0.grad();
      for (size_t i = 0; i < x0.numel(); ++i) g0[i] += (*gy)[i];
      embed_tape.backward();
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_flush(void* h) {
  static_cast<RefModel*>(h)->model->flush_shared_layer_grads();
  return 0;
}

int64_t ref_scratch_grad_bytes(void* h) { return static_cast<RefModel*>(h)->model->scratch_grad_bytes(); }

void* ref_model_delinked(void* h) {
  try {
    auto* r = static_cast<RefModel*>(h);
    auto* d = new RefModel;
    d->model = std::make_unique<Model>(r->model->delinked());
    d->index();
    return d;
  } catch (const std::exception& e) {
    fail(e);
    return nullptr;
  }
}

// ---------------- optimizer ----------------
int ref_adamw_attach(void* h, float b1, float b2, float eps, float wd) {
  auto* r = static_cast<RefModel*>(h);
  AdamWSettings s;
  s.beta1 = b1;
  s.beta2 = b2;
  s.eps = eps;
  s.weight_decay = wd;
  r->opt = std::make_unique<AdamW>(s);
  r->opt->register_model(*r->model);
  return 0;
}

int ref_adamw_step(void* h, float lr) {
  try {
    auto* r = static_cast<RefModel*>(h);
    r->opt->step(*r->model, lr);
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int64_t ref_adamw_step_count(void* h) { return static_cast<RefModel*>(h)->opt->step_count(); }
void ref_adamw_set_step_count(void* h, int64_t t) { static_cast<RefModel*>(h)->opt->set_step_count(t); }

// which = 0 -> m, 1 -> v
int ref_adamw_get_moment(void* h, const char* name, int which, float* out) {
  auto* r = static_cast<RefModel*>(h);
  auto it = r->opt->moments().find(name);
  if (it == r->opt->moments().end()) return 2;
  const auto& v = which ? it->second.v : it->second.m;
  std::memcpy(out, v.data(), v.size() * sizeof(float));
  return 0;
}
int ref_adamw_set_moment(void* h, const char* name, int which, const float* in) {
  auto* r = static_cast<RefModel*>(h);
  auto it = r->opt->moments().find(name);
  if (it == r->opt->moments().end()) return 2;
  auto& v = which ? it->second.v : it->second.m;
  std::memcpy(v.data(), in, v.size() * sizeof(float));
  return 0;
}

float ref_lr_at(float peak, double warmup_ratio, int64_t total, int64_t step) {
  return LrSchedule::cosine(peak, warmup_ratio, total).at(step);
}

// ---------------- routing (model.cpp:294-332) ----------------
// expert_rows / expert_slots are written CSR-style: offsets[E+1].
int ref_moe_dispatch(const float* logits, int T, int E, int k, float cf, int* selected,
                     uint8_t* survived, int* raw_load, int* offsets, int* rows, int* slots,
                     int* capacity, int* dropped) {
  try {
    MoEConfig moe;
    moe.n_experts = E;
    moe.n_prototypes = k;
    moe.capacity_factor = cf;
    Tensor lg = Tensor::from_data({T, E}, std::vector<float>(logits, logits + static_cast<size_t>(T) * E));
    Routing r = moe_dispatch(lg, moe);
    std::memcpy(selected, r.selected.data(), r.selected.size() * sizeof(int));
    std::memcpy(survived, r.survived.data(), r.survived.size());
    std::memcpy(raw_load, r.raw_load.data(), r.raw_load.size() * sizeof(int));
    int off = 0;
    for (int e = 0; e < E; ++e) {
      offsets[e] = off;
      for (size_t i = 0; i < r.expert_rows[static_cast<size_t>(e)].size(); ++i) {
        rows[off] = r.expert_rows[static_cast<size_t>(e)][i];
        slots[off] = r.expert_slots[static_cast<size_t>(e)][i];
        ++off;
      }
    }
    offsets[E] = off;
    *capacity = r.capacity;
    *dropped = r.dropped;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// ---------------- single primitives (fwd + bwd with a seeded output grad) ----------------
int ref_layernorm(const float* x, const float* gain, const float* bias, int rows, int d,
                  const float* gy, float* y, float* gx, float* ggain, float* gbias) {
  try {
    Tensor X = Tensor::from_data({rows, d}, std::vector<float>(x, x + static_cast<size_t>(rows) * d), true);
    Tensor G = Tensor::from_data({d}, std::vector<float>(gain, gain + d), true);
    Tensor B = Tensor::from_data({d}, std::vector<float>(bias, bias + d), true);
    GradTape tape;
    Tensor Y = layernorm(&tape, X, G, B);
    std::memcpy(y, Y.data(), Y.nbytes());
    std::memcpy(Y.grad(), gy, Y.nbytes());
    tape.backward();
    std::memcpy(gx, X.grad(), X.nbytes());
    std::memcpy(ggain, G.grad(), G.nbytes());
    std::memcpy(gbias, B.grad(), B.nbytes());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_attention(const float* q, const float* k, const float* v, int B, int H, int S, int hd,
                  int causal, const float* go, float* o, float* gq, float* gk, float* gv) {
  try {
    const size_t n = static_cast<size_t>(B) * H * S * hd;
    Tensor Q = Tensor::from_data({B, H, S, hd}, std::vector<float>(q, q + n), true);
    Tensor K = Tensor::from_data({B, H, S, hd}, std::vector<float>(k, k + n), true);
    Tensor V = Tensor::from_data({B, H, S, hd}, std::vector<float>(v, v + n), true);
    GradTape tape;
    Tensor O = masked_attention(&tape, Q, K, V, causal != 0);
    std::memcpy(o, O.data(), O.nbytes());
    std::memcpy(O.grad(), go, O.nbytes());
    tape.backward();
    std::memcpy(gq, Q.grad(), Q.nbytes());
    std::memcpy(gk, K.grad(), K.nbytes());
    std::memcpy(gv, V.grad(), V.nbytes());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_cross_entropy(const float* logits, const int* targets, const uint8_t* mask, int rows,
                      int vocab, double denom, float* loss, float* glogits) {
  try {
    Tensor L = Tensor::from_data({rows, vocab},
                                 std::vector<float>(logits, logits + static_cast<size_t>(rows) * vocab), true);
    GradTape tape;
    std::span<const uint8_t> msk;
    if (mask) msk = std::span<const uint8_t>(mask, static_cast<size_t>(rows));
    Tensor out = softmax_cross_entropy(&tape, L, std::span<const int>(targets, static_cast<size_t>(rows)), msk, denom);
    *loss = out.at(0);
    tape.backward_scalar(out);
    std::memcpy(glogits, L.grad(), L.nbytes());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_gelu(const float* x, int n, const float* gy, float* y, float* gx) {
  Tensor X = Tensor::from_data({n}, std::vector<float>(x, x + n), true);
  GradTape tape;
  Tensor Y = gelu(&tape, X);
  std::memcpy(y, Y.data(), Y.nbytes());
  std::memcpy(Y.grad(), gy, Y.nbytes());
  tape.backward();
  std::memcpy(gx, X.grad(), X.nbytes());
  return 0;
}

}  // extern "C"
