// extern "C" wrappers of the host engine (include/p2r_engine.h). No exception
// crosses this boundary: each maps to a p2r_status with the reference's message.
#include <cstring>
#include <memory>
#include <new>

#include "../p2r_internal.h"
#include "p2r/engine.hpp"
#include "comm_state.hpp"
#include "p2r_engine.h"

struct p2r_model {
  std::unique_ptr<p2r::Engine> m;
};
struct p2r_loopback {
  std::unique_ptr<p2r::LoopbackGroup> g;
};

namespace {

p2r::ModelConfig to_cfg(const p2r_model_config* c) {
  p2r::ModelConfig m;
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

template <typename F>
p2r_status guard(F&& f) {
  try {
    f();
    return P2R_OK;
  } catch (const std::invalid_argument& e) {
    return p2r::set_error(P2R_EINVAL, e.what());
  } catch (const std::out_of_range& e) {
    return p2r::set_error(P2R_ERANGE, e.what());
  } catch (const std::logic_error& e) {
    return p2r::set_error(P2R_ELOGIC, e.what());
  } catch (const std::bad_alloc&) {
    return p2r::set_error(P2R_ERUNTIME, "out of memory");
  } catch (const std::exception& e) {
    return p2r::set_error(P2R_ERUNTIME, e.what());
  }
}

p2r::AttentionMode mode_of(int causal) { return causal ? p2r::AttentionMode::Causal : p2r::AttentionMode::Full; }

}  // namespace

extern "C" {

p2r_status p2r_count_params(const p2r_model_config* cfg, int64_t* out3) {
  return guard([&] {
    p2r::ParamCounts p = p2r::count_params(to_cfg(cfg));
    out3[0] = p.embedding_params;
    out3[1] = p.per_layer_params;
    out3[2] = p.total_params;
  });
}

p2r_status p2r_model_create(const p2r_model_config* cfg, uint64_t seed, p2r_model** out) {
  return guard([&] {
    auto h = std::make_unique<p2r_model>();
    h->m = std::make_unique<p2r::Engine>(to_cfg(cfg), seed);
    *out = h.release();
  });
}

p2r_status p2r_model_destroy(p2r_model* m) {
  delete m;
  return P2R_OK;
}

int p2r_model_num_params(const p2r_model* m) { return static_cast<int>(m->m->params().size()); }

p2r_status p2r_model_param_info(const p2r_model* m, int i, char* name128, int* ndim, int* shape4,
                                int64_t* numel) {
  return guard([&] {
    const p2r::ParamView& v = m->m->params().at(static_cast<std::size_t>(i));
    std::strncpy(name128, v.name.c_str(), 127);
    name128[127] = 0;
    *ndim = static_cast<int>(v.shape.size());
    int64_t n = 1;
    for (std::size_t d = 0; d < v.shape.size() && d < 4; ++d) {
      shape4[d] = v.shape[d];
      n *= v.shape[d];
    }
    *numel = n;
  });
}

p2r_status p2r_model_get_param(const p2r_model* m, int i, float* host_out) {
  return guard([&] { m->m->get_param(i, host_out); });
}
p2r_status p2r_model_set_param(p2r_model* m, int i, const float* host_in) {
  return guard([&] { m->m->set_param(i, host_in); });
}
p2r_status p2r_model_get_grad(const p2r_model* m, int i, float* host_out) {
  return guard([&] { m->m->get_grad(i, host_out); });
}

p2r_status p2r_model_forward(p2r_model* m, const int* tokens, int batch, int seq, int causal, float* logits_out) {
  return guard([&] { m->m->forward_host(tokens, batch, seq, mode_of(causal), logits_out); });
}

p2r_status p2r_model_train_step(p2r_model* m, const int* tokens, const int* targets, const uint8_t* mask,
                                int batch, int seq, double denom, int causal, int zero, float* loss_out) {
  return guard([&] {
    const float l = m->m->train_step_host(tokens, targets, mask, batch, seq, denom, mode_of(causal), zero != 0);
    if (loss_out) *loss_out = l;
  });
}

p2r_status p2r_model_train_step_async(p2r_model* m, const int* tokens, const int* targets, const uint8_t* mask,
                                      int batch, int seq, double denom, int causal, int zero, uint64_t* ticket) {
  return guard([&] {
    const std::uint64_t t =
        m->m->train_step_host_async(tokens, targets, mask, batch, seq, denom, mode_of(causal), zero != 0);
    if (ticket) *ticket = t;
  });
}

p2r_status p2r_model_loss_wait(p2r_model* m, uint64_t ticket, float* loss_out) {
  return guard([&] {
    const float l = m->m->loss_wait(ticket);
    if (loss_out) *loss_out = l;
  });
}

p2r_status p2r_model_train_step_device(p2r_model* m, const int* d_tokens, const int* d_targets,
                                       const uint8_t* d_mask, int batch, int seq, double denom, int causal,
                                       int zero, float* loss_dev) {
  return guard([&] {
    if (denom <= 0.0) throw std::invalid_argument("softmax_cross_entropy: denominator must be > 0");
    m->m->train_step_device(d_tokens, d_targets, d_mask, batch, seq, denom, mode_of(causal), zero != 0, loss_dev);
  });
}

p2r_status p2r_model_train_step_device_graph(p2r_model* m, const int* d_tokens, const int* d_targets,
                                             const uint8_t* d_mask, int batch, int seq, double denom, int causal,
                                             int zero, float* loss_dev) {
  return guard([&] {
    if (denom <= 0.0) throw std::invalid_argument("softmax_cross_entropy: denominator must be > 0");
    m->m->train_step_device_graph(d_tokens, d_targets, d_mask, batch, seq, denom, mode_of(causal), zero != 0,
                                  loss_dev);
  });
}

p2r_status p2r_model_adamw_attach(p2r_model* m, float b1, float b2, float eps, float wd) {
  return guard([&] { m->m->adamw_attach(b1, b2, eps, wd); });
}
p2r_status p2r_model_adamw_step(p2r_model* m, float lr) {
  return guard([&] { m->m->adamw_step(lr); });
}
int64_t p2r_model_adamw_step_count(const p2r_model* m) { return m->m->step_count(); }
p2r_status p2r_model_adamw_set_step_count(p2r_model* m, int64_t t) {
  m->m->set_step_count(t);
  return P2R_OK;
}
p2r_status p2r_model_get_moment(const p2r_model* m, int i, int which, float* host_out) {
  return guard([&] { m->m->get_moment(i, which, host_out); });
}
int64_t p2r_model_state_bytes(const p2r_model* m) { return m->m->state_bytes(); }
int64_t p2r_model_grad_bytes(const p2r_model* m) { return m->m->grad_bytes(); }
int64_t p2r_model_scratch_grad_bytes(const p2r_model* m) { return m->m->scratch_grad_bytes(); }

p2r_status p2r_model_delinked(const p2r_model* m, p2r_model** out) {
  return guard([&] {
    auto h = std::make_unique<p2r_model>();
    h->m = m->m->delinked();
    *out = h.release();
  });
}

p2r_status p2r_model_set_moment(p2r_model* m, int i, int which, const float* host_in) {
  return guard([&] { m->m->set_moment(i, which, host_in); });
}

namespace {
p2r::StageState to_state(const p2r_stage_state* s) {
  p2r::StageState st;
  if (s) {
    st.stage = s->stage;
    st.global_step = s->global_step;
    st.samples_consumed = s->samples_consumed;
    st.wall_time_s = s->wall_time_s;
    st.rng_state = s->rng_state;
    st.last_eval_step = s->last_eval_step;
  }
  return st;
}
void from_state(const p2r::StageState& st, p2r_stage_state* s) {
  if (!s) return;
  s->stage = st.stage;
  s->global_step = st.global_step;
  s->samples_consumed = st.samples_consumed;
  s->wall_time_s = st.wall_time_s;
  s->rng_state = st.rng_state;
  s->last_eval_step = st.last_eval_step;
}
}  // namespace

p2r_status p2r_model_save_checkpoint(const p2r_model* m, const char* path, const p2r_stage_state* st) {
  return guard([&] {
    if (!path) throw std::invalid_argument("checkpoint: null path");
    m->m->save_checkpoint(path, to_state(st));
  });
}
p2r_status p2r_model_load_checkpoint(p2r_model* m, const char* path, p2r_stage_state* st_out) {
  return guard([&] {
    if (!path) throw std::invalid_argument("checkpoint: null path");
    from_state(m->m->load_checkpoint(path), st_out);
  });
}
p2r_status p2r_model_from_checkpoint(const char* path, p2r_model** out, p2r_stage_state* st_out) {
  return guard([&] {
    if (!path) throw std::invalid_argument("checkpoint: null path");
    p2r::StageState st;
    auto h = std::make_unique<p2r_model>();
    h->m = p2r::Engine::from_checkpoint(path, &st);
    from_state(st, st_out);
    *out = h.release();
  });
}
p2r_status p2r_delink_checkpoint(const char* in_path, const char* out_path, p2r_stage_state* st_out) {
  return guard([&] {
    if (!in_path || !out_path) throw std::invalid_argument("checkpoint: null path");
    from_state(p2r::delink_checkpoint(in_path, out_path), st_out);
  });
}

p2r_status p2r_model_expert_shard(const p2r_model* m, int expert, int* shard_out) {
  return guard([&] { *shard_out = m->m->expert_shard(expert); });
}
p2r_status p2r_model_redistribute_experts(p2r_model* m, int new_n_shards) {
  return guard([&] { m->m->redistribute_experts(new_n_shards); });
}
p2r_status p2r_redistribute_checkpoints(const char* const* in_paths, int n_in, const char* const* out_paths,
                                        int n_out) {
  return guard([&] {
    if (n_in <= 0 || n_out <= 0 || !in_paths || !out_paths)
      throw std::invalid_argument("redistribute_experts: empty shard list");
    std::vector<std::string> in(in_paths, in_paths + n_in), out(out_paths, out_paths + n_out);
    p2r::redistribute_checkpoints(in, out);
  });
}

namespace {
p2r::SwitchPolicy policy_of(const p2r_switch_policy* p) {
  if (!p) throw std::invalid_argument("switch policy: null");
  p2r::SwitchPolicy s;
  s.eval_interval_steps = p->eval_interval_steps;
  s.trial_budget_steps = p->trial_budget_steps;
  s.slope_window = p->slope_window;
  return s;
}
}  // namespace

p2r_status p2r_loss_slope(const double* time_s, const double* loss, int n, int window, double* slope_out) {
  return guard([&] {
    if (n < 0 || (n > 0 && (!time_s || !loss))) throw std::invalid_argument("loss_slope: bad series");
    *slope_out = p2r::loss_slope(std::vector<double>(time_s, time_s + n), std::vector<double>(loss, loss + n), window);
  });
}
p2r_status p2r_switch_criterion(const double* pseudo_t, const double* pseudo_loss, int n_pseudo, const double* real_t,
                                const double* real_loss, int n_real, const p2r_switch_policy* policy, int* fire_out,
                                double* pseudo_slope_out, double* real_slope_out) {
  return guard([&] {
    if (n_pseudo < 0 || n_real < 0) throw std::invalid_argument("switch: bad series");
    const p2r::SwitchDecision d = p2r::switch_criterion(
        std::vector<double>(pseudo_t, pseudo_t + n_pseudo), std::vector<double>(pseudo_loss, pseudo_loss + n_pseudo),
        std::vector<double>(real_t, real_t + n_real), std::vector<double>(real_loss, real_loss + n_real),
        policy_of(policy));
    *fire_out = d.fire ? 1 : 0;
    if (pseudo_slope_out) *pseudo_slope_out = d.pseudo_slope;
    if (real_slope_out) *real_slope_out = d.real_slope;
  });
}
p2r_status p2r_switch_evaluation_due(const p2r_switch_policy* policy, int64_t step, int* due_out) {
  return guard([&] { *due_out = p2r::switch_evaluation_due(policy_of(policy), step) ? 1 : 0; });
}

void* p2r_model_stream(p2r_model* m) { return m->m->stream(); }

p2r_status p2r_model_set_profiling(p2r_model* m, int on) {
  m->m->set_profiling(on != 0);
  return P2R_OK;
}
p2r_status p2r_model_profile(p2r_model* m, int cls, int64_t* launches, double* ms, double* flops, double* bytes) {
  return guard([&] {
    std::int64_t n = 0;
    m->m->profile(cls, &n, ms, flops, bytes);
    *launches = n;
  });
}
p2r_status p2r_model_profile_reset(p2r_model* m) {
  return guard([&] { m->m->profile_reset(); });
}
p2r_status p2r_model_buffer(p2r_model* m, int which, void** ptr, size_t* bytes) {
  return guard([&] { m->m->buffer(which, ptr, bytes); });
}

p2r_status p2r_model_routing(const p2r_model* m, int g, int* selected, uint8_t* survived, int* raw_load,
                             int* capacity, int* dropped) {
  return guard([&] { m->m->routing_host(g, selected, survived, raw_load, capacity, dropped); });
}

p2r_status p2r_model_gate_logits(const p2r_model* m, int g, float* out) {
  return guard([&] { m->m->gate_logits_host(g, out); });
}

p2r_status p2r_moe_dispatch_host(const float* logits, int T, int E, int k, float cf, int* selected,
                                 uint8_t* survived, int* raw_load, int* offsets, int* rows, int* slots,
                                 int* capacity, int* dropped) {
  return guard([&] {
    p2r::MoEConfig moe;
    moe.n_experts = E;
    moe.n_prototypes = k;
    moe.capacity_factor = cf;
    p2r::HostRouting r = p2r::moe_dispatch_host(logits, T, moe);
    std::memcpy(selected, r.selected.data(), r.selected.size() * 4);
    std::memcpy(survived, r.survived.data(), r.survived.size());
    std::memcpy(raw_load, r.raw_load.data(), r.raw_load.size() * 4);
    std::memcpy(offsets, r.offsets.data(), r.offsets.size() * 4);
    if (!r.rows.empty()) {
      std::memcpy(rows, r.rows.data(), r.rows.size() * 4);
      std::memcpy(slots, r.slots.data(), r.slots.size() * 4);
    }
    *capacity = r.capacity;
    *dropped = r.dropped;
  });
}

p2r_status p2r_comm_unique_id(char* out128) {
  return guard([&] { p2r::comm_unique_id(out128); });
}
p2r_status p2r_model_create_ep(const p2r_model_config* cfg, uint64_t seed, int world, int rank, p2r_model** out) {
  return guard([&] {
    auto h = std::make_unique<p2r_model>();
    h->m = std::make_unique<p2r::Engine>(to_cfg(cfg), seed, world, rank);
    *out = h.release();
  });
}
p2r_status p2r_model_comm_init(p2r_model* m, const char* id) {
  return guard([&] { m->m->comm_init(id); });
}
p2r_status p2r_loopback_create(int world, p2r_loopback** out) {
  return guard([&] {
    auto h = std::make_unique<p2r_loopback>();
    h->g = std::make_unique<p2r::LoopbackGroup>(world);
    *out = h.release();
  });
}
p2r_status p2r_loopback_destroy(p2r_loopback* g) {
  delete g;
  return P2R_OK;
}
p2r_status p2r_model_comm_init_loopback(p2r_model* m, p2r_loopback* g) {
  return guard([&] { m->m->comm_init_loopback(g->g.get()); });
}
p2r_status p2r_model_allreduce_grads(p2r_model* m) {
  return guard([&] { m->m->allreduce_grads(); });
}

p2r_status p2r_model_create_offload(const p2r_model_config* cfg, uint64_t seed, const int* slow, int ring_slots,
                                    p2r_model** out) {
  return guard([&] {
    const int n = cfg->n_layers_params;
    std::vector<int> pl(slow, slow + n);
    auto h = std::make_unique<p2r_model>();
    h->m = std::make_unique<p2r::Engine>(to_cfg(cfg), seed, pl, ring_slots);
    *out = h.release();
  });
}
p2r_status p2r_model_create_offload_ep(const p2r_model_config* cfg, uint64_t seed, const int* slow, int ring_slots,
                                       int world, int rank, p2r_model** out) {
  return guard([&] {
    const int n = cfg->n_layers_params;
    std::vector<int> pl(slow, slow + n);
    auto h = std::make_unique<p2r_model>();
    h->m = std::make_unique<p2r::Engine>(to_cfg(cfg), seed, pl, ring_slots, world, rank);
    *out = h.release();
  });
}
p2r_status p2r_model_set_grad_accumulation(p2r_model* m, int micro_steps) {
  return guard([&] { m->m->set_grad_accumulation(micro_steps); });
}
p2r_status p2r_model_set_activation_checkpointing(p2r_model* m, int policy) {
  return guard([&] { m->m->set_activation_checkpointing(policy); });
}
p2r_status p2r_model_set_offload_lr(p2r_model* m, float lr) {
  m->m->set_offload_lr(lr);
  return P2R_OK;
}
p2r_status p2r_model_offload_stats(p2r_model* m, double* o) {
  return guard([&] {
    const p2r::OffloadStats s = m->m->offload_stats();
    o[0] = s.fn_load;
    o[1] = s.bn_load;
    o[2] = s.opt_load;
    o[3] = s.writeback;
    o[4] = s.grad_offload;
    o[5] = s.h2d_ms;
    o[6] = s.d2h_ms;
    o[7] = s.grad_load;
  });
}
p2r_status p2r_model_offload_stats_reset(p2r_model* m) {
  return guard([&] { m->m->offload_stats_reset(); });
}
p2r_status p2r_model_set_offload_skip_copies(p2r_model* m, int skip) {
  m->m->set_offload_skip_copies(skip != 0);
  return P2R_OK;
}
int64_t p2r_model_layer_granule_bytes(const p2r_model* m) { return m->m->layer_granule_bytes(); }
int64_t p2r_model_device_param_bytes(const p2r_model* m) { return m->m->device_param_bytes(); }

p2r_status p2r_plan_offload(const int64_t* layer_bytes, int n, int64_t budget, double bandwidth, double compute_s,
                            double latency_s, int* slow_out) {
  return guard([&] {
    std::vector<std::int64_t> b(layer_bytes, layer_bytes + n);
    const std::vector<int> pl = p2r::plan_offload(b, budget, bandwidth, compute_s, latency_s);
    std::copy(pl.begin(), pl.end(), slow_out);
  });
}
double p2r_predict_step_time(const int64_t* layer_bytes, const int* slow, int n, double bandwidth, double compute_s,
                             double latency_s) {
  std::vector<std::int64_t> b(layer_bytes, layer_bytes + n);
  std::vector<int> s(slow, slow + n);
  return p2r::predict_step_time(b, s, bandwidth, compute_s, latency_s);
}

namespace {
p2r::OffloadCost cost(double h2d, double d2h, double fwd_s, double bwd_s) {
  p2r::OffloadCost c;
  c.h2d_bw = h2d;
  c.d2h_bw = d2h;
  c.fwd_s = fwd_s;
  c.bwd_s = bwd_s;
  return c;
}
}  // namespace

double p2r_predict_step_time_overlap_form(const int64_t* layer_params, const int64_t* vector_params, const int* slow,
                                          int n, double h2d_bw, double d2h_bw, double fwd_s, double bwd_s,
                                          int fn_master) {
  std::vector<std::int64_t> p(layer_params, layer_params + n), v;
  if (vector_params) v.assign(vector_params, vector_params + n);
  std::vector<int> s(slow, slow + n);
  p2r::OffloadCost c = cost(h2d_bw, d2h_bw, fwd_s, bwd_s);
  c.fn_master = fn_master != 0;
  return p2r::predict_step_time_overlap(p, v, s, c);
}
double p2r_predict_step_time_overlap_window(const int64_t* layer_params, const int64_t* vector_params, const int* slow,
                                            int n, double h2d_bw, double d2h_bw, double fwd_s, double bwd_s,
                                            int fn_master, int micro_steps, int recompute) {
  std::vector<std::int64_t> p(layer_params, layer_params + n), v;
  if (vector_params) v.assign(vector_params, vector_params + n);
  std::vector<int> s(slow, slow + n);
  p2r::OffloadCost c = cost(h2d_bw, d2h_bw, fwd_s, bwd_s);
  c.fn_master = fn_master != 0;
  c.micro_steps = micro_steps;
  c.recompute = recompute != 0;
  return p2r::predict_step_time_overlap(p, v, s, c);
}
double p2r_predict_step_time_overlap(const int64_t* layer_params, const int64_t* vector_params, const int* slow, int n,
                                     double h2d_bw, double d2h_bw, double fwd_s, double bwd_s) {
  return p2r_predict_step_time_overlap_form(layer_params, vector_params, slow, n, h2d_bw, d2h_bw, fwd_s, bwd_s, 0);
}
p2r_status p2r_plan_offload_overlap(const int64_t* layer_params, int n, int64_t budget_bytes, double h2d_bw,
                                    double d2h_bw, double fwd_s, double bwd_s, int ring_slots, int* slow_out) {
  return guard([&] {
    std::vector<std::int64_t> p(layer_params, layer_params + n);
    p2r::OffloadCost c = cost(h2d_bw, d2h_bw, fwd_s, bwd_s);
    c.ring_slots = ring_slots;
    const std::vector<int> pl = p2r::plan_offload_overlap(p, budget_bytes, c);
    std::copy(pl.begin(), pl.end(), slow_out);
  });
}

void p2r_init_normal_host(uint64_t seed, const char* name, int64_t n, float* out) {
  p2r::init_normal_host(out, static_cast<std::size_t>(n), seed, name);
}

float p2r_lr_at(float peak, double warmup_ratio, int64_t total, int64_t step) {
  try {
    return p2r::lr_at(peak, warmup_ratio, total, step);
  } catch (const std::exception& e) {
    p2r::set_error(P2R_EINVAL, e.what());
    return -1.0f;
  }
}

}  // extern "C"
