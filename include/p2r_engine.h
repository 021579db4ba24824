/*
 * p2r_engine.h — C-ABI of the step-level host engine (C++ above the kernel
 * layer of p2r_cuda.h). This is the drop-in boundary a non-C++ caller binds
 * (ctypes / cgo / JNI): it exposes exactly the reference's Model / AdamW /
 * delink / routing surface (/root/reference/proj/core/include/p2r/model.hpp,
 * optim.hpp) with host buffers in and out, plus a device-pointer fast path.
 *
 * Parameter names and order follow Model::for_each_param (model.cpp:188-198):
 * "embed.tok", "embed.pos", "final_norm.gain", "final_norm.bias",
 * "layer.<i>.ln1.gain", ..., "layer.<i>.moe.expert.<e>.b2".
 */
#ifndef P2R_ENGINE_H_
#define P2R_ENGINE_H_

#include <stddef.h>
#include <stdint.h>

#include "p2r_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ModelConfig + MoEConfig (model.hpp:13-41), same field meaning and defaults. */
typedef struct {
  int d_model, d_ff, n_layers_graph, n_layers_params, n_heads, vocab_size, seq_len;
  int n_experts, n_prototypes, n_shards;
  float capacity_factor;
} p2r_model_config;

typedef struct p2r_model p2r_model;

/* count_params (model.cpp:73-89): out3 = {embedding, per_layer, total}. */
p2r_status p2r_count_params(const p2r_model_config* cfg, int64_t* out3);
/* Model(config, seed) (model.cpp:123-179): identical std::mt19937_64 /
 * std::normal_distribution<float>(0, 0.02) init per named tensor. */
p2r_status p2r_model_create(const p2r_model_config* cfg, uint64_t seed, p2r_model** out);
p2r_status p2r_model_destroy(p2r_model* m);
int p2r_model_num_params(const p2r_model* m);
p2r_status p2r_model_param_info(const p2r_model* m, int i, char* name128, int* ndim, int* shape4,
                                int64_t* numel);
/* Host <-> device copies of one named parameter / its gradient. */
p2r_status p2r_model_get_param(const p2r_model* m, int i, float* host_out);
p2r_status p2r_model_set_param(p2r_model* m, int i, const float* host_in);
p2r_status p2r_model_get_grad(const p2r_model* m, int i, float* host_out);

/* Model::forward (model.cpp:287-292): logits [batch*seq, vocab] to host. */
p2r_status p2r_model_forward(p2r_model* m, const int* tokens, int batch, int seq, int causal,
                             float* logits_out);

/* One micro-step of the absent controller (CS-1):
 * zero_grads (if zero) -> embed -> L blocks -> head -> masked CE(denom) ->
 * backward with shared-layer grads accumulated in place. tokens/targets/mask
 * are HOST arrays (copied in on the model's stream); *loss_out is the loss.
 * Error behaviour matches the reference (out-of-range ids / targets ->
 * P2R_ERANGE with the reference's message). */
p2r_status p2r_model_train_step(p2r_model* m, const int* tokens, const int* targets,
                                const uint8_t* mask, int batch, int seq, double denom, int causal,
                                int zero, float* loss_out);
/* Pipelined form of p2r_model_train_step (a host training loop that enqueues the next
 * step / the optimizer before reading this step's loss): the inputs are staged in one
 * of two pinned slots, the step and the loss read-back are enqueued, and *ticket
 * identifies the step. p2r_model_loss_wait(ticket) waits for that step and returns
 * its loss; only the last two tickets can be waited on (older: P2R_ELOGIC). The
 * same validation and errors as p2r_model_train_step, raised before anything is enqueued. */
p2r_status p2r_model_train_step_async(p2r_model* m, const int* tokens, const int* targets,
                                      const uint8_t* mask, int batch, int seq, double denom, int causal,
                                      int zero, uint64_t* ticket);
p2r_status p2r_model_loss_wait(p2r_model* m, uint64_t ticket, float* loss_out);
/* Same, inputs already resident on the device; the loss stays on the device
 * (loss_dev, may be NULL) so steps can be enqueued / graph-captured. */
p2r_status p2r_model_train_step_device(p2r_model* m, const int* d_tokens, const int* d_targets,
                                       const uint8_t* d_mask, int batch, int seq, double denom,
                                       int causal, int zero, float* loss_dev);

/* train_step_device replayed as one CUDA graph: captured on the first call (which
 * also runs the step) and re-captured whenever an argument changes; resident,
 * MoE-free models (P2R_ELOGIC otherwise; the data-parallel all-reduce stays
 * outside the graph). Bit-identical to
 * p2r_model_train_step_device. The optimizer step stays outside the graph. */
p2r_status p2r_model_train_step_device_graph(p2r_model* m, const int* d_tokens, const int* d_targets,
                                             const uint8_t* d_mask, int batch, int seq, double denom,
                                             int causal, int zero, float* loss_dev);

/* AdamW (optim.hpp:29-54). */
p2r_status p2r_model_adamw_attach(p2r_model* m, float b1, float b2, float eps, float wd);
p2r_status p2r_model_adamw_step(p2r_model* m, float lr);
int64_t p2r_model_adamw_step_count(const p2r_model* m);
p2r_status p2r_model_adamw_set_step_count(p2r_model* m, int64_t t);
/* which: 0 = m, 1 = v */
p2r_status p2r_model_get_moment(const p2r_model* m, int i, int which, float* host_out);
int64_t p2r_model_state_bytes(const p2r_model* m);
/* Gradient bytes held on the device (one layer in Pseudo mode: no scratch copy). */
int64_t p2r_model_grad_bytes(const p2r_model* m);
int64_t p2r_model_scratch_grad_bytes(const p2r_model* m);

/* Model::delinked (model.cpp:358-377) + optimizer-moment copy (SPEC.md:279,
 * :312) as one device broadcast; logic error on a non-shared model. */
p2r_status p2r_model_delinked(const p2r_model* m, p2r_model** out);
p2r_status p2r_model_set_moment(p2r_model* m, int i, int which, const float* host_in);

/* ------------------------------------------------------------------------ */
/* Checkpoint container (SPEC.md:260-264 [TYPE] Checkpoint, :320 file format): */
/* version tag, ModelConfig, named layer-indexed fp32 parameter buffers, AdamW */
/* moments + step count, StageState; LE ints, IEEE fp32, manifest of names /   */
/* shapes / byte offsets. save -> load -> train k steps == train k steps,      */
/* bitwise. Errors: bad file -> ERUNTIME; config / shard mismatch -> EINVAL;  */
/* delink of a non-PSEUDO checkpoint -> ELOGIC.                               */
/* ------------------------------------------------------------------------ */
typedef struct {
  int stage; /* 0 = PSEUDO, 1 = REAL */
  int64_t global_step;
  int64_t samples_consumed;
  double wall_time_s;
  uint64_t rng_state;
  int64_t last_eval_step;
} p2r_stage_state;

p2r_status p2r_model_save_checkpoint(const p2r_model* m, const char* path, const p2r_stage_state* st);
/* into an existing model with the same config (attaches AdamW if the file has moments) */
p2r_status p2r_model_load_checkpoint(p2r_model* m, const char* path, p2r_stage_state* st_out);
p2r_status p2r_model_from_checkpoint(const char* path, p2r_model** out, p2r_stage_state* st_out);
/* [OP] delink(pseudo_checkpoint) -> Real checkpoint */
p2r_status p2r_delink_checkpoint(const char* in_path, const char* out_path, p2r_stage_state* st_out);

/* Expert sharding (model.cpp:334-356, SPEC redistribute_experts). In-process
 * re-sharding is bookkeeping; across GPU counts the n_in expert-parallel shard
 * checkpoints are re-sharded into n_out (weights + AdamW moments; host I/O only).
 * EINVAL when n_experts % new shard count != 0 (reference text). */
p2r_status p2r_model_expert_shard(const p2r_model* m, int expert, int* shard_out);
p2r_status p2r_model_redistribute_experts(p2r_model* m, int new_n_shards);
p2r_status p2r_redistribute_checkpoints(const char* const* in_paths, int n_in, const char* const* out_paths,
                                        int n_out);

/* Switch detector decision logic (SPEC.md:255-259 SwitchPolicy, :285-293
 * detect_switch). Slope = least-squares d loss / d wall-time over the last
 * `window` points; the switch fires when the Real trial's slope is below the
 * Pseudo continuation's (faster decrease). EINVAL on invalid policy / series. */
typedef struct {
  int eval_interval_steps, trial_budget_steps, slope_window;
} p2r_switch_policy;
p2r_status p2r_loss_slope(const double* time_s, const double* loss, int n, int window, double* slope_out);
p2r_status p2r_switch_criterion(const double* pseudo_t, const double* pseudo_loss, int n_pseudo, const double* real_t,
                                const double* real_loss, int n_real, const p2r_switch_policy* policy, int* fire_out,
                                double* pseudo_slope_out, double* real_slope_out);
p2r_status p2r_switch_evaluation_due(const p2r_switch_policy* policy, int64_t step, int* due_out);

/* Raw device stream the model enqueues on (cudaStream_t). */
void* p2r_model_stream(p2r_model* m);

/* Live per-kernel-class timing: when enabled, every kernel the engine launches
 * is bracketed by CUDA events on the model stream; p2r_model_profile reports,
 * per class, launches, summed device ms and algorithmic FLOPs / HBM bytes. */
enum {
  P2R_PROF_GEMM = 0,
  P2R_PROF_ATTN_FWD = 1,
  P2R_PROF_ATTN_BWD = 2,
  P2R_PROF_LAYERNORM = 3,
  P2R_PROF_CE = 4,
  P2R_PROF_EMBED = 5,
  P2R_PROF_ADAMW = 6,
  P2R_PROF_MOE = 7,
  P2R_PROF_BIAS = 8,
  P2R_PROF_DELINK = 9,
  P2R_PROF_NCLASSES = 10
};
p2r_status p2r_model_set_profiling(p2r_model* m, int on);
/* Synchronises the model stream, then fills the totals since the last reset. */
p2r_status p2r_model_profile(p2r_model* m, int cls, int64_t* launches, double* ms, double* flops,
                             double* bytes);
p2r_status p2r_model_profile_reset(p2r_model* m);
/* Device pointer + byte size of a parameter-side buffer: which = 0 grads of the
 * embeddings granule, 1 grads of all owned layers (for a DP allreduce). */
p2r_status p2r_model_buffer(p2r_model* m, int which, void** ptr, size_t* bytes);
/* Last routing of graph layer g (MoE): host copies of moe_dispatch outputs. */
p2r_status p2r_model_routing(const p2r_model* m, int g, int* selected, uint8_t* survived,
                             int* raw_load, int* capacity, int* dropped);

/* fp32 gate logits [T, E] of graph layer g from the last forward (MoE). */
p2r_status p2r_model_gate_logits(const p2r_model* m, int g, float* out);

/* moe_dispatch (model.cpp:294-332) on host logits [T, E]: same outputs as the
 * reference's Routing, expert_rows/slots flattened CSR (offsets[E+1]). */
p2r_status p2r_moe_dispatch_host(const float* logits, int T, int E, int k, float cf, int* selected,
                                 uint8_t* survived, int* raw_load, int* offsets, int* rows,
                                 int* slots, int* capacity, int* dropped);

/* ---- expert / data parallelism ------------------------------
 * Rank r of W holds experts [r*E/W, (r+1)*E/W) (Model::expert_shard's
 * contiguous map, model.cpp:334-340) plus a replica of everything else. MoE
 * dispatch / combine are peer-store kernels (p2r_ep_*) that write the routed rows
 * (bf16, exact counts) straight into the owner's / source's arena over NVLink;
 * completion is signalled with stream memory operations. Replicated grads are
 * summed with p2r_model_allreduce_grads. Each rank must use the GLOBAL mask count
 * as the CE denominator so the summed gradient is the large-batch mean.
 * Multi-GPU: one process per GPU, p2r_model_comm_init(NCCL unique id); the EP
 * arenas are exchanged as CUDA IPC handles at the first step (collective).
 * Loopback: W shards of ONE process on one device, each driven by its own host
 * thread, joined with p2r_model_comm_init_loopback(group) (tests / one-GPU runs). */
p2r_status p2r_comm_unique_id(char* out128);
p2r_status p2r_model_create_ep(const p2r_model_config* cfg, uint64_t seed, int world, int rank,
                               p2r_model** out);
p2r_status p2r_model_comm_init(p2r_model* m, const char* unique_id128);
typedef struct p2r_loopback p2r_loopback;
p2r_status p2r_loopback_create(int world, p2r_loopback** out);
p2r_status p2r_loopback_destroy(p2r_loopback* g);
p2r_status p2r_model_comm_init_loopback(p2r_model* m, p2r_loopback* g);
p2r_status p2r_model_allreduce_grads(p2r_model* m);

/* ---- granular CPU offload (§4.2) ---------------
 * Real model whose owned layers with slow[i] = 1 live in pinned host DRAM and
 * are streamed through `ring_slots` HBM staging slots one granule ahead of
 * compute (H2D / D2H side streams); AdamW of SLOW granules runs fused in their
 * backward with the lr given to p2r_model_set_offload_lr. */
p2r_status p2r_model_create_offload(const p2r_model_config* cfg, uint64_t seed, const int* slow,
                                    int ring_slots, p2r_model** out);
p2r_status p2r_model_set_offload_lr(p2r_model* m, float lr);
/* Expert-parallel shard (world, rank) with granular offload (C5). */
p2r_status p2r_model_create_offload_ep(const p2r_model_config* cfg, uint64_t seed, const int* slow,
                                       int ring_slots, int world, int rank, p2r_model** out);
/* Gradient accumulation over `micro_steps` train_step calls (the first with zero=1):
 * SLOW granules park partial gradients in pinned host memory between micro-steps and
 * apply the fused AdamW (lr from p2r_model_set_offload_lr) in the last backward.
 * ELOGIC for a micro-step past the window or adamw_step before its last backward. */
p2r_status p2r_model_set_grad_accumulation(p2r_model* m, int micro_steps);
/* Activation checkpointing of offloaded models: 0 off, 1 SLOW layers
 * (default), 2 every layer. Results are bit-identical to the stored activations. */
p2r_status p2r_model_set_activation_checkpointing(p2r_model* m, int policy);
/* out8 = {Fn_load, Bn_load, opt_load, writeback, grad_offload, h2d_ms, d2h_ms, grad_load} since
 * last reset (grad_load: H2D of partial SLOW gradients between accumulation micro-steps) */
p2r_status p2r_model_offload_stats(p2r_model* m, double* out8);
p2r_status p2r_model_offload_stats_reset(p2r_model* m);
p2r_status p2r_model_set_offload_skip_copies(p2r_model* m, int skip);
int64_t p2r_model_layer_granule_bytes(const p2r_model* m);
int64_t p2r_model_device_param_bytes(const p2r_model* m);
/* plan_offload: slow_out[i] = 1 for offloaded layers. */
p2r_status p2r_plan_offload(const int64_t* layer_bytes, int n, int64_t budget, double bandwidth,
                            double compute_s, double latency_s, int* slow_out);
/* predict_step_time, 4 x W per SLOW layer, no overlap. */
double p2r_predict_step_time(const int64_t* layer_bytes, const int* slow, int n, double bandwidth,
                             double compute_s, double latency_s);
/* B200 overlap model of this engine: per SLOW layer of P params
 * H2D 2P + 4*vector_params (fwd) and 12P (bwd), D2H 14P; copies on their own
 * streams overlap compute: max(C_fwd, H2D_f/h2d) + max(C_bwd, H2D_b/h2d, D2H/d2h),
 * C_* = per-layer compute x n; at least (H2D_f + H2D_b)/h2d + the first SLOW layer's
 * forward load + its write-back. vector_params may be NULL. */
double p2r_predict_step_time_overlap(const int64_t* layer_params, const int64_t* vector_params, const int* slow,
                                     int n, double h2d_bw, double d2h_bw, double fwd_s, double bwd_s);
/* the same for either forward-load form: fn_master != 0 = the engine's default (Fn loads
 * the fp32 master, 4P; D2H 12P), 0 = P2R_OFFLOAD_FN_SHADOW=1 (the formula above). */
double p2r_predict_step_time_overlap_form(const int64_t* layer_params, const int64_t* vector_params,
                                          const int* slow, int n, double h2d_bw, double d2h_bw, double fwd_s,
                                          double bwd_s, int fn_master);
/* fewest SLOW layers (18 B/param granules) under budget_bytes, spread evenly */
/* The same model over an accumulation window of micro_steps (per micro-step Fn + Bn
 * loads, partial grads parked / reloaded between micro-steps, moments + write-back
 * once) with recompute != 0 adding the SLOW layers' checkpoint recomputation. */
double p2r_predict_step_time_overlap_window(const int64_t* layer_params, const int64_t* vector_params, const int* slow,
                                            int n, double h2d_bw, double d2h_bw, double fwd_s, double bwd_s,
                                            int fn_master, int micro_steps, int recompute);
p2r_status p2r_plan_offload_overlap(const int64_t* layer_params, int n, int64_t budget_bytes, double h2d_bw,
                                    double d2h_bw, double fwd_s, double bwd_s, int ring_slots, int* slow_out);

/* init_normal (model.cpp:28-36) on the host: the exact values Model() uploads. */
void p2r_init_normal_host(uint64_t seed, const char* name, int64_t n, float* out);

/* LrSchedule::cosine(peak, warmup_ratio, total).at(step) (optim.cpp:8-24). */
float p2r_lr_at(float peak, double warmup_ratio, int64_t total, int64_t step);

#ifdef __cplusplus
}
#endif
#endif /* P2R_ENGINE_H_ */
