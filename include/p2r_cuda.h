/*
 * p2r_cuda.h — C-ABI of the B200 (sm_100a) kernel layer for the Pseudo-to-Real
 * training-step hot path.
 *
 * Every entry point takes raw device pointers + sizes + a cudaStream_t (passed
 * as void*), enqueues asynchronously and returns a p2r_status. No exceptions
 * cross this boundary; p2r_last_error() holds a thread-local message whose
 * text matches the reference's exception text where one exists.
 *
 * Each function names the reference primitive it replaces
 * (/root/reference/proj/core/...). The reference is a CPU fp32 library; here
 * GEMM operands are bf16 with fp32 accumulation, everything else is fp32.
 */
#ifndef P2R_CUDA_H_
#define P2R_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. The C++ shim maps them back to the reference exception types:
 * EINVAL -> std::invalid_argument, ERANGE -> std::out_of_range,
 * ELOGIC -> std::logic_error, ERUNTIME/ECUDA/ENCCL -> std::runtime_error. */
typedef enum {
  P2R_OK = 0,
  P2R_EINVAL = 1,
  P2R_ERANGE = 2,
  P2R_ELOGIC = 3,
  P2R_ERUNTIME = 4,
  P2R_ECUDA = 5,
  P2R_ENCCL = 6
} p2r_status;

#define P2R_MAX_ADAM_SEGS 16

const char* p2r_last_error(void);
const char* p2r_version(void);
/* Number of p2r kernels launched by this process so far (all entry points). */
uint64_t p2r_launch_count(void);

/* ------------------------------------------------------------------------ */
/* GEMM: C[m,n] = epilogue( sum_k A(m,k) * B(n,k) ) on tcgen05 + TMEM + TMA.  */
/* Replaces cblas_sgemm at tensor.cpp:138,146,149,163,171,174.               */
/* ------------------------------------------------------------------------ */
enum {
  P2R_EPI_BF16 = 0,       /* c(bf16) = acc + bias                              */
  P2R_EPI_F32 = 1,        /* c(f32)  = acc + bias + aux(f32 residual, opt.)   */
  P2R_EPI_ACC_F32 = 2,    /* c(f32) += acc      (beta=1, in-place grad accum) */
  P2R_EPI_BIAS_GELU = 3,  /* c(bf16) = gelu(acc+bias); c2(bf16) = gelu'(acc+bias) */
  P2R_EPI_DGELU = 4,      /* c(bf16) = acc * aux (bf16 GELU derivative that     */
                          /*   BIAS_GELU stored: the GELU backward of its layer) */
  P2R_EPI_F32_BF16 = 5    /* c(f32) = acc + bias + aux; c2(bf16) = same value  */
};
enum { P2R_GROUP_NONE = 0, P2R_GROUP_M = 1, P2R_GROUP_K = 2 };

typedef struct {
  int m, n, k;
  /* A(m,k): a_mn_major=0 -> stored [m][lda] (K contiguous); 1 -> stored [k][lda]. */
  const void* a;
  int lda;
  int a_mn_major;
  /* B(n,k): b_mn_major=0 -> stored [n][ldb]; 1 -> stored [k][ldb]. bf16. */
  const void* b;
  int ldb;
  int b_mn_major;
  int epi;
  void* c;
  int ldc;
  void* c2;
  int ldc2;
  const float* bias; /* [n] fp32 or NULL */
  const void* aux;   /* residual (f32) or pre-activation (bf16), [m][ldaux] */
  int ldaux;
  /* Grouping (MoE experts). GROUP_M: group g owns rows [g*seg_rows, g*seg_rows+counts[g])
   * of A/C/aux, B rows [g*n, (g+1)*n), bias + g*n. GROUP_K: group g owns K rows
   * [g*seg_rows, g*seg_rows+counts[g]) (zero-padded to 64) of A and B, C + g*m*ldc. */
  int group_mode;
  int groups;
  int seg_rows;
  const int* counts; /* device [groups] */
  /* Split-K for plain fp32-output GEMMs: >1 writes fp32 partials to workspace
   * then reduces in split order; <= 0 lets the library pick (wave fill); 1 = off. */
  int split_k;
  /* 0 = auto, 1 = one CTA per 128x256 tile, 2 = CTA pair (cluster of 2,
   * tcgen05 cta_group::2) per 256x256 tile. Pairs apply to ungrouped GEMMs. */
  int cta_group;
  /* EPI_DGELU, ungrouped: += column sums of the bf16 output into bias_grad[n]
   * (the bias gradient of the layer whose pre-activation is aux; add_bias
   * backward, tensor.cpp:227-231), from per-32-row partials the epilogue
   * writes into the workspace (p2r_gemm_workspace_bytes). NULL = off. */
  float* bias_grad;
} p2r_gemm_args;

p2r_status p2r_gemm(const p2r_gemm_args* args, void* stream);
/* Bytes of workspace the library needs for split-K / bias_grad partials (0 if none). */
size_t p2r_gemm_workspace_bytes(const p2r_gemm_args* args);
/* Supply caller-owned scratch (device) the library may use for split-K / bias-grad
 * partials of the GEMMs the CALLING THREAD launches next (thread-local). */
p2r_status p2r_set_workspace(void* ptr, size_t bytes);

/* ------------------------------------------------------------------------ */
/* Fused attention (replaces masked_attention + split/merge_heads,           */
/* tensor.cpp:400-545). qkv: bf16 [B*S, 3d] (q | k | v, heads contiguous);   */
/* o: bf16 [B*S, d]; lse: fp32 [B, H, S]. hd = d/H in {64, 128}.             */
/* ------------------------------------------------------------------------ */
p2r_status p2r_attention_fwd(const void* qkv, void* o, float* lse, int B, int H, int S, int d,
                             int causal, void* stream);
/* dsum_ws: fp32 [B, H, S] scratch. dqkv: bf16 [B*S, 3d] (overwritten). */
p2r_status p2r_attention_bwd(const void* qkv, const void* o, const float* lse, const void* dout,
                             float* dsum_ws, void* dqkv, int B, int H, int S, int d, int causal,
                             void* stream);

/* ------------------------------------------------------------------------ */
/* LayerNorm (tensor.cpp:265-336). d a multiple of 128 in [128, 2048].        */
/* ------------------------------------------------------------------------ */
p2r_status p2r_layernorm_fwd(const float* x, const float* gain, const float* bias, int rows, int d,
                             float eps, void* y_bf16, float* y_f32, float* mean, float* rstd,
                             void* stream);
size_t p2r_layernorm_bwd_workspace(int rows, int d);
/* dx = resid + LN'(dy); ggain/gbias (+=) may be NULL. */
p2r_status p2r_layernorm_bwd(const float* dy, const float* x, const float* mean, const float* rstd,
                             const float* gain, const float* resid, int rows, int d, float* dx,
                             void* dx_bf16, float* ggain, float* gbias, float* partial_ws,
                             void* stream);
/* Grid size (blocks) of the backward; the row count of its column-partial outputs.
 * flags: P2R_LN_RESID when a residual is added, P2R_LN_DY_BF16 for the bf16-dy entry. */
#define P2R_LN_RESID 1
#define P2R_LN_DY_BF16 2
int p2r_layernorm_bwd_blocks(int rows, int d, int flags);
/* p2r_layernorm_bwd plus the dense block's FFN2 bias gradient (add_bias backward,
 * tensor.cpp:227-231), which is the column sum of the residual-stream gradient this
 * call produces for the layer below:
 *  - dx_colsum_ws != NULL: dx's per-block column sums are written there
 *    ([p2r_layernorm_bwd_blocks(rows, d, resid != NULL ? P2R_LN_RESID : 0)][d] floats);
 *  - colsum_in != NULL: colsum_dst[c] += the sum of colsum_in's colsum_blocks rows
 *    (an earlier call's dx_colsum_ws), block order, in the same finish kernel as
 *    ggain/gbias. colsum_in, colsum_blocks and colsum_dst go together (else EINVAL). */
p2r_status p2r_layernorm_bwd_fused(const float* dy, const float* x, const float* mean,
                                   const float* rstd, const float* gain, const float* resid, int rows,
                                   int d, float* dx, void* dx_bf16, float* ggain, float* gbias,
                                   float* partial_ws, float* dx_colsum_ws, const float* colsum_in,
                                   int colsum_blocks, float* colsum_dst, void* stream);
/* The same with a bf16 dy ([rows][d] bf16, the dX GEMM's rounded output): the ring
 * stages half the dy bytes; everything else (fp32 statistics and accumulation) is
 * unchanged. Column partials: p2r_layernorm_bwd_blocks(..., flags | P2R_LN_DY_BF16). */
p2r_status p2r_layernorm_bwd_fused_bf16(const void* dy_bf16, const float* x, const float* mean,
                                        const float* rstd, const float* gain, const float* resid, int rows,
                                        int d, float* dx, void* dx_bf16, float* ggain, float* gbias,
                                        float* partial_ws, float* dx_colsum_ws, const float* colsum_in,
                                        int colsum_blocks, float* colsum_dst, void* stream);

/* Embeddings (embedding_lookup x2 + add, model.cpp:229-241; tensor.cpp:338-368). */
p2r_status p2r_embed_fwd(const int* ids, const float* tok, const float* pos, int T, int S, int d,
                         float* x, void* stream);
/* dtok rows are summed in ascending token order (stable radix sort of ids);
 * ws >= p2r_embed_bwd_workspace(B*S, V) bytes when dtok != NULL. */
size_t p2r_embed_bwd_workspace(int T, int V);
p2r_status p2r_embed_bwd(const int* ids, const float* dx, int B, int S, int d, int V, float* dtok,
                         float* dpos, void* ws, size_t ws_bytes, void* stream);

/* Softmax cross-entropy fwd+bwd (tensor.cpp:670-723). logits fp32 [rows][ld];
 * dlogits bf16 [rows][ldg] = (p - onehot) * loss_grad / denom, zero on masked
 * rows and pad columns; *loss (device) = sum(-log p_t) / denom. */
size_t p2r_cross_entropy_workspace(int rows);
p2r_status p2r_cross_entropy(const float* logits, int rows, int V, int ld, const int* targets,
                             const uint8_t* mask, double denom, float loss_grad,
                             void* dlogits_bf16, int ldg, float* loss, double* loss_sum,
                             double* partial_ws, void* stream);

/* AdamW over one granule (optim.cpp:41-63), bit-exact given equal grads.
 * Segments give (offset, length, decay) inside the granule; bc1/bc2 are the
 * host-computed float bias corrections 1 - powf(beta, t). */
p2r_status p2r_adamw_step(float* p, const float* g, float* m, float* v, void* p_bf16,
                          const long long* seg_off, const long long* seg_len,
                          const int* seg_decay, int nseg, float b1, float b2, float eps, float wd,
                          float lr, float bc1, float bc2, void* stream);
p2r_status p2r_cast_bf16(const float* src, void* dst, long long n, void* stream);

/* Delink broadcast (model.cpp:358-377): dst + l*dst_stride_bytes = src, l < L. */
p2r_status p2r_delink_broadcast(const void* src, void* dst, size_t bytes, size_t dst_stride_bytes,
                                int L, void* stream);

/* Bias gradient column sums (add_bias backward, tensor.cpp:227-231). */
size_t p2r_colsum_workspace(int rows, int n, int groups);
p2r_status p2r_bias_grad(const void* x, int dtype, int ld, int rows, int n, int groups,
                         int seg_rows, const int* counts, float* out, long long out_group_stride,
                         float* ws, void* stream);

/* ------------------------------------------------------------------------ */
/* MoE (model.cpp:248-332; tensor.cpp:370-398, 547-664).                     */
/* ------------------------------------------------------------------------ */
int p2r_moe_capacity(float capacity_factor, int n_tokens, int n_experts, int n_prototypes);
p2r_status p2r_moe_gate_logits(const float* b, const float* gate, int T, int d, int E,
                               float* logits, void* stream);
/* Bit-exact moe_dispatch. pos[t*k+g] = slot row inside the expert segment or -1
 * (dropped); rows_pad/slots_pad: [E*seg_rows] token / group of each admitted
 * row (expert-major, token order); counts[e] = admitted rows. */
p2r_status p2r_moe_route(const float* logits, int T, int E, int k, int capacity, int seg_rows,
                         int* selected, uint8_t* survived, int* pos, int* raw_load, int* counts,
                         int* rows_pad, int* slots_pad, int* dropped, void* stream);
p2r_status p2r_moe_combine_weights(const float* logits, int T, int E, int k, const int* selected,
                                   const uint8_t* survived, float* w, void* stream);
p2r_status p2r_moe_dispatch(const void* src, int src_dtype, int d, int E, int seg_rows,
                            const int* rows_pad, const int* slots_pad, const int* counts,
                            const float* w, int k, void* xe_bf16, int pad_full, void* stream);
/* out[t] = resid[t] + sum over the token's surviving slots (group order) of
 * w * ye[row]; ye: bf16 expert outputs [E][seg_rows][d] (moe_combine, tensor.cpp:609-641). */
p2r_status p2r_moe_combine(const void* ye_bf16, int T, int d, int k, int seg_rows, const int* selected,
                           const int* pos, const float* w, const float* resid, float* out,
                           void* stream);
/* dw[t,g] = <dout[t], ye[row(t,g)]> (moe_combine backward, tensor.cpp:643-662). */
p2r_status p2r_moe_combine_bwd_weights(const float* dout, const void* ye_bf16, int T, int d, int k,
                                       int seg_rows, const int* selected, const int* pos,
                                       float* dw, void* stream);
p2r_status p2r_moe_gate_bwd(const float* b, const float* w, const float* gw, int T, int d, int E,
                            int k, const int* selected, const uint8_t* survived, float* glogits,
                            float* dgate, void* stream);
/* db[t] (+)= sum of the token's expert-input gradients (bf16 dxe [E][seg_rows][d], slots
 * in reverse group order) + glogits . gate^T (gather_rows backward, tensor.cpp:386-396). */
p2r_status p2r_moe_dispatch_bwd(const void* dxe_bf16, int T, int d, int k, int seg_rows,
                                const int* selected, const int* pos, const float* glogits,
                                const float* gate, int E, float* db, int accumulate, void* stream);

/* ------------------------------------------------------------------------ */
/* Expert-parallel exchange over peer memory (model.cpp:334-340 expert map:  */
/* expert e on rank e / (E/W)). Kernels store rows straight into the peer    */
/* ranks' buffers (NVLink peer pointers, or local pointers for a loopback    */
/* group); completion is signalled by the caller (stream memory operations). */
/* Layouts: source [E][seg][d]; owner slots [El][W][seg][d] + counts [El][W];*/
/* owner compact [El][W*seg][d] (zero-padded to 128 rows per expert).        */
/* ------------------------------------------------------------------------ */
/* Source side: admitted rows of every expert (src bf16 (dtype 1), or fp32 (0) scaled
 * by w[t*k + slot] when w != NULL) -> peer_slots[e / El] at [e % El][rank][row];
 * counts[e] -> peer_counts[e / El][(e % El) * W + rank]. */
p2r_status p2r_ep_send_rows(const void* src, int src_dtype, int d, int E, int seg, const int* rows_pad,
                            const int* slots_pad, const int* counts, const float* w, int k, int W, int rank,
                            void* const* peer_slots, int* const* peer_counts, void* stream);
/* Owner side: slots + counts -> compact rows, tot[El] rows per local expert and
 * prefix[El][W+1] (row offset of each source inside the compact segment). */
p2r_status p2r_ep_pack(const void* slots, const int* counts, int d, int seg, int El, int W, void* compact,
                       int* tot, int* prefix, void* stream);
/* Owner side: compact rows -> each source's [E][seg] layout (peer_dst[source]). */
p2r_status p2r_ep_return_rows(const void* compact, const int* prefix, int d, int seg, int El, int W, int rank,
                              void* const* peer_dst, void* stream);

/* ------------------------------------------------------------------------ */
/* Primitive layer of the drop-in tensor API (include/p2r/tensor.hpp):       */
/* generic-shape fp32 kernels for the reference's primitives and their        */
/* backward (tensor.cpp:131-723), deterministic reduction order. Not on the   */
/* training hot path (that is the fused bf16 layer above).                    */
/* ------------------------------------------------------------------------ */
/* C = op(A) op(B) + beta C; op = transpose when ta / tb; batched with strides */
p2r_status p2r_prim_gemm_f32(int ta, int tb, int m, int n, int k, const float* a, int lda, const float* b, int ldb,
                             float* c, int ldc, float beta, int batch, long long sa, long long sb, long long sc,
                             void* stream);
/* op 0: out = a + b; 1: out += a; 2: out = gelu(a); 3: out += b * gelu'(a) */
p2r_status p2r_prim_ew(int op, long long n, const float* a, const float* b, float* out, void* stream);
p2r_status p2r_prim_bias(int rows, int n, const float* x, const float* b, float* out, void* stream);
p2r_status p2r_prim_colsum_acc(int rows, int n, const float* g, float* out, void* stream);
p2r_status p2r_prim_layernorm_fwd(int rows, int d, const float* x, const float* gain, const float* bias, float eps,
                                  float* y, float* xhat, float* inv, void* stream);
p2r_status p2r_prim_layernorm_bwd(int rows, int d, const float* gy, const float* xhat, const float* inv,
                                  const float* gain, float* gx, float* ggain, float* gbias, void* stream);
p2r_status p2r_prim_gather_rows(int n_out, int d, const float* x, const int* rows, float* out, void* stream);
p2r_status p2r_prim_scatter_rows_acc(int n, int d, const float* g, const int* rows, float* gx, void* stream);
/* dir 0: [B*S, H*hd] -> [B, H, S, hd]; 1: inverse; acc: out += */
p2r_status p2r_prim_permute_heads(int dir, int acc, int B, int H, int S, int hd, const float* in, float* out,
                                  void* stream);
p2r_status p2r_prim_softmax_rows(long long rows, int n, int causal_S, float* x, void* stream);
p2r_status p2r_prim_softmax_bwd_rows(long long rows, int n, const float* p, const float* dp, float* ds, void* stream);
/* dir 0: out = weights from logits; dir 1: out(glogits) += backward of w given gw */
p2r_status p2r_prim_selected_softmax(int dir, int T, int E, int k, const float* logits_or_w, const float* gw,
                                     const int* sel, const uint8_t* surv, float* out, void* stream);
p2r_status p2r_prim_combine_fwd(int T, int d, int k, const int* off, const int* crow, const int* cslot,
                                const float* y, const float* w, float* out, void* stream);
p2r_status p2r_prim_combine_bwd(int R, int d, int k, const int* rtok, const int* rslot, const float* dout,
                                const float* y, const float* w, float* dy, float* dw, void* stream);
p2r_status p2r_prim_cross_entropy(int rows, int V, const float* logits, const int* targets, const uint8_t* mask,
                                  double denom, double* row_loss_ws, float* loss, float* glogits, void* stream);

/* out = stage[0] + stage[1] + ... + stage[W-1] (fp32 [W][n], rank order): the
 * deterministic sum of a loopback group's data-parallel all-reduce. */
p2r_status p2r_sum_ranks(const float* stage, int W, long long n, float* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* P2R_CUDA_H_ */
