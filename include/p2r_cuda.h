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
  P2R_EPI_BIAS_GELU = 3,  /* c(bf16) = gelu(acc+bias); c2(bf16) = acc+bias    */
  P2R_EPI_DGELU = 4,      /* c(bf16) = acc * gelu'(aux bf16 pre-activation)   */
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
  /* Split-K for plain GEMMs: >1 writes fp32 partials to workspace then reduces. */
  int split_k;
} p2r_gemm_args;

p2r_status p2r_gemm(const p2r_gemm_args* args, void* stream);
/* Bytes of workspace the library needs for split-K on this GEMM (0 if none). */
size_t p2r_gemm_workspace_bytes(const p2r_gemm_args* args);
/* Supply caller-owned scratch (device) the library may use for split-K. */
p2r_status p2r_set_workspace(void* ptr, size_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* P2R_CUDA_H_ */
