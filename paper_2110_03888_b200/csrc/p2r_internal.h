// Internal helpers shared by the C-ABI translation units (error state, launch
// accounting). Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <utility>

#include "../../include/p2r_cuda.h"

namespace p2r {

p2r_status set_error(p2r_status code, const char* msg);
p2r_status set_cuda_error(cudaError_t e, const char* where);
void count_launch();
void count_launches(uint64_t n);  // graph replays: the kernels a captured graph launches
p2r_status attention_fwd_tc(const void* qkv, void* o, float* lse, int B, int H, int S, int d, int causal,
                            cudaStream_t s);
p2r_status attention_bwd_tc(const void* qkv, const void* o, const float* lse, const void* dout, float* dsum,
                            void* dqkv, int B, int H, int S, int d, int causal, cudaStream_t s);

// Launch with programmatic dependent launch (and an optional cluster size). The
// kernel must call pdl_wait() before reading data produced earlier in the stream.
// P2R_PDL=0 falls back to plain stream-ordered launches (A/B diagnostics).
// out[g * out_group_stride + col] += sum over c < nchunks of partial[(g * nchunks + c) * n + col]
// (fixed order; optim_delink.cu). Shared by p2r_bias_grad and the GELU' GEMM epilogue.
cudaError_t colsum_finish_launch(const float* partial, int nchunks, int n, int groups, float* out,
                                 long long out_group_stride, cudaStream_t s);

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("P2R_PDL");
    return e == nullptr || e[0] != '0';
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, int cluster_x,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  unsigned n = 0;
  if (pdl_enabled()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_x > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = static_cast<unsigned>(cluster_x);
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = n ? at : nullptr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace p2r

// launch_k(...) + error mapping + launch accounting
#define P2R_LAUNCH_K(where, ...)                                        \
  do {                                                                 \
    cudaError_t le__ = ::p2r::launch_k(__VA_ARGS__);                   \
    if (le__ != cudaSuccess) return ::p2r::set_cuda_error(le__, where); \
  } while (0);                                                         \
  P2R_CHECK_LAUNCH(where)

#define P2R_CHECK_LAUNCH(where)                                        \
  do {                                                                 \
    ::p2r::count_launch();                                             \
    cudaError_t e__ = cudaGetLastError();                              \
    if (e__ != cudaSuccess) return ::p2r::set_cuda_error(e__, where);  \
  } while (0)
