// Internal helpers shared by the C-ABI translation units (error state, launch
// accounting). Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/p2r_cuda.h"

namespace p2r {

p2r_status set_error(p2r_status code, const char* msg);
p2r_status set_cuda_error(cudaError_t e, const char* where);
void count_launch();
p2r_status attention_fwd_tc(const void* qkv, void* o, float* lse, int B, int H, int S, int d, int causal,
                            cudaStream_t s);
p2r_status attention_bwd_tc(const void* qkv, const void* o, const float* lse, const void* dout, float* dsum,
                            void* dqkv, int B, int H, int S, int d, int causal, cudaStream_t s);

}  // namespace p2r

#define P2R_CHECK_LAUNCH(where)                                        \
  do {                                                                 \
    ::p2r::count_launch();                                             \
    cudaError_t e__ = cudaGetLastError();                              \
    if (e__ != cudaSuccess) return ::p2r::set_cuda_error(e__, where);  \
  } while (0)
