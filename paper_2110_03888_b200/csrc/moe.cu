// MoE sublayer kernels (model.cpp:248-332, tensor.cpp:370-398, :547-664).
//
//   gate logits (fp32)     matmul(b, gate)                model.cpp:250
//   routing                moe_dispatch                   model.cpp:294-332  (bit-exact)
//   combine weights        selected_softmax fwd/bwd       tensor.cpp:547-607
//   dispatch               gather_rows fwd                tensor.cpp:370-382
//   combine (+ residual)   moe_combine fwd/bwd            tensor.cpp:609-664
//   dispatch backward      gather_rows bwd                tensor.cpp:386-395
//
// Expert-major buffers use a static padded layout: expert e owns rows
// [e*seg, e*seg + count[e]) with seg = roundup(capacity, 128); rows up to the
// next 128 boundary are zero so grouped GEMMs can treat them as K padding.
#include <cmath>

#include "../../include/p2r_cuda.h"
#include "common.cuh"
#include "p2r_internal.h"

namespace p2r {

// logits[t][e] = sum_c b[t][c] * gate[c][e]   (fp32, smem tiled: 32 tokens x E)
template <int E>
__global__ void __launch_bounds__(256) gate_logits_kernel(const float* __restrict__ b,
                                                         const float* __restrict__ gate, int T,
                                                         int d, float* __restrict__ logits) {
  constexpr int TT = 32, KC = 64;
  __shared__ float sb[TT][KC + 1];
  __shared__ float sg[KC][E];
  const int t0 = blockIdx.x * TT;
  constexpr int OUT = TT * E;
  constexpr int PER = (OUT + 255) / 256;
  float acc[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) acc[i] = 0.f;
  for (int k0 = 0; k0 < d; k0 += KC) {
    for (int i = threadIdx.x; i < TT * KC; i += 256) {
      const int r = i / KC, c = i % KC;
      sb[r][c] = (t0 + r < T && k0 + c < d) ? b[static_cast<long long>(t0 + r) * d + k0 + c] : 0.f;
    }
    for (int i = threadIdx.x; i < KC * E; i += 256) {
      const int r = i / E, c = i % E;
      sg[r][c] = (k0 + r < d) ? gate[static_cast<long long>(k0 + r) * E + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int o = threadIdx.x + 256 * i;
      if (o < OUT) {
        const int r = o / E, e = o % E;
        float s = acc[i];
#pragma unroll 8
        for (int c = 0; c < KC; ++c) s += sb[r][c] * sg[c][e];
        acc[i] = s;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int o = threadIdx.x + 256 * i;
    if (o < OUT) {
      const int r = o / E, e = o % E;
      if (t0 + r < T) logits[static_cast<long long>(t0 + r) * E + e] = acc[i];
    }
  }
}

// Routing: one CTA of 1024 threads walks the T*k (token, group) entries in
// order, chunk by chunk, computing each entry's rank among earlier entries
// that picked the same expert (warp match + per-warp counts + ordered scan).
// Admission = rank < capacity reproduces the FCFS counters of model.cpp:321-328.
__global__ void __launch_bounds__(1024) route_kernel(const float* __restrict__ logits, int T, int E,
                                                    int k, int capacity, int seg_rows,
                                                    int* __restrict__ selected,
                                                    uint8_t* __restrict__ survived,
                                                    int* __restrict__ pos_out,
                                                    int* __restrict__ raw_load,
                                                    int* __restrict__ counts,
                                                    int* __restrict__ rows_pad,
                                                    int* __restrict__ slots_pad,
                                                    int* __restrict__ dropped_out) {
  extern __shared__ int sm[];
  int* base = sm;                 // [E]  running count per expert
  int* wcnt = sm + E;             // [32][E] per-warp counts in this chunk
  const int gs = E / k;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int e = threadIdx.x; e < E; e += blockDim.x) base[e] = 0;
  const int N = T * k;
  for (int c0 = 0; c0 < N; c0 += 1024) {
    for (int i = threadIdx.x; i < 32 * E; i += blockDim.x) wcnt[i] = 0;
    __syncthreads();
    const int i = c0 + threadIdx.x;
    int best = -1;
    if (i < N) {
      const int t = i / k, g = i % k;
      const float* row = logits + static_cast<long long>(t) * E;
      best = g * gs;
      float bv = row[best];
      for (int e = g * gs + 1; e < (g + 1) * gs; ++e) {
        const float v = row[e];
        if (v > bv) {  // strict '>': ties keep the lowest index; NaN never wins
          bv = v;
          best = e;
        }
      }
    }
    const unsigned active = __ballot_sync(0xffffffffu, i < N);
    unsigned peers = 0;
    int rank_w = 0;
    if (i < N) {
      peers = __match_any_sync(active, best);
      rank_w = __popc(peers & ((1u << lane) - 1u));
      if (rank_w == 0) wcnt[warp * E + best] = __popc(peers);
    }
    __syncthreads();
    // exclusive scan over warps per expert (ordered), then advance base
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      int run = base[e];
      for (int w = 0; w < 32; ++w) {
        const int c = wcnt[w * E + e];
        wcnt[w * E + e] = run;
        run += c;
      }
      base[e] = run;
    }
    __syncthreads();
    if (i < N) {
      const int rank = wcnt[warp * E + best] + rank_w;
      selected[i] = best;
      const bool ok = rank < capacity;
      survived[i] = ok ? 1 : 0;
      pos_out[i] = ok ? rank : -1;
      if (ok) {
        rows_pad[static_cast<long long>(best) * seg_rows + rank] = i / k;
        slots_pad[static_cast<long long>(best) * seg_rows + rank] = i % k;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int dr = 0;
    for (int e = 0; e < E; ++e) dr += base[e] > capacity ? base[e] - capacity : 0;
    *dropped_out = dr;
  }
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    raw_load[e] = base[e];
    counts[e] = base[e] < capacity ? base[e] : capacity;
  }
}

// selected_softmax forward, one thread per token, reference op order.
__global__ void sel_softmax_kernel(const float* __restrict__ logits, int T, int E, int k,
                                   const int* __restrict__ selected,
                                   const uint8_t* __restrict__ survived, float* __restrict__ w) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  float mx = -1e30f;
  for (int j = 0; j < k; ++j)
    if (survived[t * k + j]) mx = fmaxf(mx, logits[static_cast<long long>(t) * E + selected[t * k + j]]);
  float sum = 0.f;
  for (int j = 0; j < k; ++j) {
    const int s = t * k + j;
    float e = 0.f;
    if (survived[s]) {
      e = expf(logits[static_cast<long long>(t) * E + selected[s]] - mx);
      sum += e;
    }
    w[s] = e;
  }
  if (sum > 0.f) {
    const float inv = 1.0f / sum;
    for (int j = 0; j < k; ++j)
      if (survived[t * k + j]) w[t * k + j] *= inv;
  }
}

// xe[e*seg + r] = src[rows_pad[e*seg + r]] for r < count[e]; zero rows up to the
// next 128 boundary. One block per padded row, bf16 out (fp32 or bf16 in).
template <typename Tin>
__global__ void dispatch_kernel(const Tin* __restrict__ src, int d, const int* __restrict__ rows_pad,
                                const int* __restrict__ counts, int seg_rows,
                                const float* __restrict__ w, const int* __restrict__ slots_pad,
                                int k, __nv_bfloat16* __restrict__ xe, int pad_full) {
  const int e = blockIdx.y, r = blockIdx.x;
  const int cnt = counts[e];
  // pad_full: zero the whole segment (expert-parallel owners run full-capacity groups)
  const int top = pad_full ? seg_rows : min(seg_rows, (cnt + 127) / 128 * 128);
  if (r >= top) return;
  __nv_bfloat16* dst = xe + (static_cast<long long>(e) * seg_rows + r) * d;
  if (r >= cnt) {
    for (int c = threadIdx.x; c < d; c += blockDim.x) dst[c] = __float2bfloat16_rn(0.f);
    return;
  }
  const int t = rows_pad[static_cast<long long>(e) * seg_rows + r];
  float scale = 1.f;
  if (w) scale = w[t * k + slots_pad[static_cast<long long>(e) * seg_rows + r]];
  const Tin* s = src + static_cast<long long>(t) * d;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float v;
    if constexpr (sizeof(Tin) == 4)
      v = s[c];
    else
      v = __bfloat162float(s[c]);
    dst[c] = __float2bfloat16_rn(w ? scale * v : v);
  }
}

// out[t] = resid[t] + sum_{g asc, survived} w[t,g] * ye[sel*seg + pos]   (fp32)
__global__ void combine_kernel(const float* __restrict__ ye, int d, int seg_rows,
                               const int* __restrict__ selected, const int* __restrict__ pos,
                               const float* __restrict__ w, int k,
                               const float* __restrict__ resid, float* __restrict__ out) {
  const int t = blockIdx.x;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float acc = 0.f;
    for (int j = 0; j < k; ++j) {
      const int s = t * k + j;
      const int p = pos[s];
      if (p < 0) continue;
      acc += w[s] * ye[(static_cast<long long>(selected[s]) * seg_rows + p) * d + c];
    }
    out[static_cast<long long>(t) * d + c] = (resid ? resid[static_cast<long long>(t) * d + c] : 0.f) + acc;
  }
}

// dw[t,g] = <dout[t], ye[row(t,g)]>  (warp per (t,g)); 0 for dropped slots
__global__ void combine_bwd_w_kernel(const float* __restrict__ dout, const float* __restrict__ ye,
                                     int T, int d, int k, int seg_rows,
                                     const int* __restrict__ selected, const int* __restrict__ pos,
                                     float* __restrict__ dw) {
  const int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= T * k) return;
  const int p = pos[s];
  float acc = 0.f;
  if (p >= 0) {
    const int t = s / k;
    const float* a = dout + static_cast<long long>(t) * d;
    const float* y = ye + (static_cast<long long>(selected[s]) * seg_rows + p) * d;
    for (int c = lane; c < d; c += 32) acc += a[c] * y[c];
  }
  acc = warp_sum(acc);
  if (lane == 0) dw[s] = acc;
}

// selected_softmax backward: glogits[t][sel] = w * (gw - sum_j w_j gw_j) (0 elsewhere)
__global__ void sel_softmax_bwd_kernel(const float* __restrict__ w, const float* __restrict__ gw,
                                       int T, int E, int k, const int* __restrict__ selected,
                                       const uint8_t* __restrict__ survived,
                                       float* __restrict__ glogits) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  float* gl = glogits + static_cast<long long>(t) * E;
  for (int e = 0; e < E; ++e) gl[e] = 0.f;
  float dot = 0.f;
  for (int j = 0; j < k; ++j)
    if (survived[t * k + j]) dot += w[t * k + j] * gw[t * k + j];
  for (int j = 0; j < k; ++j) {
    const int s = t * k + j;
    if (survived[s]) gl[selected[s]] += w[s] * (gw[s] - dot);
  }
}

// db[t] = (accumulate ? db[t] : 0) + sum over the token's slots (g DESC, the
// tape's reverse expert order) of dxe[row] + glogits[t] . gate^T
__global__ void dispatch_bwd_kernel(const float* __restrict__ dxe, int d, int k, int seg_rows,
                                    const int* __restrict__ selected, const int* __restrict__ pos,
                                    const float* __restrict__ glogits, const float* __restrict__ gate,
                                    int E, float* __restrict__ db, int accumulate) {
  const int t = blockIdx.x;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float acc = accumulate ? db[static_cast<long long>(t) * d + c] : 0.f;
    for (int j = k - 1; j >= 0; --j) {
      const int s = t * k + j;
      const int p = pos[s];
      if (p < 0) continue;
      acc += dxe[(static_cast<long long>(selected[s]) * seg_rows + p) * d + c];
    }
    if (glogits) {
      float g = 0.f;
      for (int e = 0; e < E; ++e) g += glogits[static_cast<long long>(t) * E + e] * gate[static_cast<long long>(c) * E + e];
      acc += g;
    }
    db[static_cast<long long>(t) * d + c] = acc;
  }
}

// dgate[c][e] += sum_t b[t][c] * glogits[t][e]   (deterministic, thread per output)
__global__ void gate_bwd_kernel(const float* __restrict__ b, const float* __restrict__ glogits, int T,
                                int d, int E, float* __restrict__ dgate) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= d * E) return;
  const int c = o / E, e = o % E;
  float s = 0.f;
  for (int t = 0; t < T; ++t) s += b[static_cast<long long>(t) * d + c] * glogits[static_cast<long long>(t) * E + e];
  dgate[o] += s;
}

}  // namespace p2r

using namespace p2r;

extern "C" int p2r_moe_capacity(float capacity_factor, int n_tokens, int n_experts, int n_prototypes) {
  // model.cpp:308-309: computed in double, then ceil
  const int gs = n_experts / n_prototypes;
  return static_cast<int>(
      std::ceil(static_cast<double>(capacity_factor) * n_tokens / static_cast<double>(gs)));
}

extern "C" p2r_status p2r_moe_gate_logits(const float* b, const float* gate, int T, int d, int E,
                                          float* logits, void* stream) {
  if (T <= 0) return P2R_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int blocks = (T + 31) / 32;
  switch (E) {
    case 2: gate_logits_kernel<2><<<blocks, 256, 0, s>>>(b, gate, T, d, logits); break;
    case 4: gate_logits_kernel<4><<<blocks, 256, 0, s>>>(b, gate, T, d, logits); break;
    case 8: gate_logits_kernel<8><<<blocks, 256, 0, s>>>(b, gate, T, d, logits); break;
    case 16: gate_logits_kernel<16><<<blocks, 256, 0, s>>>(b, gate, T, d, logits); break;
    case 32: gate_logits_kernel<32><<<blocks, 256, 0, s>>>(b, gate, T, d, logits); break;
    case 64: gate_logits_kernel<64><<<blocks, 256, 0, s>>>(b, gate, T, d, logits); break;
    default: return set_error(P2R_EINVAL, "moe gate: n_experts must be 2,4,8,16,32 or 64");
  }
  P2R_CHECK_LAUNCH("moe gate logits");
  return P2R_OK;
}

extern "C" p2r_status p2r_moe_route(const float* logits, int T, int E, int k, int capacity,
                                    int seg_rows, int* selected, uint8_t* survived, int* pos,
                                    int* raw_load, int* counts, int* rows_pad, int* slots_pad,
                                    int* dropped, void* stream) {
  if (k <= 0 || E % k != 0)
    return set_error(P2R_EINVAL, "moe config: n_experts must be divisible by n_prototypes");
  if (seg_rows < (capacity < T ? capacity : T))
    return set_error(P2R_EINVAL, "moe route: seg_rows must be >= capacity");
  if (E > 1024) return set_error(P2R_EINVAL, "moe route: at most 1024 experts per rank");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int smem = (E + 32 * E) * static_cast<int>(sizeof(int));
  if (smem > 48 * 1024) {
    static cudaError_t e = cudaFuncSetAttribute(route_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e != cudaSuccess) return set_cuda_error(e, "route attr");
  }
  route_kernel<<<1, 1024, smem, s>>>(logits, T, E, k, capacity, seg_rows, selected, survived, pos,
                                     raw_load, counts, rows_pad, slots_pad, dropped);
  P2R_CHECK_LAUNCH("moe route");
  return P2R_OK;
}

extern "C" p2r_status p2r_moe_combine_weights(const float* logits, int T, int E, int k,
                                              const int* selected, const uint8_t* survived,
                                              float* w, void* stream) {
  if (T <= 0) return P2R_OK;
  sel_softmax_kernel<<<(T + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(logits, T, E, k, selected, survived, w);
  P2R_CHECK_LAUNCH("moe combine weights");
  return P2R_OK;
}

// src_dtype: 0 fp32, 1 bf16. w != NULL scales each gathered row by its combine weight.
extern "C" p2r_status p2r_moe_dispatch(const void* src, int src_dtype, int d, int E, int seg_rows,
                                       const int* rows_pad, const int* slots_pad, const int* counts,
                                       const float* w, int k, void* xe_bf16, int pad_full, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  dim3 grid(seg_rows, E);
  if (src_dtype == 0)
    dispatch_kernel<float><<<grid, 128, 0, s>>>(static_cast<const float*>(src), d, rows_pad, counts, seg_rows, w, slots_pad, k,
                                                static_cast<__nv_bfloat16*>(xe_bf16), pad_full);
  else
    dispatch_kernel<__nv_bfloat16><<<grid, 128, 0, s>>>(static_cast<const __nv_bfloat16*>(src), d, rows_pad, counts, seg_rows, w,
                                                        slots_pad, k, static_cast<__nv_bfloat16*>(xe_bf16), pad_full);
  P2R_CHECK_LAUNCH("moe dispatch");
  return P2R_OK;
}

extern "C" p2r_status p2r_moe_combine(const float* ye, int T, int d, int k, int seg_rows,
                                      const int* selected, const int* pos, const float* w,
                                      const float* resid, float* out, void* stream) {
  if (T <= 0) return P2R_OK;
  combine_kernel<<<T, 256, 0, static_cast<cudaStream_t>(stream)>>>(ye, d, seg_rows, selected, pos, w, k, resid, out);
  P2R_CHECK_LAUNCH("moe combine");
  return P2R_OK;
}

extern "C" p2r_status p2r_moe_combine_bwd_weights(const float* dout, const float* ye, int T, int d,
                                                  int k, int seg_rows, const int* selected,
                                                  const int* pos, float* dw, void* stream) {
  if (T <= 0) return P2R_OK;
  const long long warps = static_cast<long long>(T) * k;
  combine_bwd_w_kernel<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      dout, ye, T, d, k, seg_rows, selected, pos, dw);
  P2R_CHECK_LAUNCH("moe combine bwd w");
  return P2R_OK;
}

extern "C" p2r_status p2r_moe_gate_bwd(const float* b, const float* w, const float* gw, int T,
                                       int d, int E, int k, const int* selected,
                                       const uint8_t* survived, float* glogits, float* dgate,
                                       void* stream) {
  if (T <= 0) return P2R_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  sel_softmax_bwd_kernel<<<(T + 255) / 256, 256, 0, s>>>(w, gw, T, E, k, selected, survived, glogits);
  P2R_CHECK_LAUNCH("moe selected softmax bwd");
  gate_bwd_kernel<<<(d * E + 255) / 256, 256, 0, s>>>(b, glogits, T, d, E, dgate);
  P2R_CHECK_LAUNCH("moe gate bwd");
  return P2R_OK;
}

extern "C" p2r_status p2r_moe_dispatch_bwd(const float* dxe, int T, int d, int k, int seg_rows,
                                           const int* selected, const int* pos,
                                           const float* glogits, const float* gate, int E,
                                           float* db, int accumulate, void* stream) {
  if (T <= 0) return P2R_OK;
  dispatch_bwd_kernel<<<T, 256, 0, static_cast<cudaStream_t>(stream)>>>(dxe, d, k, seg_rows, selected, pos, glogits, gate, E, db,
                                                                         accumulate);
  P2R_CHECK_LAUNCH("moe dispatch bwd");
  return P2R_OK;
}
