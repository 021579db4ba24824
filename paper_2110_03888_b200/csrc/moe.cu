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
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>

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

// Register-tiled form for E in {8, 16, 32, 64} and d % 32 == 0: TT tokens x E
// experts per block, TT*E/(4*TM) threads, each a TM x 4 (token x expert) micro-tile
// (TM = 4 for E >= 32; TM = 1 for E = 8, 16 keeps 2-4 warps per block) fed by
// two 16-byte shared loads per 16 FFMAs; the next k-chunk is prefetched into
// registers while the current one is consumed. Every output is still one FFMA
// chain over c = 0, 1, ..., d-1, so the logits are bit-identical to the plain
// kernel above (and routing decisions with them).
template <int E, int TT, int TM>
__global__ void __launch_bounds__(TT * E / (4 * TM)) gate_logits_rt_kernel(const float* __restrict__ b,
                                                                          const float* __restrict__ gate, int T,
                                                                          int d, float* __restrict__ logits) {
  constexpr int KC = 32, NT = TT * E / (4 * TM), LDT = TT + 4;
  constexpr int BV = TT * KC / 4 / NT;  // float4 of b per thread per chunk
  constexpr int GV = KC * E / 4 / NT;   // float4 of gate per thread per chunk
  __shared__ __align__(16) float sbT[KC][LDT];
  __shared__ __align__(16) float sg[KC][E];
  pdl_trigger();
  pdl_wait();
  const int t0 = blockIdx.x * TT;
  const int te = threadIdx.x % (E / 4), tq = threadIdx.x / (E / 4);
  static_assert(TT * KC % (4 * NT) == 0 && KC * E % (4 * NT) == 0, "gate tile");
  float acc[TM][4];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  float4 rb[BV], rg[GV];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int v = 0; v < BV; ++v) {
      const int idx = threadIdx.x + NT * v, r = idx / (KC / 4), c4 = idx % (KC / 4);
      rb[v] = t0 + r < T ? __ldg(reinterpret_cast<const float4*>(b + static_cast<long long>(t0 + r) * d + k0) + c4)
                         : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int v = 0; v < GV; ++v) {
      const int idx = threadIdx.x + NT * v;
      rg[v] = __ldg(reinterpret_cast<const float4*>(gate + static_cast<long long>(k0) * E) + idx);
    }
  };
  fetch(0);
  for (int k0 = 0; k0 < d; k0 += KC) {
#pragma unroll
    for (int v = 0; v < BV; ++v) {
      const int idx = threadIdx.x + NT * v, r = idx / (KC / 4), c = 4 * (idx % (KC / 4));
      sbT[c][r] = rb[v].x;
      sbT[c + 1][r] = rb[v].y;
      sbT[c + 2][r] = rb[v].z;
      sbT[c + 3][r] = rb[v].w;
    }
#pragma unroll
    for (int v = 0; v < GV; ++v) reinterpret_cast<float4*>(&sg[0][0])[threadIdx.x + NT * v] = rg[v];
    __syncthreads();
    if (k0 + KC < d) fetch(k0 + KC);
#pragma unroll 8
    for (int c = 0; c < KC; ++c) {
      float av[TM];
      if constexpr (TM == 4) {
        const float4 a = *reinterpret_cast<const float4*>(&sbT[c][4 * tq]);
        av[0] = a.x, av[1] = a.y, av[2] = a.z, av[3] = a.w;
      } else {
        av[0] = sbT[c][tq];
      }
      const float4 g = *reinterpret_cast<const float4*>(&sg[c][4 * te]);
      const float gv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], gv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int t = t0 + TM * tq + i;
    if (t < T)
      *reinterpret_cast<float4*>(logits + static_cast<long long>(t) * E + 4 * te) =
          make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
  }
}

// Routing (model.cpp:294-332), two kernels over chunks of 256 (token, group)
// entries in entry order i = t*k + g:
//  1. route_chunk_kernel: each thread scans its entry's expert group with the
//     reference's strict '>' seeded at the group's first expert (ties keep the
//     lowest index; a NaN never displaces the best; a leading NaN is kept), then
//     ranks the entry among the chunk's earlier entries on the same expert (warp
//     match + per-warp counts + an ordered scan over the 8 warps) and writes the
//     chunk's per-expert histogram.
//  2. route_finish_kernel: the chunk's base per expert = the histograms of all
//     earlier chunks (integer sums, order-free); rank = base + in-chunk rank is the
//     FCFS admission counter of model.cpp:321-328, admitted iff rank < capacity.
//     The last chunk's block also writes raw_load, counts and dropped.
constexpr int kRouteChunk = 256;

__global__ void __launch_bounds__(kRouteChunk) route_chunk_kernel(const float* __restrict__ logits, int T, int E,
                                                                  int k, int* __restrict__ selected,
                                                                  int* __restrict__ rank_tmp,
                                                                  int* __restrict__ hist) {
  extern __shared__ int wcnt[];  // [8][E]
  pdl_trigger();
  pdl_wait();
  constexpr int NW = kRouteChunk / 32;
  const int N = T * k, gs = E / k;
  const int i = blockIdx.x * kRouteChunk + threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int x = threadIdx.x; x < NW * E; x += kRouteChunk) wcnt[x] = 0;
  int best = -1;
  if (i < N) {
    const int t = i / k, g = i % k;
    const float* row = logits + static_cast<long long>(t) * E + static_cast<long long>(g) * gs;
    int b = 0;
    float bv = __ldg(row);
#pragma unroll 8
    for (int e = 1; e < gs; ++e) {
      const float v = __ldg(row + e);
      if (v > bv) {  // strict '>': ties keep the lowest index; NaN never wins
        bv = v;
        b = e;
      }
    }
    best = g * gs + b;
  }
  __syncthreads();  // wcnt zeroed
  const unsigned active = __ballot_sync(0xffffffffu, i < N);
  int rank_w = 0;
  if (i < N) {
    const unsigned peers = __match_any_sync(active, best);
    rank_w = __popc(peers & ((1u << lane) - 1u));
    if (rank_w == 0) wcnt[warp * E + best] = __popc(peers);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += kRouteChunk) {  // exclusive scan over warps, in warp order
    int run = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const int c = wcnt[w * E + e];
      wcnt[w * E + e] = run;
      run += c;
    }
    hist[static_cast<long long>(blockIdx.x) * E + e] = run;
  }
  __syncthreads();
  if (i < N) {
    selected[i] = best;
    rank_tmp[i] = wcnt[warp * E + best] + rank_w;
  }
}

__global__ void __launch_bounds__(kRouteChunk) route_finish_kernel(
    const int* __restrict__ hist, int nchunks, int T, int E, int k, int capacity, int seg_rows,
    const int* __restrict__ selected, int* __restrict__ pos_out, uint8_t* __restrict__ survived,
    int* __restrict__ raw_load, int* __restrict__ counts, int* __restrict__ rows_pad, int* __restrict__ slots_pad,
    int* __restrict__ dropped_out) {
  extern __shared__ int rs[];  // base [E], then partial sums [P][E]
  __shared__ int drop_sh;
  pdl_trigger();
  pdl_wait();
  const int c = blockIdx.x;
  const int P = E >= kRouteChunk ? 1 : kRouteChunk / E;  // partitions of the earlier-chunk range
  int* base = rs;
  int* part = rs + E;
  for (int x = threadIdx.x; x < P * E; x += kRouteChunk) {
    const int e = x % E, p = x / E;
    int sum = 0;
    for (int j = p; j < c; j += P) sum += hist[static_cast<long long>(j) * E + e];
    part[x] = sum;
  }
  if (threadIdx.x == 0) drop_sh = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += kRouteChunk) {
    int sum = 0;
    for (int p = 0; p < P; ++p) sum += part[p * E + e];
    base[e] = sum;
  }
  __syncthreads();
  const int i = c * kRouteChunk + threadIdx.x;
  if (i < T * k) {
    const int best = selected[i];
    const int rank = base[best] + pos_out[i];
    const bool ok = rank < capacity;
    survived[i] = ok ? 1 : 0;
    pos_out[i] = ok ? rank : -1;
    if (ok) {
      rows_pad[static_cast<long long>(best) * seg_rows + rank] = i / k;
      slots_pad[static_cast<long long>(best) * seg_rows + rank] = i % k;
    }
  }
  if (c == nchunks - 1) {
    int dr = 0;
    for (int e = threadIdx.x; e < E; e += kRouteChunk) {
      const int tot = base[e] + hist[static_cast<long long>(c) * E + e];
      raw_load[e] = tot;
      counts[e] = tot < capacity ? tot : capacity;
      dr += tot > capacity ? tot - capacity : 0;
    }
    atomicAdd(&drop_sh, dr);  // integer: exact in any order
    __syncthreads();
    if (threadIdx.x == 0) *dropped_out = drop_sh;
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

// out[t] = resid[t] + sum_{g asc, survived} w[t,g] * ye[sel*seg + pos]   (fp32 sum of bf16 rows)
__global__ void combine_kernel(const __nv_bfloat16* __restrict__ ye, int d, int seg_rows,
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
      acc += w[s] * __bfloat162float(ye[(static_cast<long long>(selected[s]) * seg_rows + p) * d + c]);
    }
    out[static_cast<long long>(t) * d + c] = (resid ? resid[static_cast<long long>(t) * d + c] : 0.f) + acc;
  }
}

// 4-wide forms of dispatch / combine / dispatch backward (d % 4 == 0): 16-byte
// fp32 accesses (8-byte bf16), element arithmetic identical to the scalar kernels.
P2R_DEVICE float4 ld_src4(const float* p) { return *reinterpret_cast<const float4*>(p); }
P2R_DEVICE float4 ld_src4(const __nv_bfloat16* p) {
  const uint2 u = *reinterpret_cast<const uint2*>(p);
  const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x), b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
  return make_float4(__low2float(a), __high2float(a), __low2float(b), __high2float(b));
}
P2R_DEVICE void st_bf4(__nv_bfloat16* p, float x, float y, float z, float w) {
  __nv_bfloat162 a = __floats2bfloat162_rn(x, y), b = __floats2bfloat162_rn(z, w);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&a);
  u.y = *reinterpret_cast<uint32_t*>(&b);
  *reinterpret_cast<uint2*>(p) = u;
}

template <typename Tin>
__global__ void dispatch4_kernel(const Tin* __restrict__ src, int d, const int* __restrict__ rows_pad,
                                 const int* __restrict__ counts, int seg_rows, const float* __restrict__ w,
                                 const int* __restrict__ slots_pad, int k, __nv_bfloat16* __restrict__ xe,
                                 int pad_full) {
  const int e = blockIdx.y, r = blockIdx.x;
  const int cnt = counts[e];
  const int top = pad_full ? seg_rows : min(seg_rows, (cnt + 127) / 128 * 128);
  if (r >= top) return;
  __nv_bfloat16* dst = xe + (static_cast<long long>(e) * seg_rows + r) * d;
  if (r >= cnt) {
    for (int c = 4 * threadIdx.x; c < d; c += 4 * blockDim.x) st_bf4(dst + c, 0.f, 0.f, 0.f, 0.f);
    return;
  }
  const int t = rows_pad[static_cast<long long>(e) * seg_rows + r];
  float scale = 1.f;
  if (w) scale = w[t * k + slots_pad[static_cast<long long>(e) * seg_rows + r]];
  const Tin* sp = src + static_cast<long long>(t) * d;
  for (int c = 4 * threadIdx.x; c < d; c += 4 * blockDim.x) {
    const float4 v = ld_src4(sp + c);
    if (w)
      st_bf4(dst + c, scale * v.x, scale * v.y, scale * v.z, scale * v.w);
    else
      st_bf4(dst + c, v.x, v.y, v.z, v.w);
  }
}

__global__ void combine4_kernel(const __nv_bfloat16* __restrict__ ye, int d, int seg_rows, const int* __restrict__ selected,
                                const int* __restrict__ pos, const float* __restrict__ w, int k,
                                const float* __restrict__ resid, float* __restrict__ out) {
  const int t = blockIdx.x;
  for (int c = 4 * threadIdx.x; c < d; c += 4 * blockDim.x) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j < k; ++j) {
      const int s = t * k + j;
      const int p = pos[s];
      if (p < 0) continue;
      const float ws = w[s];
      const float4 y = ld_src4(ye + (static_cast<long long>(selected[s]) * seg_rows + p) * d + c);
      acc.x += ws * y.x;
      acc.y += ws * y.y;
      acc.z += ws * y.z;
      acc.w += ws * y.w;
    }
    const long long o = static_cast<long long>(t) * d + c;
    const float4 rr = resid ? *reinterpret_cast<const float4*>(resid + o) : make_float4(0.f, 0.f, 0.f, 0.f);
    *reinterpret_cast<float4*>(out + o) = make_float4(rr.x + acc.x, rr.y + acc.y, rr.z + acc.z, rr.w + acc.w);
  }
}

// k-sum of the routed rows only (no gate term: glogits == NULL)
__global__ void dispatch_bwd4_kernel(const __nv_bfloat16* __restrict__ dxe, int d, int k, int seg_rows,
                                     const int* __restrict__ selected, const int* __restrict__ pos,
                                     float* __restrict__ db, int accumulate) {
  const int t = blockIdx.x;
  for (int c = 4 * threadIdx.x; c < d; c += 4 * blockDim.x) {
    const long long o = static_cast<long long>(t) * d + c;
    float4 acc = accumulate ? *reinterpret_cast<const float4*>(db + o) : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = k - 1; j >= 0; --j) {
      const int s = t * k + j;
      const int p = pos[s];
      if (p < 0) continue;
      const float4 g = ld_src4(dxe + (static_cast<long long>(selected[s]) * seg_rows + p) * d + c);
      acc.x += g.x;
      acc.y += g.y;
      acc.z += g.z;
      acc.w += g.w;
    }
    *reinterpret_cast<float4*>(db + o) = acc;
  }
}

// dw[t,g] = <dout[t], ye[row(t,g)]>  (warp per (t,g)); 0 for dropped slots
__global__ void combine_bwd_w_kernel(const float* __restrict__ dout, const __nv_bfloat16* __restrict__ ye,
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
    const __nv_bfloat16* y = ye + (static_cast<long long>(selected[s]) * seg_rows + p) * d;
    for (int c = lane; c < d; c += 32) acc += a[c] * __bfloat162float(y[c]);
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
__global__ void dispatch_bwd_kernel(const __nv_bfloat16* __restrict__ dxe, int d, int k, int seg_rows,
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
      acc += __bfloat162float(dxe[(static_cast<long long>(selected[s]) * seg_rows + p) * d + c]);
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

// Per-(device, stream) scratch for the routing histograms, grown on demand (the
// C-ABI of p2r_moe_route has no workspace argument; growth synchronises).
cudaError_t route_scratch(cudaStream_t s, size_t bytes, int** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<void*, size_t>> pool;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  auto& slot = pool[{dev, s}];
  if (slot.second < bytes) {
    if (slot.first) {
      e = cudaStreamSynchronize(s);
      if (e == cudaSuccess) e = cudaFree(slot.first);
      if (e != cudaSuccess) return e;
      slot = {nullptr, 0};
    }
    e = cudaMalloc(&slot.first, bytes);
    if (e != cudaSuccess) return e;
    slot.second = bytes;
  }
  *out = static_cast<int*>(slot.first);
  return cudaSuccess;
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
#ifdef P2R_DIAG  // diagnostic build: P2R_GATE_PLAIN=1 forces the plain kernel (tests compare the two bit for bit)
  static const bool plain = [] {
    const char* e = std::getenv("P2R_GATE_PLAIN");
    return e != nullptr && e[0] == '1';
  }();
#else
  constexpr bool plain = false;
#endif
  if (!plain && d % 32 == 0 && (E == 8 || E == 16 || E == 32 || E == 64)) {
    cudaError_t le = cudaSuccess;
    if (E == 8) le = launch_k(gate_logits_rt_kernel<8, 32, 1>, dim3(blocks), dim3(64), 0, s, 1, b, gate, T, d, logits);
    if (E == 16)
      le = launch_k(gate_logits_rt_kernel<16, 32, 1>, dim3(blocks), dim3(128), 0, s, 1, b, gate, T, d, logits);
    if (E == 32)
      le = launch_k(gate_logits_rt_kernel<32, 32, 4>, dim3(blocks), dim3(64), 0, s, 1, b, gate, T, d, logits);
    if (E == 64)
      le = launch_k(gate_logits_rt_kernel<64, 32, 4>, dim3(blocks), dim3(128), 0, s, 1, b, gate, T, d, logits);
    if (le != cudaSuccess) return set_cuda_error(le, "moe gate logits");
    P2R_CHECK_LAUNCH("moe gate logits");
    return P2R_OK;
  }
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
  const int N = T * k;
  if (N <= 0) {  // nothing routed: zero loads / counts / drops
    if (E > 0) {
      cudaError_t e = cudaMemsetAsync(raw_load, 0, static_cast<size_t>(E) * sizeof(int), s);
      if (e == cudaSuccess) e = cudaMemsetAsync(counts, 0, static_cast<size_t>(E) * sizeof(int), s);
      if (e == cudaSuccess) e = cudaMemsetAsync(dropped, 0, sizeof(int), s);
      if (e != cudaSuccess) return set_cuda_error(e, "moe route");
    }
    return P2R_OK;
  }
  const int nchunks = (N + kRouteChunk - 1) / kRouteChunk;
  int* hist = nullptr;
  {
    const cudaError_t e = route_scratch(s, static_cast<size_t>(nchunks) * E * sizeof(int), &hist);
    if (e != cudaSuccess) return set_cuda_error(e, "moe route scratch");
  }
  const int smem1 = (kRouteChunk / 32) * E * static_cast<int>(sizeof(int));
  const int P = E >= kRouteChunk ? 1 : kRouteChunk / E;
  const int smem2 = (E + P * E) * static_cast<int>(sizeof(int));
  static const cudaError_t a1 =
      cudaFuncSetAttribute(route_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  static const cudaError_t a2 =
      cudaFuncSetAttribute(route_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  if (a1 != cudaSuccess || a2 != cudaSuccess) return set_cuda_error(a1 != cudaSuccess ? a1 : a2, "route attr");
  cudaError_t le = launch_k(route_chunk_kernel, dim3(nchunks), dim3(kRouteChunk), smem1, s, 1, logits, T, E, k,
                            selected, pos, hist);
  if (le == cudaSuccess)
    le = launch_k(route_finish_kernel, dim3(nchunks), dim3(kRouteChunk), smem2, s, 1,
                  static_cast<const int*>(hist), nchunks, T, E, k, capacity, seg_rows,
                  static_cast<const int*>(selected), pos, survived, raw_load, counts, rows_pad, slots_pad, dropped);
  if (le != cudaSuccess) return set_cuda_error(le, "moe route");
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
  if (d % 4 == 0) {
    const int thr = d >= 2048 ? 256 : 128;
    if (src_dtype == 0)
      dispatch4_kernel<float><<<grid, thr, 0, s>>>(static_cast<const float*>(src), d, rows_pad, counts, seg_rows, w,
                                                   slots_pad, k, static_cast<__nv_bfloat16*>(xe_bf16), pad_full);
    else
      dispatch4_kernel<__nv_bfloat16><<<grid, thr, 0, s>>>(static_cast<const __nv_bfloat16*>(src), d, rows_pad, counts,
                                                           seg_rows, w, slots_pad, k,
                                                           static_cast<__nv_bfloat16*>(xe_bf16), pad_full);
  } else if (src_dtype == 0)
    dispatch_kernel<float><<<grid, 128, 0, s>>>(static_cast<const float*>(src), d, rows_pad, counts, seg_rows, w, slots_pad, k,
                                                static_cast<__nv_bfloat16*>(xe_bf16), pad_full);
  else
    dispatch_kernel<__nv_bfloat16><<<grid, 128, 0, s>>>(static_cast<const __nv_bfloat16*>(src), d, rows_pad, counts, seg_rows, w,
                                                        slots_pad, k, static_cast<__nv_bfloat16*>(xe_bf16), pad_full);
  P2R_CHECK_LAUNCH("moe dispatch");
  return P2R_OK;
}

extern "C" p2r_status p2r_moe_combine(const void* ye_bf16, int T, int d, int k, int seg_rows,
                                      const int* selected, const int* pos, const float* w,
                                      const float* resid, float* out, void* stream) {
  if (T <= 0) return P2R_OK;
  const __nv_bfloat16* ye = static_cast<const __nv_bfloat16*>(ye_bf16);
  if (d % 4 == 0)
    combine4_kernel<<<T, d >= 2048 ? 256 : 128, 0, static_cast<cudaStream_t>(stream)>>>(ye, d, seg_rows, selected, pos,
                                                                                       w, k, resid, out);
  else
    combine_kernel<<<T, 256, 0, static_cast<cudaStream_t>(stream)>>>(ye, d, seg_rows, selected, pos, w, k, resid, out);
  P2R_CHECK_LAUNCH("moe combine");
  return P2R_OK;
}

extern "C" p2r_status p2r_moe_combine_bwd_weights(const float* dout, const void* ye_bf16, int T, int d,
                                                  int k, int seg_rows, const int* selected,
                                                  const int* pos, float* dw, void* stream) {
  if (T <= 0) return P2R_OK;
  const __nv_bfloat16* ye = static_cast<const __nv_bfloat16*>(ye_bf16);
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

extern "C" p2r_status p2r_moe_dispatch_bwd(const void* dxe_bf16, int T, int d, int k, int seg_rows,
                                           const int* selected, const int* pos,
                                           const float* glogits, const float* gate, int E,
                                           float* db, int accumulate, void* stream) {
  if (T <= 0) return P2R_OK;
  const __nv_bfloat16* dxe = static_cast<const __nv_bfloat16*>(dxe_bf16);
  if (glogits == nullptr && d % 4 == 0)
    dispatch_bwd4_kernel<<<T, d >= 2048 ? 256 : 128, 0, static_cast<cudaStream_t>(stream)>>>(dxe, d, k, seg_rows,
                                                                                            selected, pos, db, accumulate);
  else
    dispatch_bwd_kernel<<<T, 256, 0, static_cast<cudaStream_t>(stream)>>>(dxe, d, k, seg_rows, selected, pos, glogits,
                                                                           gate, E, db, accumulate);
  P2R_CHECK_LAUNCH("moe dispatch bwd");
  return P2R_OK;
}
