// LayerNorm fwd/bwd, token+position embedding fwd/bwd, fused softmax-CE fwd/bwd.
//
//   layernorm            tensor.cpp:265-336 (two-pass mean / biased var, eps 1e-5)
//   embedding_lookup+add tensor.cpp:338-368, model.cpp:229-241
//   softmax_cross_entropy tensor.cpp:670-723 (fp64 loss sum, / denom, masked rows)
// All reductions are deterministic (fixed-order trees, no float atomics).
#include <cub/device/device_radix_sort.cuh>

#include "../../include/p2r_cuda.h"
#include "common.cuh"
#include "p2r_internal.h"

namespace p2r {

// ------------------------------- LayerNorm -----------------------------------
// One warp per row; NV float4 per lane (d = 128 * NV).
template <int NV>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const float* __restrict__ x,
                                                    const float* __restrict__ gain,
                                                    const float* __restrict__ bias, int rows,
                                                    float eps, __nv_bfloat16* __restrict__ y16,
                                                    float* __restrict__ y32,
                                                    float* __restrict__ mean_out,
                                                    float* __restrict__ rstd_out) {
  constexpr int D = 128 * NV;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const float4* xr = reinterpret_cast<const float4*>(x + static_cast<long long>(warp) * D);
  float4 v[NV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    v[i] = xr[lane + 32 * i];
    s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  }
  s = warp_sum(s);
  const float mean = s / static_cast<float>(D);
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float a = v[i].x - mean, b = v[i].y - mean, c = v[i].z - mean, d = v[i].w - mean;
    q += (a * a + b * b) + (c * c + d * d);
  }
  q = warp_sum(q);
  const float var = q / static_cast<float>(D);
  const float inv = 1.0f / sqrtf(var + eps);
  if (lane == 0) {
    mean_out[warp] = mean;
    rstd_out[warp] = inv;
  }
  const float4* g4 = reinterpret_cast<const float4*>(gain);
  const float4* b4 = reinterpret_cast<const float4*>(bias);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    const float4 g = g4[c4], bb = b4[c4];
    float4 o;
    o.x = (v[i].x - mean) * inv * g.x + bb.x;
    o.y = (v[i].y - mean) * inv * g.y + bb.y;
    o.z = (v[i].z - mean) * inv * g.z + bb.z;
    o.w = (v[i].w - mean) * inv * g.w + bb.w;
    const long long off = static_cast<long long>(warp) * D + 4LL * c4;
    if (y16) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
      uint2 w;
      w.x = *reinterpret_cast<uint32_t*>(&lo);
      w.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(y16 + off) = w;
    }
    if (y32) *reinterpret_cast<float4*>(y32 + off) = o;
  }
}

// dx = resid + inv * (gy - mean(gy) - xhat * mean(gy * xhat)), gy = dy * gain.
// Per-block partial sums of dy*xhat and dy (for dgain/dbias) go to `partial`
// ([gridDim.x][2][D]); ln_param_grad_reduce adds them into the grads in order.
template <int NV>
__global__ void __launch_bounds__(256) ln_bwd_kernel(
    const float* __restrict__ dy, const float* __restrict__ x, const float* __restrict__ mean_in,
    const float* __restrict__ rstd_in, const float* __restrict__ gain,
    const float* __restrict__ resid, int rows, int rows_per_block, float* __restrict__ dx32,
    __nv_bfloat16* __restrict__ dx16, float* __restrict__ partial) {
  constexpr int D = 128 * NV;
  __shared__ float red[8][2][128];  // per-warp partials, one float4-slice at a time
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(rows, r0 + rows_per_block);
  float4 pg[NV], pb[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) pg[i] = pb[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  const float4* g4 = reinterpret_cast<const float4*>(gain);
  for (int r = r0 + warp; r < r1; r += 8) {
    const float4* dyr = reinterpret_cast<const float4*>(dy + static_cast<long long>(r) * D);
    const float4* xr = reinterpret_cast<const float4*>(x + static_cast<long long>(r) * D);
    const float mean = mean_in[r], inv = rstd_in[r];
    float4 h[NV], gy[NV];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c4 = lane + 32 * i;
      const float4 d = dyr[c4], xv = xr[c4], g = g4[c4];
      h[i] = make_float4((xv.x - mean) * inv, (xv.y - mean) * inv, (xv.z - mean) * inv,
                         (xv.w - mean) * inv);
      pg[i].x += d.x * h[i].x;
      pg[i].y += d.y * h[i].y;
      pg[i].z += d.z * h[i].z;
      pg[i].w += d.w * h[i].w;
      pb[i].x += d.x;
      pb[i].y += d.y;
      pb[i].z += d.z;
      pb[i].w += d.w;
      gy[i] = make_float4(d.x * g.x, d.y * g.y, d.z * g.z, d.w * g.w);
      s1 += (gy[i].x + gy[i].y) + (gy[i].z + gy[i].w);
      s2 += (gy[i].x * h[i].x + gy[i].y * h[i].y) + (gy[i].z * h[i].z + gy[i].w * h[i].w);
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    const float inv_d = 1.0f / static_cast<float>(D);
    const float a1 = inv_d * s1, a2 = inv_d * s2;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c4 = lane + 32 * i;
      const long long off = static_cast<long long>(r) * D + 4LL * c4;
      float4 o = make_float4(inv * (gy[i].x - a1 - h[i].x * a2), inv * (gy[i].y - a1 - h[i].y * a2),
                             inv * (gy[i].z - a1 - h[i].z * a2), inv * (gy[i].w - a1 - h[i].w * a2));
      if (resid) {
        const float4 rr = *reinterpret_cast<const float4*>(resid + off);
        o.x += rr.x;
        o.y += rr.y;
        o.z += rr.z;
        o.w += rr.w;
      }
      *reinterpret_cast<float4*>(dx32 + off) = o;
      if (dx16) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&lo);
        w.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(dx16 + off) = w;
      }
    }
  }
  // block reduce of the per-warp column partials (fixed order: warp 0..7)
  float* out = partial + static_cast<long long>(blockIdx.x) * 2 * D;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    red[warp][0][4 * lane + 0] = pg[i].x;
    red[warp][0][4 * lane + 1] = pg[i].y;
    red[warp][0][4 * lane + 2] = pg[i].z;
    red[warp][0][4 * lane + 3] = pg[i].w;
    red[warp][1][4 * lane + 0] = pb[i].x;
    red[warp][1][4 * lane + 1] = pb[i].y;
    red[warp][1][4 * lane + 2] = pb[i].z;
    red[warp][1][4 * lane + 3] = pb[i].w;
    __syncthreads();
    const int t = threadIdx.x;  // 256 threads: t<128 gain, else bias
    const int which = t >> 7, c = t & 127;
    float s = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][which][c];
    out[which * D + 4 * (32 * i) + c] = s;
    (void)c4;
    __syncthreads();
  }
}

// grad_gain[c] += sum_b partial[b][0][c]; grad_bias[c] += sum_b partial[b][1][c].
// Block of 8 warps per 32 flattened columns: warp w sums partial rows w, w+8, ...
// (coalesced 128-byte rows), then the 8 warp sums are added in warp order.
__global__ void __launch_bounds__(256) ln_param_grad_reduce(const float* __restrict__ partial, int nblk,
                                                            int D, float* __restrict__ ggain,
                                                            float* __restrict__ gbias) {
  __shared__ float red[8][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 32 + lane;  // flattened [2][D] column
  float s = 0.f;
  if (c < 2 * D) {
#pragma unroll 4
    for (int b = warp; b < nblk; b += 8) s += partial[static_cast<long long>(b) * 2 * D + c];
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && c < 2 * D) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
    const int which = c / D, col = c % D;
    float* dst = which ? gbias : ggain;
    if (dst) dst[col] += t;
  }
}

// ------------------------------- embeddings ----------------------------------
__global__ void embed_fwd_kernel(const int* __restrict__ ids, const float* __restrict__ tok,
                                 const float* __restrict__ pos, int T, int S, int d,
                                 float* __restrict__ x) {
  const int t = blockIdx.x;
  if (t >= T) return;
  const int id = ids[t];
  const int s = t % S;
  const float4* a = reinterpret_cast<const float4*>(tok + static_cast<long long>(id) * d);
  const float4* b = reinterpret_cast<const float4*>(pos + static_cast<long long>(s) * d);
  float4* o = reinterpret_cast<float4*>(x + static_cast<long long>(t) * d);
  for (int c = threadIdx.x; c < d / 4; c += blockDim.x) {
    const float4 u = a[c], v = b[c];
    o[c] = make_float4(u.x + v.x, u.y + v.y, u.z + v.z, u.w + v.w);
  }
}

// dtok[v] += sum_{t: ids[t]==v, t ascending} dx[t]  (token-order scatter-add, tensor.cpp:356-365).
// The ids are stably radix-sorted (positions as values), so each id's run lists
// its tokens in ascending order; one block per id sums its run in that order.
__global__ void iota_kernel(int* __restrict__ v, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

__global__ void run_bounds_kernel(const int* __restrict__ keys, int n, int* __restrict__ start,
                                  int* __restrict__ end) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int k = keys[i];
  if (i == 0 || keys[i - 1] != k) start[k] = i;
  if (i == n - 1 || keys[i + 1] != k) end[k] = i + 1;
}

__global__ void embed_tok_bwd_kernel(const int* __restrict__ order, const int* __restrict__ start,
                                     const int* __restrict__ end, const float* __restrict__ dx, int d,
                                     float* __restrict__ dtok) {
  const int v = blockIdx.x;
  const int b = start[v], e = end[v];
  if (b >= e) return;
  const int c0 = (blockIdx.y * blockDim.x + threadIdx.x) * 4;
  if (c0 >= d) return;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = b; i < e; ++i) {
    const float4 g = *reinterpret_cast<const float4*>(dx + static_cast<long long>(order[i]) * d + c0);
    acc.x += g.x;
    acc.y += g.y;
    acc.z += g.z;
    acc.w += g.w;
  }
  float4* o = reinterpret_cast<float4*>(dtok + static_cast<long long>(v) * d + c0);
  const float4 cur = *o;
  *o = make_float4(cur.x + acc.x, cur.y + acc.y, cur.z + acc.z, cur.w + acc.w);
}

// dpos[s] += sum_b dx[b*S + s]
__global__ void embed_pos_bwd_kernel(const float* __restrict__ dx, int B, int S, int d,
                                     float* __restrict__ dpos) {
  const int s = blockIdx.x;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    float acc = 0.f;
    for (int b = 0; b < B; ++b) acc += dx[(static_cast<long long>(b) * S + s) * d + c];
    dpos[static_cast<long long>(s) * d + c] += acc;
  }
}

// ------------------------------- cross-entropy --------------------------------
// Warp per row over logits [rows][ld] (fp32, V valid columns). Writes bf16
// dlogits = (p - onehot) * (1/denom) (0 for masked rows and pad columns) and a
// per-block fp64 partial of sum(-log p[target]).
__global__ void __launch_bounds__(256) ce_kernel(const float* __restrict__ logits, int rows, int V,
                                                int ld, const int* __restrict__ targets,
                                                const uint8_t* __restrict__ mask, float scale,
                                                __nv_bfloat16* __restrict__ dlogits, int ldg,
                                                double* __restrict__ partial) {
  __shared__ double wsum[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + warp;
  double lossv = 0.0;
  if (r < rows) {
    const float* row = logits + static_cast<long long>(r) * ld;
    float mx = -INFINITY;
    for (int c = lane; c < V; c += 32) mx = fmaxf(mx, row[c]);
    mx = warp_max(mx);
    float s = 0.f;
    for (int c = lane; c < V; c += 32) s += expf(row[c] - mx);
    s = warp_sum(s);
    const float inv = 1.0f / s;
    const bool active = mask == nullptr || mask[r] != 0;
    const int t = targets[r];
    __nv_bfloat16* g = dlogits + static_cast<long long>(r) * ldg;
    for (int c = lane; c < ldg; c += 32) {
      float v = 0.f;
      if (active && c < V) {
        const float p = expf(row[c] - mx) * inv;
        v = (p - (c == t ? 1.0f : 0.0f)) * scale;
      }
      g[c] = __float2bfloat16_rn(v);
    }
    if (active && lane == 0) {
      const float pt = expf(row[t] - mx) * inv;
      lossv = -log(static_cast<double>(pt));
    }
  }
  if (lane == 0) wsum[warp] = lossv;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += wsum[w];
    partial[blockIdx.x] = s;
  }
}

__global__ void ce_finalize(const double* __restrict__ partial, int n, double denom,
                            float* __restrict__ loss, double* __restrict__ loss_sum) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += partial[i];
    if (loss_sum) *loss_sum = s;
    *loss = static_cast<float>(s / denom);
  }
}

}  // namespace p2r

using namespace p2r;

extern "C" p2r_status p2r_layernorm_fwd(const float* x, const float* gain, const float* bias,
                                        int rows, int d, float eps, void* y_bf16, float* y_f32,
                                        float* mean, float* rstd, void* stream) {
  if (rows <= 0) return P2R_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int blocks = (rows + 7) / 8;
  auto* y16 = static_cast<__nv_bfloat16*>(y_bf16);
  switch (d) {
    case 128: ln_fwd_kernel<1><<<blocks, 256, 0, s>>>(x, gain, bias, rows, eps, y16, y_f32, mean, rstd); break;
    case 256: ln_fwd_kernel<2><<<blocks, 256, 0, s>>>(x, gain, bias, rows, eps, y16, y_f32, mean, rstd); break;
    case 512: ln_fwd_kernel<4><<<blocks, 256, 0, s>>>(x, gain, bias, rows, eps, y16, y_f32, mean, rstd); break;
    case 1024: ln_fwd_kernel<8><<<blocks, 256, 0, s>>>(x, gain, bias, rows, eps, y16, y_f32, mean, rstd); break;
    case 2048: ln_fwd_kernel<16><<<blocks, 256, 0, s>>>(x, gain, bias, rows, eps, y16, y_f32, mean, rstd); break;
    default: return set_error(P2R_EINVAL, "layernorm: d_model must be one of 128/256/512/1024/2048");
  }
  P2R_CHECK_LAUNCH("layernorm fwd");
  return P2R_OK;
}

// 16 rows per block (2 per warp): ~512 blocks at T = 8192 keeps every SM busy.
constexpr int kLnBwdRows = 16;

// partial_ws: >= ceil(rows / rows_per_block) * 2 * d floats
extern "C" size_t p2r_layernorm_bwd_workspace(int rows, int d) {
  const int rpb = kLnBwdRows;
  return static_cast<size_t>((rows + rpb - 1) / rpb) * 2 * d * sizeof(float);
}

extern "C" p2r_status p2r_layernorm_bwd(const float* dy, const float* x, const float* mean,
                                        const float* rstd, const float* gain, const float* resid,
                                        int rows, int d, float* dx, void* dx_bf16, float* ggain,
                                        float* gbias, float* partial_ws, void* stream) {
  if (rows <= 0) return P2R_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int rpb = kLnBwdRows;
  const int blocks = (rows + rpb - 1) / rpb;
  auto* d16 = static_cast<__nv_bfloat16*>(dx_bf16);
  switch (d) {
    case 128: ln_bwd_kernel<1><<<blocks, 256, 0, s>>>(dy, x, mean, rstd, gain, resid, rows, rpb, dx, d16, partial_ws); break;
    case 256: ln_bwd_kernel<2><<<blocks, 256, 0, s>>>(dy, x, mean, rstd, gain, resid, rows, rpb, dx, d16, partial_ws); break;
    case 512: ln_bwd_kernel<4><<<blocks, 256, 0, s>>>(dy, x, mean, rstd, gain, resid, rows, rpb, dx, d16, partial_ws); break;
    case 1024: ln_bwd_kernel<8><<<blocks, 256, 0, s>>>(dy, x, mean, rstd, gain, resid, rows, rpb, dx, d16, partial_ws); break;
    case 2048: ln_bwd_kernel<16><<<blocks, 256, 0, s>>>(dy, x, mean, rstd, gain, resid, rows, rpb, dx, d16, partial_ws); break;
    default: return set_error(P2R_EINVAL, "layernorm: d_model must be one of 128/256/512/1024/2048");
  }
  P2R_CHECK_LAUNCH("layernorm bwd");
  if (ggain || gbias) {
    ln_param_grad_reduce<<<(2 * d + 31) / 32, 256, 0, s>>>(partial_ws, blocks, d, ggain, gbias);
    P2R_CHECK_LAUNCH("layernorm param grad");
  }
  return P2R_OK;
}

extern "C" p2r_status p2r_embed_fwd(const int* ids, const float* tok, const float* pos, int T,
                                    int S, int d, float* x, void* stream) {
  if (T <= 0) return P2R_OK;
  if (d % 4) return set_error(P2R_EINVAL, "embedding: d_model must be a multiple of 4");
  embed_fwd_kernel<<<T, 128, 0, static_cast<cudaStream_t>(stream)>>>(ids, tok, pos, T, S, d, x);
  P2R_CHECK_LAUNCH("embed fwd");
  return P2R_OK;
}

namespace {
int key_bits(int V) {
  int b = 1;
  while ((1LL << b) < V) ++b;
  return b;
}
size_t align256(size_t x) { return (x + 255) & ~static_cast<size_t>(255); }
size_t cub_sort_bytes(int T, int V) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const int*>(nullptr), static_cast<int*>(nullptr),
                                  static_cast<const int*>(nullptr), static_cast<int*>(nullptr), T, 0, key_bits(V));
  return bytes;
}
}  // namespace

extern "C" size_t p2r_embed_bwd_workspace(int T, int V) {
  if (T <= 0 || V <= 0) return 0;
  return align256(cub_sort_bytes(T, V)) + 3 * align256(static_cast<size_t>(T) * sizeof(int)) +
         2 * align256(static_cast<size_t>(V) * sizeof(int));
}

extern "C" p2r_status p2r_embed_bwd(const int* ids, const float* dx, int B, int S, int d, int V,
                                    float* dtok, float* dpos, void* ws, size_t ws_bytes, void* stream) {
  const int T = B * S;
  if (T <= 0) return P2R_OK;
  if (d % 4) return set_error(P2R_EINVAL, "embedding: d_model must be a multiple of 4");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtok) {
    if (ws == nullptr || ws_bytes < p2r_embed_bwd_workspace(T, V))
      return set_error(P2R_EINVAL, "embed bwd: workspace too small (see p2r_embed_bwd_workspace)");
    char* w = static_cast<char*>(ws);
    size_t tmp_bytes = cub_sort_bytes(T, V);
    void* tmp = w;
    w += align256(tmp_bytes);
    int* keys = reinterpret_cast<int*>(w);
    w += align256(static_cast<size_t>(T) * sizeof(int));
    int* pos_in = reinterpret_cast<int*>(w);
    w += align256(static_cast<size_t>(T) * sizeof(int));
    int* order = reinterpret_cast<int*>(w);
    w += align256(static_cast<size_t>(T) * sizeof(int));
    int* start = reinterpret_cast<int*>(w);
    w += align256(static_cast<size_t>(V) * sizeof(int));
    int* end = reinterpret_cast<int*>(w);
    iota_kernel<<<(T + 255) / 256, 256, 0, s>>>(pos_in, T);
    P2R_CHECK_LAUNCH("embed bwd iota");
    cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, ids, keys, pos_in, order, T, 0, key_bits(V), s);
    if (e != cudaSuccess) return set_cuda_error(e, "embed bwd sort");
    count_launch();
    e = cudaMemsetAsync(start, 0, 2 * align256(static_cast<size_t>(V) * sizeof(int)), s);
    if (e != cudaSuccess) return set_cuda_error(e, "embed bwd memset");
    run_bounds_kernel<<<(T + 255) / 256, 256, 0, s>>>(keys, T, start, end);
    P2R_CHECK_LAUNCH("embed bwd bounds");
    dim3 grid(V, (d / 4 + 127) / 128);
    embed_tok_bwd_kernel<<<grid, 128, 0, s>>>(order, start, end, dx, d, dtok);
    P2R_CHECK_LAUNCH("embed tok bwd");
  }
  if (dpos) {
    embed_pos_bwd_kernel<<<S, 256, 0, s>>>(dx, B, S, d, dpos);
    P2R_CHECK_LAUNCH("embed pos bwd");
  }
  return P2R_OK;
}

extern "C" size_t p2r_cross_entropy_workspace(int rows) {
  return static_cast<size_t>((rows + 7) / 8) * sizeof(double);
}

extern "C" p2r_status p2r_cross_entropy(const float* logits, int rows, int V, int ld,
                                        const int* targets, const uint8_t* mask, double denom,
                                        float loss_grad, void* dlogits_bf16, int ldg, float* loss,
                                        double* loss_sum, double* partial_ws, void* stream) {
  if (denom <= 0.0) return set_error(P2R_EINVAL, "softmax_cross_entropy: denominator must be > 0");
  if (rows <= 0) return P2R_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int blocks = (rows + 7) / 8;
  const float scale = loss_grad / static_cast<float>(denom);
  ce_kernel<<<blocks, 256, 0, s>>>(logits, rows, V, ld, targets, mask, scale,
                                   static_cast<__nv_bfloat16*>(dlogits_bf16), ldg, partial_ws);
  P2R_CHECK_LAUNCH("cross entropy");
  ce_finalize<<<1, 32, 0, s>>>(partial_ws, blocks, denom, loss, loss_sum);
  P2R_CHECK_LAUNCH("cross entropy finalize");
  return P2R_OK;
}
