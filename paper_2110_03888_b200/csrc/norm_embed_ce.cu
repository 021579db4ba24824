// LayerNorm fwd/bwd, token+position embedding fwd/bwd, fused softmax-CE fwd/bwd.
//
//   layernorm            tensor.cpp:265-336 (two-pass mean / biased var, eps 1e-5)
//   embedding_lookup+add tensor.cpp:338-368, model.cpp:229-241
//   softmax_cross_entropy tensor.cpp:670-723 (fp64 loss sum, / denom, masked rows)
// All reductions are deterministic (fixed-order trees, no float atomics).
#include <cstdlib>

#include <cub/device/device_radix_sort.cuh>

#include "../../include/p2r_cuda.h"
#include "common.cuh"
#include "p2r_internal.h"

namespace p2r {

// ------------------------------- LayerNorm -----------------------------------
// Warp-per-row with warp-private bulk-copy pipelines: each warp owns rows
// gw, gw + W, ... (W = warps in the grid) and a ring of `nst` shared-memory row
// slots filled by 1-D cp.async.bulk copies that its lane 0 issues `nst` rows
// ahead (completion on the warp's own mbarriers). Row statistics are warp
// shuffles, so no block-level barrier sits on the per-row path; lane l owns the
// float4 columns l, l+32, ... (NV = d/128 of them). gain/bias live in shared
// memory. All reductions have a fixed order (deterministic).
constexpr int kLnMaxStages = 3;

P2R_DEVICE float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }

P2R_DEVICE void ln_row_issue(uint64_t* bar, uint32_t dst, const float* const* src, int ntens, int row, int D) {
  const uint32_t bytes = static_cast<uint32_t>(D) * 4;
  mbar_arrive_expect_tx(bar, bytes * ntens);
  for (int t = 0; t < ntens; ++t) bulk_load(dst + t * bytes, src[t] + static_cast<long long>(row) * D, bytes, bar);
}

// One row of each of ntens tensors into a ring slot; tensor 0 has b0 bytes per
// row (bf16 or fp32 dy), the others are fp32 rows of D floats packed behind it.
P2R_DEVICE void ln_row_issue_b(uint64_t* bar, uint32_t dst, const void* const* src, int ntens, int row, int D,
                               uint32_t b0) {
  const uint32_t bytes = static_cast<uint32_t>(D) * 4;
  mbar_arrive_expect_tx(bar, b0 + bytes * (ntens - 1));
  bulk_load(dst, static_cast<const uint8_t*>(src[0]) + static_cast<long long>(row) * b0, b0, bar);
  for (int t = 1; t < ntens; ++t)
    bulk_load(dst + b0 + (t - 1) * bytes, static_cast<const float*>(src[t]) + static_cast<long long>(row) * D, bytes,
              bar);
}

// four consecutive dy values of a ring row, fp32 or bf16 (8-byte shared load)
template <bool DY16>
P2R_DEVICE float4 ln_lds_dy(uint32_t row, int c4) {
  if constexpr (DY16) {
    uint32_t lo, hi;
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(row + c4 * 8));
    const float2 a = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&lo));
    const float2 b = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&hi));
    return make_float4(a.x, a.y, b.x, b.y);
  } else {
    return lds128f(row + c4 * 16);
  }
}

P2R_DEVICE void st_bf16x4(__nv_bfloat16* p, float4 o) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
  uint2 w;
  w.x = *reinterpret_cast<uint32_t*>(&lo);
  w.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(p) = w;
}

template <int NV>
__global__ void __launch_bounds__(256) ln_fwd_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                                                    const float* __restrict__ bias, int rows, float eps,
                                                    __nv_bfloat16* __restrict__ y16, float* __restrict__ y32,
                                                    float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                    int nst) {
  pdl_trigger();
  pdl_wait();
  constexpr int D = 128 * NV;
  extern __shared__ __align__(128) uint8_t ln_smem[];
  __shared__ uint64_t bars[8][kLnMaxStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  float* sg = reinterpret_cast<float*>(ln_smem);  // gain | bias
  for (int i = threadIdx.x; i < 2 * D; i += blockDim.x) sg[i] = i < D ? gain[i] : bias[i - D];
  const uint32_t ring = smem_u32(ln_smem) + 2 * D * 4 + warp * nst * D * 4;
  uint64_t* bar = bars[warp];
  const int W = gridDim.x * nw, gw = blockIdx.x * nw + warp;
  const int nrows = gw < rows ? (rows - gw + W - 1) / W : 0;
  const float* src[1] = {x};
  if (lane == 0) {
    for (int i = 0; i < nst; ++i) mbar_init(bar + i, 1);
    fence_barrier_init();
    for (int k = 0; k < nst && k < nrows; ++k) ln_row_issue(bar + k, ring + k * D * 4, src, 1, gw + k * W, D);
  }
  __syncthreads();  // gain/bias staged, barriers initialised
  const float inv_d = 1.0f / static_cast<float>(D);
  for (int k = 0; k < nrows; ++k) {
    const int st = k % nst, r = gw + k * W;
    mbar_wait(bar + st, (k / nst) & 1);
    float4 v[NV];
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      v[i] = lds128f(ring + st * D * 4 + (lane + 32 * i) * 16);
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
    s = warp_sum(s);  // consumes every lane's smem reads
    if (lane == 0 && k + nst < nrows) ln_row_issue(bar + st, ring + st * D * 4, src, 1, r + nst * W, D);
    const float mu = s * inv_d;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const float a = v[i].x - mu, b = v[i].y - mu, c = v[i].z - mu, d = v[i].w - mu;
      q += (a * a + b * b) + (c * c + d * d);
    }
    q = warp_sum(q);  // two-pass (biased) variance, tensor.cpp:265-336
    const float inv = 1.0f / sqrtf(q * inv_d + eps);
    if (lane == 0) {
      mean_out[r] = mu;
      rstd_out[r] = inv;
    }
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c4 = lane + 32 * i;
      const float4 g = reinterpret_cast<const float4*>(sg)[c4], bb = reinterpret_cast<const float4*>(sg + D)[c4];
      float4 o;
      o.x = (v[i].x - mu) * inv * g.x + bb.x;
      o.y = (v[i].y - mu) * inv * g.y + bb.y;
      o.z = (v[i].z - mu) * inv * g.z + bb.z;
      o.w = (v[i].w - mu) * inv * g.w + bb.w;
      const long long off = static_cast<long long>(r) * D + 4LL * c4;
      if (y16) st_bf16x4(y16 + off, o);
      if (y32) *reinterpret_cast<float4*>(y32 + off) = o;
    }
  }
}

// Register variant: one warp per row, the row held in registers (NV float4 per
// lane, 16-byte loads), no shared memory. A small register footprint gives 40+
// resident warps per SM whose loads are all in flight at once -- the memory
// system, not a per-warp pipeline, hides the latency (the bulk-ring kernel
// above keeps 16 warps per SM and spends its time in per-row latency).
template <int NV>
__global__ void __launch_bounds__(256) ln_fwd_reg_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                                                        const float* __restrict__ bias, int rows, float eps,
                                                        __nv_bfloat16* __restrict__ y16, float* __restrict__ y32,
                                                        float* __restrict__ mean_out, float* __restrict__ rstd_out) {
  pdl_trigger();
  pdl_wait();
  constexpr int D = 128 * NV;
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float* xr = x + static_cast<long long>(r) * D;
  float4 v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = ld4(xr + 4 * (lane + 32 * i));
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  s = warp_sum(s);
  const float inv_d = 1.0f / static_cast<float>(D);
  const float mu = s * inv_d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const float a = v[i].x - mu, b = v[i].y - mu, c = v[i].z - mu, d = v[i].w - mu;
    q += (a * a + b * b) + (c * c + d * d);
  }
  q = warp_sum(q);  // two-pass (biased) variance, tensor.cpp:265-336
  const float inv = 1.0f / sqrtf(q * inv_d + eps);
  if (lane == 0) {
    mean_out[r] = mu;
    rstd_out[r] = inv;
  }
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    const float4 g = __ldg(reinterpret_cast<const float4*>(gain) + c4), bb = __ldg(reinterpret_cast<const float4*>(bias) + c4);
    float4 o;
    o.x = (v[i].x - mu) * inv * g.x + bb.x;
    o.y = (v[i].y - mu) * inv * g.y + bb.y;
    o.z = (v[i].z - mu) * inv * g.z + bb.z;
    o.w = (v[i].w - mu) * inv * g.w + bb.w;
    const long long off = static_cast<long long>(r) * D + 4LL * c4;
    if (y16) st_bf16x4(y16 + off, o);
    if (y32) *reinterpret_cast<float4*>(y32 + off) = o;
  }
}

// dx = resid + inv * (gy - mean(gy) - xhat * mean(gy * xhat)), gy = dy * gain.
// dgain/dbias: per-lane column accumulators over the warp's rows, combined per
// block (warp order) into partial[blockIdx.x][2][D]; ln_param_grad_reduce adds
// the block partials into the grads in block order. COLSUM: the column sums of
// dx itself are accumulated the same way into cpartial[blockIdx.x][D] (the dense
// block backward takes the FFN2 bias gradient of the layer below from them,
// add_bias backward tensor.cpp:227-231, instead of re-reading dx).
template <int NV, bool COLSUM, bool DY16>
__global__ void __launch_bounds__(128) ln_bwd_kernel(
    const void* __restrict__ dy, const float* __restrict__ x, const float* __restrict__ mean_in,
    const float* __restrict__ rstd_in, const float* __restrict__ gain, const float* __restrict__ resid, int rows,
    float* __restrict__ dx32, __nv_bfloat16* __restrict__ dx16, float* __restrict__ partial, int nst,
    float* __restrict__ cpartial) {
  pdl_trigger();
  pdl_wait();
  constexpr int D = 128 * NV;
  extern __shared__ __align__(128) uint8_t ln_smem[];
  __shared__ uint64_t bars[4][kLnMaxStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int ntens = resid ? 3 : 2;
  float* sg = reinterpret_cast<float*>(ln_smem);
  for (int i = threadIdx.x; i < D; i += blockDim.x) sg[i] = gain[i];
  constexpr uint32_t kDyBytes = D * (DY16 ? 2 : 4);
  const uint32_t slot = kDyBytes + (ntens - 1) * D * 4;  // one row of each tensor
  const uint32_t ring = smem_u32(ln_smem) + D * 4 + warp * nst * slot;
  uint64_t* bar = bars[warp];
  const int W = gridDim.x * nw, gw = blockIdx.x * nw + warp;
  const int nrows = gw < rows ? (rows - gw + W - 1) / W : 0;
  const void* src[3] = {dy, x, resid};
  if (lane == 0) {
    for (int i = 0; i < nst; ++i) mbar_init(bar + i, 1);
    fence_barrier_init();
    for (int k = 0; k < nst && k < nrows; ++k)
      ln_row_issue_b(bar + k, ring + k * slot, src, ntens, gw + k * W, D, kDyBytes);
  }
  __syncthreads();
  const float inv_d = 1.0f / static_cast<float>(D);
  float4 pg[NV], pb[NV], pc[COLSUM ? NV : 1];
#pragma unroll
  for (int i = 0; i < NV; ++i) pg[i] = pb[i] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int i = 0; i < (COLSUM ? NV : 1); ++i) pc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  float mu_n = 0.f, inv_n = 0.f;
  if (nrows > 0) {
    mu_n = mean_in[gw];
    inv_n = rstd_in[gw];
  }
  for (int k = 0; k < nrows; ++k) {
    const int st = k % nst, r = gw + k * W;
    const float mu = mu_n, inv = inv_n;
    if (k + 1 < nrows) {  // next row's statistics, off the critical path
      mu_n = mean_in[r + W];
      inv_n = rstd_in[r + W];
    }
    mbar_wait(bar + st, (k / nst) & 1);
    const uint32_t sd = ring + st * slot, sx = sd + kDyBytes, sr = sx + D * 4;
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const uint32_t o = (lane + 32 * i) * 16;
      const float4 d = ln_lds_dy<DY16>(sd, lane + 32 * i), xv = lds128f(sx + o),
                   g = reinterpret_cast<const float4*>(sg)[lane + 32 * i];
      const float4 h = make_float4((xv.x - mu) * inv, (xv.y - mu) * inv, (xv.z - mu) * inv, (xv.w - mu) * inv);
      const float4 gy = make_float4(d.x * g.x, d.y * g.y, d.z * g.z, d.w * g.w);
      s1 += (gy.x + gy.y) + (gy.z + gy.w);
      s2 += (gy.x * h.x + gy.y * h.y) + (gy.z * h.z + gy.w * h.w);
      pg[i].x += d.x * h.x;
      pg[i].y += d.y * h.y;
      pg[i].z += d.z * h.z;
      pg[i].w += d.w * h.w;
      pb[i].x += d.x;
      pb[i].y += d.y;
      pb[i].z += d.z;
      pb[i].w += d.w;
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    const float a1 = inv_d * s1, a2 = inv_d * s2;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c4 = lane + 32 * i;
      const uint32_t o = c4 * 16;
      const float4 d = ln_lds_dy<DY16>(sd, c4), xv = lds128f(sx + o), g = reinterpret_cast<const float4*>(sg)[c4];
      const float4 rr = resid ? lds128f(sr + o) : make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 h = make_float4((xv.x - mu) * inv, (xv.y - mu) * inv, (xv.z - mu) * inv, (xv.w - mu) * inv);
      float4 out;
      out.x = inv * (d.x * g.x - a1 - h.x * a2) + rr.x;
      out.y = inv * (d.y * g.y - a1 - h.y * a2) + rr.y;
      out.z = inv * (d.z * g.z - a1 - h.z * a2) + rr.z;
      out.w = inv * (d.w * g.w - a1 - h.w * a2) + rr.w;
      const long long off = static_cast<long long>(r) * D + 4LL * c4;
      *reinterpret_cast<float4*>(dx32 + off) = out;
      if (dx16) st_bf16x4(dx16 + off, out);
      if constexpr (COLSUM) {
        pc[i].x += out.x;
        pc[i].y += out.y;
        pc[i].z += out.z;
        pc[i].w += out.w;
      }
    }
    __syncwarp();  // every lane's reads of this slot are done before it is refilled
    if (lane == 0 && k + nst < nrows) ln_row_issue_b(bar + st, ring + st * slot, src, ntens, r + nst * W, D, kDyBytes);
  }
  // combine the warps' column partials in warp order (the ring is drained)
  __syncthreads();
  constexpr int NACC = COLSUM ? 3 : 2;
  float* red = reinterpret_cast<float*>(ln_smem + D * 4);  // [nw][NACC][D]
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c4 = lane + 32 * i;
    reinterpret_cast<float4*>(red + (warp * NACC) * D)[c4] = pg[i];
    reinterpret_cast<float4*>(red + (warp * NACC + 1) * D)[c4] = pb[i];
    if constexpr (COLSUM) reinterpret_cast<float4*>(red + (warp * NACC + 2) * D)[c4] = pc[i];
  }
  __syncthreads();
  float* out = partial + static_cast<long long>(blockIdx.x) * 2 * D;
  for (int c = threadIdx.x; c < NACC * D; c += blockDim.x) {
    float t = 0.f;
    for (int w = 0; w < nw; ++w) t += red[w * NACC * D + c];
    if (c < 2 * D) {
      out[c] = t;
    } else if constexpr (COLSUM) {
      cpartial[static_cast<long long>(blockIdx.x) * D + (c - 2 * D)] = t;
    }
  }
}

// grad_gain[c] += sum_b partial[b][0][c]; grad_bias[c] += sum_b partial[b][1][c];
// and, when cin != NULL, cdst[c] += sum_b cin[b][c] (a previous backward's dx
// column partials, see ln_bwd_kernel COLSUM). 1024 threads per 32 flattened
// columns: warp w sums partial rows w, w+32, ... (coalesced 128-byte rows, all
// loads of a warp in flight together), then the 32 warp sums are added in warp order.
__global__ void __launch_bounds__(1024) ln_param_grad_reduce(const float* __restrict__ partial, int nblk, int D,
                                                             float* __restrict__ ggain, float* __restrict__ gbias,
                                                             const float* __restrict__ cin, int cblk,
                                                             float* __restrict__ cdst) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[32][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 32 + lane;  // flattened [2][D] (+ [D]) column
  const int ncol = cin ? 3 * D : 2 * D;
  float s = 0.f;
  if (c < 2 * D) {
#pragma unroll 8
    for (int b = warp; b < nblk; b += 32) s += partial[static_cast<long long>(b) * 2 * D + c];
  } else if (c < ncol) {
#pragma unroll 8
    for (int b = warp; b < cblk; b += 32) s += cin[static_cast<long long>(b) * D + (c - 2 * D)];
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && c < ncol) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 32; ++w) t += red[w][lane];
    const int which = c / D, col = c % D;
    float* dst = which == 0 ? ggain : (which == 1 ? gbias : cdst);
    if (dst) dst[col] += t;
  }
}

// ------------------------------- embeddings ----------------------------------
__global__ void embed_fwd_kernel(const int* __restrict__ ids, const float* __restrict__ tok,
                                 const float* __restrict__ pos, int T, int S, int d,
                                 float* __restrict__ x) {
  pdl_trigger();
  pdl_wait();
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
  pdl_trigger();
  pdl_wait();
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
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += partial[i];
    if (loss_sum) *loss_sum = s;
    *loss = static_cast<float>(s / denom);
  }
}

}  // namespace p2r

using namespace p2r;

namespace {
bool ln_dim_ok(int d) { return d >= 128 && d <= 2048 && d % 128 == 0; }

constexpr int kLnFwdWarps = 8, kLnBwdWarps = 4;
constexpr int kSmemPerSM = 227 * 1024;
constexpr int kLnSmemAttr = 200 * 1024;  // opt-in dynamic limit (leaves room for static smem)

// stages per warp ring (<= 3) and blocks: as many resident blocks as the
// staging allows, at most 4 per SM (fwd) / 2 per SM (bwd).
struct LnLaunch {
  int nst, smem, blocks, warps;
};
[[maybe_unused]] LnLaunch ln_fwd_launch(int rows, int d) {  // (the bulk-ring forward: diagnostic build)
  LnLaunch l{};
  l.nst = kLnMaxStages;
  while (l.nst > 1 && 2 * d * 4 + kLnFwdWarps * l.nst * d * 4 > 110 * 1024) --l.nst;
  l.smem = 2 * d * 4 + kLnFwdWarps * l.nst * d * 4;
  int per_sm = kSmemPerSM / (l.smem + 1024);
  per_sm = per_sm < 1 ? 1 : (per_sm > 4 ? 4 : per_sm);
  const int need = (rows + kLnFwdWarps - 1) / kLnFwdWarps;
  l.blocks = need < per_sm * kNumSMs ? need : per_sm * kNumSMs;
  return l;
}
int ln_env(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e != nullptr && e[0] != 0 ? std::atoi(e) : dflt;
}
// row_floats: ring bytes per row / 4 (dy + x [+ resid]; a bf16 dy counts d/2)
LnLaunch ln_bwd_launch(int rows, int d, int row_floats) {
  // tuning knobs (measurement only): rows in flight per warp, warps per block, smem cap, blocks per SM
  static const int k_nst = ln_env("P2R_LN_BWD_NST", 2), k_warps = ln_env("P2R_LN_BWD_WARPS", kLnBwdWarps),
                   k_cap = ln_env("P2R_LN_BWD_SMEM_KB", 110), k_persm = ln_env("P2R_LN_BWD_PERSM", 2);
  LnLaunch l{};
  l.warps = k_warps < 1 ? 1 : (k_warps > 4 ? 4 : k_warps);
  l.nst = k_nst < 1 ? 1 : (k_nst > kLnMaxStages ? kLnMaxStages : k_nst);
  while (l.nst > 1 && d * 4 + l.warps * l.nst * row_floats * 4 > k_cap * 1024) --l.nst;
  const int ring = l.warps * l.nst * row_floats * 4, red = l.warps * 3 * d * 4;
  l.smem = d * 4 + (ring > red ? ring : red);
  int per_sm = kSmemPerSM / (l.smem + 1024);
  per_sm = per_sm < 1 ? 1 : (per_sm > k_persm ? k_persm : per_sm);
  const int need = (rows + l.warps - 1) / l.warps;
  l.blocks = need < per_sm * kNumSMs ? need : per_sm * kNumSMs;
  return l;
}

#define P2R_LN_NV_CASES(X) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(16)
}  // namespace

extern "C" p2r_status p2r_layernorm_fwd(const float* x, const float* gain, const float* bias,
                                        int rows, int d, float eps, void* y_bf16, float* y_f32,
                                        float* mean, float* rstd, void* stream) {
  if (rows <= 0) return P2R_OK;
  if (!ln_dim_ok(d)) return set_error(P2R_EINVAL, "layernorm: d_model must be a multiple of 128 in [128, 2048]");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* y16 = static_cast<__nv_bfloat16*>(y_bf16);
#ifdef P2R_DIAG  // diagnostic build: P2R_LN_FWD_RING=1 selects the bulk-ring forward
  static const bool ring = [] {
    const char* e = std::getenv("P2R_LN_FWD_RING");
    return e != nullptr && e[0] == '1';
  }();
#else
  constexpr bool ring = false;
#endif
  if (!ring) {
    switch (d / 128) {
#define P2R_LN_FWD_REG(NV)                                                                                  \
  case NV: {                                                                                               \
    const cudaError_t le = launch_k(ln_fwd_reg_kernel<NV>, dim3((rows + 7) / 8), dim3(256), 0, s, 1, x, gain, bias, \
                                    rows, eps, y16, y_f32, mean, rstd);                                   \
    if (le != cudaSuccess) return set_cuda_error(le, "layernorm fwd");                                     \
    break;                                                                                                 \
  }
      P2R_LN_NV_CASES(P2R_LN_FWD_REG)
#undef P2R_LN_FWD_REG
      default: break;
    }
    P2R_CHECK_LAUNCH("layernorm fwd");
    return P2R_OK;
  }
#ifdef P2R_DIAG
  const LnLaunch l = ln_fwd_launch(rows, d);
  switch (d / 128) {
#define P2R_LN_FWD(NV)                                                                                     \
  case NV: {                                                                                               \
    static cudaError_t a = cudaFuncSetAttribute(ln_fwd_kernel<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                                kLnSmemAttr);                                                \
    if (a != cudaSuccess) return set_cuda_error(a, "layernorm fwd attr");                                  \
    const cudaError_t le = launch_k(ln_fwd_kernel<NV>, dim3(l.blocks), dim3(32 * kLnFwdWarps), l.smem, s, 1, x, gain, bias, rows, eps, \
                 y16, y_f32, mean, rstd, l.nst);                                                            \
    if (le != cudaSuccess) return set_cuda_error(le, "layernorm fwd");                                       \
    break;                                                                                                 \
  }
    P2R_LN_NV_CASES(P2R_LN_FWD)
#undef P2R_LN_FWD
    default: break;
  }
  P2R_CHECK_LAUNCH("layernorm fwd");
#endif
  return P2R_OK;
}

namespace {
// ring floats per row for a launch: dy (fp32, or bf16 = half) + x (+ resid)
int ln_bwd_row_floats(int d, bool resid, bool dy16) { return (dy16 ? d / 2 : d) + d + (resid ? d : 0); }

p2r_status ln_bwd_fused(const void* dy, bool dy16, const float* x, const float* mean, const float* rstd,
                        const float* gain, const float* resid, int rows, int d, float* dx, void* dx_bf16,
                        float* ggain, float* gbias, float* partial_ws, float* dx_colsum_ws, const float* colsum_in,
                        int colsum_blocks, float* colsum_dst, void* stream) {
  if (rows <= 0) return P2R_OK;
  if (!ln_dim_ok(d)) return set_error(P2R_EINVAL, "layernorm: d_model must be a multiple of 128 in [128, 2048]");
  if ((colsum_in == nullptr) != (colsum_dst == nullptr) || (colsum_in && colsum_blocks <= 0))
    return set_error(P2R_EINVAL, "layernorm bwd: colsum_in, colsum_blocks and colsum_dst go together");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const LnLaunch l = ln_bwd_launch(rows, d, ln_bwd_row_floats(d, resid != nullptr, dy16));
  auto* d16 = static_cast<__nv_bfloat16*>(dx_bf16);
  switch (d / 128) {
#define P2R_LN_BWD_ONE(NV, CS, DY)                                                                            \
  {                                                                                                        \
    static cudaError_t a = cudaFuncSetAttribute(ln_bwd_kernel<NV, CS, DY>,                                  \
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, kLnSmemAttr);  \
    if (a != cudaSuccess) return set_cuda_error(a, "layernorm bwd attr");                                  \
    const cudaError_t le = launch_k(ln_bwd_kernel<NV, CS, DY>, dim3(l.blocks), dim3(32 * l.warps), l.smem, s, 1, dy, \
                                    x, mean, rstd, gain, resid, rows, dx, d16, partial_ws, l.nst, dx_colsum_ws); \
    if (le != cudaSuccess) return set_cuda_error(le, "layernorm bwd");                                       \
  }
#define P2R_LN_BWD(NV)                                  \
  case NV:                                              \
    if (dy16) {                                         \
      if (dx_colsum_ws) P2R_LN_BWD_ONE(NV, true, true)  \
      else P2R_LN_BWD_ONE(NV, false, true)              \
    } else {                                            \
      if (dx_colsum_ws) P2R_LN_BWD_ONE(NV, true, false) \
      else P2R_LN_BWD_ONE(NV, false, false)             \
    }                                                   \
    break;
    P2R_LN_NV_CASES(P2R_LN_BWD)
#undef P2R_LN_BWD
#undef P2R_LN_BWD_ONE
    default: break;
  }
  P2R_CHECK_LAUNCH("layernorm bwd");
  if (ggain || gbias || colsum_dst) {
    const int ncol = colsum_in ? 3 * d : 2 * d;
    P2R_LAUNCH_K("layernorm param grad", ln_param_grad_reduce, dim3((ncol + 31) / 32), dim3(1024), 0, s, 1,
                 static_cast<const float*>(partial_ws), l.blocks, d, ggain, gbias, colsum_in, colsum_blocks,
                 colsum_dst);
  }
  return P2R_OK;
}
}  // namespace

// partial_ws: >= blocks * 2 * d floats for every launch variant (residual or not, fp32 or bf16 dy)
extern "C" size_t p2r_layernorm_bwd_workspace(int rows, int d) {
  if (rows <= 0 || !ln_dim_ok(d)) return 0;
  int b = 0;
  for (int v = 0; v < 4; ++v) {
    const int bv = ln_bwd_launch(rows, d, ln_bwd_row_floats(d, v & 1, v & 2)).blocks;
    b = bv > b ? bv : b;
  }
  return static_cast<size_t>(b) * 2 * d * sizeof(float);
}

extern "C" int p2r_layernorm_bwd_blocks(int rows, int d, int flags) {
  if (rows <= 0 || !ln_dim_ok(d)) return 0;
  return ln_bwd_launch(rows, d, ln_bwd_row_floats(d, flags & P2R_LN_RESID, flags & P2R_LN_DY_BF16)).blocks;
}

extern "C" p2r_status p2r_layernorm_bwd_fused(const float* dy, const float* x, const float* mean,
                                              const float* rstd, const float* gain, const float* resid,
                                              int rows, int d, float* dx, void* dx_bf16, float* ggain,
                                              float* gbias, float* partial_ws, float* dx_colsum_ws,
                                              const float* colsum_in, int colsum_blocks, float* colsum_dst,
                                              void* stream) {
  return ln_bwd_fused(dy, false, x, mean, rstd, gain, resid, rows, d, dx, dx_bf16, ggain, gbias, partial_ws,
                      dx_colsum_ws, colsum_in, colsum_blocks, colsum_dst, stream);
}

extern "C" p2r_status p2r_layernorm_bwd_fused_bf16(const void* dy_bf16, const float* x, const float* mean,
                                                   const float* rstd, const float* gain, const float* resid,
                                                   int rows, int d, float* dx, void* dx_bf16, float* ggain,
                                                   float* gbias, float* partial_ws, float* dx_colsum_ws,
                                                   const float* colsum_in, int colsum_blocks, float* colsum_dst,
                                                   void* stream) {
  return ln_bwd_fused(dy_bf16, true, x, mean, rstd, gain, resid, rows, d, dx, dx_bf16, ggain, gbias, partial_ws,
                      dx_colsum_ws, colsum_in, colsum_blocks, colsum_dst, stream);
}

extern "C" p2r_status p2r_layernorm_bwd(const float* dy, const float* x, const float* mean,
                                        const float* rstd, const float* gain, const float* resid,
                                        int rows, int d, float* dx, void* dx_bf16, float* ggain,
                                        float* gbias, float* partial_ws, void* stream) {
  return p2r_layernorm_bwd_fused(dy, x, mean, rstd, gain, resid, rows, d, dx, dx_bf16, ggain, gbias, partial_ws,
                                 nullptr, nullptr, 0, nullptr, stream);
}

extern "C" p2r_status p2r_embed_fwd(const int* ids, const float* tok, const float* pos, int T,
                                    int S, int d, float* x, void* stream) {
  if (T <= 0) return P2R_OK;
  if (d % 4) return set_error(P2R_EINVAL, "embedding: d_model must be a multiple of 4");
  P2R_LAUNCH_K("embed fwd", embed_fwd_kernel, dim3(T), dim3(128), 0, static_cast<cudaStream_t>(stream), 1, ids, tok,
               pos, T, S, d, x);
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
  P2R_LAUNCH_K("cross entropy", ce_kernel, dim3(blocks), dim3(256), 0, s, 1, logits, rows, V, ld, targets, mask, scale,
               static_cast<__nv_bfloat16*>(dlogits_bf16), ldg, partial_ws);
  P2R_LAUNCH_K("cross entropy finalize", ce_finalize, dim3(1), dim3(32), 0, s, 1,
               static_cast<const double*>(partial_ws), blocks, denom, loss, loss_sum);
  return P2R_OK;
}
