// AdamW (bit-exact with optim.cpp:41-63 given equal grads), the Pseudo-to-Real
// delink broadcast (model.cpp:358-377 + moment copy SPEC.md:279,:312), bias
// gradient column sums (add_bias backward, tensor.cpp:227-231) and small
// utilities. All HBM-bound; float4-vectorised, grid-stride, deterministic.
#include "../../include/p2r_cuda.h"
#include "common.cuh"
#include "p2r_internal.h"

namespace p2r {

struct AdamSeg {
  long long off;  // element offset inside the granule
  long long len;
  int decay;      // weight decay on ndim >= 2 tensors only (optim.cpp:437)
};
struct AdamArgs {
  float* p;
  const float* g;
  float* m;
  float* v;
  __nv_bfloat16* p16;  // bf16 shadow used by the GEMMs (may be null)
  float b1, b2, omb1, omb2, bc1, bc2, eps, wd, lr;
  int nseg;
  AdamSeg seg[P2R_MAX_ADAM_SEGS];
};

// Exactly the reference operation order, every op individually rounded (no
// FMA contraction; the reference is compiled for baseline x86-64 = SSE).
P2R_DEVICE void adam_elem(float& p, float g, float& m, float& v, const AdamArgs& a, bool decay) {
  m = __fadd_rn(__fmul_rn(a.b1, m), __fmul_rn(a.omb1, g));
  v = __fadd_rn(__fmul_rn(a.b2, v), __fmul_rn(__fmul_rn(a.omb2, g), g));
  const float mhat = __fdiv_rn(m, a.bc1);
  const float vhat = __fdiv_rn(v, a.bc2);
  float upd = __fdiv_rn(mhat, __fadd_rn(__fsqrt_rn(vhat), a.eps));
  if (decay) upd = __fadd_rn(upd, __fmul_rn(a.wd, p));
  p = __fsub_rn(p, __fmul_rn(a.lr, upd));
}

__global__ void __launch_bounds__(256) adamw_kernel(const __grid_constant__ AdamArgs a) {
  pdl_trigger();
  pdl_wait();
  const AdamSeg sg = a.seg[blockIdx.y];
  const bool decay = sg.decay != 0;
  const long long n4 = sg.len / 4;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  float* P = a.p + sg.off;
  const float* G = a.g + sg.off;
  float* M = a.m + sg.off;
  float* V = a.v + sg.off;
  __nv_bfloat16* P16 = a.p16 ? a.p16 + sg.off : nullptr;
  const bool aligned = ((sg.off & 3) == 0);
  if (aligned) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
      float4 p = reinterpret_cast<float4*>(P)[i];
      const float4 g = reinterpret_cast<const float4*>(G)[i];
      float4 m = reinterpret_cast<float4*>(M)[i];
      float4 v = reinterpret_cast<float4*>(V)[i];
      adam_elem(p.x, g.x, m.x, v.x, a, decay);
      adam_elem(p.y, g.y, m.y, v.y, a, decay);
      adam_elem(p.z, g.z, m.z, v.z, a, decay);
      adam_elem(p.w, g.w, m.w, v.w, a, decay);
      reinterpret_cast<float4*>(P)[i] = p;
      reinterpret_cast<float4*>(M)[i] = m;
      reinterpret_cast<float4*>(V)[i] = v;
      if (P16) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(p.x, p.y), hi = __floats2bfloat162_rn(p.z, p.w);
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&lo);
        w.y = *reinterpret_cast<uint32_t*>(&hi);
        reinterpret_cast<uint2*>(P16)[i] = w;
      }
    }
  }
  const long long start = aligned ? n4 * 4 : 0;
  for (long long i = start + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < sg.len; i += stride) {
    float p = P[i], m = M[i], v = V[i];
    adam_elem(p, G[i], m, v, a, decay);
    P[i] = p;
    M[i] = m;
    V[i] = v;
    if (P16) P16[i] = __float2bfloat16_rn(p);
  }
}

// fp32 -> bf16 shadow copy
__global__ void cast_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, long long n) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride)
    dst[i] = __float2bfloat16_rn(src[i]);
}

// Delink broadcast: 1 read of the shared granule, L writes (dst_l = dst + l*dst_stride).
__global__ void __launch_bounds__(256) delink_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                     long long n16, long long dst_stride16, int L) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n16; i += stride) {
    const uint4 v = src[i];
    for (int l = 0; l < L; ++l) dst[l * dst_stride16 + i] = v;
  }
}

// Column sums for bias gradients. Stage 1: partial[chunk][col] over a row chunk
// (rows in ascending order per thread-row, then a fixed-order tree over the 8
// thread-rows). Grouped mode: group g covers rows [g*seg, g*seg+counts[g]) and
// writes group-separated partials.
template <typename T>
P2R_DEVICE float to_f(T v);
template <>
P2R_DEVICE float to_f<float>(float v) { return v; }
template <>
P2R_DEVICE float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

// 16-byte vectors: VEC = 4 fp32 or 8 bf16 columns per thread, so one warp reads
// a 512-byte (fp32) / 512-byte (bf16) row segment per load; 8 warps split the
// chunk's rows and the warp partials are added in warp order (deterministic).
template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  static constexpr int N = 4;
  P2R_DEVICE static void load(const float* p, float* o) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    o[0] = v.x, o[1] = v.y, o[2] = v.z, o[3] = v.w;
  }
};
template <>
struct Vec16<__nv_bfloat16> {
  static constexpr int N = 8;
  P2R_DEVICE static void load(const __nv_bfloat16* p, float* o) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[i]));
      o[2 * i] = f.x, o[2 * i + 1] = f.y;
    }
  }
};

template <typename T>
__global__ void __launch_bounds__(256) colsum_partial_kernel(const T* __restrict__ x, int ld, int rows, int n,
                                                             int chunk_rows, int seg_rows,
                                                             const int* __restrict__ counts,
                                                             float* __restrict__ partial) {
  pdl_trigger();
  pdl_wait();
  constexpr int V = Vec16<T>::N;
  __shared__ float red[8][32 * V];
  const int lane = threadIdx.x & 31;
  const int tr = threadIdx.x >> 5;  // 0..7
  const int col = (blockIdx.x * 32 + lane) * V;
  const int chunk = blockIdx.y;
  const int g = blockIdx.z;
  int r0, r1;
  if (counts) {
    r0 = g * seg_rows + chunk * chunk_rows;
    r1 = min(g * seg_rows + counts[g], r0 + chunk_rows);
  } else {
    r0 = chunk * chunk_rows;
    r1 = min(rows, r0 + chunk_rows);
  }
  float s[V];
#pragma unroll
  for (int i = 0; i < V; ++i) s[i] = 0.f;
  if (col < n) {
#pragma unroll 4
    for (int r = r0 + tr; r < r1; r += 8) {
      float v[V];
      Vec16<T>::load(x + static_cast<long long>(r) * ld + col, v);
#pragma unroll
      for (int i = 0; i < V; ++i) s[i] += v[i];
    }
  }
#pragma unroll
  for (int i = 0; i < V; ++i) red[tr][lane * V + i] = s[i];
  __syncthreads();
  for (int c = threadIdx.x; c < 32 * V; c += 256) {
    const int gc = blockIdx.x * 32 * V + c;
    if (gc >= n) continue;
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][c];
    partial[(static_cast<long long>(g) * gridDim.y + chunk) * n + gc] = t;
  }
}

// out[g*stride + col] += sum_c partial[g][c][col]: 32 columns x 32 warps per
// block, warp w adds chunks w, w+32, ...; warp sums combined in warp order.
__global__ void __launch_bounds__(1024) colsum_finish_kernel(const float* __restrict__ partial, int nchunks, int n,
                                                             int groups, float* __restrict__ out,
                                                             long long out_group_stride) {
  pdl_trigger();
  pdl_wait();
  __shared__ float red[32][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int col = blockIdx.x * 32 + lane, g = blockIdx.y;
  float s = 0.f;
  if (col < n)
    for (int c = warp; c < nchunks; c += 32) s += partial[(static_cast<long long>(g) * nchunks + c) * n + col];
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && col < n) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 32; ++w) t += red[w][lane];
    out[g * out_group_stride + col] += t;
  }
}

cudaError_t colsum_finish_launch(const float* partial, int nchunks, int n, int groups, float* out,
                                 long long out_group_stride, cudaStream_t s) {
  const cudaError_t e = launch_k(colsum_finish_kernel, dim3((n + 31) / 32, groups), dim3(1024), 0, s, 1, partial,
                                 nchunks, n, groups, out, out_group_stride);
  return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace p2r

using namespace p2r;

extern "C" p2r_status p2r_adamw_step(float* p, const float* g, float* m, float* v, void* p_bf16,
                                     const long long* seg_off, const long long* seg_len,
                                     const int* seg_decay, int nseg, float b1, float b2, float eps,
                                     float wd, float lr, float bc1, float bc2, void* stream) {
  if (nseg <= 0) return P2R_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int base = 0; base < nseg; base += P2R_MAX_ADAM_SEGS) {
    AdamArgs a{};
    a.p = p;
    a.g = g;
    a.m = m;
    a.v = v;
    a.p16 = static_cast<__nv_bfloat16*>(p_bf16);
    a.b1 = b1;
    a.b2 = b2;
    a.omb1 = 1.0f - b1;
    a.omb2 = 1.0f - b2;
    a.bc1 = bc1;
    a.bc2 = bc2;
    a.eps = eps;
    a.wd = wd;
    a.lr = lr;
    a.nseg = nseg - base < P2R_MAX_ADAM_SEGS ? nseg - base : P2R_MAX_ADAM_SEGS;
    long long maxlen = 0;
    for (int i = 0; i < a.nseg; ++i) {
      a.seg[i].off = seg_off[base + i];
      a.seg[i].len = seg_len[base + i];
      a.seg[i].decay = seg_decay[base + i];
      if (a.seg[i].len > maxlen) maxlen = a.seg[i].len;
    }
    long long bx = (maxlen / 4 + 255) / 256;
    if (bx < 1) bx = 1;
    if (bx > 4 * kNumSMs) bx = 4 * kNumSMs;
    P2R_LAUNCH_K("adamw", adamw_kernel, dim3(static_cast<unsigned>(bx), a.nseg), dim3(256), 0, s, 1, a);
  }
  return P2R_OK;
}

extern "C" p2r_status p2r_cast_bf16(const float* src, void* dst, long long n, void* stream) {
  if (n <= 0) return P2R_OK;
  long long blocks = (n + 255) / 256;
  if (blocks > 8 * kNumSMs) blocks = 8 * kNumSMs;
  cast_bf16_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      src, static_cast<__nv_bfloat16*>(dst), n);
  P2R_CHECK_LAUNCH("cast bf16");
  return P2R_OK;
}

extern "C" p2r_status p2r_delink_broadcast(const void* src, void* dst, size_t bytes,
                                           size_t dst_stride_bytes, int L, void* stream) {
  if (L <= 0 || bytes == 0) return P2R_OK;
  if ((bytes % 16) || (dst_stride_bytes % 16) || (reinterpret_cast<uintptr_t>(src) % 16) ||
      (reinterpret_cast<uintptr_t>(dst) % 16))
    return set_error(P2R_EINVAL, "delink: buffers must be 16-byte aligned and sized");
  const long long n16 = static_cast<long long>(bytes / 16);
  long long blocks = (n16 + 255) / 256;
  if (blocks > 8 * kNumSMs) blocks = 8 * kNumSMs;
  delink_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(src), static_cast<uint4*>(dst), n16,
      static_cast<long long>(dst_stride_bytes / 16), L);
  P2R_CHECK_LAUNCH("delink");
  return P2R_OK;
}

// 128-row chunks: ~1000 blocks at T = 8192 keep every SM's loads in flight
constexpr int kColsumChunk = 128;

extern "C" size_t p2r_colsum_workspace(int rows, int n, int groups) {
  const int chunk_rows = kColsumChunk;
  return static_cast<size_t>(groups) * ((rows + chunk_rows - 1) / chunk_rows) * n * sizeof(float);
}

// out[g*out_group_stride + c] += sum over the group's rows of x[r][c].
// dtype: 0 = fp32, 1 = bf16. counts == NULL -> one group of `rows` rows.
extern "C" p2r_status p2r_bias_grad(const void* x, int dtype, int ld, int rows, int n, int groups,
                                    int seg_rows, const int* counts, float* out,
                                    long long out_group_stride, float* ws, void* stream) {
  if (rows <= 0 || n <= 0) return P2R_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int chunk_rows = kColsumChunk;
  const int span = counts ? seg_rows : rows;
  const int nchunks = (span + chunk_rows - 1) / chunk_rows;
  const int G = counts ? groups : 1;
  const int vec = dtype == 0 ? 4 : 8;
  if ((n % vec) || (ld % vec) || (reinterpret_cast<uintptr_t>(x) % 16))
    return set_error(P2R_EINVAL, "bias grad: n, ld must be multiples of 16 bytes and x 16-byte aligned");
  dim3 grid((n / vec + 31) / 32, nchunks, G);
  if (dtype == 0) {
    P2R_LAUNCH_K("bias grad partial", colsum_partial_kernel<float>, grid, dim3(256), 0, s, 1,
                 static_cast<const float*>(x), ld, rows, n, chunk_rows, seg_rows, counts, ws);
  } else {
    P2R_LAUNCH_K("bias grad partial", colsum_partial_kernel<__nv_bfloat16>, grid, dim3(256), 0, s, 1,
                 static_cast<const __nv_bfloat16*>(x), ld, rows, n, chunk_rows, seg_rows, counts, ws);
  }
  P2R_LAUNCH_K("bias grad finish", colsum_finish_kernel, dim3((n + 31) / 32, G), dim3(1024), 0, s, 1,
               static_cast<const float*>(ws), nchunks, n, G, out, out_group_stride);
  return P2R_OK;
}
