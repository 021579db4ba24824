// Primitive layer of the drop-in tensor API (include/p2r/tensor.hpp): generic-shape
// fp32 kernels for the reference's fourteen differentiable primitives and their
// backward (/root/reference/proj/core/src/tensor.cpp:131-723). These keep the
// reference's fp32 arithmetic (the SPEC.md:46-66 known-answer tests hold at
// 1e-6); the training hot path does not use them -- the model layer runs the
// fused bf16 tcgen05 kernels (gemm_sm100.cu, attention_*.cu, ...). Every entry
// point takes device pointers and a stream; reductions run in a fixed order.
#include <cuda_runtime.h>

#include "common.cuh"
#include "p2r_cuda.h"
#include "p2r_internal.h"

namespace p2r {
namespace {

constexpr int kT = 16;  // SIMT GEMM tile

// C = op(A) op(B) + beta C, batched (blockIdx.z) with element strides
__global__ void gemm_f32_kernel(int ta, int tb, int m, int n, int k, const float* __restrict__ A, int lda,
                                const float* __restrict__ B, int ldb, float* __restrict__ C, int ldc, float beta,
                                long long sA, long long sB, long long sC) {
  __shared__ float As[kT][kT + 1], Bs[kT][kT + 1];
  const long long z = blockIdx.z;
  A += z * sA;
  B += z * sB;
  C += z * sC;
  const int row = blockIdx.y * kT + threadIdx.y, col = blockIdx.x * kT + threadIdx.x;
  float acc = 0.f;
  for (int k0 = 0; k0 < k; k0 += kT) {
    const int ka = k0 + threadIdx.x, kb = k0 + threadIdx.y;
    As[threadIdx.y][threadIdx.x] =
        (row < m && ka < k) ? (ta ? A[static_cast<long long>(ka) * lda + row] : A[static_cast<long long>(row) * lda + ka]) : 0.f;
    Bs[threadIdx.y][threadIdx.x] =
        (col < n && kb < k) ? (tb ? B[static_cast<long long>(col) * ldb + kb] : B[static_cast<long long>(kb) * ldb + col]) : 0.f;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kT; ++i) acc += As[threadIdx.y][i] * Bs[i][threadIdx.x];
    __syncthreads();
  }
  if (row < m && col < n) {
    float* c = C + static_cast<long long>(row) * ldc + col;
    *c = beta == 0.f ? acc : beta * *c + acc;
  }
}

// op 0: out = a + b; 1: out += a; 2: out = gelu(a); 3: out += b * gelu'(a)
__global__ void ew_kernel(int op, long long n, const float* __restrict__ a, const float* __restrict__ b,
                          float* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float x = a[i];
  switch (op) {
    case 0: out[i] = x + b[i]; break;
    case 1: out[i] += x; break;
    case 2: out[i] = 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); break;
    default: {
      const float cdf = 0.5f * (1.0f + erff(x * 0.70710678118654752f));
      const float pdf = 0.39894228040143268f * expf(-0.5f * x * x);
      out[i] += b[i] * (cdf + x * pdf);
    }
  }
}

__global__ void bias_kernel(int rows, int n, const float* __restrict__ x, const float* __restrict__ b,
                            float* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long long>(rows) * n) return;
  out[i] = x[i] + b[i % n];
}

// out[c] += sum over rows (in row order) of g[r][c]
__global__ void colsum_acc_kernel(int rows, int n, const float* __restrict__ g, float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  float s = 0.f;
  for (int r = 0; r < rows; ++r) s += g[static_cast<long long>(r) * n + c];
  out[c] += s;
}

// one warp per row: two-pass mean / biased variance (tensor.cpp:265-298)
__global__ void ln_fwd_kernel(int rows, int d, const float* __restrict__ x, const float* __restrict__ gain,
                              const float* __restrict__ bias, float eps, float* __restrict__ y,
                              float* __restrict__ xhat, float* __restrict__ inv) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* xr = x + static_cast<long long>(r) * d;
  float s = 0.f;
  for (int c = lane; c < d; c += 32) s += xr[c];
  s = warp_sum(s);
  const float mean = s / static_cast<float>(d);
  float v = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float t = xr[c] - mean;
    v += t * t;
  }
  v = warp_sum(v);
  const float iv = 1.0f / sqrtf(v / static_cast<float>(d) + eps);
  for (int c = lane; c < d; c += 32) {
    const float h = (xr[c] - mean) * iv;
    xhat[static_cast<long long>(r) * d + c] = h;
    y[static_cast<long long>(r) * d + c] = h * gain[c] + bias[c];
  }
  if (lane == 0) inv[r] = iv;
}

// gx += inv (g - mean(g) - xhat mean(g xhat)), g = gy * gain (tensor.cpp:302-331)
__global__ void ln_bwd_kernel(int rows, int d, const float* __restrict__ gy, const float* __restrict__ xhat,
                              const float* __restrict__ inv, const float* __restrict__ gain, float* __restrict__ gx) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const long long o = static_cast<long long>(r) * d;
  float s1 = 0.f, s2 = 0.f;
  for (int c = lane; c < d; c += 32) {
    const float g = gy[o + c] * gain[c];
    s1 += g;
    s2 += g * xhat[o + c];
  }
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  const float id = 1.0f / static_cast<float>(d);
  for (int c = lane; c < d; c += 32) {
    const float g = gy[o + c] * gain[c];
    gx[o + c] += inv[r] * (g - id * s1 - xhat[o + c] * (id * s2));
  }
}

// ggain[c] += sum_r gy xhat, gbias[c] += sum_r gy (row order)
__global__ void ln_param_grad_kernel(int rows, int d, const float* __restrict__ gy, const float* __restrict__ xhat,
                                     float* __restrict__ ggain, float* __restrict__ gbias) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  float a = 0.f, b = 0.f;
  for (int r = 0; r < rows; ++r) {
    const float g = gy[static_cast<long long>(r) * d + c];
    a += g * xhat[static_cast<long long>(r) * d + c];
    b += g;
  }
  ggain[c] += a;
  gbias[c] += b;
}

__global__ void gather_rows_kernel(int n_out, int d, const float* __restrict__ x, const int* __restrict__ rows,
                                   float* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long long>(n_out) * d) return;
  const int r = static_cast<int>(i / d), c = static_cast<int>(i % d);
  out[i] = x[static_cast<long long>(rows[r]) * d + c];
}

// gx[rows[i]] += g[i] in i order (one thread per column: deterministic)
__global__ void scatter_rows_acc_kernel(int n, int d, const float* __restrict__ g, const int* __restrict__ rows,
                                        float* __restrict__ gx) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  for (int i = 0; i < n; ++i) gx[static_cast<long long>(rows[i]) * d + c] += g[static_cast<long long>(i) * d + c];
}

// dir 0: [B*S, H*hd] -> [B, H, S, hd]; dir 1: the inverse. acc: out += instead of =
__global__ void permute_heads_kernel(int dir, int acc, int B, int H, int S, int hd, const float* __restrict__ in,
                                     float* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long long n = static_cast<long long>(B) * H * S * hd;
  if (i >= n) return;
  // i indexes the split layout [b][h][s][e]
  const int e = static_cast<int>(i % hd);
  long long t = i / hd;
  const int s = static_cast<int>(t % S);
  t /= S;
  const int h = static_cast<int>(t % H);
  const int b = static_cast<int>(t / H);
  const long long m = (static_cast<long long>(b) * S + s) * (static_cast<long long>(H) * hd) + static_cast<long long>(h) * hd + e;
  const long long src = dir == 0 ? m : i, dst = dir == 0 ? i : m;
  if (acc)
    out[dst] += in[src];
  else
    out[dst] = in[src];
}

// row-wise softmax in place over n columns; causal rows (row index % S = i) keep j <= i
// and zero the rest (tensor.cpp:487-502). One warp per row.
__global__ void softmax_rows_kernel(long long rows, int n, int causal_S, float* __restrict__ x) {
  const long long r = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  float* xr = x + r * n;
  const int lim = causal_S > 0 ? static_cast<int>(r % causal_S) + 1 : n;
  float mx = -INFINITY;
  for (int c = lane; c < lim; c += 32) mx = fmaxf(mx, xr[c]);
  mx = warp_max(mx);
  float s = 0.f;
  for (int c = lane; c < lim; c += 32) {
    const float e = expf(xr[c] - mx);
    xr[c] = e;
    s += e;
  }
  s = warp_sum(s);
  for (int c = lane; c < n; c += 32) xr[c] = c < lim ? xr[c] / s : 0.f;
}

// ds = p (dp - sum_j p dp) per row (tensor.cpp:526-533)
__global__ void softmax_bwd_rows_kernel(long long rows, int n, const float* __restrict__ p, const float* __restrict__ dp,
                                        float* __restrict__ ds) {
  const long long r = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* pr = p + r * n;
  const float* dr = dp + r * n;
  float dot = 0.f;
  for (int c = lane; c < n; c += 32) dot += pr[c] * dr[c];
  dot = warp_sum(dot);
  for (int c = lane; c < n; c += 32) ds[r * n + c] = pr[c] * (dr[c] - dot);
}

// selected_softmax forward (tensor.cpp:547-580): thread per token
__global__ void sel_softmax_fwd_kernel(int T, int E, int k, const float* __restrict__ logits,
                                       const int* __restrict__ sel, const uint8_t* __restrict__ surv,
                                       float* __restrict__ w) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  float mx = -1e30f;
  for (int j = 0; j < k; ++j)
    if (surv[t * k + j]) mx = fmaxf(mx, logits[static_cast<long long>(t) * E + sel[t * k + j]]);
  float s = 0.f;
  for (int j = 0; j < k; ++j) {
    float e = 0.f;
    if (surv[t * k + j]) {
      e = expf(logits[static_cast<long long>(t) * E + sel[t * k + j]] - mx);
      s += e;
    }
    w[t * k + j] = e;
  }
  if (s > 0.f) {
    const float inv = 1.0f / s;
    for (int j = 0; j < k; ++j)
      if (surv[t * k + j]) w[t * k + j] *= inv;
  }
}

// selected_softmax backward (tensor.cpp:586-603): gl[t][sel] += w (gw - sum w gw)
__global__ void sel_softmax_bwd_kernel2(int T, int E, int k, const float* __restrict__ w, const float* __restrict__ gw,
                                        const int* __restrict__ sel, const uint8_t* __restrict__ surv,
                                        float* __restrict__ gl) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  float dot = 0.f;
  for (int j = 0; j < k; ++j)
    if (surv[t * k + j]) dot += w[t * k + j] * gw[t * k + j];
  for (int j = 0; j < k; ++j)
    if (surv[t * k + j]) gl[static_cast<long long>(t) * E + sel[t * k + j]] += w[t * k + j] * (gw[t * k + j] - dot);
}

// moe_combine forward: out[t] += w[t, slot] * y[row] over the token's contributions,
// listed in (expert asc, row asc) order in [off[t], off[t+1])
__global__ void combine_fwd_kernel(int T, int d, int k, const int* __restrict__ off, const int* __restrict__ crow,
                                   const int* __restrict__ cslot, const float* __restrict__ y, const float* __restrict__ w,
                                   float* __restrict__ out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long long>(T) * d) return;
  const int t = static_cast<int>(i / d), c = static_cast<int>(i % d);
  float acc = out[i];
  for (int q = off[t]; q < off[t + 1]; ++q) acc += w[t * k + cslot[q]] * y[static_cast<long long>(crow[q]) * d + c];
  out[i] = acc;
}

// moe_combine backward: dy[r] += w[t, slot] dout[t]; dw[t, slot] += <dout[t], y[r]>
__global__ void combine_bwd_kernel(int R, int d, int k, const int* __restrict__ rtok, const int* __restrict__ rslot,
                                   const float* __restrict__ dout, const float* __restrict__ y, const float* __restrict__ w,
                                   float* __restrict__ dy, float* __restrict__ dw) {
  const int r = blockIdx.x;
  const int t = rtok[r], s = rslot[r];
  const float ws = w[t * k + s];
  float dot = 0.f;
  for (int c = threadIdx.x; c < d; c += blockDim.x) {
    const float g = dout[static_cast<long long>(t) * d + c];
    if (dy) dy[static_cast<long long>(r) * d + c] += ws * g;
    dot += g * y[static_cast<long long>(r) * d + c];
  }
  __shared__ float red[32];
  dot = warp_sum(dot);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dot;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s2 = 0.f;
    for (int i = 0; i < static_cast<int>(blockDim.x >> 5); ++i) s2 += red[i];
    if (dw) dw[t * k + s] += s2;
  }
}

// softmax cross entropy (tensor.cpp:670-723): per row -log p[target] (double), and
// glogits = (p - onehot) / denom for active rows. One warp per row.
__global__ void ce_kernel(int rows, int V, const float* __restrict__ logits, const int* __restrict__ tgt,
                          const uint8_t* __restrict__ mask, float scale, double* __restrict__ row_loss,
                          float* __restrict__ gl) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* x = logits + static_cast<long long>(r) * V;
  const bool active = mask == nullptr || mask[r] != 0;
  float mx = -INFINITY;
  for (int c = lane; c < V; c += 32) mx = fmaxf(mx, x[c]);
  mx = warp_max(mx);
  float s = 0.f;
  for (int c = lane; c < V; c += 32) s += expf(x[c] - mx);
  s = warp_sum(s);
  const float inv = 1.0f / s;
  const int t = active ? tgt[r] : 0;
  for (int c = lane; c < V; c += 32) {
    const float p = expf(x[c] - mx) * inv;
    gl[static_cast<long long>(r) * V + c] = active ? (p - (c == t ? 1.f : 0.f)) * scale : 0.f;
  }
  if (lane == 0) row_loss[r] = active ? -log(static_cast<double>(expf(x[t] - mx) * inv)) : 0.0;
}

// loss = sum_r row_loss (row order, double) / denom
__global__ void ce_finish_kernel(int rows, const double* __restrict__ row_loss, double denom, float* __restrict__ loss) {
  double s = 0.0;
  for (int r = 0; r < rows; ++r) s += row_loss[r];
  *loss = static_cast<float>(s / denom);
}

unsigned nblk(long long n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace
}  // namespace p2r

using namespace p2r;
#define S_ static_cast<cudaStream_t>(stream)

extern "C" p2r_status p2r_prim_gemm_f32(int ta, int tb, int m, int n, int k, const float* a, int lda, const float* b,
                                        int ldb, float* c, int ldc, float beta, int batch, long long sa, long long sb,
                                        long long sc, void* stream) {
  if (m <= 0 || n <= 0 || batch <= 0) return P2R_OK;
  const dim3 grid((n + kT - 1) / kT, (m + kT - 1) / kT, batch), block(kT, kT);
  gemm_f32_kernel<<<grid, block, 0, S_>>>(ta, tb, m, n, k, a, lda, b, ldb, c, ldc, beta, sa, sb, sc);
  P2R_CHECK_LAUNCH("prim gemm");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_ew(int op, long long n, const float* a, const float* b, float* out, void* stream) {
  if (n <= 0) return P2R_OK;
  ew_kernel<<<nblk(n, 256), 256, 0, S_>>>(op, n, a, b, out);
  P2R_CHECK_LAUNCH("prim elementwise");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_bias(int rows, int n, const float* x, const float* b, float* out, void* stream) {
  if (rows <= 0 || n <= 0) return P2R_OK;
  bias_kernel<<<nblk(static_cast<long long>(rows) * n, 256), 256, 0, S_>>>(rows, n, x, b, out);
  P2R_CHECK_LAUNCH("prim bias");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_colsum_acc(int rows, int n, const float* g, float* out, void* stream) {
  if (n <= 0) return P2R_OK;
  colsum_acc_kernel<<<nblk(n, 128), 128, 0, S_>>>(rows, n, g, out);
  P2R_CHECK_LAUNCH("prim colsum");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_layernorm_fwd(int rows, int d, const float* x, const float* gain, const float* bias,
                                             float eps, float* y, float* xhat, float* inv, void* stream) {
  if (rows <= 0) return P2R_OK;
  ln_fwd_kernel<<<nblk(rows, 4), 128, 0, S_>>>(rows, d, x, gain, bias, eps, y, xhat, inv);
  P2R_CHECK_LAUNCH("prim layernorm fwd");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_layernorm_bwd(int rows, int d, const float* gy, const float* xhat, const float* inv,
                                             const float* gain, float* gx, float* ggain, float* gbias, void* stream) {
  if (rows <= 0) return P2R_OK;
  if (gx) {
    ln_bwd_kernel<<<nblk(rows, 4), 128, 0, S_>>>(rows, d, gy, xhat, inv, gain, gx);
    P2R_CHECK_LAUNCH("prim layernorm bwd");
  }
  if (ggain && gbias) {
    ln_param_grad_kernel<<<nblk(d, 128), 128, 0, S_>>>(rows, d, gy, xhat, ggain, gbias);
    P2R_CHECK_LAUNCH("prim layernorm param grad");
  }
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_gather_rows(int n_out, int d, const float* x, const int* rows, float* out, void* stream) {
  if (n_out <= 0 || d <= 0) return P2R_OK;
  gather_rows_kernel<<<nblk(static_cast<long long>(n_out) * d, 256), 256, 0, S_>>>(n_out, d, x, rows, out);
  P2R_CHECK_LAUNCH("prim gather rows");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_scatter_rows_acc(int n, int d, const float* g, const int* rows, float* gx, void* stream) {
  if (n <= 0 || d <= 0) return P2R_OK;
  scatter_rows_acc_kernel<<<nblk(d, 128), 128, 0, S_>>>(n, d, g, rows, gx);
  P2R_CHECK_LAUNCH("prim scatter rows");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_permute_heads(int dir, int acc, int B, int H, int S, int hd, const float* in, float* out,
                                             void* stream) {
  const long long n = static_cast<long long>(B) * H * S * hd;
  if (n <= 0) return P2R_OK;
  permute_heads_kernel<<<nblk(n, 256), 256, 0, S_>>>(dir, acc, B, H, S, hd, in, out);
  P2R_CHECK_LAUNCH("prim permute heads");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_softmax_rows(long long rows, int n, int causal_S, float* x, void* stream) {
  if (rows <= 0) return P2R_OK;
  softmax_rows_kernel<<<nblk(rows, 4), 128, 0, S_>>>(rows, n, causal_S, x);
  P2R_CHECK_LAUNCH("prim softmax rows");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_softmax_bwd_rows(long long rows, int n, const float* p, const float* dp, float* ds,
                                                void* stream) {
  if (rows <= 0) return P2R_OK;
  softmax_bwd_rows_kernel<<<nblk(rows, 4), 128, 0, S_>>>(rows, n, p, dp, ds);
  P2R_CHECK_LAUNCH("prim softmax bwd");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_selected_softmax(int dir, int T, int E, int k, const float* logits_or_w,
                                                const float* gw, const int* sel, const uint8_t* surv, float* out,
                                                void* stream) {
  if (T <= 0) return P2R_OK;
  if (dir == 0)
    sel_softmax_fwd_kernel<<<nblk(T, 128), 128, 0, S_>>>(T, E, k, logits_or_w, sel, surv, out);
  else
    sel_softmax_bwd_kernel2<<<nblk(T, 128), 128, 0, S_>>>(T, E, k, logits_or_w, gw, sel, surv, out);
  P2R_CHECK_LAUNCH("prim selected softmax");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_combine_fwd(int T, int d, int k, const int* off, const int* crow, const int* cslot,
                                           const float* y, const float* w, float* out, void* stream) {
  if (T <= 0 || d <= 0) return P2R_OK;
  combine_fwd_kernel<<<nblk(static_cast<long long>(T) * d, 256), 256, 0, S_>>>(T, d, k, off, crow, cslot, y, w, out);
  P2R_CHECK_LAUNCH("prim combine");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_combine_bwd(int R, int d, int k, const int* rtok, const int* rslot, const float* dout,
                                           const float* y, const float* w, float* dy, float* dw, void* stream) {
  if (R <= 0) return P2R_OK;
  combine_bwd_kernel<<<R, 128, 0, S_>>>(R, d, k, rtok, rslot, dout, y, w, dy, dw);
  P2R_CHECK_LAUNCH("prim combine bwd");
  return P2R_OK;
}

extern "C" p2r_status p2r_prim_cross_entropy(int rows, int V, const float* logits, const int* targets,
                                             const uint8_t* mask, double denom, double* row_loss_ws, float* loss,
                                             float* glogits, void* stream) {
  if (rows <= 0) return P2R_OK;
  ce_kernel<<<nblk(rows, 4), 128, 0, S_>>>(rows, V, logits, targets, mask, static_cast<float>(1.0 / denom),
                                           row_loss_ws, glogits);
  P2R_CHECK_LAUNCH("prim cross entropy");
  ce_finish_kernel<<<1, 1, 0, S_>>>(rows, row_loss_ws, denom, loss);
  P2R_CHECK_LAUNCH("prim cross entropy finish");
  return P2R_OK;
}
#undef S_
