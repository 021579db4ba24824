// Expert-parallel exchange over peer memory (the reference's
// expert_shard map, model.cpp:334-340: expert e lives on rank e / (E / W)).
//
// The MoE dispatch and combine of a rank's tokens are fused with the all-to-all:
// instead of packing send buffers for a collective, the kernels below write
// token rows straight into the owner rank's receive buffers (NVLink / NVSwitch
// peer stores on a multi-GPU node; local stores for a loopback group of shards on
// one device), and the host signals completion with stream memory operations
// (csrc/engine/comm.cpp). Only admitted rows cross the link, in bf16, so the bytes
// per direction are the routed rows x d x 2 (no capacity padding).
//
// Layouts (W ranks, E experts, El = E / W local experts, seg = per-expert rows):
//   source, local   [E][seg][d]        expert-major rows of this rank's tokens
//   owner, slots    [El][W][seg][d]    rows from each source rank, per local expert
//   owner, counts   [El][W]            rows each source sent to each local expert
//   owner, compact  [El][W*seg][d]     per local expert: source 0's rows, then
//                                      source 1's, ...; zero-padded to 128 rows,
//                                      the operand layout of the grouped GEMMs
#include <cuda_bf16.h>

#include "common.cuh"
#include "p2r_cuda.h"
#include "p2r_internal.h"

namespace p2r {
namespace {

constexpr int kMaxPeers = 64;
struct PeerTable {
  void* p[kMaxPeers];
};
struct PeerCounts {
  int* p[kMaxPeers];
};

P2R_DEVICE void copy_row_bf16(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst, int d) {
  // 16-byte vectors (d % 8 == 0 for every supported d_model)
  const uint4* s = reinterpret_cast<const uint4*>(src);
  uint4* o = reinterpret_cast<uint4*>(dst);
  for (int c = threadIdx.x; c < d / 8; c += blockDim.x) o[c] = s[c];
}

// Source side: the admitted rows of every expert, gathered from the token-major
// activations (bf16 rows; or fp32 rows scaled by the combine weight in the
// backward), stored into the owner's slot layout [El][W][seg] at this rank's
// slot, plus this rank's count per expert. grid (seg, E).
template <typename Tin>
__global__ void ep_send_rows_kernel(const Tin* __restrict__ src, int d, const int* __restrict__ rows_pad,
                                    const int* __restrict__ slots_pad, const int* __restrict__ counts,
                                    const float* __restrict__ w, int k, int seg, int El, int W, int rank,
                                    PeerTable slots, PeerCounts peer_counts) {
  const int e = blockIdx.y, r = blockIdx.x;
  const int q = e / El, j = e % El;
  const int cnt = counts[e];
  if (r == 0 && threadIdx.x == 0) peer_counts.p[q][j * W + rank] = cnt;
  if (r >= cnt) return;
  const long long li = static_cast<long long>(e) * seg + r;
  const int t = rows_pad[li];
  __nv_bfloat16* dst = static_cast<__nv_bfloat16*>(slots.p[q]) + (static_cast<long long>(j * W + rank) * seg + r) * d;
  if constexpr (sizeof(Tin) == 2) {
    copy_row_bf16(reinterpret_cast<const __nv_bfloat16*>(src) + static_cast<long long>(t) * d, dst, d);
  } else {
    const float scale = w ? w[t * k + slots_pad[li]] : 1.f;
    const float* s = reinterpret_cast<const float*>(src) + static_cast<long long>(t) * d;
    for (int c = 4 * threadIdx.x; c < d; c += 4 * blockDim.x) {
      const float4 v = *reinterpret_cast<const float4*>(s + c);
      __nv_bfloat162 a = __floats2bfloat162_rn(scale * v.x, scale * v.y), b = __floats2bfloat162_rn(scale * v.z, scale * v.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&a);
      u.y = *reinterpret_cast<uint32_t*>(&b);
      *reinterpret_cast<uint2*>(dst + c) = u;
    }
  }
}

// Owner side: slots [El][W][seg] -> compact [El][gseg] (gseg = W*seg), rows of
// source 0 first; rows past the total up to the next 128 are zeroed (the grouped
// GEMMs read whole 128-row tiles). tot[j] and prefix[j][0..W] describe the layout.
// grid (gseg, El).
__global__ void ep_pack_kernel(const __nv_bfloat16* __restrict__ slots, const int* __restrict__ cnt, int d, int seg,
                               int W, __nv_bfloat16* __restrict__ compact, int* __restrict__ tot,
                               int* __restrict__ prefix) {
  const int j = blockIdx.y, i = blockIdx.x;
  const int gseg = W * seg;
  int total = 0, src = -1, row = 0;
  for (int w = 0; w < W; ++w) {
    const int c = cnt[j * W + w];
    if (src < 0 && i < total + c) {
      src = w;
      row = i - total;
    }
    total += c;
  }
  if (i == 0 && threadIdx.x == 0) {
    tot[j] = total;
    int acc = 0;
    for (int w = 0; w < W; ++w) {
      prefix[j * (W + 1) + w] = acc;
      acc += cnt[j * W + w];
    }
    prefix[j * (W + 1) + W] = acc;
  }
  __nv_bfloat16* dst = compact + (static_cast<long long>(j) * gseg + i) * d;
  if (src >= 0) {
    copy_row_bf16(slots + (static_cast<long long>(j * W + src) * seg + row) * d, dst, d);
  } else if (i < (total + 127) / 128 * 128) {
    uint4* o = reinterpret_cast<uint4*>(dst);
    for (int c = threadIdx.x; c < d / 8; c += blockDim.x) o[c] = make_uint4(0, 0, 0, 0);
  }
}

// Owner side: compact rows [El][gseg] (expert outputs / input gradients, bf16)
// back to their source ranks, into the source's local layout [E][seg] at the
// row the source dispatched them from. grid (gseg, El).
__global__ void ep_return_rows_kernel(const __nv_bfloat16* __restrict__ compact, const int* __restrict__ prefix, int d,
                                      int seg, int W, int El, int rank, PeerTable dst) {
  const int j = blockIdx.y, i = blockIdx.x;
  const int* pf = prefix + j * (W + 1);
  if (i >= pf[W]) return;
  int w = 0;
  while (i >= pf[w + 1]) ++w;
  const int r = i - pf[w];
  const int e = rank * El + j;  // global expert id
  __nv_bfloat16* out = static_cast<__nv_bfloat16*>(dst.p[w]) + (static_cast<long long>(e) * seg + r) * d;
  copy_row_bf16(compact + (static_cast<long long>(j) * W * seg + i) * d, out, d);
}

int row_threads(int d) { return d >= 2048 ? 256 : 128; }

}  // namespace
}  // namespace p2r

using namespace p2r;

extern "C" p2r_status p2r_ep_send_rows(const void* src, int src_dtype, int d, int E, int seg,
                                       const int* rows_pad, const int* slots_pad, const int* counts,
                                       const float* w, int k, int W, int rank, void* const* peer_slots,
                                       int* const* peer_counts, void* stream) {
  if (W < 1 || W > kMaxPeers || E % W != 0 || d % 8 != 0) return set_error(P2R_EINVAL, "ep send: bad shape");
  PeerTable pt{};
  PeerCounts pc{};
  for (int q = 0; q < W; ++q) {
    pt.p[q] = peer_slots[q];
    pc.p[q] = peer_counts[q];
  }
  const dim3 grid(seg, E);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (src_dtype == 1)
    ep_send_rows_kernel<__nv_bfloat16><<<grid, row_threads(d), 0, s>>>(
        static_cast<const __nv_bfloat16*>(src), d, rows_pad, slots_pad, counts, w, k, seg, E / W, W, rank, pt, pc);
  else
    ep_send_rows_kernel<float><<<grid, row_threads(d), 0, s>>>(static_cast<const float*>(src), d, rows_pad, slots_pad,
                                                               counts, w, k, seg, E / W, W, rank, pt, pc);
  P2R_CHECK_LAUNCH("ep send rows");
  return P2R_OK;
}

extern "C" p2r_status p2r_ep_pack(const void* slots, const int* cnt, int d, int seg, int El, int W, void* compact,
                                  int* tot, int* prefix, void* stream) {
  if (W < 1 || d % 8 != 0) return set_error(P2R_EINVAL, "ep pack: bad shape");
  const dim3 grid(W * seg, El);
  ep_pack_kernel<<<grid, row_threads(d), 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(slots), cnt, d, seg, W, static_cast<__nv_bfloat16*>(compact), tot, prefix);
  P2R_CHECK_LAUNCH("ep pack");
  return P2R_OK;
}

extern "C" p2r_status p2r_ep_return_rows(const void* compact, const int* prefix, int d, int seg, int El, int W,
                                         int rank, void* const* peer_dst, void* stream) {
  if (W < 1 || W > kMaxPeers || d % 8 != 0) return set_error(P2R_EINVAL, "ep return: bad shape");
  PeerTable pt{};
  for (int q = 0; q < W; ++q) pt.p[q] = peer_dst[q];
  const dim3 grid(W * seg, El);
  ep_return_rows_kernel<<<grid, row_threads(d), 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(compact), prefix, d, seg, W, El, rank, pt);
  P2R_CHECK_LAUNCH("ep return rows");
  return P2R_OK;
}

namespace p2r {
namespace {
// out[i] = stage[0][i] + stage[1][i] + ... (rank order: deterministic)
__global__ void sum_ranks_kernel(const float* __restrict__ stage, int W, long long n, float* __restrict__ out) {
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    float acc = stage[i];
    for (int w = 1; w < W; ++w) acc += stage[static_cast<long long>(w) * n + i];
    out[i] = acc;
  }
}
}  // namespace
}  // namespace p2r

extern "C" p2r_status p2r_sum_ranks(const float* stage, int W, long long n, float* out, void* stream) {
  if (n <= 0) return P2R_OK;
  long long blocks = (n + 255) / 256;
  if (blocks > 8LL * kNumSMs) blocks = 8LL * kNumSMs;
  sum_ranks_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(stage, W, n, out);
  P2R_CHECK_LAUNCH("sum ranks");
  return P2R_OK;
}
