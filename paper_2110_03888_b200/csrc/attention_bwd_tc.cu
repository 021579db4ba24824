// Flash-attention BACKWARD on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Replaces masked_attention's backward (tensor.cpp:510-541). P is recomputed
// from the saved row log-sum-exp (no S x S matrix). Deterministic: no atomics.
//   dQ kernel   (CTA = 128 queries, loop over 64-key blocks):
//       S = Q.K^T, dP = dO.V^T (TMEM, double-buffered) -> softmax warps (thread =
//       query row) form dS = P o (dP - D) in a SWIZZLE_128B smem tile ->
//       dQ += dS.K (K tile re-read MN-major). Its prologue also computes
//       D = rowsum(dO o O) (tensor.cpp:526-533) for the dK/dV kernel.
//   dK/dV kernel (CTA = 128 keys, loop over 64-query blocks):
//       S^T = K.Q^T, dP^T = V.dO^T -> thread = key row forms P^T and dS^T ->
//       dV += P^T.dO, dK += dS^T.Q (Q / dO tiles re-read MN-major).
// The same swizzled smem bytes serve as a K-major operand for one MMA and as
// an MN-major operand for the next, so no transposes are materialised.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "../../include/p2r_cuda.h"
#include "common.cuh"
#include "p2r_internal.h"

namespace p2r {
namespace attn_bwd_tc {

constexpr float kLog2e = 1.4426950408889634f;

P2R_DEVICE uint32_t sw128_off(int row, int chunk16) {
  return static_cast<uint32_t>(row * 128 + ((chunk16 ^ (row & 7)) << 4));
}
P2R_DEVICE float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// SW128 descriptors are advanced by adding (bytes >> 4) to the start-address
// field: precomputed once, so the single MMA-issuing thread does one add per
// MMA instead of rebuilding the 64-bit descriptor (which made 128x64 MMAs
// issue-bound at ~80 cycles).
P2R_DEVICE uint64_t dadd(uint64_t d, uint32_t bytes) { return d + (bytes >> 4); }
P2R_DEVICE void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
P2R_DEVICE void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct BwdParams {
  const __nv_bfloat16* o;     // [T, d]
  const __nv_bfloat16* dout;  // [T, d]
  const float* lse;           // [B, H, S]
  float* dsum;                // [B, H, S]
  __nv_bfloat16* dqkv;        // [T, 3d]
  int B, H, S, d;
  int causal;
  float scale, sl2;
};

// write a row of 64 bf16 values (from fp32 pairs) into a [rows x 64] SW128 atom
P2R_DEVICE void store_row64(uint32_t atom, int row, const float* v) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[c * 8 + 2 * i], v[c * 8 + 2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    sts128(atom + sw128_off(row, c), make_uint4(w[0], w[1], w[2], w[3]));
  }
}

// write 32 bf16 values (4 x 16-B chunks starting at chunk c0) of one row of a SW128 atom
P2R_DEVICE void store_row32(uint32_t atom, int row, int c0, const float* v) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[c * 8 + 2 * i], v[c * 8 + 2 * i + 1]);
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    sts128(atom + sw128_off(row, c0 + c), make_uint4(w[0], w[1], w[2], w[3]));
  }
}

// S and dP rows of one block: both TMEM loads in flight before a single wait
P2R_DEVICE void ld32x2(uint32_t ta, uint32_t tb, float* a, float* b) {
  uint32_t ra[32], rb[32];
  tmem_ld_32x32b_x32(ta, ra);
  tmem_ld_32x32b_x32(tb, rb);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    a[i] = __uint_as_float(ra[i]);
    b[i] = __uint_as_float(rb[i]);
  }
}

// ============================================================================ dQ
template <int HD>
struct DqCfg {
  static constexpr int BQ = 128, BKV = 64, KA = HD / 64;
  static constexpr int NS = HD == 64 ? 4 : 2;  // K/V TMA ring depth (hides load latency behind 2+ blocks)
  static constexpr int QT = BQ * HD * 2;     // Q / dO tile
  static constexpr int KT = BKV * HD * 2;    // K / V tile
  static constexpr int DST = BQ * BKV * 2;   // dS tile (one 64-key atom)
  static constexpr int OFF_Q = 0, OFF_DO = QT, OFF_K = 2 * QT, OFF_V = OFF_K + NS * KT, OFF_DS = OFF_V + NS * KT;
  static constexpr int OFF_BAR = OFF_DS + 2 * DST;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int T_S = 0, T_DP = 128, T_DQ = 256;  // S[2] at 0/64, dP[2] at 128/192
};

template <int HD>
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq_tc(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                   const __grid_constant__ CUtensorMap tm_do, const BwdParams p) {
  using C = DqCfg<HD>;
#ifdef P2R_ATTN_TRACE
  // diagnostic build only: clock64 timeline of CTA (0,0,0) (the heaviest causal
  // tile), dumped over the start of `o` at exit; see scripts/attn_trace.py
  __shared__ long long s_tr[512];
  const bool tr_cta = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
#define TR(slot) do { if (tr_cta) s_tr[(slot)] = clock64(); } while (0)
#else
#define TR(slot) do {} while (0)
#endif
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar;          // Q + dO
  uint64_t* s_full = bar + 1;      // [2]  S and dP of block j
  uint64_t* ds_full = bar + 3;     // [2]  dS of block j in smem
  uint64_t* dq_done = bar + 5;     // [2]  dQ += dS_j.K_j completed
  uint64_t* kv_full = bar + 7;     // [NS]
  uint64_t* kv_empty = kv_full + C::NS;  // [NS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kv_empty + C::NS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // causal: the last query tiles see the most keys -> launch them first
  const int qb = p.causal ? gridDim.x - 1 - blockIdx.x : blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int q0 = qb * C::BQ, row0 = b * p.S;
  const int kend = p.causal ? min(p.S, q0 + C::BQ) : p.S;
  const int nkv = (kend + C::BKV - 1) / C::BKV;
  if (threadIdx.x == 0) TR(0);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_do);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(ds_full + i, 256);
      mbar_init(dq_done + i, 1);
    }
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // dkdv reads the dq kernel's D (dsum)
  const uint32_t sb = smem_u32(smem);
  if (threadIdx.x == 0) TR(1);

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * C::QT);
      for (int a = 0; a < C::KA; ++a) {
        tma_load_2d(smem + C::OFF_Q + a * C::BQ * 128, &tm_q, q_full, h * HD + 64 * a, row0 + q0);
        tma_load_2d(smem + C::OFF_DO + a * C::BQ * 128, &tm_do, q_full, h * HD + 64 * a, row0 + q0);
      }
      for (int j = 0; j < nkv; ++j) {
        const int st = j % C::NS;
        mbar_wait(kv_empty + st, ((j / C::NS) & 1) ^ 1);
        mbar_arrive_expect_tx(kv_full + st, 2 * C::KT);
        for (int a = 0; a < C::KA; ++a) {
          tma_load_2d(smem + C::OFF_K + st * C::KT + a * C::BKV * 128, &tm_kv, kv_full + st, p.d + h * HD + 64 * a,
                      row0 + j * C::BKV);
          tma_load_2d(smem + C::OFF_V + st * C::KT + a * C::BKV * 128, &tm_kv, kv_full + st,
                      2 * p.d + h * HD + 64 * a, row0 + j * C::BKV);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = make_idesc_bf16(C::BQ, C::BKV, false, false);
      constexpr uint32_t id_q = make_idesc_bf16(C::BQ, HD, false, true);
      mbar_wait(q_full, 0);
      tc_fence_after();
      TR(2);
      auto issue_dq = [&](int jj) {
        mbar_wait(ds_full + (jj & 1), (jj >> 1) & 1);
        tc_fence_after();
        TR(16 + 4 * jj + 2);
        const uint32_t sds = sb + C::OFF_DS + (jj & 1) * C::DST;
        const uint32_t sk = sb + C::OFF_K + (jj % C::NS) * C::KT;
#pragma unroll
        for (int k = 0; k < C::BKV / 16; ++k)
          umma_bf16(tmem + C::T_DQ, make_sw128_desc(sds + k * 32, 16, 1024),
                    make_sw128_desc(sk + k * 2048, C::BKV * 128, 1024), id_q, (jj > 0 || k > 0) ? 1u : 0u);
        umma_commit(kv_empty + jj % C::NS);
        umma_commit(dq_done + (jj & 1));
        TR(16 + 4 * jj + 3);
      };
      for (int j = 0; j < nkv; ++j) {
        const int st = j % C::NS;
        mbar_wait(kv_full + st, (j / C::NS) & 1);
        tc_fence_after();
        TR(16 + 4 * j);
        const uint32_t sk = sb + C::OFF_K + st * C::KT, sv = sb + C::OFF_V + st * C::KT;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t ka = (k >> 2), kk = (k & 3) * 32;
          umma_bf16(tmem + C::T_S + (j & 1) * 64, make_sw128_desc(sb + C::OFF_Q + ka * C::BQ * 128 + kk, 16, 1024),
                    make_sw128_desc(sk + ka * C::BKV * 128 + kk, 16, 1024), id_s, k > 0 ? 1u : 0u);
          umma_bf16(tmem + C::T_DP + (j & 1) * 64, make_sw128_desc(sb + C::OFF_DO + ka * C::BQ * 128 + kk, 16, 1024),
                    make_sw128_desc(sv + ka * C::BKV * 128 + kk, 16, 1024), id_s, k > 0 ? 1u : 0u);
        }
        umma_commit(s_full + (j & 1));
        TR(16 + 4 * j + 1);
        if (j > 0) issue_dq(j - 1);
      }
      issue_dq(nkv - 1);
    }
  } else if (warp >= 4) {
    // 8 warps: two per TMEM lane quadrant, each owning 32 of the 64 key columns
    const int r = (warp & 3) * 32 + lane;
    const int half = (warp - 4) >> 2;
    const int q = q0 + r;
    const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const long long bh = static_cast<long long>(b) * p.H + h;
    // D = rowsum(dO o O) for this row (fp32 accumulate), published for the dK/dV kernel
    float D = 0.0f;
    if (q < p.S) {
      const uint4* a4 = reinterpret_cast<const uint4*>(p.dout + static_cast<long long>(row0 + q) * p.d + h * HD);
      const uint4* o4 = reinterpret_cast<const uint4*>(p.o + static_cast<long long>(row0 + q) * p.d + h * HD);
#pragma unroll
      for (int c = 0; c < HD / 8; ++c) {
        const uint4 x = a4[c], y = o4[c];
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 u = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[i]));
          const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ys[i]));
          D += u.x * v.x + u.y * v.y;
        }
      }
      if (half == 0) p.dsum[bh * p.S + q] = D;
    }
    const float lse2 = q < p.S ? p.lse[bh * p.S + q] * kLog2e : 0.0f;
    const float sl2 = p.sl2;
    const bool trw = warp == 4 && lane == 0;  // trace writer (P2R_ATTN_TRACE builds)
    if (trw) TR(3);
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(s_full + (j & 1), (j >> 1) & 1);
      tc_fence_after();
      if (trw) TR(100 + 6 * j);
      float s[32], dp[32];
      ld32x2(tmem + la + C::T_S + (j & 1) * 64 + half * 32, tmem + la + C::T_DP + (j & 1) * 64 + half * 32, s, dp);
      if (trw) TR(100 + 6 * j + 1);
      const int k0 = j * C::BKV + half * 32;
      int lim = 32;
      if (q >= p.S) lim = 0;
      else if (p.causal || k0 + 32 > p.S) lim = min(p.causal ? q + 1 : p.S, p.S) - k0;
      // exponentials unconditionally (no per-element predication); the causal /
      // tail mask is a select on the few blocks that need it (discards any inf)
#pragma unroll
      for (int i = 0; i < 32; ++i) s[i] = ex2_approx(fmaf(s[i], sl2, -lse2));
      if (lim < 32) {
#pragma unroll
        for (int i = 0; i < 32; ++i) s[i] = i < lim ? s[i] : 0.0f;
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) s[i] = s[i] * (dp[i] - D);
      if (trw) TR(100 + 6 * j + 2);
      if (j >= 2) mbar_wait(dq_done + (j & 1), ((j - 2) >> 1) & 1);
      if (trw) TR(100 + 6 * j + 3);
      store_row32(sb + C::OFF_DS + (j & 1) * C::DST, r, half * 4, s);
      fence_async_smem();
      tc_fence_before();
      if (trw) TR(100 + 6 * j + 4);
      mbar_arrive(ds_full + (j & 1));
      if (trw) TR(100 + 6 * j + 5);
    }
    mbar_wait(dq_done + ((nkv - 1) & 1), ((nkv - 1) >> 1) & 1);
    tc_fence_after();
    __nv_bfloat16* dq = p.dqkv + static_cast<long long>(row0 + q) * 3 * p.d + h * HD;
#pragma unroll
    for (int c = half; c < HD / 32; c += 2) {
      uint32_t rr[32];
      tmem_ld_32x32b_x32(tmem + la + C::T_DQ + c * 32, rr);
      tmem_ld_wait();
      if (q < p.S) {
        uint32_t w[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          __nv_bfloat162 hh = __floats2bfloat162_rn(__uint_as_float(rr[2 * i]) * p.scale, __uint_as_float(rr[2 * i + 1]) * p.scale);
          w[i] = *reinterpret_cast<uint32_t*>(&hh);
        }
        uint4* dst = reinterpret_cast<uint4*>(dq + c * 32);
#pragma unroll
        for (int i = 0; i < 4; ++i) dst[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef P2R_ATTN_TRACE
  if (threadIdx.x == 0) TR(4);
  __syncthreads();
  if (tr_cta)
    for (int i = threadIdx.x; i < 512; i += blockDim.x) reinterpret_cast<long long*>(const_cast<__nv_bfloat16*>(p.o))[i] = s_tr[i];
#endif
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}
#undef TR

// ============================================================================ dK / dV
template <int HD>
struct KvCfg {
  static constexpr int BK = 128, BQ = 64, KA = HD / 64;
  static constexpr int NS = HD == 64 ? 4 : 2;  // Q/dO TMA ring depth
  static constexpr int KT = BK * HD * 2;     // K / V tile
  static constexpr int QT = BQ * HD * 2;     // Q / dO tile
  static constexpr int PT = BK * BQ * 2;     // P^T / dS^T tile (one 64-query atom)
  static constexpr int OFF_K = 0, OFF_V = KT, OFF_Q = 2 * KT, OFF_DO = OFF_Q + NS * QT;
  static constexpr int OFF_P = OFF_DO + NS * QT, OFF_DS = OFF_P + 2 * PT;
  static constexpr int OFF_LD = OFF_DS + 2 * PT;  // [2][2][64] floats: lse2, D
  static constexpr int OFF_BAR = OFF_LD + 1024;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int T_S = 0, T_DP = 128, T_DV = 256, T_DK = 256 + HD;
};

template <int HD>
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dkdv_tc(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                     const __grid_constant__ CUtensorMap tm_do, const BwdParams p) {
  using C = KvCfg<HD>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bar;
  uint64_t* s_full = bar + 1;    // [2]
  uint64_t* p_full = bar + 3;    // [2]
  uint64_t* pv_done = bar + 5;   // [2]
  uint64_t* q_full = bar + 7;    // [NS]
  uint64_t* q_empty = q_full + C::NS;  // [NS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_empty + C::NS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int k0 = kb * C::BK, row0 = b * p.S;
  const int qstart = p.causal ? k0 : 0;
  const int nq = (p.S - qstart + C::BQ - 1) / C::BQ;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    mbar_init(kv_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(p_full + i, 256);
      mbar_init(pv_done + i, 1);
    }
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // dkdv reads the dq kernel's D (dsum)
  const uint32_t sb = smem_u32(smem);

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * C::KT);
      for (int a = 0; a < C::KA; ++a) {
        tma_load_2d(smem + C::OFF_K + a * C::BK * 128, &tm_kv, kv_full, p.d + h * HD + 64 * a, row0 + k0);
        tma_load_2d(smem + C::OFF_V + a * C::BK * 128, &tm_kv, kv_full, 2 * p.d + h * HD + 64 * a, row0 + k0);
      }
      for (int i = 0; i < nq; ++i) {
        const int st = i % C::NS;
        const int q1 = qstart + i * C::BQ;
        mbar_wait(q_empty + st, ((i / C::NS) & 1) ^ 1);
        mbar_arrive_expect_tx(q_full + st, 2 * C::QT);
        for (int a = 0; a < C::KA; ++a) {
          tma_load_2d(smem + C::OFF_Q + st * C::QT + a * C::BQ * 128, &tm_q, q_full + st, h * HD + 64 * a, row0 + q1);
          tma_load_2d(smem + C::OFF_DO + st * C::QT + a * C::BQ * 128, &tm_do, q_full + st, h * HD + 64 * a, row0 + q1);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = make_idesc_bf16(C::BK, C::BQ, false, false);
      constexpr uint32_t id_o = make_idesc_bf16(C::BK, HD, false, true);
      mbar_wait(kv_full, 0);
      tc_fence_after();
      auto issue_kv = [&](int ii) {
        mbar_wait(p_full + (ii & 1), (ii >> 1) & 1);
        tc_fence_after();
        const int st = ii & 1, qs = ii % C::NS;
        const uint32_t spt = sb + C::OFF_P + st * C::PT, sds = sb + C::OFF_DS + st * C::PT;
        const uint32_t sq = sb + C::OFF_Q + qs * C::QT, sdo = sb + C::OFF_DO + qs * C::QT;
#pragma unroll
        for (int k = 0; k < C::BQ / 16; ++k) {
          // dV += P^T dO ; dK += dS^T Q   (dO / Q tiles re-read MN-major: rows = queries)
          umma_bf16(tmem + C::T_DV, make_sw128_desc(spt + k * 32, 16, 1024),
                    make_sw128_desc(sdo + k * 2048, C::BQ * 128, 1024), id_o, (ii > 0 || k > 0) ? 1u : 0u);
          umma_bf16(tmem + C::T_DK, make_sw128_desc(sds + k * 32, 16, 1024),
                    make_sw128_desc(sq + k * 2048, C::BQ * 128, 1024), id_o, (ii > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit(q_empty + qs);
        umma_commit(pv_done + st);
      };
      for (int i = 0; i < nq; ++i) {
        const int st = i & 1, qs = i % C::NS;
        mbar_wait(q_full + qs, (i / C::NS) & 1);
        tc_fence_after();
        const uint32_t sq = sb + C::OFF_Q + qs * C::QT, sdo = sb + C::OFF_DO + qs * C::QT;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t ka = (k >> 2), kk = (k & 3) * 32;
          umma_bf16(tmem + C::T_S + st * 64, make_sw128_desc(sb + C::OFF_K + ka * C::BK * 128 + kk, 16, 1024),
                    make_sw128_desc(sq + ka * C::BQ * 128 + kk, 16, 1024), id_s, k > 0 ? 1u : 0u);
          umma_bf16(tmem + C::T_DP + st * 64, make_sw128_desc(sb + C::OFF_V + ka * C::BK * 128 + kk, 16, 1024),
                    make_sw128_desc(sdo + ka * C::BQ * 128 + kk, 16, 1024), id_s, k > 0 ? 1u : 0u);
        }
        umma_commit(s_full + st);
        if (i > 0) issue_kv(i - 1);
      }
      issue_kv(nq - 1);
    }
  } else if (warp >= 4) {
    // 8 warps: two per TMEM lane quadrant, each owning 32 of the 64 query columns
    const int t = threadIdx.x - 128;  // 0..255
    const int kr = (warp & 3) * 32 + lane;  // key row == TMEM lane
    const int half = (warp - 4) >> 2;
    const int key = k0 + kr;
    const float sl2 = p.sl2;
    const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const long long bh = static_cast<long long>(b) * p.H + h;
    // lse2 / D of query block i staged in sLD[i & 1] (threads 0..63: lse, 64..127: D);
    // block i+1's values are loaded into a register while block i is processed.
    // (raw values in the register; the log2(e) scale is applied at the smem store
    // so no instruction waits on the load before the block's named barrier)
    auto fetch_ld = [&](int i) -> float {
      const int qq = qstart + i * C::BQ + (t & 63);
      if (t >= 128 || i >= nq || qq >= p.S) return 0.0f;
      return t < 64 ? p.lse[bh * p.S + qq] : p.dsum[bh * p.S + qq];
    };
    const float ld_scale = t < 64 ? kLog2e : 1.0f;
    if (t < 128) sts32f(sb + C::OFF_LD + 4 * ((t >> 6) * 64 + (t & 63)), fetch_ld(0) * ld_scale);
    for (int i = 0; i < nq; ++i) {
      const int st = i & 1;
      const int q1 = qstart + i * C::BQ;
      const float ld_next = fetch_ld(i + 1);
      named_sync(1, 256);
      mbar_wait(s_full + st, (i >> 1) & 1);
      tc_fence_after();
      float s[32], dp[32];
      ld32x2(tmem + la + C::T_S + st * 64 + half * 32, tmem + la + C::T_DP + st * 64 + half * 32, s, dp);
      // this warp's 32 query columns: lse2 at +0, D at +64 floats (warp-uniform broadcasts)
      const uint32_t lda = sb + C::OFF_LD + (st * 128 + half * 32) * 4;
      // visible: query q >= key (causal), q < S, key < S
      const int qb1 = q1 + half * 32;
      int lo = 0, hi = min(32, p.S - qb1);
      if (p.causal) lo = max(0, key - qb1);
      if (key >= p.S) hi = 0;
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        const float4 l4 = lds128f(lda + 16 * c4);
        s[4 * c4 + 0] = ex2_approx(fmaf(s[4 * c4 + 0], sl2, -l4.x));
        s[4 * c4 + 1] = ex2_approx(fmaf(s[4 * c4 + 1], sl2, -l4.y));
        s[4 * c4 + 2] = ex2_approx(fmaf(s[4 * c4 + 2], sl2, -l4.z));
        s[4 * c4 + 3] = ex2_approx(fmaf(s[4 * c4 + 3], sl2, -l4.w));
      }
      if (lo > 0 || hi < 32) {  // diagonal / tail blocks only
#pragma unroll
        for (int c = 0; c < 32; ++c) s[c] = (c >= lo && c < hi) ? s[c] : 0.0f;
      }
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        const float4 d4 = lds128f(lda + 256 + 16 * c4);
        dp[4 * c4 + 0] = s[4 * c4 + 0] * (dp[4 * c4 + 0] - d4.x);
        dp[4 * c4 + 1] = s[4 * c4 + 1] * (dp[4 * c4 + 1] - d4.y);
        dp[4 * c4 + 2] = s[4 * c4 + 2] * (dp[4 * c4 + 2] - d4.z);
        dp[4 * c4 + 3] = s[4 * c4 + 3] * (dp[4 * c4 + 3] - d4.w);
      }
      if (i >= 2) mbar_wait(pv_done + st, ((i - 2) >> 1) & 1);
      store_row32(sb + C::OFF_P + st * C::PT, kr, half * 4, s);
      store_row32(sb + C::OFF_DS + st * C::PT, kr, half * 4, dp);
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(p_full + st);
      // every thread passed this iteration's named_sync, so block i-1's slot is free
      if (t < 128) sts32f(sb + C::OFF_LD + 4 * (((st ^ 1) * 2 + (t >> 6)) * 64 + (t & 63)), ld_next * ld_scale);
    }
    mbar_wait(pv_done + ((nq - 1) & 1), ((nq - 1) >> 1) & 1);
    tc_fence_after();
    // half 0 stores dK (scaled), half 1 stores dV
    __nv_bfloat16* dst_row = p.dqkv + static_cast<long long>(row0 + key) * 3 * p.d + (half == 0 ? p.d : 2 * p.d) + h * HD;
    const float sc = half == 0 ? p.scale : 1.0f;
    const uint32_t col = half == 0 ? C::T_DK : C::T_DV;
#pragma unroll
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t rr[32];
      tmem_ld_32x32b_x32(tmem + la + col + c * 32, rr);
      tmem_ld_wait();
      if (key < p.S) {
        uint32_t w[16];
#pragma unroll
        for (int i2 = 0; i2 < 16; ++i2) {
          __nv_bfloat162 hh = __floats2bfloat162_rn(__uint_as_float(rr[2 * i2]) * sc, __uint_as_float(rr[2 * i2 + 1]) * sc);
          w[i2] = *reinterpret_cast<uint32_t*>(&hh);
        }
        uint4* dst = reinterpret_cast<uint4*>(dst_row + c * 32);
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) dst[i2] = make_uint4(w[4 * i2], w[4 * i2 + 1], w[4 * i2 + 2], w[4 * i2 + 3]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ============================================================================
// Ping-pong variants (hd = 64): each CTA owns TWO 128-row tiles that share one
// TMA stream of K/V (dQ kernel) or Q/dO (dK/dV kernel) blocks. Two softmax
// groups of 4 warps (thread = one row, all 64 columns of the block, processed
// as two 32-column halves) each own one tile, so while one group turns S/dP
// into P/dS the tensor core runs the other tile's MMAs and the next block's
// S/dP — the per-block MMA <-> softmax hand-off no longer serialises the CTA.
// S/dP are single-buffered per tile in TMEM: the group releases them (s_free)
// as soon as both halves are in registers. Still deterministic (fixed order).
// ============================================================================
struct DqPP {
  static constexpr int HD = 64, BQ = 128, BKV = 64, NS = 4;
  static constexpr int QT = BQ * HD * 2;    // one Q or dO tile (16 KB)
  static constexpr int KT = BKV * HD * 2;   // one K or V block (8 KB)
  static constexpr int DST = BQ * BKV * 2;  // one dS tile (16 KB)
  static constexpr int OFF_Q = 0, OFF_DO = 2 * QT, OFF_K = 4 * QT, OFF_V = OFF_K + NS * KT;
  static constexpr int OFF_DS = OFF_V + NS * KT;   // [tile][buf]
  static constexpr int OFF_BAR = OFF_DS + 4 * DST;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int T_TILE = 192;  // TMEM per tile: S +0, dP +64, dQ +128
};

__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq_pp(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                   const __grid_constant__ CUtensorMap tm_do, const BwdParams p) {
  using C = DqPP;
#ifdef P2R_ATTN_TRACE
  __shared__ long long s_tr[512];
  const bool tr_cta = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0;
#define TRP(slot) do { if (tr_cta) s_tr[(slot)] = clock64(); } while (0)
#else
#define TRP(slot) do {} while (0)
#endif
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar;
  uint64_t* kv_full = bar + 1;            // [NS]
  uint64_t* kv_empty = kv_full + C::NS;   // [NS]
  uint64_t* s_full = kv_empty + C::NS;    // [tile]
  uint64_t* s_free = s_full + 2;          // [tile]
  uint64_t* ds_full = s_free + 2;         // [tile][buf]
  uint64_t* dq_done = ds_full + 4;        // [tile][buf]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // causal: the last query pairs see the most keys -> launch them first
  const int pq = p.causal ? gridDim.x - 1 - blockIdx.x : blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int q0 = pq * 2 * C::BQ, row0 = b * p.S;
  int nkvt[2];
#pragma unroll
  for (int X = 0; X < 2; ++X) {
    const int qs = q0 + X * C::BQ;
    const int kend = p.causal ? min(p.S, qs + C::BQ) : p.S;
    nkvt[X] = qs < p.S ? (kend + C::BKV - 1) / C::BKV : 0;
  }
  const int nkv = max(nkvt[0], nkvt[1]);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_do);
    mbar_init(q_full, 1);
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 2);  // S/dP issuer (warp 1) + dQ issuer (warp 3)
    }
    for (int X = 0; X < 2; ++X) {
      mbar_init(s_full + X, 1);
      mbar_init(s_free + X, 4);  // one arrive per warp of the group
      for (int u = 0; u < 2; ++u) {
        mbar_init(ds_full + 2 * X + u, 128);
        mbar_init(dq_done + 2 * X + u, 1);
      }
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  const uint32_t sb = smem_u32(smem);

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 4 * C::QT);
      for (int X = 0; X < 2; ++X) {
        tma_load_2d(smem + C::OFF_Q + X * C::QT, &tm_q, q_full, h * C::HD, row0 + q0 + X * C::BQ);
        tma_load_2d(smem + C::OFF_DO + X * C::QT, &tm_do, q_full, h * C::HD, row0 + q0 + X * C::BQ);
      }
      for (int j = 0; j < nkv; ++j) {
        const int st = j % C::NS;
        mbar_wait(kv_empty + st, ((j / C::NS) & 1) ^ 1);
        mbar_arrive_expect_tx(kv_full + st, 2 * C::KT);
        tma_load_2d(smem + C::OFF_K + st * C::KT, &tm_kv, kv_full + st, p.d + h * C::HD, row0 + j * C::BKV);
        tma_load_2d(smem + C::OFF_V + st * C::KT, &tm_kv, kv_full + st, 2 * p.d + h * C::HD, row0 + j * C::BKV);
      }
    }
  } else if (warp == 1) {
    {  // whole warp: uniform control flow, one elected lane issues each MMA
      constexpr uint32_t id_s = make_idesc_bf16(C::BQ, C::BKV, false, false);
      mbar_wait(q_full, 0);
      tc_fence_after();
      // base descriptors (K-major: +32 B per 16-wide k step; MN-major K: +2048 B)
      const uint64_t dQ0 = make_sw128_desc(sb + C::OFF_Q, 16, 1024), dO0 = make_sw128_desc(sb + C::OFF_DO, 16, 1024);
      const uint64_t dK0 = make_sw128_desc(sb + C::OFF_K, 16, 1024), dV0 = make_sw128_desc(sb + C::OFF_V, 16, 1024);
      auto issue_s = [&](int X, int j) {
        if (j >= 1) {
          mbar_wait(s_free + X, (j - 1) & 1);  // the group holds S/dP(j-1) in registers
          tc_fence_after();
        }
        const uint32_t st = j % C::NS;
        const uint64_t a = dadd(dQ0, X * C::QT), ao = dadd(dO0, X * C::QT);
        const uint64_t bk = dadd(dK0, st * C::KT), bv = dadd(dV0, st * C::KT);
        const uint32_t tS = tmem + X * C::T_TILE;
#pragma unroll
        for (int k = 0; k < C::HD / 16; ++k) {
          umma_bf16_warp(tS, dadd(a, k * 32), dadd(bk, k * 32), id_s, k > 0 ? 1u : 0u);
          umma_bf16_warp(tS + 64, dadd(ao, k * 32), dadd(bv, k * 32), id_s, k > 0 ? 1u : 0u);
        }
        umma_commit_warp(s_full + X);
      };

      // S/dP issuer: one K/V block after another, each as soon as the group
      // released the previous S/dP (dQ MMAs are issued by warp 3)
      for (int j = 0; j < nkv; ++j) {
        mbar_wait(kv_full + j % C::NS, (j / C::NS) & 1);
        tc_fence_after();
        TRP(16 + 4 * j);
        for (int X = 0; X < 2; ++X)
          if (j < nkvt[X]) issue_s(X, j);
        TRP(16 + 4 * j + 1);
        umma_commit_warp(kv_empty + j % C::NS);
      }
    }
  } else if (warp == 3) {
    {  // dQ issuer (whole warp, one elected lane issues)
      constexpr uint32_t id_q = make_idesc_bf16(C::BQ, C::HD, false, true);
      const uint64_t dS0 = make_sw128_desc(sb + C::OFF_DS, 16, 1024);
      const uint64_t dKm0 = make_sw128_desc(sb + C::OFF_K, C::BKV * 128, 1024);
      for (int j = 0; j < nkv; ++j) {
        for (int X = 0; X < 2; ++X) {
          if (j < nkvt[X]) {
            const int u = j & 1;
            mbar_wait(ds_full + 2 * X + u, (j >> 1) & 1);  // implies S(j) done, so K_j is in smem
            tc_fence_after();
            const uint64_t a = dadd(dS0, (2 * X + u) * C::DST), bk = dadd(dKm0, (j % C::NS) * C::KT);
            const uint32_t tQ = tmem + X * C::T_TILE + 128;
#pragma unroll
            for (int k = 0; k < C::BKV / 16; ++k)
              umma_bf16_warp(tQ, dadd(a, k * 32), dadd(bk, k * 2048), id_q, (j > 0 || k > 0) ? 1u : 0u);
            umma_commit_warp(dq_done + 2 * X + u);
          }
          TRP(16 + 4 * j + 2 + X);
        }
        umma_commit_warp(kv_empty + j % C::NS);
      }
    }
  } else if (warp >= 4) {
    const int X = (warp - 4) >> 2;           // tile owned by this softmax group
    const int r = (warp & 3) * 32 + lane;    // query row in the tile == TMEM lane
    const int q = q0 + X * C::BQ + r;
    const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + la + X * C::T_TILE, tP = tS + 64, tQ = tS + 128;
    const long long bh = static_cast<long long>(b) * p.H + h;
    const int nkvX = nkvt[X];
    // D = rowsum(dO o O) for this row (fp32 accumulate), published for the dK/dV kernel
    float D = 0.0f;
    if (q < p.S) {
      const uint4* a4 = reinterpret_cast<const uint4*>(p.dout + static_cast<long long>(row0 + q) * p.d + h * C::HD);
      const uint4* o4 = reinterpret_cast<const uint4*>(p.o + static_cast<long long>(row0 + q) * p.d + h * C::HD);
#pragma unroll
      for (int c = 0; c < C::HD / 8; ++c) {
        const uint4 x = a4[c], y = o4[c];
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 u = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[i]));
          const float2 v = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ys[i]));
          D += u.x * v.x + u.y * v.y;
        }
      }
      p.dsum[bh * p.S + q] = D;
    }
    const float lse2 = q < p.S ? p.lse[bh * p.S + q] * kLog2e : 0.0f;
    const float sl2 = p.sl2;
    const bool trw = (warp == 4 || warp == 8) && lane == 0;  // trace writers (P2R_ATTN_TRACE builds)
    const int trb = 100 + X * 100;
    (void)trw;
    (void)trb;
    for (int j = 0; j < nkvX; ++j) {
      const int u = j & 1;
      const uint32_t dsb = sb + C::OFF_DS + (2 * X + u) * C::DST;
      mbar_wait(s_full + X, j & 1);
      tc_fence_after();
      if (trw) TRP(trb + 4 * j);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float s[32], dp[32];
        ld32x2(tS + hh * 32, tP + hh * 32, s, dp);
        if (hh == 1) {  // S/dP(j) fully in registers: the MMA may overwrite them
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_free + X);
          if (trw) TRP(trb + 4 * j + 1);
        }
        const int k0 = j * C::BKV + hh * 32;
        int lim = 32;
        if (q >= p.S) lim = 0;
        else if (p.causal || k0 + 32 > p.S) lim = min(p.causal ? q + 1 : p.S, p.S) - k0;
#pragma unroll
        for (int i = 0; i < 32; ++i) s[i] = ex2_approx(fmaf(s[i], sl2, -lse2));
        if (lim < 32) {
#pragma unroll
          for (int i = 0; i < 32; ++i) s[i] = i < lim ? s[i] : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) s[i] = s[i] * (dp[i] - D);
        if (hh == 0 && j >= 2) mbar_wait(dq_done + 2 * X + u, ((j - 2) >> 1) & 1);  // dS buffer reuse
        store_row32(dsb, r, hh * 4, s);
      }
      if (trw) TRP(trb + 4 * j + 2);
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(ds_full + 2 * X + u);
      if (trw) TRP(trb + 4 * j + 3);
    }
    if (nkvX > 0) {
      mbar_wait(dq_done + 2 * X + ((nkvX - 1) & 1), ((nkvX - 1) >> 1) & 1);
      tc_fence_after();
      __nv_bfloat16* dq = p.dqkv + static_cast<long long>(row0 + q) * 3 * p.d + h * C::HD;
#pragma unroll
      for (int c = 0; c < C::HD / 32; ++c) {
        uint32_t rr[32];
        tmem_ld_32x32b_x32(tQ + c * 32, rr);
        tmem_ld_wait();
        if (q < p.S) {
          uint32_t w[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            __nv_bfloat162 hh2 = __floats2bfloat162_rn(__uint_as_float(rr[2 * i]) * p.scale,
                                                      __uint_as_float(rr[2 * i + 1]) * p.scale);
            w[i] = *reinterpret_cast<uint32_t*>(&hh2);
          }
          uint4* dst = reinterpret_cast<uint4*>(dq + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef P2R_ATTN_TRACE
  if (tr_cta)
    for (int i = threadIdx.x; i < 512; i += blockDim.x) reinterpret_cast<long long*>(const_cast<__nv_bfloat16*>(p.o))[i] = s_tr[i];
#endif
#undef TRP
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

struct KvPP {
  static constexpr int HD = 64, BK = 128, BQ = 64, NS = 4;
  static constexpr int KT = BK * HD * 2;   // one K or V tile (16 KB)
  static constexpr int QT = BQ * HD * 2;   // one Q or dO block (8 KB)
  static constexpr int PT = BK * BQ * 2;   // one P^T or dS^T tile (16 KB)
  static constexpr int OFF_K = 0, OFF_V = 2 * KT, OFF_Q = 4 * KT, OFF_DO = OFF_Q + NS * QT;
  static constexpr int OFF_P = OFF_DO + NS * QT, OFF_DS = OFF_P + 2 * PT;
  static constexpr int OFF_LD = OFF_DS + 2 * PT;  // [tile][slot][lse2 | D][64] floats
  static constexpr int OFF_BAR = OFF_LD + 2 * 2 * 2 * 64 * 4;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int T_TILE = 256;  // TMEM per tile: S^T +0, dP^T +64, dV +128, dK +192
};

__global__ void __launch_bounds__(384, 1)
    attn_bwd_dkdv_pp(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                     const __grid_constant__ CUtensorMap tm_do, const BwdParams p) {
  using C = KvPP;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bar;
  uint64_t* q_full = bar + 1;           // [NS]
  uint64_t* q_empty = q_full + C::NS;   // [NS]
  uint64_t* s_full = q_empty + C::NS;   // [tile]
  uint64_t* s_free = s_full + 2;        // [tile]
  uint64_t* p_full = s_free + 2;        // [tile]
  uint64_t* pv_done = p_full + 2;       // [tile]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pk = blockIdx.x, h = blockIdx.y, b = blockIdx.z;  // causal: low pk = most queries = first
  const int k0 = pk * 2 * C::BK, row0 = b * p.S;
  const int nq = (p.S + C::BQ - 1) / C::BQ;
  int i0t[2];  // first query block of each key tile (causal: queries >= keys)
#pragma unroll
  for (int X = 0; X < 2; ++X) {
    const int ks = k0 + X * C::BK;
    i0t[X] = ks >= p.S ? nq : (p.causal ? ks / C::BQ : 0);
  }
  const int i0 = min(i0t[0], i0t[1]);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    mbar_init(kv_full, 1);
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 2);  // S^T/dP^T issuer (warp 1) + dV/dK issuer (warp 3)
    }
    for (int X = 0; X < 2; ++X) {
      mbar_init(s_full + X, 1);
      mbar_init(s_free + X, 4);
      mbar_init(p_full + X, 128);
      mbar_init(pv_done + X, 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // reads the dq kernel's D (dsum)
  const uint32_t sb = smem_u32(smem);

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 4 * C::KT);
      for (int X = 0; X < 2; ++X) {
        tma_load_2d(smem + C::OFF_K + X * C::KT, &tm_kv, kv_full, p.d + h * C::HD, row0 + k0 + X * C::BK);
        tma_load_2d(smem + C::OFF_V + X * C::KT, &tm_kv, kv_full, 2 * p.d + h * C::HD, row0 + k0 + X * C::BK);
      }
      for (int i = i0; i < nq; ++i) {
        const int n = i - i0, st = n % C::NS;
        mbar_wait(q_empty + st, ((n / C::NS) & 1) ^ 1);
        mbar_arrive_expect_tx(q_full + st, 2 * C::QT);
        tma_load_2d(smem + C::OFF_Q + st * C::QT, &tm_q, q_full + st, h * C::HD, row0 + i * C::BQ);
        tma_load_2d(smem + C::OFF_DO + st * C::QT, &tm_do, q_full + st, h * C::HD, row0 + i * C::BQ);
      }
    }
  } else if (warp == 1) {
    {  // whole warp: uniform control flow, one elected lane issues each MMA
      constexpr uint32_t id_s = make_idesc_bf16(C::BK, C::BQ, false, false);
      mbar_wait(kv_full, 0);
      tc_fence_after();
      const uint64_t dK0 = make_sw128_desc(sb + C::OFF_K, 16, 1024), dV0 = make_sw128_desc(sb + C::OFF_V, 16, 1024);
      const uint64_t dQ0 = make_sw128_desc(sb + C::OFF_Q, 16, 1024), dO0 = make_sw128_desc(sb + C::OFF_DO, 16, 1024);
      auto issue_s = [&](int X, int i) {
        const int n = i - i0t[X];
        if (n >= 1) {
          mbar_wait(s_free + X, (n - 1) & 1);
          tc_fence_after();
        }
        const uint32_t st = (i - i0) % C::NS;
        const uint64_t ak = dadd(dK0, X * C::KT), av = dadd(dV0, X * C::KT);
        const uint64_t bq = dadd(dQ0, st * C::QT), bo = dadd(dO0, st * C::QT);
        const uint32_t tS = tmem + X * C::T_TILE;
#pragma unroll
        for (int k = 0; k < C::HD / 16; ++k) {
          umma_bf16_warp(tS, dadd(ak, k * 32), dadd(bq, k * 32), id_s, k > 0 ? 1u : 0u);
          umma_bf16_warp(tS + 64, dadd(av, k * 32), dadd(bo, k * 32), id_s, k > 0 ? 1u : 0u);
        }
        umma_commit_warp(s_full + X);
      };

      for (int i = i0; i < nq; ++i) {
        const int n = i - i0;
        mbar_wait(q_full + n % C::NS, (n / C::NS) & 1);
        tc_fence_after();
        for (int X = 0; X < 2; ++X)
          if (i >= i0t[X]) issue_s(X, i);
        umma_commit_warp(q_empty + n % C::NS);
      }
    }
  } else if (warp == 3) {
    {  // dV/dK issuer (whole warp, one elected lane issues)
      constexpr uint32_t id_o = make_idesc_bf16(C::BK, C::HD, false, true);
      const uint64_t dQm0 = make_sw128_desc(sb + C::OFF_Q, C::BQ * 128, 1024);
      const uint64_t dOm0 = make_sw128_desc(sb + C::OFF_DO, C::BQ * 128, 1024);
      const uint64_t dP0 = make_sw128_desc(sb + C::OFF_P, 16, 1024), dS0 = make_sw128_desc(sb + C::OFF_DS, 16, 1024);
      for (int i = i0; i < nq; ++i) {
        const uint32_t st = (i - i0) % C::NS;
        for (int X = 0; X < 2; ++X) {
          if (i < i0t[X]) continue;
          const int n = i - i0t[X];
          mbar_wait(p_full + X, n & 1);  // implies S^T(i) done, so Q_i / dO_i are in smem
          tc_fence_after();
          const uint64_t ap = dadd(dP0, X * C::PT), as = dadd(dS0, X * C::PT);
          const uint64_t bo = dadd(dOm0, st * C::QT), bq = dadd(dQm0, st * C::QT);
          const uint32_t tS = tmem + X * C::T_TILE;
#pragma unroll
          for (int k = 0; k < C::BQ / 16; ++k) {
            // dV += P^T dO ; dK += dS^T Q   (dO / Q blocks re-read MN-major: rows = queries)
            umma_bf16_warp(tS + 128, dadd(ap, k * 32), dadd(bo, k * 2048), id_o, (n > 0 || k > 0) ? 1u : 0u);
            umma_bf16_warp(tS + 192, dadd(as, k * 32), dadd(bq, k * 2048), id_o, (n > 0 || k > 0) ? 1u : 0u);
          }
          umma_commit_warp(pv_done + X);
        }
        umma_commit_warp(q_empty + st);
      }
    }
  } else if (warp >= 4) {
    const int X = (warp - 4) >> 2;
    const int t = threadIdx.x - 128 - X * 128;  // 0..127 within the group
    const int kr = (warp & 3) * 32 + lane;       // key row in the tile == TMEM lane
    const int key = k0 + X * C::BK + kr;
    const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + la + X * C::T_TILE, tP = tS + 64;
    const long long bh = static_cast<long long>(b) * p.H + h;
    const float sl2 = p.sl2;
    const int iX0 = i0t[X];
    const uint32_t ldb = sb + C::OFF_LD + X * (2 * 2 * 64 * 4);  // this group's [slot][lse2 | D][64]
    // lse2 / D of query block i staged in slot (i - iX0) & 1 (threads 0..63: lse, 64..127: D);
    // block i+1's values are loaded into a register while block i is processed.
    auto fetch_ld = [&](int i) -> float {
      const int qq = i * C::BQ + (t & 63);
      if (i >= nq || qq >= p.S) return 0.0f;
      return t < 64 ? p.lse[bh * p.S + qq] : p.dsum[bh * p.S + qq];
    };
    const float ld_scale = t < 64 ? kLog2e : 1.0f;
    if (iX0 < nq) sts32f(ldb + 4 * ((t >> 6) * 64 + (t & 63)), fetch_ld(iX0) * ld_scale);
    for (int i = iX0; i < nq; ++i) {
      const int n = i - iX0, slot = n & 1;
      const float ld_next = fetch_ld(i + 1);
      named_sync(1 + X, 128);
      mbar_wait(s_full + X, n & 1);
      tc_fence_after();
      const int q1 = i * C::BQ;
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        float s[32], dp[32];
        ld32x2(tS + hh * 32, tP + hh * 32, s, dp);
        if (hh == 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_free + X);
        }
        const uint32_t lda = ldb + (slot * 128 + hh * 32) * 4;
        // visible: query q >= key (causal), q < S, key < S
        const int qb1 = q1 + hh * 32;
        int lo = 0, hi = min(32, p.S - qb1);
        if (p.causal) lo = max(0, key - qb1);
        if (key >= p.S) hi = 0;
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          const float4 l4 = lds128f(lda + 16 * c4);
          s[4 * c4 + 0] = ex2_approx(fmaf(s[4 * c4 + 0], sl2, -l4.x));
          s[4 * c4 + 1] = ex2_approx(fmaf(s[4 * c4 + 1], sl2, -l4.y));
          s[4 * c4 + 2] = ex2_approx(fmaf(s[4 * c4 + 2], sl2, -l4.z));
          s[4 * c4 + 3] = ex2_approx(fmaf(s[4 * c4 + 3], sl2, -l4.w));
        }
        if (lo > 0 || hi < 32) {
#pragma unroll
          for (int c = 0; c < 32; ++c) s[c] = (c >= lo && c < hi) ? s[c] : 0.0f;
        }
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
          const float4 d4 = lds128f(lda + 256 + 16 * c4);
          dp[4 * c4 + 0] = s[4 * c4 + 0] * (dp[4 * c4 + 0] - d4.x);
          dp[4 * c4 + 1] = s[4 * c4 + 1] * (dp[4 * c4 + 1] - d4.y);
          dp[4 * c4 + 2] = s[4 * c4 + 2] * (dp[4 * c4 + 2] - d4.z);
          dp[4 * c4 + 3] = s[4 * c4 + 3] * (dp[4 * c4 + 3] - d4.w);
        }
        if (hh == 0 && n >= 1) mbar_wait(pv_done + X, (n - 1) & 1);  // P^T / dS^T buffer reuse
        store_row32(sb + C::OFF_P + X * C::PT, kr, hh * 4, s);
        store_row32(sb + C::OFF_DS + X * C::PT, kr, hh * 4, dp);
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(p_full + X);
      // every thread of the group passed this iteration's barrier: slot ^ 1 is free
      sts32f(ldb + 4 * (((slot ^ 1) * 2 + (t >> 6)) * 64 + (t & 63)), ld_next * ld_scale);
    }
    const int nX = nq - iX0;
    if (nX > 0) {
      mbar_wait(pv_done + X, (nX - 1) & 1);
      tc_fence_after();
      // dK (scaled) then dV for this key row
#pragma unroll
      for (int which = 0; which < 2; ++which) {
        __nv_bfloat16* dst_row =
            p.dqkv + static_cast<long long>(row0 + key) * 3 * p.d + (which == 0 ? p.d : 2 * p.d) + h * C::HD;
        const float sc = which == 0 ? p.scale : 1.0f;
        const uint32_t col = which == 0 ? 192 : 128;
#pragma unroll
        for (int c = 0; c < C::HD / 32; ++c) {
          uint32_t rr[32];
          tmem_ld_32x32b_x32(tS + col + c * 32, rr);
          tmem_ld_wait();
          if (key < p.S) {
            uint32_t w[16];
#pragma unroll
            for (int i2 = 0; i2 < 16; ++i2) {
              __nv_bfloat162 hh2 = __floats2bfloat162_rn(__uint_as_float(rr[2 * i2]) * sc,
                                                        __uint_as_float(rr[2 * i2 + 1]) * sc);
              w[i2] = *reinterpret_cast<uint32_t*>(&hh2);
            }
            uint4* dst = reinterpret_cast<uint4*>(dst_row + c * 32);
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2) dst[i2] = make_uint4(w[4 * i2], w[4 * i2 + 1], w[4 * i2 + 2], w[4 * i2 + 3]);
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

bool map2d(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int HD>
p2r_status run(const void* qkv, const BwdParams& p, cudaStream_t s) {
  const uint64_t T = static_cast<uint64_t>(p.B) * p.S;
  CUtensorMap qkv128, qkv64, do128, do64;
  if (!map2d(&qkv128, qkv, T, 3ull * p.d, 128) || !map2d(&qkv64, qkv, T, 3ull * p.d, 64) ||
      !map2d(&do128, p.dout, T, p.d, 128) || !map2d(&do64, p.dout, T, p.d, 64))
    return set_error(P2R_ECUDA, "attention bwd: tensor map encode failed");
  static cudaError_t a1 = cudaFuncSetAttribute(attn_bwd_dq_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, DqCfg<HD>::SMEM);
  static cudaError_t a2 = cudaFuncSetAttribute(attn_bwd_dkdv_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, KvCfg<HD>::SMEM);
  if (a1 != cudaSuccess || a2 != cudaSuccess) return set_cuda_error(a1 ? a1 : a2, "attention bwd attr");
  static const bool v1 = std::getenv("P2R_ATTN_BWD_V1") != nullptr;
  if (HD == 64 && !v1) {  // ping-pong kernels: two 128-row tiles per CTA
    static cudaError_t a3 = cudaFuncSetAttribute(attn_bwd_dq_pp, cudaFuncAttributeMaxDynamicSharedMemorySize, DqPP::SMEM);
    static cudaError_t a4 =
        cudaFuncSetAttribute(attn_bwd_dkdv_pp, cudaFuncAttributeMaxDynamicSharedMemorySize, KvPP::SMEM);
    if (a3 != cudaSuccess || a4 != cudaSuccess) return set_cuda_error(a3 ? a3 : a4, "attention bwd attr");
    const dim3 grid2((p.S + 255) / 256, p.H, p.B);
    P2R_LAUNCH_K("attention bwd dq (tcgen05, 2 tiles)", attn_bwd_dq_pp, grid2, dim3(384), DqPP::SMEM, s, 1, qkv128,
                 qkv64, do128, p);
    P2R_LAUNCH_K("attention bwd dkdv (tcgen05, 2 tiles)", attn_bwd_dkdv_pp, grid2, dim3(384), KvPP::SMEM, s, 1,
                 qkv128, qkv64, do64, p);
    return P2R_OK;
  }
  const dim3 grid((p.S + 127) / 128, p.H, p.B);
  P2R_LAUNCH_K("attention bwd dq (tcgen05)", attn_bwd_dq_tc<HD>, grid, dim3(384), DqCfg<HD>::SMEM, s, 1, qkv128,
               qkv64, do128, p);
  P2R_LAUNCH_K("attention bwd dkdv (tcgen05)", attn_bwd_dkdv_tc<HD>, grid, dim3(384), KvCfg<HD>::SMEM, s, 1, qkv128,
               qkv64, do64, p);
  return P2R_OK;
}

}  // namespace attn_bwd_tc

p2r_status attention_bwd_tc(const void* qkv, const void* o, const float* lse, const void* dout, float* dsum,
                            void* dqkv, int B, int H, int S, int d, int causal, cudaStream_t s) {
  attn_bwd_tc::BwdParams p{};
  p.o = static_cast<const __nv_bfloat16*>(o);
  p.dout = static_cast<const __nv_bfloat16*>(dout);
  p.lse = lse;
  p.dsum = dsum;
  p.dqkv = static_cast<__nv_bfloat16*>(dqkv);
  p.B = B;
  p.H = H;
  p.S = S;
  p.d = d;
  p.causal = causal;
  const int hd = d / H;
  p.scale = 1.0f / sqrtf(static_cast<float>(hd));
  p.sl2 = p.scale * attn_bwd_tc::kLog2e;
  if (hd == 64) return attn_bwd_tc::run<64>(qkv, p, s);
  if (hd == 128) return attn_bwd_tc::run<128>(qkv, p, s);
  return set_error(P2R_EINVAL, "attention: head_dim must be 64 or 128");
}

}  // namespace p2r
