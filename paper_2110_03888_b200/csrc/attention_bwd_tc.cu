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

// 16 registers -> 32 lanes x 16 consecutive 32-bit TMEM columns
P2R_DEVICE void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
// D (+)= A.B with A (M rows = TMEM lanes, K packed bf16 pairs along columns) read from TMEM
P2R_DEVICE void umma_bf16_ta_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                  uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
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
// S/dP are single-buffered per tile in TMEM, and the group writes its bf16 dS
// (dQ kernel) / P^T and dS^T (dK/dV kernel) back over the first 32 columns of
// those blocks (tcgen05.st), where the dQ / dV / dK MMAs read them as their A
// operand straight from TMEM: no smem round trip; the next block's S/dP MMA
// waits for those MMAs. Still deterministic (fixed order).
// ============================================================================
// Exponentials of the recomputed P moved from the SFU (16 ex2 / clk / SM, the
// softmax groups' bound) to the FMA pipe: this many of every 16 pairs of a 32-key
// half row (dQ) or 32-query half row (dK/dV) use exp2_fma2.
#ifndef P2R_BWD_FMA_PAIRS
#define P2R_BWD_FMA_PAIRS 5
#endif
constexpr int kBwdFmaPairs = P2R_BWD_FMA_PAIRS;

#ifndef P2R_BWD_NS
#define P2R_BWD_NS 4
#endif
// (dS and P^T / dS^T live in TMEM as MMA A operands: no smem tiles for them)
struct DqPP {
  static constexpr int HD = 64, BQ = 128, BKV = 64, NS = P2R_BWD_NS;
  static constexpr int QT = BQ * HD * 2;    // one Q or dO tile (16 KB)
  static constexpr int KT = BKV * HD * 2;   // one K or V block (8 KB)
  static constexpr int OFF_Q = 0, OFF_DO = 2 * QT, OFF_K = 4 * QT, OFF_V = OFF_K + NS * KT;
  static constexpr int OFF_BAR = OFF_V + NS * KT;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int T_TILE = 192;  // TMEM per tile: S +0, dP +64, dQ(item parity 0) +128
  static constexpr int T_DQ1 = 384;   // dQ(item parity 1) of tile X at T_DQ1 + 64 X
};

// Persistent over (query-tile pair, head, batch) work items, heaviest causal
// pairs first: every pipeline counter runs across items, the dQ accumulator is
// double-buffered by item parity, an item's dQ epilogue is deferred until the
// next item's first block is handed to the MMA, and the next item's D / LSE
// rows are fetched while the tensor core starts on it.
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dq_pp(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kv,
                   const __grid_constant__ CUtensorMap tm_do, const BwdParams p) {
  using C = DqPP;
#ifdef P2R_ATTN_TRACE
  __shared__ long long s_tr[512];
  const bool tr_cta = blockIdx.x == 0;
#define TRP(slot) do { if (tr_cta && (slot) < 512) s_tr[(slot)] = clock64(); } while (0)
#else
#define TRP(slot) do {} while (0)
#endif
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar;
  uint64_t* q_empty = bar + 1;
  uint64_t* kv_full = bar + 2;            // [NS]
  uint64_t* kv_empty = kv_full + C::NS;   // [NS]
  uint64_t* s_full = kv_empty + C::NS;    // [tile]
  uint64_t* ds_full = s_full + 2;         // [tile][buf]
  uint64_t* dq_done = ds_full + 4;        // [tile][buf]
  uint64_t* dq_empty = dq_done + 4;       // [tile][item parity]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_empty + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npq = (p.S + 2 * C::BQ - 1) / (2 * C::BQ);
  const int n_items = npq * p.H * p.B;
  struct Item {
    int h, b, q0, nkvt[2], nkv;
  };
  auto item = [&](int w) {
    Item I;
    const int hb = p.H * p.B, g = w / hb, rem = w - g * hb;
    const int pq = p.causal ? npq - 1 - g : g;  // causal: the last query pairs see the most keys
    I.h = rem % p.H;
    I.b = rem / p.H;
    I.q0 = pq * 2 * C::BQ;
#pragma unroll
    for (int X = 0; X < 2; ++X) {
      const int qs = I.q0 + X * C::BQ;
      const int kend = p.causal ? min(p.S, qs + C::BQ) : p.S;
      I.nkvt[X] = qs < p.S ? (kend + C::BKV - 1) / C::BKV : 0;
    }
    I.nkv = max(I.nkvt[0], I.nkvt[1]);
    return I;
  };
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_do);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 2);  // S/dP issuer (warp 1) + dQ issuer (warp 3)
    }
    for (int X = 0; X < 2; ++X) {
      mbar_init(s_full + X, 1);
      for (int u = 0; u < 2; ++u) {
        mbar_init(ds_full + 2 * X + u, 128);
        mbar_init(dq_done + 2 * X + u, 1);
        mbar_init(dq_empty + 2 * X + u, 128);
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
      int G = 0, it = 0;
      for (int k = 0, w = blockIdx.x; w < n_items; w = snake_item(++k, blockIdx.x, gridDim.x), ++it) {
        const Item I = item(w);
        const int row0 = I.b * p.S;
        mbar_wait(q_empty, (it & 1) ^ 1);  // the previous item's S/dP MMAs are done with Q / dO
        mbar_arrive_expect_tx(q_full, 4 * C::QT);
        for (int X = 0; X < 2; ++X) {
          tma_load_2d(smem + C::OFF_Q + X * C::QT, &tm_q, q_full, I.h * C::HD, row0 + I.q0 + X * C::BQ);
          tma_load_2d(smem + C::OFF_DO + X * C::QT, &tm_do, q_full, I.h * C::HD, row0 + I.q0 + X * C::BQ);
        }
        for (int j = 0; j < I.nkv; ++j, ++G) {
          const int st = G % C::NS;
          mbar_wait(kv_empty + st, ((G / C::NS) & 1) ^ 1);
          mbar_arrive_expect_tx(kv_full + st, 2 * C::KT);
          tma_load_2d(smem + C::OFF_K + st * C::KT, &tm_kv, kv_full + st, p.d + I.h * C::HD, row0 + j * C::BKV);
          tma_load_2d(smem + C::OFF_V + st * C::KT, &tm_kv, kv_full + st, 2 * p.d + I.h * C::HD, row0 + j * C::BKV);
        }
      }
    }
  } else if (warp == 1) {
    {  // whole warp: uniform control flow, one elected lane issues each MMA
      constexpr uint32_t id_s = make_idesc_bf16(C::BQ, C::BKV, false, false);
      // base descriptors (K-major: +32 B per 16-wide k step; MN-major K: +2048 B)
      const uint64_t dQ0 = make_sw128_desc(sb + C::OFF_Q, 16, 1024), dO0 = make_sw128_desc(sb + C::OFF_DO, 16, 1024);
      const uint64_t dK0 = make_sw128_desc(sb + C::OFF_K, 16, 1024), dV0 = make_sw128_desc(sb + C::OFF_V, 16, 1024);
      int G = 0, it = 0, cX[2] = {0, 0};
      for (int k = 0, w = blockIdx.x; w < n_items; w = snake_item(++k, blockIdx.x, gridDim.x), ++it) {
        const Item I = item(w);
        mbar_wait(q_full, it & 1);
        tc_fence_after();
        // S/dP issuer: one K/V block after another, each as soon as the group
        // released the previous S/dP (dQ MMAs are issued by warp 3)
        for (int j = 0; j < I.nkv; ++j, ++G) {
          const uint32_t st = G % C::NS;
          mbar_wait(kv_full + st, (G / C::NS) & 1);
          tc_fence_after();
          TRP(16 + 4 * G);
          for (int X = 0; X < 2; ++X) {
            if (j >= I.nkvt[X]) continue;
            if (cX[X] >= 1) {  // dS(j-1) sits in this tile's S columns until the dQ MMA read it
              const int c = cX[X] - 1;
              mbar_wait(dq_done + 2 * X + (c & 1), (c >> 1) & 1);
              tc_fence_after();
            }
            const uint64_t a = dadd(dQ0, X * C::QT), ao = dadd(dO0, X * C::QT);
            const uint64_t bk = dadd(dK0, st * C::KT), bv = dadd(dV0, st * C::KT);
            const uint32_t tS = tmem + X * C::T_TILE;
#pragma unroll
            for (int k = 0; k < C::HD / 16; ++k) {
              umma_bf16_warp(tS, dadd(a, k * 32), dadd(bk, k * 32), id_s, k > 0 ? 1u : 0u);
              umma_bf16_warp(tS + 64, dadd(ao, k * 32), dadd(bv, k * 32), id_s, k > 0 ? 1u : 0u);
            }
            umma_commit_warp(s_full + X);
            ++cX[X];
          }
          TRP(16 + 4 * G + 1);
          if (j == I.nkv - 1) umma_commit_warp(q_empty);  // this item's Q / dO are no longer read
          umma_commit_warp(kv_empty + st);
        }
      }
    }
  } else if (warp == 3) {
    {  // dQ issuer (whole warp, one elected lane issues)
      constexpr uint32_t id_q = make_idesc_bf16(C::BQ, C::HD, false, true);
      const uint64_t dKm0 = make_sw128_desc(sb + C::OFF_K, C::BKV * 128, 1024);
      int G = 0, it = 0, cX[2] = {0, 0};
      for (int k = 0, w = blockIdx.x; w < n_items; w = snake_item(++k, blockIdx.x, gridDim.x), ++it) {
        const Item I = item(w);
        const int par = it & 1;
        for (int j = 0; j < I.nkv; ++j, ++G) {
          for (int X = 0; X < 2; ++X) {
            if (j < I.nkvt[X]) {
              const int u = cX[X] & 1;
              mbar_wait(ds_full + 2 * X + u, (cX[X] >> 1) & 1);  // implies S(j) done, so K_j is in smem
              tc_fence_after();
              if (j == 0) {  // this dQ buffer was last drained by the group for item it - 2
                mbar_wait(dq_empty + 2 * X + par, ((it >> 1) & 1) ^ 1);
                tc_fence_after();
              }
              const uint64_t bk = dadd(dKm0, (G % C::NS) * C::KT);
              const uint32_t tQ = tmem + (par ? C::T_DQ1 + 64 * X : X * C::T_TILE + 128);
              const uint32_t tA = tmem + X * C::T_TILE;  // dS: bf16 pairs over the S block's first 32 columns
#pragma unroll
              for (int k = 0; k < C::BKV / 16; ++k)
                umma_bf16_ta_warp(tQ, tA + k * 8, dadd(bk, k * 2048), id_q, (j > 0 || k > 0) ? 1u : 0u);
              umma_commit_warp(dq_done + 2 * X + u);
              ++cX[X];
            }
            TRP(16 + 4 * G + 2 + X);
          }
          umma_commit_warp(kv_empty + G % C::NS);
        }
      }
    }
  } else if (warp >= 4) {
    const int X = (warp - 4) >> 2;           // tile owned by this softmax group
    const int r = (warp & 3) * 32 + lane;    // query row in the tile == TMEM lane
    const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + la + X * C::T_TILE, tP = tS + 64;
    const float sl2 = p.sl2;
    const bool trw = (warp == 4 || warp == 8) && lane == 0;  // trace writers (P2R_ATTN_TRACE builds)
    const int trb = 100 + X * 200;
    (void)trw;
    (void)trb;
    // D = rowsum(dO o O) of this row (fp32 accumulate), published for the dK/dV kernel, + its LSE
    auto row_stats = [&](const Item& I, float& D, float& lse2) {
      const int q = I.q0 + X * C::BQ + r;
      D = 0.0f;
      lse2 = 0.0f;
      if (q >= p.S) return;
      const long long bh = static_cast<long long>(I.b) * p.H + I.h;
      const long long off = static_cast<long long>(I.b * p.S + q) * p.d + I.h * C::HD;
      const uint4* a4 = reinterpret_cast<const uint4*>(p.dout + off);
      const uint4* o4 = reinterpret_cast<const uint4*>(p.o + off);
      lse2 = p.lse[bh * p.S + q] * kLog2e;
#pragma unroll
      for (int c = 0; c < C::HD / 8; ++c) {
        const uint4 x = a4[c], y = o4[c];
        const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 u2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[i]));
          const float2 v2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ys[i]));
          D += u2.x * v2.x + u2.y * v2.y;
        }
      }
      p.dsum[bh * p.S + q] = D;
    };
    struct Pend {
      bool valid;
      int par, c_last, q, h, b;
    } pend{};
    auto epilogue = [&](const Pend& e) {
      mbar_wait(dq_done + 2 * X + (e.c_last & 1), (e.c_last >> 1) & 1);
      tc_fence_after();
      const uint32_t tQ = tmem + la + (e.par ? C::T_DQ1 + 64 * X : X * C::T_TILE + 128);
      uint32_t rr[C::HD];
#pragma unroll
      for (int c = 0; c < C::HD / 32; ++c) tmem_ld_32x32b_x32(tQ + c * 32, rr + 32 * c);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(dq_empty + 2 * X + e.par);
      if (e.q < p.S) {
        __nv_bfloat16* dq = p.dqkv + static_cast<long long>(e.b * p.S + e.q) * 3 * p.d + e.h * C::HD;
#pragma unroll
        for (int c = 0; c < C::HD / 32; ++c) {
          uint32_t wv[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            __nv_bfloat162 hh2 = __floats2bfloat162_rn(__uint_as_float(rr[32 * c + 2 * i]) * p.scale,
                                                      __uint_as_float(rr[32 * c + 2 * i + 1]) * p.scale);
            wv[i] = *reinterpret_cast<uint32_t*>(&hh2);
          }
          uint4* dst = reinterpret_cast<uint4*>(dq + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_uint4(wv[4 * i], wv[4 * i + 1], wv[4 * i + 2], wv[4 * i + 3]);
        }
      }
    };
    int it = 0, cX = 0;
    float D = 0.0f, lse2 = 0.0f;
    if (static_cast<int>(blockIdx.x) < n_items) row_stats(item(blockIdx.x), D, lse2);
    for (int k = 0, w = blockIdx.x; w < n_items; w = snake_item(++k, blockIdx.x, gridDim.x), ++it) {
      const Item I = item(w);
      const int q = I.q0 + X * C::BQ + r;
      const int nkvX = I.nkvt[X];
      for (int j = 0; j < nkvX; ++j, ++cX) {
        const int u = cX & 1;
        mbar_wait(s_full + X, cX & 1);
        tc_fence_after();
        if (trw) TRP(trb + 4 * cX);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float s[32], dp[32];
          ld32x2(tS + hh * 32, tP + hh * 32, s, dp);
          if (hh == 1 && trw) TRP(trb + 4 * cX + 1);
          const int k0 = j * C::BKV + hh * 32;
          int lim = 32;
          if (q >= p.S) lim = 0;
          else if (p.causal || k0 + 32 > p.S) lim = min(p.causal ? q + 1 : p.S, p.S) - k0;
          {  // FP32x2: s * scale - lse, then P * (dP - D) (same per-element rounding as the scalar form)
            const float2 sl2p = make_float2(sl2, sl2), nl = make_float2(-lse2, -lse2);
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float2 z = __ffma2_rn(make_float2(s[i], s[i + 1]), sl2p, nl);
              if (i / 2 >= 16 - kBwdFmaPairs) {
                const float2 e = exp2_fma2(z);
                s[i] = e.x;
                s[i + 1] = e.y;
              } else {
                s[i] = ex2_approx(z.x);
                s[i + 1] = ex2_approx(z.y);
              }
            }
          }
          if (lim < 32) {
#pragma unroll
            for (int i = 0; i < 32; ++i) s[i] = i < lim ? s[i] : 0.0f;
          }
          {
            const float2 nD = make_float2(-D, -D);
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
              const float2 v = __fmul2_rn(make_float2(s[i], s[i + 1]), __fadd2_rn(make_float2(dp[i], dp[i + 1]), nD));
              s[i] = v.x;
              s[i + 1] = v.y;
            }
          }
          // dS of these 32 keys -> bf16 pairs over columns [16 hh, 16 hh + 16) of this tile's
          // S block (the dQ MMA's A operand; the other half's columns are not touched)
          uint32_t wv[16];
#pragma unroll
          for (int i2 = 0; i2 < 16; ++i2) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(s[2 * i2], s[2 * i2 + 1]);
            wv[i2] = *reinterpret_cast<uint32_t*>(&h2);
          }
          tmem_st_32x32b_x16(tS + hh * 16, wv);
        }
        if (trw) TRP(trb + 4 * cX + 2);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(ds_full + 2 * X + u);
        if (trw) TRP(trb + 4 * cX + 3);
        if (j == 0 && pend.valid) {  // the previous item's dQ epilogue, off the critical path
          epilogue(pend);
          pend.valid = false;
        }
      }
      if (nkvX > 0) pend = Pend{true, it & 1, cX - 1, q, I.h, I.b};
      // the next item's row statistics (global loads overlap its Q / dO TMA)
      if (const int wn = snake_item(k + 1, blockIdx.x, gridDim.x); wn < n_items) row_stats(item(wn), D, lse2);
    }
    if (pend.valid) epilogue(pend);
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
  static constexpr int HD = 64, BK = 128, BQ = 64, NS = P2R_BWD_NS;
  static constexpr int KT = BK * HD * 2;   // one K or V tile (16 KB)
  static constexpr int QT = BQ * HD * 2;   // one Q or dO block (8 KB)
  static constexpr int OFF_K = 0, OFF_V = 2 * KT, OFF_Q = 4 * KT, OFF_DO = OFF_Q + NS * QT;
  static constexpr int OFF_LD = OFF_DO + NS * QT;  // [tile][slot][lse2 | D][64] floats
  static constexpr int OFF_BAR = OFF_LD + 2 * 2 * 2 * 64 * 4;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
  static constexpr int T_TILE = 256;  // TMEM per tile: S^T +0, dP^T +64, dV +128, dK +192
};

// Persistent over (key-tile pair, head, batch) work items (causal: the first
// key pairs see the most queries -> first). The dV/dK accumulators fill TMEM,
// so an item's first dV/dK MMA waits (acc_empty) for the previous item's
// epilogue, which the group runs right after handing over the next item's
// first block; the staged LSE/D slots run on a per-tile global block parity.
__global__ void __launch_bounds__(384, 1)
    attn_bwd_dkdv_pp(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                     const __grid_constant__ CUtensorMap tm_do, const BwdParams p) {
  using C = KvPP;
#ifdef P2R_ATTN_TRACE
  // diagnostic build only: CTA 0's timeline, dumped after the dq kernel's (o + 4 KB)
  __shared__ long long s_tr[512];
  const bool tr_cta = blockIdx.x == 0;
#define TRK(slot) do { if (tr_cta && (slot) < 512) s_tr[(slot)] = clock64(); } while (0)
#else
#define TRK(slot) do {} while (0)
#endif
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* kv_full = bar;
  uint64_t* kv_empty = bar + 1;
  uint64_t* q_full = bar + 2;           // [NS]
  uint64_t* q_empty = q_full + C::NS;   // [NS]
  uint64_t* s_full = q_empty + C::NS;   // [tile]
  uint64_t* p_full = s_full + 2;        // [tile]
  uint64_t* pv_done = p_full + 2;       // [tile]
  uint64_t* acc_empty = pv_done + 2;    // [tile]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = (p.S + C::BQ - 1) / C::BQ;
  const int npk = (p.S + 2 * C::BK - 1) / (2 * C::BK);
  const int n_items = npk * p.H * p.B;
  struct Item {
    int h, b, k0, i0t[2], i0;
  };
  auto item = [&](int w) {
    Item I;
    const int hb = p.H * p.B, pk = w / hb, rem = w - pk * hb;
    I.h = rem % p.H;
    I.b = rem / p.H;
    I.k0 = pk * 2 * C::BK;
#pragma unroll
    for (int X = 0; X < 2; ++X) {  // first query block of each key tile (causal: queries >= keys)
      const int ks = I.k0 + X * C::BK;
      I.i0t[X] = ks >= p.S ? nq : (p.causal ? ks / C::BQ : 0);
    }
    I.i0 = min(I.i0t[0], I.i0t[1]);
    return I;
  };
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_kv);
    tma_prefetch_desc(&tm_q);
    tma_prefetch_desc(&tm_do);
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 2);  // S^T/dP^T issuer (warp 1) + dV/dK issuer (warp 3)
    }
    for (int X = 0; X < 2; ++X) {
      mbar_init(s_full + X, 1);
      mbar_init(p_full + X, 128);
      mbar_init(pv_done + X, 1);
      mbar_init(acc_empty + X, 128);
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
      int G = 0, it = 0;
      for (int k = 0, w = blockIdx.x; w < n_items; w = snake_item(++k, blockIdx.x, gridDim.x), ++it) {
        const Item I = item(w);
        const int row0 = I.b * p.S;
        mbar_wait(kv_empty, (it & 1) ^ 1);  // the previous item's S^T/dP^T MMAs are done with K / V
        mbar_arrive_expect_tx(kv_full, 4 * C::KT);
        for (int X = 0; X < 2; ++X) {
          tma_load_2d(smem + C::OFF_K + X * C::KT, &tm_kv, kv_full, p.d + I.h * C::HD, row0 + I.k0 + X * C::BK);
          tma_load_2d(smem + C::OFF_V + X * C::KT, &tm_kv, kv_full, 2 * p.d + I.h * C::HD, row0 + I.k0 + X * C::BK);
        }
        for (int i = I.i0; i < nq; ++i, ++G) {
          const int st = G % C::NS;
          mbar_wait(q_empty + st, ((G / C::NS) & 1) ^ 1);
          mbar_arrive_expect_tx(q_full + st, 2 * C::QT);
          tma_load_2d(smem + C::OFF_Q + st * C::QT, &tm_q, q_full + st, I.h * C::HD, row0 + i * C::BQ);
          tma_load_2d(smem + C::OFF_DO + st * C::QT, &tm_do, q_full + st, I.h * C::HD, row0 + i * C::BQ);
        }
      }
    }
  } else if (warp == 1) {
    {  // whole warp: uniform control flow, one elected lane issues each MMA
      constexpr uint32_t id_s = make_idesc_bf16(C::BK, C::BQ, false, false);
      const uint64_t dK0 = make_sw128_desc(sb + C::OFF_K, 16, 1024), dV0 = make_sw128_desc(sb + C::OFF_V, 16, 1024);
      const uint64_t dQ0 = make_sw128_desc(sb + C::OFF_Q, 16, 1024), dO0 = make_sw128_desc(sb + C::OFF_DO, 16, 1024);
      int G = 0, it = 0, cX[2] = {0, 0};
      for (int k = 0, w = blockIdx.x; w < n_items; w = snake_item(++k, blockIdx.x, gridDim.x), ++it) {
        const Item I = item(w);
        mbar_wait(kv_full, it & 1);
        tc_fence_after();
        for (int i = I.i0; i < nq; ++i, ++G) {
          const uint32_t st = G % C::NS;
          mbar_wait(q_full + st, (G / C::NS) & 1);
          tc_fence_after();
          if (lane == 0 && G < 24) TRK(16 + 4 * G);
          for (int X = 0; X < 2; ++X) {
            if (i < I.i0t[X]) continue;
            if (cX[X] >= 1) {  // P^T / dS^T(i-1) sit in this tile's S^T / dP^T columns until dV/dK(i-1) read them
              mbar_wait(pv_done + X, (cX[X] - 1) & 1);
              tc_fence_after();
            }
            if (lane == 0 && G < 24) TRK(16 + 4 * G + 1 + X);
            const uint64_t ak = dadd(dK0, X * C::KT), av = dadd(dV0, X * C::KT);
            const uint64_t bq = dadd(dQ0, st * C::QT), bo = dadd(dO0, st * C::QT);
            const uint32_t tS = tmem + X * C::T_TILE;
#pragma unroll
            for (int k = 0; k < C::HD / 16; ++k) {
              umma_bf16_warp(tS, dadd(ak, k * 32), dadd(bq, k * 32), id_s, k > 0 ? 1u : 0u);
              umma_bf16_warp(tS + 64, dadd(av, k * 32), dadd(bo, k * 32), id_s, k > 0 ? 1u : 0u);
            }
            umma_commit_warp(s_full + X);
            ++cX[X];
          }
          if (i == nq - 1) umma_commit_warp(kv_empty);  // this item's K / V are no longer read
          umma_commit_warp(q_empty + st);
        }
      }
    }
  } else if (warp == 3) {
    {  // dV/dK issuer (whole warp, one elected lane issues)
      constexpr uint32_t id_o = make_idesc_bf16(C::BK, C::HD, false, true);
      const uint64_t dQm0 = make_sw128_desc(sb + C::OFF_Q, C::BQ * 128, 1024);
      const uint64_t dOm0 = make_sw128_desc(sb + C::OFF_DO, C::BQ * 128, 1024);
      int G = 0, it = 0, cX[2] = {0, 0};
      for (int k = 0, w = blockIdx.x; w < n_items; w = snake_item(++k, blockIdx.x, gridDim.x), ++it) {
        const Item I = item(w);
        for (int i = I.i0; i < nq; ++i, ++G) {
          const uint32_t st = G % C::NS;
          for (int X = 0; X < 2; ++X) {
            if (i < I.i0t[X]) continue;
            const int n = i - I.i0t[X];
            mbar_wait(p_full + X, cX[X] & 1);  // implies S^T(i) done, so Q_i / dO_i are in smem
            tc_fence_after();
            if (n == 0) {  // the previous item's dV/dK of this tile were drained by its epilogue
              mbar_wait(acc_empty + X, (it & 1) ^ 1);
              tc_fence_after();
            }
            const uint64_t bo = dadd(dOm0, st * C::QT), bq = dadd(dQm0, st * C::QT);
            const uint32_t tS = tmem + X * C::T_TILE;
#pragma unroll
            for (int k = 0; k < C::BQ / 16; ++k) {
              // dV += P^T dO ; dK += dS^T Q with A = P^T / dS^T from TMEM (bf16 pairs packed over
              // the first 32 columns of the S^T / dP^T blocks: 16 queries = 8 columns per MMA);
              // dO / Q blocks re-read MN-major from smem (rows = queries)
              umma_bf16_ta_warp(tS + 128, tS + k * 8, dadd(bo, k * 2048), id_o, (n > 0 || k > 0) ? 1u : 0u);
              umma_bf16_ta_warp(tS + 192, tS + 64 + k * 8, dadd(bq, k * 2048), id_o, (n > 0 || k > 0) ? 1u : 0u);
            }
            umma_commit_warp(pv_done + X);
            if (lane == 0 && cX[X] < 48) TRK(120 + 48 * X + cX[X]);
            ++cX[X];
          }
          umma_commit_warp(q_empty + st);
        }
      }
    }
  } else if (warp >= 4) {
    const int X = (warp - 4) >> 2;
    const int t = threadIdx.x - 128 - X * 128;  // 0..127 within the group
    const int kr = (warp & 3) * 32 + lane;       // key row in the tile == TMEM lane
    const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + la + X * C::T_TILE, tP = tS + 64;
    const float sl2 = p.sl2;
    const uint32_t ldb = sb + C::OFF_LD + X * (2 * 2 * 64 * 4);  // this group's [slot][lse2 | D][64]
    // lse2 / D of a query block staged in slot (tile block count) & 1 (threads 0..63: lse, 64..127: D);
    // the next block's values are loaded into a register while the current one is processed
    // (raw: consuming the load here would put its DRAM latency on every block).
    auto fetch_ld = [&](const Item& I, int i) -> float {
      const int qq = i * C::BQ + (t & 63);
      if (i >= nq || qq >= p.S) return 0.0f;
      const long long bh = static_cast<long long>(I.b) * p.H + I.h;
      return t < 64 ? p.lse[bh * p.S + qq] : p.dsum[bh * p.S + qq];
    };
    const float ld_scale = t < 64 ? -kLog2e : -1.0f;  // staged negated: -lse*log2e | -D (FP32x2 adds)
    struct Pend {
      bool valid;
      int c_last, key, h, b;
    } pend{};
    auto epilogue = [&](const Pend& e) {
      mbar_wait(pv_done + X, e.c_last & 1);
      tc_fence_after();
      uint32_t rr[2 * C::HD];  // dV | dK columns of this key row
#pragma unroll
      for (int c = 0; c < 2 * C::HD / 32; ++c) tmem_ld_32x32b_x32(tS + 128 + c * 32, rr + 32 * c);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(acc_empty + X);
      if (e.key < p.S) {
#pragma unroll
        for (int which = 0; which < 2; ++which) {  // dK (scaled) then dV
          __nv_bfloat16* dst_row =
              p.dqkv + static_cast<long long>(e.b * p.S + e.key) * 3 * p.d + (which == 0 ? p.d : 2 * p.d) + e.h * C::HD;
          const float sc = which == 0 ? p.scale : 1.0f;
          const int base = which == 0 ? C::HD : 0;
#pragma unroll
          for (int c = 0; c < C::HD / 32; ++c) {
            uint32_t wv[16];
#pragma unroll
            for (int i2 = 0; i2 < 16; ++i2) {
              __nv_bfloat162 hh2 = __floats2bfloat162_rn(__uint_as_float(rr[base + 32 * c + 2 * i2]) * sc,
                                                        __uint_as_float(rr[base + 32 * c + 2 * i2 + 1]) * sc);
              wv[i2] = *reinterpret_cast<uint32_t*>(&hh2);
            }
            uint4* dst = reinterpret_cast<uint4*>(dst_row + c * 32);
#pragma unroll
            for (int i2 = 0; i2 < 4; ++i2) dst[i2] = make_uint4(wv[4 * i2], wv[4 * i2 + 1], wv[4 * i2 + 2], wv[4 * i2 + 3]);
          }
        }
      }
    };
    int cX = 0;
    if (static_cast<int>(blockIdx.x) < n_items) {
      const Item I0 = item(blockIdx.x);
      if (I0.i0t[X] < nq) sts32f(ldb + 4 * ((t >> 6) * 64 + (t & 63)), fetch_ld(I0, I0.i0t[X]) * ld_scale);
    }
    for (int k = 0, w = blockIdx.x; w < n_items; w = snake_item(++k, blockIdx.x, gridDim.x)) {
      const Item I = item(w);
      const int key = I.k0 + X * C::BK + kr;
      const int iX0 = I.i0t[X];
      const int wn = snake_item(k + 1, blockIdx.x, gridDim.x);
      const bool has_next = wn < n_items;
      Item In{};
      if (has_next) In = item(wn);
      for (int i = iX0; i < nq; ++i, ++cX) {
        const int n = i - iX0, slot = cX & 1;
        // the value staged for this tile's next block: the next query block, or the next item's first
        const float ld_next = i + 1 < nq ? fetch_ld(I, i + 1) : (has_next && In.i0t[X] < nq ? fetch_ld(In, In.i0t[X]) : 0.0f);
        named_sync(1 + X, 128);
        mbar_wait(s_full + X, cX & 1);
        tc_fence_after();
        const bool trw = (warp == 4 || warp == 8) && lane == 0 && cX < 48;
        if (trw) TRK(240 + 128 * X + 2 * cX);
        const int q1 = i * C::BQ;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          float s[32], dp[32];
          ld32x2(tS + hh * 32, tP + hh * 32, s, dp);
          const uint32_t lda = ldb + (slot * 128 + hh * 32) * 4;
          // visible: query q >= key (causal), q < S, key < S
          const int qb1 = q1 + hh * 32;
          int lo = 0, hi = min(32, p.S - qb1);
          if (p.causal) lo = max(0, key - qb1);
          if (key >= p.S) hi = 0;
          const float2 sl2p = make_float2(sl2, sl2);
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {  // FP32x2 (same per-element rounding as the scalar form)
            const float4 l4 = lds128f(lda + 16 * c4);
            const float2 z0 = __ffma2_rn(make_float2(s[4 * c4 + 0], s[4 * c4 + 1]), sl2p, make_float2(l4.x, l4.y));
            const float2 z1 = __ffma2_rn(make_float2(s[4 * c4 + 2], s[4 * c4 + 3]), sl2p, make_float2(l4.z, l4.w));
            if (2 * c4 >= 16 - kBwdFmaPairs) {
              const float2 e0 = exp2_fma2(z0);
              s[4 * c4 + 0] = e0.x;
              s[4 * c4 + 1] = e0.y;
            } else {
              s[4 * c4 + 0] = ex2_approx(z0.x);
              s[4 * c4 + 1] = ex2_approx(z0.y);
            }
            if (2 * c4 + 1 >= 16 - kBwdFmaPairs) {
              const float2 e1 = exp2_fma2(z1);
              s[4 * c4 + 2] = e1.x;
              s[4 * c4 + 3] = e1.y;
            } else {
              s[4 * c4 + 2] = ex2_approx(z1.x);
              s[4 * c4 + 3] = ex2_approx(z1.y);
            }
          }
          if (lo > 0 || hi < 32) {
#pragma unroll
            for (int c = 0; c < 32; ++c) s[c] = (c >= lo && c < hi) ? s[c] : 0.0f;
          }
#pragma unroll
          for (int c4 = 0; c4 < 8; ++c4) {
            const float4 d4 = lds128f(lda + 256 + 16 * c4);
            const float2 v0 = __fmul2_rn(make_float2(s[4 * c4 + 0], s[4 * c4 + 1]),
                                         __fadd2_rn(make_float2(dp[4 * c4 + 0], dp[4 * c4 + 1]), make_float2(d4.x, d4.y)));
            const float2 v1 = __fmul2_rn(make_float2(s[4 * c4 + 2], s[4 * c4 + 3]),
                                         __fadd2_rn(make_float2(dp[4 * c4 + 2], dp[4 * c4 + 3]), make_float2(d4.z, d4.w)));
            dp[4 * c4 + 0] = v0.x;
            dp[4 * c4 + 1] = v0.y;
            dp[4 * c4 + 2] = v1.x;
            dp[4 * c4 + 3] = v1.y;
          }
          // P^T / dS^T of these 32 queries -> bf16 pairs over columns [16 hh, 16 hh + 16) of the
          // S^T / dP^T blocks (already in registers; the other half's columns are not touched)
          uint32_t wp[16], wd[16];
#pragma unroll
          for (int i2 = 0; i2 < 16; ++i2) {
            __nv_bfloat162 a2 = __floats2bfloat162_rn(s[2 * i2], s[2 * i2 + 1]);
            __nv_bfloat162 b2 = __floats2bfloat162_rn(dp[2 * i2], dp[2 * i2 + 1]);
            wp[i2] = *reinterpret_cast<uint32_t*>(&a2);
            wd[i2] = *reinterpret_cast<uint32_t*>(&b2);
          }
          tmem_st_32x32b_x16(tS + hh * 16, wp);
          tmem_st_32x32b_x16(tP + hh * 16, wd);
        }
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full + X);
        if (trw) TRK(240 + 128 * X + 2 * cX + 1);
        // every thread of the group passed this iteration's barrier: slot ^ 1 is free
        sts32f(ldb + 4 * (((slot ^ 1) * 2 + (t >> 6)) * 64 + (t & 63)), ld_next * ld_scale);
        if (n == 0 && pend.valid) {  // the previous item's dK/dV epilogue, off the critical path
          epilogue(pend);
          pend.valid = false;
        }
      }
      if (nq - iX0 > 0) pend = Pend{true, cX - 1, key, I.h, I.b};
    }
    if (pend.valid) epilogue(pend);
  }
  tc_fence_before();
  __syncthreads();
#ifdef P2R_ATTN_TRACE
  if (threadIdx.x == 0) TRK(0);
  if (tr_cta)
    for (int i = threadIdx.x; i < 512; i += blockDim.x)
      reinterpret_cast<long long*>(const_cast<__nv_bfloat16*>(p.o))[512 + i] = s_tr[i];
#endif
#undef TRK
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
#ifdef P2R_DIAG  // diagnostic build: P2R_ATTN_BWD_V1=1 runs the one-tile kernels at hd 64 too
  static const bool v1 = std::getenv("P2R_ATTN_BWD_V1") != nullptr;
#else
  constexpr bool v1 = false;
#endif
  if (HD == 64 && !v1) {  // ping-pong kernels: two 128-row tiles per CTA
    static cudaError_t a3 = cudaFuncSetAttribute(attn_bwd_dq_pp, cudaFuncAttributeMaxDynamicSharedMemorySize, DqPP::SMEM);
    static cudaError_t a4 =
        cudaFuncSetAttribute(attn_bwd_dkdv_pp, cudaFuncAttributeMaxDynamicSharedMemorySize, KvPP::SMEM);
    if (a3 != cudaSuccess || a4 != cudaSuccess) return set_cuda_error(a3 ? a3 : a4, "attention bwd attr");
    const int n_dq = (p.S + 255) / 256 * p.H * p.B;
    P2R_LAUNCH_K("attention bwd dq (tcgen05, 2 tiles, persistent)", attn_bwd_dq_pp,
                 dim3(n_dq < kNumSMs ? n_dq : kNumSMs), dim3(384), DqPP::SMEM, s, 1, qkv128, qkv64, do128, p);
    P2R_LAUNCH_K("attention bwd dkdv (tcgen05, 2 tiles, persistent)", attn_bwd_dkdv_pp,
                 dim3(n_dq < kNumSMs ? n_dq : kNumSMs), dim3(384), KvPP::SMEM, s, 1, qkv128, qkv64, do64, p);
    return P2R_OK;
  }
#ifndef P2R_DIAG
  if constexpr (HD == 64) return P2R_OK;  // (unreachable: hd 64 always runs the ping-pong kernels)
#endif
  static cudaError_t a1 = cudaFuncSetAttribute(attn_bwd_dq_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, DqCfg<HD>::SMEM);
  static cudaError_t a2 = cudaFuncSetAttribute(attn_bwd_dkdv_tc<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, KvCfg<HD>::SMEM);
  if (a1 != cudaSuccess || a2 != cudaSuccess) return set_cuda_error(a1 ? a1 : a2, "attention bwd attr");
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
