// Flash-attention FORWARD on 5th-gen tensor cores (tcgen05 + TMEM + TMA).
//
// Replaces masked_attention's forward (tensor.cpp:464-506) + split/merge_heads
// (tensor.cpp:400-462): Q, K, V are read by TMA straight from the fused QKV
// projection [T, 3d]; O is written merged-head [T, d]; the row log-sum-exp is
// saved for the backward instead of the S x S probability matrix.
//
// Persistent: one CTA per SM walks (query tile, head, batch) work items,
// heaviest causal tiles first, round-robin over CTAs; every pipeline counter
// runs across items, so the next item's Q/K/V loads, S MMAs and PVs overlap
// the current item's tail (O is double-buffered in TMEM). 12 warps:
//   warp 0     TMA producer: Q per item (double-buffered for hd 64), K/V tiles
//              (128 keys) through an NKV-stage ring
//   warp 1     MMA issuer (whole warp, elected lane): S_g = Q.K_g^T into a
//              double-buffered TMEM S tile, then O += P_{g-1}.V_{g-1}
//   warp 2     TMEM allocator (S0 | S1 | O0 | O1 columns)
//   warps 4-11 softmax: two warps per TMEM lane quadrant (query row), each
//              owning half the keys of a block: causal mask, online softmax
//              with CONDITIONAL rescaling of O (only when the running max grows
//              by > 2^8), bf16 P written back over the S block in TMEM (the PV
//              MMA's A operand); per item, normalise O and store O / LSE.
#include <cudaTypedefs.h>

#include <mutex>

#include "../../include/p2r_cuda.h"
#include "common.cuh"
#include "p2r_internal.h"

namespace p2r {
namespace attn_tc {

#ifndef P2R_FWD_NKV64
#define P2R_FWD_NKV64 3
#endif
#ifndef P2R_FWD_NKV128
#define P2R_FWD_NKV128 2
#endif
// O (+)= P.V with P (bf16 pairs packed along TMEM columns, rows = lanes) read from TMEM
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

constexpr int BQ = 128, BKV = 128;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kRescaleThresh = 8.0f;  // log2 units: P stays <= 256 in bf16
#ifndef P2R_ATTN_FMA_CHUNKS
#define P2R_ATTN_FMA_CHUNKS 2
#endif
// of each half-row's 8 eight-key chunks, this many take exp2 on the FMA pipe
constexpr int kFmaChunks = P2R_ATTN_FMA_CHUNKS;

template <int HD>
struct Cfg {
  static constexpr int KATOMS = HD / 64;                 // 128-B K atoms per row
  static constexpr int TILE = BQ * HD * 2;               // Q / K / V tile bytes
  // P never touches smem: the softmax writes it (bf16 pairs) over its S block in TMEM,
  // where the PV MMA reads it as the A operand
  // K/V ring depth: with 2 stages the load of block j+2 waits for PV(j) and its
  // latency lands on every block (trace: ~1.9k vs ~1.4k softmax cycles/block)
  static constexpr int NKV = HD == 64 ? P2R_FWD_NKV64 : P2R_FWD_NKV128;
  static constexpr int NQ = HD == 64 ? 2 : 1;  // Q buffers (the next item's Q loads early)
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + NQ * TILE;
  static constexpr int OFF_V = OFF_K + NKV * TILE;
  static constexpr int OFF_BAR = OFF_V + NKV * TILE;
  static constexpr int XCH = (2 * 2 + 2) * 128 * 4;   // row-max exchange [2][2][128] + sums [2][128]
  static constexpr int SMEM = OFF_BAR + 256 + XCH + 1024;
  static constexpr int TMEM_S0 = 0, TMEM_S1 = 128, TMEM_O = 256;  // O buffer ob at TMEM_O + ob * HD
};

struct FwdParams {
  __nv_bfloat16* o;
  float* lse;
  int B, H, S, d;
  int causal;
  float sl2;  // softmax scale * log2(e)
};

// 2^x on the FMA pipe (FA4-style MUFU offload, exp2_fma2 in common.cuh): x = n + f with
// n = round(x) via the 1.5*2^23 magic add, 2^f by a degree-3 fit on [-1/2, 1/2] (max rel.
// error 1.4e-4, far below P's bf16 rounding), the exponent added with integer ops; pair
// form on the FP32x2 pipe (FFMA2/FADD2): the softmax is issue-bound.
P2R_DEVICE float max3f(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
P2R_DEVICE void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// 2^x on the SFU (inputs here are <= 8, outputs feed a bf16 MMA operand)
P2R_DEVICE float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int HD>
__global__ void __launch_bounds__(384, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const FwdParams p) {
  using C = Cfg<HD>;
#ifdef P2R_ATTN_TRACE
  // diagnostic build only: clock64 timeline of CTA 0's first blocks dumped over the start of `lse`
  __shared__ long long s_tr[256];
  const bool tr_cta = blockIdx.x == 0;
#define TRF(slot) do { if (tr_cta) s_tr[(slot)] = clock64(); } while (0)
#else
#define TRF(slot) do {} while (0)
#endif
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bar + 0;    // [NQ <= 2]
  uint64_t* q_empty = bar + 2;   // [NQ]
  uint64_t* kv_full = bar + 4;   // [NKV <= 4]
  uint64_t* kv_empty = bar + 8;  // [NKV]
  uint64_t* s_full = bar + 12;   // [2]
  uint64_t* p_full = bar + 14;   // [2]
  uint64_t* o_done = bar + 16;   // [2] one commit per PV
  uint64_t* o_empty = bar + 18;  // [2] O buffer drained by the softmax warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 20);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nqb = (p.S + BQ - 1) / BQ;
  const int n_items = nqb * p.H * p.B;
  // item w: heaviest (last) causal query tiles first
  auto item = [&](int w, int& qb, int& h, int& b) {
    const int hb = p.H * p.B;
    qb = nqb - 1 - w / hb;
    const int rem = w - (w / hb) * hb;
    h = rem % p.H;
    b = rem / p.H;
  };
  auto nkv_of = [&](int qb) { return p.causal ? min(qb + 1, nqb) : nqb; };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    for (int i = 0; i < C::NQ; ++i) {
      mbar_init(q_full + i, 1);
      mbar_init(q_empty + i, 1);
    }
    for (int i = 0; i < C::NKV; ++i) {
      mbar_init(kv_full + i, 1);
      mbar_init(kv_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(s_full + i, 1);
      mbar_init(p_full + i, 256);  // 8 softmax warps
      mbar_init(o_done + i, 1);
      mbar_init(o_empty + i, 256);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TRF(0);
  pdl_trigger();
  pdl_wait();
  const uint32_t sbase = smem_u32(smem);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int g = 0, it = 0;
      for (int k = 0, w = blockIdx.x; w < n_items; w = snake_item(++k, blockIdx.x, gridDim.x), ++it) {
        int qb, h, b;
        item(w, qb, h, b);
        const int row0 = b * p.S, nkv = nkv_of(qb);
        const int qs = it % C::NQ;
        mbar_wait(q_empty + qs, ((it / C::NQ) & 1) ^ 1);
        mbar_arrive_expect_tx(q_full + qs, C::TILE);
        for (int a = 0; a < C::KATOMS; ++a)
          tma_load_2d(smem + C::OFF_Q + qs * C::TILE + a * BQ * 128, &tm_qkv, q_full + qs, h * HD + 64 * a,
                      row0 + qb * BQ);
        for (int j = 0; j < nkv; ++j, ++g) {
          const int st = g % C::NKV;
          mbar_wait(kv_empty + st, ((g / C::NKV) & 1) ^ 1);
          mbar_arrive_expect_tx(kv_full + st, 2 * C::TILE);
          for (int a = 0; a < C::KATOMS; ++a) {
            tma_load_2d(smem + C::OFF_K + st * C::TILE + a * BKV * 128, &tm_qkv, kv_full + st,
                        p.d + h * HD + 64 * a, row0 + j * BKV);
            tma_load_2d(smem + C::OFF_V + st * C::TILE + a * BKV * 128, &tm_qkv, kv_full + st,
                        2 * p.d + h * HD + 64 * a, row0 + j * BKV);
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // ---------------- MMA issuer (whole warp, one elected lane issues) ----------------
      constexpr uint32_t idesc_s = make_idesc_bf16(BQ, BKV, false, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(BQ, HD, false, true);
      // precomputed base descriptors, advanced by byte offsets (desc_add)
      const uint64_t dQ0 = make_sw128_desc(sbase + C::OFF_Q, 16, 1024);
      const uint64_t dK0 = make_sw128_desc(sbase + C::OFF_K, 16, 1024);
      const uint64_t dV0 = make_sw128_desc(sbase + C::OFF_V, BKV * 128, 1024);
      // PV of global block gg (block jj of item iit): O[iit & 1] (+)= P_gg . V_gg
      auto issue_pv = [&](int gg, int jj, int iit) {
        const int ob = iit & 1;
        if (jj == 0) {  // first PV of an item: its O buffer must have been drained (item iit - 2)
          mbar_wait(o_empty + ob, ((iit >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        mbar_wait(p_full + (gg & 1), (gg >> 1) & 1);
        tc_fence_after();
        if (lane == 0 && gg < 22) TRF(8 + 4 * gg + 2);
        const uint32_t st = gg % C::NKV;
        const uint64_t bv = desc_add(dV0, st * C::TILE);
        const uint32_t tp = tmem + ((gg & 1) ? C::TMEM_S1 : C::TMEM_S0);  // P_gg over S_gg's first 64 columns
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k)
          // A = P from TMEM (16 keys = 8 columns per MMA), B = V (MN-major: rows = keys, 64 hd per 128-B row).
          // S_{gg+2} reuses this TMEM block: it is issued after this PV, and the tensor pipe runs in order
          umma_bf16_ta_warp(tmem + C::TMEM_O + ob * HD, tp + k * 8, desc_add(bv, k * 2048), idesc_o,
                            (jj > 0 || k > 0) ? 1u : 0u);
        umma_commit_warp(kv_empty + st);
        umma_commit_warp(o_done + (gg & 1));
        if (lane == 0 && gg < 22) TRF(8 + 4 * gg + 3);
      };
      int g = 0, it = 0;
      int pg = -1, pj = 0, pit = 0;  // the PV still to issue
      for (int k = 0, w = blockIdx.x; w < n_items; w = snake_item(++k, blockIdx.x, gridDim.x), ++it) {
        int qb, h, b;
        item(w, qb, h, b);
        const int nkv = nkv_of(qb);
        const int qs = it % C::NQ;
        mbar_wait(q_full + qs, (it / C::NQ) & 1);
        tc_fence_after();
        const uint64_t dQ = desc_add(dQ0, qs * C::TILE);
        for (int j = 0; j < nkv; ++j, ++g) {
          const uint32_t st = g % C::NKV;
          mbar_wait(kv_full + st, (g / C::NKV) & 1);
          tc_fence_after();
          if (lane == 0 && g < 22) TRF(8 + 4 * g);
          const uint64_t bk = desc_add(dK0, st * C::TILE);
          const uint32_t dS = tmem + ((g & 1) ? C::TMEM_S1 : C::TMEM_S0);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k)
            umma_bf16_warp(dS, desc_add(dQ, (k >> 2) * (BQ * 128) + (k & 3) * 32),
                           desc_add(bk, (k >> 2) * (BKV * 128) + (k & 3) * 32), idesc_s, k > 0 ? 1u : 0u);
          umma_commit_warp(s_full + (g & 1));
          if (j == nkv - 1) umma_commit_warp(q_empty + qs);  // this item's Q is no longer read
          if (lane == 0 && g < 22) TRF(8 + 4 * g + 1);
          if (pg >= 0) issue_pv(pg, pj, pit);
          pg = g;
          pj = j;
          pit = it;
        }
      }
      if (pg >= 0) issue_pv(pg, pj, pit);
    }
  } else if (warp >= 4) {
    // ---------------- softmax / correction / epilogue ----------------
    // 8 warps: two per TMEM lane quadrant; warp half `hf` owns key columns
    // [64 hf, 64 hf + 64) of each block and O columns [HD/2 hf, HD/2 (hf + 1)).
    // The two halves of a row exchange their partial maxima through shared
    // memory (double-buffered by block parity) behind a 64-thread named barrier.
    const int qd = warp & 3, hf = (warp - 4) >> 2;
    const int r = qd * 32 + lane;  // query row within the tile == TMEM lane
    const uint32_t lane_addr = static_cast<uint32_t>(qd * 32) << 16;
    constexpr int KH = BKV / 2, OH = HD / 2;
    // [parity][half][row] partial maxima, then [half][row] partial sums (after the barriers area)
    const uint32_t xch = smem_u32(smem) + C::OFF_BAR + 256;
    const bool trw = warp == 4 && lane == 0;
    (void)trw;
    // An item's epilogue (wait for its last PV, normalise O, store O / LSE) is
    // deferred until the next item's first block is handed to the MMA: the
    // softmax warps would otherwise idle on the last PV while S of the next
    // item is already waiting. O is double-buffered, so the deferred O survives.
    struct Pend {
      bool valid;
      float l, m;
      int ob, g_last, b, h, q;
    } pend{};
    auto epilogue = [&](const Pend& e) {
      mbar_wait(o_done + (e.g_last & 1), (e.g_last >> 1) & 1);
      tc_fence_after();
      const float inv = e.l > 0.0f ? 1.0f / e.l : 0.0f;
      const bool row_ok = e.q < p.S;
      const uint32_t tO = tmem + lane_addr + C::TMEM_O + e.ob * HD + hf * OH;
      uint32_t rr[OH];
#pragma unroll
      for (int c = 0; c < OH / 32; ++c) tmem_ld_32x32b_x32(tO + c * 32, rr + 32 * c);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(o_empty + e.ob);  // O buffer ob is free for item it + 2
      if (row_ok) {
        __nv_bfloat16* orow = p.o + static_cast<long long>(e.b * p.S + e.q) * p.d + e.h * HD + hf * OH;
#pragma unroll
        for (int c = 0; c < OH / 32; ++c) {
          uint32_t wv[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            __nv_bfloat162 hh = __floats2bfloat162_rn(__uint_as_float(rr[32 * c + 2 * i]) * inv,
                                                      __uint_as_float(rr[32 * c + 2 * i + 1]) * inv);
            wv[i] = *reinterpret_cast<uint32_t*>(&hh);
          }
          uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_uint4(wv[4 * i], wv[4 * i + 1], wv[4 * i + 2], wv[4 * i + 3]);
        }
#ifndef P2R_ATTN_TRACE  // trace builds dump the timeline over lse instead
        if (hf == 0) p.lse[(static_cast<long long>(e.b) * p.H + e.h) * p.S + e.q] = (e.m + log2f(e.l)) * 0.6931471805599453f;
#endif
      }
    };
    int g = 0, it = 0;
    for (int k = 0, w = blockIdx.x; w < n_items; w = snake_item(++k, blockIdx.x, gridDim.x), ++it) {
      int qb, h, b;
      item(w, qb, h, b);
      const int nkv = nkv_of(qb), q0 = qb * BQ;
      const int q = q0 + r;
      const int ob = it & 1;
      const uint32_t tO = tmem + lane_addr + C::TMEM_O + ob * HD + hf * OH;
      float m_used = -INFINITY, l = 0.0f;
      for (int j = 0; j < nkv; ++j, ++g) {
        mbar_wait(s_full + (g & 1), (g >> 1) & 1);
        tc_fence_after();
        if (trw && g < 22) TRF(100 + 4 * g);
        const uint32_t tS = tmem + lane_addr + ((g & 1) ? C::TMEM_S1 : C::TMEM_S0) + hf * KH;
        float x[KH];
        {
          uint32_t ra[32], rb[32];
          tmem_ld_32x32b_x32(tS, ra);
          tmem_ld_32x32b_x32(tS + 32, rb);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            x[i] = __uint_as_float(ra[i]);
            x[32 + i] = __uint_as_float(rb[i]);
          }
        }
        const int k0 = j * BKV + hf * KH;
        const bool diag = p.causal && (j * BKV + BKV > q0);
        const bool tail = j * BKV + BKV > p.S;
        if (diag || tail) {  // warp-uniform: only the diagonal / ragged-tail blocks mask
          const int lim = min(diag ? q + 1 : p.S, p.S) - k0;  // keys [0, lim) of this half are visible
#pragma unroll
          for (int i = 0; i < KH; ++i)
            if (i >= lim) x[i] = -INFINITY;
        }
        // max on raw scores (scale > 0), combined with the other half of the row
        float mr0 = max3f(x[0], x[1], x[2]), mr1 = max3f(x[3], x[4], x[5]);
#pragma unroll
        for (int i = 6; i + 3 < KH; i += 4) {
          mr0 = max3f(mr0, x[i], x[i + 1]);
          mr1 = max3f(mr1, x[i + 2], x[i + 3]);
        }
        mr0 = max3f(mr0, x[KH - 2], x[KH - 1]);
        const uint32_t slot = xch + 4 * (((g & 1) * 2) * 128 + r);
        sts32f(slot + 4 * 128 * hf, fmaxf(mr0, mr1));
        if (trw && g < 22) TRF(100 + 4 * g + 1);
        named_sync(1 + qd, 64);
        float other;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(other) : "r"(slot + 4 * 128 * (hf ^ 1)) : "memory");
        const float mx = fmaxf(fmaxf(mr0, mr1), other) * p.sl2;
        // Lazy rescale. Both halves of a row take the same decision, but rows (lanes)
        // differ, and the TMEM load / store below are warp-collective (.sync.aligned):
        // the warp enters the branch together when any of its rows needs it, and rows
        // that do not keep their max (factor 1). A lane-divergent branch here hung the
        // kernel once scores grew during training.
        const bool need = mx > m_used + kRescaleThresh;
        if (__any_sync(0xffffffffu, need)) {
          if (j > 0) {
            // O holds sum_{<j} 2^(x - m_used) V: rescale this half's O columns to the new max
            mbar_wait(o_done + ((g - 1) & 1), ((g - 1) >> 1) & 1);
            tc_fence_after();
            const float f = need ? exp2f(m_used - mx) : 1.0f;
#pragma unroll
            for (int c = 0; c < OH / 32; ++c) {
              uint32_t rr[32];
              tmem_ld_32x32b_x32(tO + c * 32, rr);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) rr[i] = __float_as_uint(__uint_as_float(rr[i]) * f);
              tmem_st_32x32b_x32(tO + c * 32, rr);
            }
            tmem_st_wait();
            if (need) l *= f;
          }
          if (need) m_used = mx;
        }
        // P_g goes over S_g's TMEM block (its 64 keys -> 32 packed columns at 32 hf); both halves
        // of the row finished reading S_g before the max exchange above, and S_g's completion
        // implies PV_{g-2} (the previous reader of this block) completed: the pipe runs in order
        const uint32_t tPw = tmem + lane_addr + ((g & 1) ? C::TMEM_S1 : C::TMEM_S0) + 32 * hf;
        uint32_t pw[32];
        float2 ls = make_float2(0.0f, 0.0f);
        const float2 sl2 = make_float2(p.sl2, p.sl2), nm = make_float2(-m_used, -m_used);
#pragma unroll
        for (int c16 = 0; c16 < KH / 8; ++c16) {
          uint32_t wv[4];
          // the softmax is MUFU-bound (16 ex2/clk/SM): a quarter of the exponentials go to the FMA pipe
          const bool fma_pipe = c16 >= KH / 8 - kFmaChunks;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 z = __ffma2_rn(make_float2(x[c16 * 8 + 2 * i], x[c16 * 8 + 2 * i + 1]), sl2, nm);
            const float2 e = fma_pipe ? exp2_fma2(z) : make_float2(ex2_approx(z.x), ex2_approx(z.y));
            ls = __fadd2_rn(ls, e);
            __nv_bfloat162 hh = __floats2bfloat162_rn(e.x, e.y);
            wv[i] = *reinterpret_cast<uint32_t*>(&hh);
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) pw[4 * c16 + i] = wv[i];
        }
        tmem_st_32x32b_x32(tPw, pw);
        l += ls.x + ls.y;
        if (trw && g < 22) TRF(100 + 4 * g + 2);
        tmem_st_wait();
        tc_fence_before();
        mbar_arrive(p_full + (g & 1));
        if (trw && g < 22) TRF(100 + 4 * g + 3);
        if (j == 0 && pend.valid) {  // the previous item's epilogue, off the critical path
          epilogue(pend);
          pend.valid = false;
        }
      }
      // row sum = both halves' partial sums
      const uint32_t lslot = xch + 4 * (4 * 128 + r);
      sts32f(lslot + 4 * 128 * hf, l);
      named_sync(1 + qd, 64);
      float lo;
      asm volatile("ld.shared.f32 %0, [%1];" : "=f"(lo) : "r"(lslot + 4 * 128 * (hf ^ 1)) : "memory");
      l += lo;
      pend = Pend{true, l, m_used, ob, g - 1, b, h, q};
    }
    if (pend.valid) epilogue(pend);
  }
  tc_fence_before();
  __syncthreads();
#ifdef P2R_ATTN_TRACE
  if (threadIdx.x == 0) TRF(1);
  if (tr_cta)
    for (int i = threadIdx.x; i < 256; i += blockDim.x) reinterpret_cast<long long*>(p.lse)[i] = s_tr[i];
#endif
#undef TRF
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

template <int HD>
p2r_status run(const void* qkv, const FwdParams& p, cudaStream_t s) {
  using C = Cfg<HD>;
  auto fn = encode_fn();
  if (!fn) return set_error(P2R_ECUDA, "attention: cuTensorMapEncodeTiled unavailable");
  CUtensorMap tm;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(3) * p.d, static_cast<cuuint64_t>(p.B) * p.S};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(3) * p.d * 2};
  const cuuint32_t box[2] = {64, 128};
  const cuuint32_t es[2] = {1, 1};
  if (fn(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qkv), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return set_error(P2R_ECUDA, "attention: tensor map encode failed");
  static cudaError_t attr = cudaFuncSetAttribute(attn_fwd_tc_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (attr != cudaSuccess) return set_cuda_error(attr, "attention tc attr");
  const int n_items = (p.S + BQ - 1) / BQ * p.H * p.B;
  const dim3 grid(n_items < kNumSMs ? n_items : kNumSMs);  // persistent: one CTA per SM
  P2R_LAUNCH_K("attention fwd (tcgen05)", attn_fwd_tc_kernel<HD>, grid, dim3(384), C::SMEM, s, 1, tm, p);
  return P2R_OK;
}

}  // namespace attn_tc

// Used by p2r_attention_fwd (attention.cu) when the shape qualifies.
p2r_status attention_fwd_tc(const void* qkv, void* o, float* lse, int B, int H, int S, int d, int causal,
                            cudaStream_t s) {
  attn_tc::FwdParams p{};
  p.o = static_cast<__nv_bfloat16*>(o);
  p.lse = lse;
  p.B = B;
  p.H = H;
  p.S = S;
  p.d = d;
  p.causal = causal;
  const int hd = d / H;
  p.sl2 = (1.0f / sqrtf(static_cast<float>(hd))) * attn_tc::kLog2e;
  if (hd == 64) return attn_tc::run<64>(qkv, p, s);
  if (hd == 128) return attn_tc::run<128>(qkv, p, s);
  return set_error(P2R_EINVAL, "attention: head_dim must be 64 or 128");
}

}  // namespace p2r
