// Fused causal/full softmax attention, forward and backward (flash style).
//
// Replaces masked_attention (tensor.cpp:464-545) together with split_heads /
// merge_heads (tensor.cpp:400-462): Q, K, V are read straight from the fused
// QKV projection output [T, 3d] (head h at columns h*hd, d+h*hd, 2d+h*hd) and
// O is written merged-head [T, d], so the permutations disappear. The S x S
// probability matrix the reference keeps for backward (tensor.cpp:472-474) is
// never materialised: forward saves the row log-sum-exp, backward recomputes P.
// Scale 1/sqrt(hd) is applied to Q.K^T exactly where the reference applies it
// (tensor.cpp:483). Backward is deterministic (no float atomics): one kernel
// produces dQ (+ the rowsum(dO*O) term), a second produces dK/dV.
//
// The kernels are tcgen05/TMEM (attention_tc.cu, attention_bwd_tc.cu); this file
// holds the C-ABI entry points. The round-1 bf16 mma.sync.m16n8k16 kernels below
// are compiled only into the diagnostic build (-DP2R_DIAG, build/libp2r_diag.so,
// P2R_ATTN_MMA_SYNC=1) for A/B measurements; the product library does not carry them.
#include <cstdlib>

#include "../../include/p2r_cuda.h"
#include "common.cuh"
#include "p2r_internal.h"

#ifdef P2R_DIAG
namespace p2r {
namespace attn {

constexpr float kLog2e = 1.4426950408889634f;

P2R_DEVICE void mma16816(float* c, const uint32_t* a, const uint32_t* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}
P2R_DEVICE void ldsm_x4(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
P2R_DEVICE void ldsm_x4_t(uint32_t* r, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
P2R_DEVICE uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
P2R_DEVICE void cp_async16(uint32_t dst, const void* src, bool pred) {
  const int n = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n));
}
P2R_DEVICE void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
P2R_DEVICE void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

// Row-major [rows x HD] bf16 tile in smem; 16-byte chunks XOR-swizzled by row
// so ldmatrix (8 rows x 16 B) is conflict-free.
template <int HD>
P2R_DEVICE uint32_t tile_off(int row, int chunk) {
  constexpr int CH = HD / 8;  // 16-byte chunks per row
  return static_cast<uint32_t>((row * CH + (chunk ^ (row & 7))) * 16);
}

// Async-load `rows` rows of a head slice (row stride ld elements) into a tile.
template <int HD, int ROWS, int NTHREADS>
P2R_DEVICE void load_tile(uint32_t smem_base, const __nv_bfloat16* g, long long ld, int valid_rows) {
  constexpr int CH = HD / 8;
  for (int i = threadIdx.x; i < ROWS * CH; i += NTHREADS) {
    const int r = i / CH, c = i % CH;
    const bool ok = r < valid_rows;
    const __nv_bfloat16* src = g + (ok ? r : 0) * ld + c * 8;
    cp_async16(smem_base + tile_off<HD>(r, c), src, ok);
  }
}

// A-operand fragments (16 rows x HD) of a row-major smem tile starting at row r0.
template <int HD>
P2R_DEVICE void load_a_frags(uint32_t (*a)[4], uint32_t base, int r0, int lane) {
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    const int row = r0 + (lane & 15);
    const int chunk = kk * 2 + (lane >> 4);
    ldsm_x4(a[kk], base + tile_off<HD>(row, chunk));
  }
}

// acc[16 x 8*NT] += A(16 x HD, regs) * B where B[k=hd][n=row of tile] (tile rows n0..)
template <int HD, int NT>
P2R_DEVICE void mma_a_tileT(float (*acc)[4], const uint32_t (*a)[4], uint32_t tile, int n0, int lane) {
#pragma unroll
  for (int nt = 0; nt < NT; nt += 2) {
#pragma unroll
    for (int kk = 0; kk < HD / 16; ++kk) {
      // x4: matrices (n-tile nt, k lo), (nt, k hi), (nt+1, k lo), (nt+1, k hi)
      const int mi = lane >> 3;
      const int row = n0 + nt * 8 + ((mi >> 1) << 3) + (lane & 7);
      const int chunk = kk * 2 + (mi & 1);
      uint32_t b[4];
      ldsm_x4(b, tile + tile_off<HD>(row, chunk));
      mma16816(acc[nt], a[kk], b);
      mma16816(acc[nt + 1], a[kk], b + 2);
    }
  }
}

// acc[16 x HD] += P(16 x 8*KT keys, as bf16 A frags from C layout) * tile[keys][hd]
template <int HD, int KT>
P2R_DEVICE void mma_p_tile(float (*acc)[4], const float (*p)[4], uint32_t tile, int k0, int lane) {
#pragma unroll
  for (int kk = 0; kk < KT / 2; ++kk) {
    uint32_t a[4];
    a[0] = pack_bf16(p[2 * kk][0], p[2 * kk][1]);
    a[1] = pack_bf16(p[2 * kk][2], p[2 * kk][3]);
    a[2] = pack_bf16(p[2 * kk + 1][0], p[2 * kk + 1][1]);
    a[3] = pack_bf16(p[2 * kk + 1][2], p[2 * kk + 1][3]);
#pragma unroll
    for (int nt = 0; nt < HD / 8; nt += 2) {
      // trans x4: matrices (k lo, n nt), (k hi, n nt), (k lo, nt+1), (k hi, nt+1)
      const int mi = lane >> 3;
      const int row = k0 + kk * 16 + ((mi & 1) << 3) + (lane & 7);
      const int chunk = nt + (mi >> 1);
      uint32_t b[4];
      ldsm_x4_t(b, tile + tile_off<HD>(row, chunk));
      mma16816(acc[nt], a, b);
      mma16816(acc[nt + 1], a, b + 2);
    }
  }
}

struct AttnParams {
  const __nv_bfloat16* qkv;  // [B*S, 3d]
  __nv_bfloat16* o;          // [B*S, d]
  float* lse;                // [B, H, S]
  const __nv_bfloat16* dout; // [B*S, d]
  float* dsum;               // [B, H, S] rowsum(dO * O)
  __nv_bfloat16* dqkv;       // [B*S, 3d]
  int B, H, S, d;
  int causal;
  float scale;
};

// ------------------------------- forward -------------------------------------
template <int HD>
__global__ void __launch_bounds__(256) attn_fwd_kernel(const AttnParams p) {
  constexpr int BR = 128, BC = 64;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sK0 = sQ + BR * HD * 2;
  const uint32_t sV0 = sK0 + 2 * BC * HD * 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const long long ld = 3LL * p.d;
  const __nv_bfloat16* base = p.qkv + static_cast<long long>(b) * p.S * ld;
  const __nv_bfloat16* Qg = base + h * HD;
  const __nv_bfloat16* Kg = base + p.d + h * HD;
  const __nv_bfloat16* Vg = base + 2 * p.d + h * HD;
  const int q0 = qb * BR;
  const int nq = min(BR, p.S - q0);

  load_tile<HD, BR, 256>(sQ, Qg + q0 * ld, ld, nq);
  cp_commit();
  const int kend = p.causal ? min(p.S, q0 + BR) : p.S;
  const int nkb = (kend + BC - 1) / BC;
  load_tile<HD, BC, 256>(sK0, Kg, ld, min(BC, p.S));
  load_tile<HD, BC, 256>(sV0, Vg, ld, min(BC, p.S));
  cp_commit();

  float o_acc[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o_acc[i][0] = o_acc[i][1] = o_acc[i][2] = o_acc[i][3] = 0.f;
  float m_r[2] = {-INFINITY, -INFINITY}, l_r[2] = {0.f, 0.f};
  uint32_t qa[HD / 16][4];
  const float sl2 = p.scale * kLog2e;
  const int row_a = q0 + warp * 16 + (lane >> 2);  // query index of c0/c1
  const int row_b = row_a + 8;

  for (int j = 0; j < nkb; ++j) {
    if (j + 1 < nkb) {
      const int k1 = (j + 1) * BC;
      load_tile<HD, BC, 256>(sK0 + ((j + 1) & 1) * BC * HD * 2, Kg + k1 * ld, ld, min(BC, p.S - k1));
      load_tile<HD, BC, 256>(sV0 + ((j + 1) & 1) * BC * HD * 2, Vg + k1 * ld, ld, min(BC, p.S - k1));
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (j == 0) load_a_frags<HD>(qa, sQ, warp * 16, lane);
    const uint32_t sK = sK0 + (j & 1) * BC * HD * 2;
    const uint32_t sV = sV0 + (j & 1) * BC * HD * 2;
    float s[BC / 8][4];
#pragma unroll
    for (int i = 0; i < BC / 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
    mma_a_tileT<HD, BC / 8>(s, qa, sK, 0, lane);
    const int k0 = j * BC;
    float mx[2] = {m_r[0], m_r[1]};
#pragma unroll
    for (int nt = 0; nt < BC / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + nt * 8 + (lane & 3) * 2 + (e & 1);
        const int q = (e < 2) ? row_a : row_b;
        const bool masked = key >= p.S || (p.causal && key > q);
        s[nt][e] = masked ? -INFINITY : s[nt][e] * sl2;
        mx[e >> 1] = fmaxf(mx[e >> 1], s[nt][e]);
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
      mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
    }
    float corr[2], rs[2] = {0.f, 0.f};
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const float mnew = mx[r];
      corr[r] = (m_r[r] == -INFINITY) ? 0.f : exp2f(m_r[r] - mnew);
      m_r[r] = mnew;
    }
#pragma unroll
    for (int nt = 0; nt < BC / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float mm = m_r[e >> 1];
        const float v = (mm == -INFINITY) ? 0.f : exp2f(s[nt][e] - mm);
        s[nt][e] = v;
        rs[e >> 1] += v;
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 1);
      rs[r] += __shfl_xor_sync(0xffffffffu, rs[r], 2);
      l_r[r] = l_r[r] * corr[r] + rs[r];
    }
#pragma unroll
    for (int i = 0; i < HD / 8; ++i) {
      o_acc[i][0] *= corr[0];
      o_acc[i][1] *= corr[0];
      o_acc[i][2] *= corr[1];
      o_acc[i][3] *= corr[1];
    }
    mma_p_tile<HD, BC / 8>(o_acc, s, sV, 0, lane);
    __syncthreads();
  }
  // epilogue: normalise, store O (merged heads) and LSE (natural log)
  const float inv0 = l_r[0] > 0.f ? 1.f / l_r[0] : 0.f;
  const float inv1 = l_r[1] > 0.f ? 1.f / l_r[1] : 0.f;
  __nv_bfloat16* Og = p.o + static_cast<long long>(b) * p.S * p.d + h * HD;
#pragma unroll
  for (int nt = 0; nt < HD / 8; ++nt) {
    const int col = nt * 8 + (lane & 3) * 2;
    if (row_a < p.S)
      *reinterpret_cast<uint32_t*>(Og + static_cast<long long>(row_a) * p.d + col) =
          pack_bf16(o_acc[nt][0] * inv0, o_acc[nt][1] * inv0);
    if (row_b < p.S)
      *reinterpret_cast<uint32_t*>(Og + static_cast<long long>(row_b) * p.d + col) =
          pack_bf16(o_acc[nt][2] * inv1, o_acc[nt][3] * inv1);
  }
  if ((lane & 3) == 0) {
    float* L = p.lse + (static_cast<long long>(b) * p.H + h) * p.S;
    if (row_a < p.S) L[row_a] = (m_r[0] / kLog2e) + logf(l_r[0]);
    if (row_b < p.S) L[row_b] = (m_r[1] / kLog2e) + logf(l_r[1]);
  }
}

// ------------------------------- backward: dQ --------------------------------
// Also writes dsum[i] = sum_c dO[i,c] * O[i,c] (the rowsum(dP*P) term of
// tensor.cpp:526-533) for the dK/dV kernel.
template <int HD>
__global__ void __launch_bounds__(256) attn_bwd_dq_kernel(const AttnParams p) {
  constexpr int BR = 128, BC = 64;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = smem_u32(smem);
  const uint32_t sdO = sQ + BR * HD * 2;
  const uint32_t sK0 = sdO + BR * HD * 2;
  const uint32_t sV0 = sK0 + 2 * BC * HD * 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const long long ld = 3LL * p.d;
  const __nv_bfloat16* base = p.qkv + static_cast<long long>(b) * p.S * ld;
  const __nv_bfloat16* Qg = base + h * HD;
  const __nv_bfloat16* Kg = base + p.d + h * HD;
  const __nv_bfloat16* Vg = base + 2 * p.d + h * HD;
  const __nv_bfloat16* dOg = p.dout + static_cast<long long>(b) * p.S * p.d + h * HD;
  const __nv_bfloat16* Og = p.o + static_cast<long long>(b) * p.S * p.d + h * HD;
  const int q0 = qb * BR;
  const int nq = min(BR, p.S - q0);

  load_tile<HD, BR, 256>(sQ, Qg + q0 * ld, ld, nq);
  load_tile<HD, BR, 256>(sdO, dOg + static_cast<long long>(q0) * p.d, p.d, nq);
  cp_commit();
  const int kend = p.causal ? min(p.S, q0 + BR) : p.S;
  const int nkb = (kend + BC - 1) / BC;
  load_tile<HD, BC, 256>(sK0, Kg, ld, min(BC, p.S));
  load_tile<HD, BC, 256>(sV0, Vg, ld, min(BC, p.S));
  cp_commit();

  const int row_a = q0 + warp * 16 + (lane >> 2);
  const int row_b = row_a + 8;
  const long long bh = static_cast<long long>(b) * p.H + h;
  // rowsum(dO * O) for this thread's two rows (direct from global, fp32 accumulate)
  float dsum[2] = {0.f, 0.f};
  {
    // each of the 4 lanes of a row handles HD/4 columns
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int row = r ? row_b : row_a;
      float acc = 0.f;
      if (row < p.S) {
        const __nv_bfloat16* a = dOg + static_cast<long long>(row) * p.d;
        const __nv_bfloat16* o = Og + static_cast<long long>(row) * p.d;
        for (int c = (lane & 3) * 2; c < HD; c += 8) {
          const float2 x = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(a + c));
          const float2 y = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(o + c));
          acc += x.x * y.x + x.y * y.y;
        }
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      dsum[r] = acc;
    }
    if ((lane & 3) == 0) {
      if (row_a < p.S) p.dsum[bh * p.S + row_a] = dsum[0];
      if (row_b < p.S) p.dsum[bh * p.S + row_b] = dsum[1];
    }
  }
  const float lse_a = row_a < p.S ? p.lse[bh * p.S + row_a] * kLog2e : 0.f;
  const float lse_b = row_b < p.S ? p.lse[bh * p.S + row_b] * kLog2e : 0.f;
  const float sl2 = p.scale * kLog2e;

  float dq[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) dq[i][0] = dq[i][1] = dq[i][2] = dq[i][3] = 0.f;
  uint32_t qa[HD / 16][4], da[HD / 16][4];

  for (int j = 0; j < nkb; ++j) {
    if (j + 1 < nkb) {
      const int k1 = (j + 1) * BC;
      load_tile<HD, BC, 256>(sK0 + ((j + 1) & 1) * BC * HD * 2, Kg + k1 * ld, ld, min(BC, p.S - k1));
      load_tile<HD, BC, 256>(sV0 + ((j + 1) & 1) * BC * HD * 2, Vg + k1 * ld, ld, min(BC, p.S - k1));
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (j == 0) {
      load_a_frags<HD>(qa, sQ, warp * 16, lane);
      load_a_frags<HD>(da, sdO, warp * 16, lane);
    }
    const uint32_t sK = sK0 + (j & 1) * BC * HD * 2;
    const uint32_t sV = sV0 + (j & 1) * BC * HD * 2;
    float s[BC / 8][4], dp[BC / 8][4];
#pragma unroll
    for (int i = 0; i < BC / 8; ++i) {
      s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
      dp[i][0] = dp[i][1] = dp[i][2] = dp[i][3] = 0.f;
    }
    mma_a_tileT<HD, BC / 8>(s, qa, sK, 0, lane);
    mma_a_tileT<HD, BC / 8>(dp, da, sV, 0, lane);
    const int k0 = j * BC;
#pragma unroll
    for (int nt = 0; nt < BC / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = k0 + nt * 8 + (lane & 3) * 2 + (e & 1);
        const int q = (e < 2) ? row_a : row_b;
        const bool masked = key >= p.S || q >= p.S || (p.causal && key > q);
        const float pv = masked ? 0.f : exp2f(s[nt][e] * sl2 - ((e < 2) ? lse_a : lse_b));
        s[nt][e] = pv * (dp[nt][e] - dsum[e >> 1]);  // dS
      }
    }
    mma_p_tile<HD, BC / 8>(dq, s, sK, 0, lane);
    __syncthreads();
  }
  __nv_bfloat16* dQg = p.dqkv + static_cast<long long>(b) * p.S * ld + h * HD;
#pragma unroll
  for (int nt = 0; nt < HD / 8; ++nt) {
    const int col = nt * 8 + (lane & 3) * 2;
    if (row_a < p.S)
      *reinterpret_cast<uint32_t*>(dQg + row_a * ld + col) = pack_bf16(dq[nt][0] * p.scale, dq[nt][1] * p.scale);
    if (row_b < p.S)
      *reinterpret_cast<uint32_t*>(dQg + row_b * ld + col) = pack_bf16(dq[nt][2] * p.scale, dq[nt][3] * p.scale);
  }
}

// ------------------------------- backward: dK, dV -----------------------------
template <int HD>
__global__ void __launch_bounds__(256) attn_bwd_dkdv_kernel(const AttnParams p) {
  constexpr int BKEY = 128, BQ = 64;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sK = smem_u32(smem);
  const uint32_t sV = sK + BKEY * HD * 2;
  const uint32_t sQ0 = sV + BKEY * HD * 2;
  const uint32_t sdO0 = sQ0 + 2 * BQ * HD * 2;
  float* sL = reinterpret_cast<float*>(smem + (2 * BKEY + 4 * BQ) * HD * 2);  // [2][BQ]
  float* sD = sL + 2 * BQ;                                                     // [2][BQ]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const long long ld = 3LL * p.d;
  const __nv_bfloat16* base = p.qkv + static_cast<long long>(b) * p.S * ld;
  const __nv_bfloat16* Qg = base + h * HD;
  const __nv_bfloat16* Kg = base + p.d + h * HD;
  const __nv_bfloat16* Vg = base + 2 * p.d + h * HD;
  const __nv_bfloat16* dOg = p.dout + static_cast<long long>(b) * p.S * p.d + h * HD;
  const long long bh = static_cast<long long>(b) * p.H + h;
  const float* Lg = p.lse + bh * p.S;
  const float* Dg = p.dsum + bh * p.S;
  const int k0 = kb * BKEY;
  const int nk = min(BKEY, p.S - k0);

  load_tile<HD, BKEY, 256>(sK, Kg + k0 * ld, ld, nk);
  load_tile<HD, BKEY, 256>(sV, Vg + k0 * ld, ld, nk);
  cp_commit();
  const int qstart = p.causal ? (k0 / BQ) * BQ : 0;
  const int nqb = (p.S - qstart + BQ - 1) / BQ;
  auto issue_q = [&](int i, int buf) {
    const int q1 = qstart + i * BQ;
    const int nv = min(BQ, p.S - q1);
    load_tile<HD, BQ, 256>(sQ0 + buf * BQ * HD * 2, Qg + q1 * ld, ld, nv);
    load_tile<HD, BQ, 256>(sdO0 + buf * BQ * HD * 2, dOg + static_cast<long long>(q1) * p.d, p.d, nv);
    for (int t = threadIdx.x; t < BQ; t += 256) {
      const int q = q1 + t;
      sL[buf * BQ + t] = q < p.S ? Lg[q] * kLog2e : 0.f;
      sD[buf * BQ + t] = q < p.S ? Dg[q] : 0.f;
    }
  };
  issue_q(0, 0);
  cp_commit();

  const int key_a = k0 + warp * 16 + (lane >> 2);
  const int key_b = key_a + 8;
  const float sl2 = p.scale * kLog2e;
  float dk[HD / 8][4], dv[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) {
    dk[i][0] = dk[i][1] = dk[i][2] = dk[i][3] = 0.f;
    dv[i][0] = dv[i][1] = dv[i][2] = dv[i][3] = 0.f;
  }
  uint32_t ka[HD / 16][4], va[HD / 16][4];

  for (int i = 0; i < nqb; ++i) {
    __syncthreads();  // buffer (i+1)&1 is free (consumed in iteration i-1)
    if (i + 1 < nqb) issue_q(i + 1, (i + 1) & 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (i == 0) {
      load_a_frags<HD>(ka, sK, warp * 16, lane);
      load_a_frags<HD>(va, sV, warp * 16, lane);
    }
    const int buf = i & 1;
    const uint32_t sQ = sQ0 + buf * BQ * HD * 2;
    const uint32_t sdO = sdO0 + buf * BQ * HD * 2;
    const float* L = sL + buf * BQ;
    const float* D = sD + buf * BQ;
    const int q1 = qstart + i * BQ;
    float st[BQ / 8][4], dpt[BQ / 8][4];
#pragma unroll
    for (int t = 0; t < BQ / 8; ++t) {
      st[t][0] = st[t][1] = st[t][2] = st[t][3] = 0.f;
      dpt[t][0] = dpt[t][1] = dpt[t][2] = dpt[t][3] = 0.f;
    }
    mma_a_tileT<HD, BQ / 8>(st, ka, sQ, 0, lane);   // S^T = K Q^T
    mma_a_tileT<HD, BQ / 8>(dpt, va, sdO, 0, lane); // dP^T = V dO^T
#pragma unroll
    for (int nt = 0; nt < BQ / 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ql = nt * 8 + (lane & 3) * 2 + (e & 1);
        const int q = q1 + ql;
        const int key = (e < 2) ? key_a : key_b;
        const bool masked = q >= p.S || key >= p.S || (p.causal && key > q);
        const float pv = masked ? 0.f : exp2f(st[nt][e] * sl2 - L[ql]);
        st[nt][e] = pv;                       // P^T
        dpt[nt][e] = pv * (dpt[nt][e] - D[ql]);  // dS^T
      }
    }
    mma_p_tile<HD, BQ / 8>(dv, st, sdO, 0, lane);   // dV += P^T dO
    mma_p_tile<HD, BQ / 8>(dk, dpt, sQ, 0, lane);   // dK += dS^T Q
  }
  __nv_bfloat16* dKg = p.dqkv + static_cast<long long>(b) * p.S * ld + p.d + h * HD;
  __nv_bfloat16* dVg = dKg + p.d;
#pragma unroll
  for (int nt = 0; nt < HD / 8; ++nt) {
    const int col = nt * 8 + (lane & 3) * 2;
    if (key_a < p.S) {
      *reinterpret_cast<uint32_t*>(dKg + key_a * ld + col) = pack_bf16(dk[nt][0] * p.scale, dk[nt][1] * p.scale);
      *reinterpret_cast<uint32_t*>(dVg + key_a * ld + col) = pack_bf16(dv[nt][0], dv[nt][1]);
    }
    if (key_b < p.S) {
      *reinterpret_cast<uint32_t*>(dKg + key_b * ld + col) = pack_bf16(dk[nt][2] * p.scale, dk[nt][3] * p.scale);
      *reinterpret_cast<uint32_t*>(dVg + key_b * ld + col) = pack_bf16(dv[nt][2], dv[nt][3]);
    }
  }
}

template <typename K>
cudaError_t set_smem(K kern, int bytes) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

template <int HD>
p2r_status run_fwd(const AttnParams& p, cudaStream_t s) {
  const int smem = (128 + 4 * 64) * HD * 2;
  static cudaError_t e0 = set_smem(attn_fwd_kernel<HD>, smem);
  if (e0 != cudaSuccess) return set_cuda_error(e0, "attention fwd attr");
  dim3 grid((p.S + 127) / 128, p.H, p.B);
  attn_fwd_kernel<HD><<<grid, 256, smem, s>>>(p);
  P2R_CHECK_LAUNCH("attention fwd");
  return P2R_OK;
}

template <int HD>
p2r_status run_bwd(const AttnParams& p, cudaStream_t s) {
  const int smem_q = (2 * 128 + 4 * 64) * HD * 2;
  const int smem_kv = (2 * 128 + 4 * 64) * HD * 2 + 4 * 64 * 4;
  static cudaError_t e0 = set_smem(attn_bwd_dq_kernel<HD>, smem_q);
  static cudaError_t e1 = set_smem(attn_bwd_dkdv_kernel<HD>, smem_kv);
  if (e0 != cudaSuccess || e1 != cudaSuccess) return set_cuda_error(e0 ? e0 : e1, "attention bwd attr");
  dim3 grid((p.S + 127) / 128, p.H, p.B);
  attn_bwd_dq_kernel<HD><<<grid, 256, smem_q, s>>>(p);
  P2R_CHECK_LAUNCH("attention bwd dq");
  attn_bwd_dkdv_kernel<HD><<<grid, 256, smem_kv, s>>>(p);
  P2R_CHECK_LAUNCH("attention bwd dkdv");
  return P2R_OK;
}

p2r_status legacy_fwd(const void* qkv, void* o, float* lse, int B, int H, int S, int d, int causal,
                      cudaStream_t s) {
  AttnParams p{};
  p.qkv = static_cast<const __nv_bfloat16*>(qkv);
  p.o = static_cast<__nv_bfloat16*>(o);
  p.lse = lse;
  p.B = B;
  p.H = H;
  p.S = S;
  p.d = d;
  p.causal = causal;
  const int hd = d / H;
  p.scale = 1.0f / sqrtf(static_cast<float>(hd));
  return hd == 64 ? run_fwd<64>(p, s) : run_fwd<128>(p, s);
}

p2r_status legacy_bwd(const void* qkv, const void* o, const float* lse, const void* dout, float* dsum_ws, void* dqkv,
                      int B, int H, int S, int d, int causal, cudaStream_t s) {
  AttnParams p{};
  p.qkv = static_cast<const __nv_bfloat16*>(qkv);
  p.o = const_cast<__nv_bfloat16*>(static_cast<const __nv_bfloat16*>(o));
  p.lse = const_cast<float*>(lse);
  p.dout = static_cast<const __nv_bfloat16*>(dout);
  p.dsum = dsum_ws;
  p.dqkv = static_cast<__nv_bfloat16*>(dqkv);
  p.B = B;
  p.H = H;
  p.S = S;
  p.d = d;
  p.causal = causal;
  const int hd = d / H;
  p.scale = 1.0f / sqrtf(static_cast<float>(hd));
  return hd == 64 ? run_bwd<64>(p, s) : run_bwd<128>(p, s);
}

}  // namespace attn
}  // namespace p2r

#endif  // P2R_DIAG

using namespace p2r;

extern "C" p2r_status p2r_attention_fwd(const void* qkv, void* o, float* lse, int B, int H, int S,
                                        int d, int causal, void* stream) {
  if (B < 0 || H <= 0 || S < 0 || d <= 0 || d % H != 0)
    return set_error(P2R_EINVAL, "masked_attention: q/k/v must share a [B,H,S,hd] shape");
  if (B == 0 || S == 0) return P2R_OK;  // empty batch / sequence: nothing to compute
  const int hd = d / H;
  if (hd != 64 && hd != 128) return set_error(P2R_EINVAL, "attention: head_dim must be 64 or 128");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
#ifdef P2R_DIAG
  static const bool legacy = std::getenv("P2R_ATTN_MMA_SYNC") != nullptr;
  if (legacy) return attn::legacy_fwd(qkv, o, lse, B, H, S, d, causal, s);
#endif
  return attention_fwd_tc(qkv, o, lse, B, H, S, d, causal, s);
}

extern "C" p2r_status p2r_attention_bwd(const void* qkv, const void* o, const float* lse,
                                        const void* dout, float* dsum_ws, void* dqkv, int B, int H,
                                        int S, int d, int causal, void* stream) {
  if (B < 0 || H <= 0 || S < 0 || d <= 0 || d % H != 0)
    return set_error(P2R_EINVAL, "masked_attention: q/k/v must share a [B,H,S,hd] shape");
  if (B == 0 || S == 0) return P2R_OK;  // empty batch / sequence: nothing to compute
  const int hd = d / H;
  if (hd != 64 && hd != 128) return set_error(P2R_EINVAL, "attention: head_dim must be 64 or 128");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
#ifdef P2R_DIAG
  static const bool legacy = std::getenv("P2R_ATTN_MMA_SYNC") != nullptr;
  if (legacy) return attn::legacy_bwd(qkv, o, lse, dout, dsum_ws, dqkv, B, H, S, d, causal, s);
#endif
  return attention_bwd_tc(qkv, o, lse, dout, dsum_ws, dqkv, B, H, S, d, causal, s);
}
