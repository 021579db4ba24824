// tcgen05 / TMEM / TMA GEMM for sm_100a.
//
// Replaces every cblas_sgemm call of the reference (tensor.cpp:138 matmul fwd,
// :146/:149 matmul bwd dA/dB, :163/:171/:174 matmul_nt) for the QKV / O / FFN /
// expert / tied-head projections. bf16 operands, fp32 accumulation in TMEM,
// fused epilogues (bias, exact GELU, GELU', fp32 residual add, beta=1 fp32
// accumulation straight into the shared-layer gradient buffer).
//
// Structure (one CTA per SM, persistent, 8 warps):
//   warp 0      : TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1      : MMA issuer (one lane), tcgen05.mma M=128 N=BN K=16
//   warp 2      : TMEM allocator (2 x BN fp32 columns: double-buffered accum)
//   warps 4..7  : epilogue, TMEM -> registers -> global
// Operands may be K-major or MN-major (both SWIZZLE_128B), so forward
// (X.W), dX (dY.W^T) and dW (X^T.dY) all run without transposed copies of
// activations.
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <utility>
#include <vector>

#include "../../include/p2r_cuda.h"

#include "common.cuh"
#include "p2r_internal.h"

namespace p2r {

constexpr int BM = 128;
constexpr int BK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B row

struct GemmParams {
  int m, n, k;
  int num_m_blk, num_n_blk, num_k_blk;
  int epi;
  void* c;
  int ldc;
  void* c2;
  int ldc2;
  const float* bias;
  const void* aux;
  int ldaux;
  int group_mode, groups, seg_rows;
  const int* counts;
  int split_k;
  int tiles_total;
  long long c_split_stride;  // elements between split-K partial outputs
  int vec4;                  // all epilogue leading dims / bases allow 4-wide accesses
  int raster_g;              // ungrouped tile order: groups of raster_g m-blocks x all n-blocks
  int tma_c;                 // bf16 epilogues: stage 32x32 tiles in smem, TMA-store them (tmC / tmC2)
  float* colsum;             // GELU' bias grad: per-32-row column partials [ceil(m/32)][n] of the bf16 output
  // serial split-K (C += A.B only): split ks of tile r accumulates straight into C
  // once counters[r * CG + rank] == ks, then releases the next split
  int serial;
  int* counters;
};

struct Tile {
  bool valid;
  int m_blk, n_blk;
  int a_row;    // first m row of this CTA's A slice (K-major: tensor row; MN-major: column)
  int b_row;    // K-major B: first row (n)
  int b_col;    // MN-major B: first column (n) of this CTA's B slice
  int kbase;    // MN-major operands: first K row
  int kb0, kb1; // k-block range
  int g;
  int ks;
  int r;  // tile index within its split (serial split-K counter slot)
};

// CG = CTAs per tile (2: CTA pair, 256-row tile; rank picks the CTA's 128-row
// A slice and its BN/2-row B slice). Grouped modes run with CG = 1.
P2R_DEVICE Tile get_tile(const GemmParams& p, int t, int BN, int CG = 1, int rank = 0) {
  Tile T;
  T.valid = true;
  T.g = 0;
  T.ks = 0;
  T.r = t;
  if (p.group_mode == P2R_GROUP_M) {
    const int mt = p.seg_rows / BM;
    const int per_g = mt * p.num_n_blk;
    T.g = t / per_g;
    const int r = t - T.g * per_g;
    T.n_blk = r / mt;
    T.m_blk = r - T.n_blk * mt;
    const int cnt = __ldg(p.counts + T.g);
    T.valid = T.m_blk * BM < cnt;
    T.a_row = T.g * p.seg_rows + T.m_blk * BM;
    T.b_row = T.g * p.n + T.n_blk * BN;
    T.b_col = T.n_blk * BN;
    T.kbase = T.g * p.k;  // MN-major B: stacked [groups*k, n]
    T.kb0 = 0;
    T.kb1 = p.num_k_blk;
  } else if (p.group_mode == P2R_GROUP_K) {
    const int per_g = p.num_m_blk * p.num_n_blk;
    T.g = t / per_g;
    const int r = t - T.g * per_g;
    T.n_blk = r / p.num_m_blk;
    T.m_blk = r - T.n_blk * p.num_m_blk;
    const int cnt = __ldg(p.counts + T.g);
    T.valid = cnt > 0;
    T.a_row = T.m_blk * BM;
    T.b_row = T.n_blk * BN;
    T.b_col = T.n_blk * BN;
    T.kbase = T.g * p.seg_rows;
    T.kb0 = 0;
    T.kb1 = (cnt + BK - 1) / BK;
  } else {
    // Grouped raster: consecutive tiles (= CTAs running concurrently) sweep
    // raster_g m-blocks x every n-block, so each A and B block is shared by a
    // bounded number of concurrent tiles (no L2 hot spot, fewer DRAM re-reads).
    const int per_s = p.num_m_blk * p.num_n_blk;
    T.ks = t / per_s;
    const int r = t - T.ks * per_s;
    T.r = r;
    const int gsz = p.raster_g * p.num_n_blk;
    const int grp = r / gsz;
    const int m0 = grp * p.raster_g;
    const int gm = min(p.raster_g, p.num_m_blk - m0);
    const int w = r - grp * gsz;
    T.m_blk = m0 + w % gm;
    T.n_blk = w / gm;
    T.a_row = T.m_blk * BM * CG + rank * BM;
    T.b_row = T.n_blk * BN + rank * (BN / CG);
    T.b_col = T.b_row;
    T.kbase = 0;
    T.kb0 = static_cast<int>((static_cast<long long>(T.ks) * p.num_k_blk) / p.split_k);
    T.kb1 = static_cast<int>((static_cast<long long>(T.ks + 1) * p.num_k_blk) / p.split_k);
    T.valid = T.kb1 > T.kb0;
  }
  return T;
}

#ifndef P2R_GEMM_EPI_WARPS
#define P2R_GEMM_EPI_WARPS 8
#endif
constexpr int kEpiWarps = P2R_GEMM_EPI_WARPS;       // kEpiWarps / 4 per TMEM lane quadrant
constexpr int kGemmThreads = 128 + 32 * kEpiWarps;  // 4 control warps + epilogue

template <int BN, int CG = 1>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (BN / CG) * BK * 2;  // a pair splits B's rows between its CTAs
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = ((229376 - kEpiWarps * 4096) / STAGE_BYTES) > 8 ? 8
                                                                               : ((229376 - kEpiWarps * 4096) / STAGE_BYTES);
  static constexpr int TMEM_COLS = (2 * BN) < 32 ? 32 : (2 * BN);
  static constexpr int STG_BYTES = kEpiWarps * 4096;  // per epilogue warp: transpose tile / two TMA-store slots
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + STG_BYTES + 256 /*barriers*/;
};

// Epilogue for ONE element: lane = column, so every global access of a warp is
// row-contiguous (coalesced). `zero` stores zeros (padding rows of a grouped
// segment) so later grouped-K GEMMs see clean K padding.
// Returns the GELU' value (fp32, before bf16 rounding; feeds the bias-grad column sums).
template <int EPI>
P2R_DEVICE float epilogue_elem(const GemmParams& p, float v, long long row, int col, bool zero,
                               float b, char* cbase, int ldc) {
  constexpr int epi = EPI;
  if (zero) v = 0.0f;
  switch (epi) {
    case P2R_EPI_BF16:
      reinterpret_cast<__nv_bfloat16*>(cbase)[row * ldc + col] = __float2bfloat16_rn(zero ? 0.0f : v + b);
      break;
    case P2R_EPI_F32:
    case P2R_EPI_F32_BF16: {
      if (!zero) {
        v += b;
        if (p.aux != nullptr) v += reinterpret_cast<const float*>(p.aux)[row * p.ldaux + col];
      }
      reinterpret_cast<float*>(cbase)[row * ldc + col] = v;
      if (epi == P2R_EPI_F32_BF16)
        reinterpret_cast<__nv_bfloat16*>(p.c2)[row * p.ldc2 + col] = __float2bfloat16_rn(v);
      break;
    }
    case P2R_EPI_ACC_F32: {
      if (zero) break;
      float* d = reinterpret_cast<float*>(cbase) + row * ldc + col;
      *d = *d + v;
      break;
    }
    case P2R_EPI_BIAS_GELU: {
      const float pre = zero ? 0.0f : v + b;
      float gd;
      const float g = gelu_pair_f(pre, gd);
      reinterpret_cast<__nv_bfloat16*>(p.c2)[row * p.ldc2 + col] = __float2bfloat16_rn(zero ? 0.0f : gd);
      reinterpret_cast<__nv_bfloat16*>(cbase)[row * ldc + col] = __float2bfloat16_rn(zero ? 0.0f : g);
      break;
    }
    case P2R_EPI_DGELU: {  // aux = the GELU derivative the forward epilogue stored
      float o = 0.0f;
      if (!zero) o = v * __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p.aux)[row * p.ldaux + col]);
      reinterpret_cast<__nv_bfloat16*>(cbase)[row * ldc + col] = __float2bfloat16_rn(o);
      return o;
    }
    default:
      break;
  }
  return 0.0f;
}

P2R_DEVICE uint32_t pack2_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}
P2R_DEVICE uint2 pack4_bf16(float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 w;
  w.x = *reinterpret_cast<uint32_t*>(&lo);
  w.y = *reinterpret_cast<uint32_t*>(&hi);
  return w;
}
P2R_DEVICE float4 unpack4_bf16(uint2 w) {
  const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.x));
  const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.y));
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

// Epilogue for 4 consecutive columns of one row (16 B fp32 / 8 B bf16 accesses).
// EPI is a compile-time kind so each kernel instance carries only its own math.
// Returns the 4 GELU' values (fp32; 0 for columns past n), else zeros.
template <int EPI>
P2R_DEVICE float4 epilogue_vec4(const GemmParams& p, float4 v, long long row, int col, int nc, bool zero,
                                float4 b, char* cbase, int ldc) {
  if (nc < 4 || !p.vec4) {
    const float vv[4] = {v.x, v.y, v.z, v.w};
    const float bb[4] = {b.x, b.y, b.z, b.w};
    float out[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (j < nc) out[j] = epilogue_elem<EPI>(p, vv[j], row, col + j, zero, bb[j], cbase, ldc);
    return make_float4(out[0], out[1], out[2], out[3]);
  }
  const long long o = row * ldc + col;
  switch (EPI) {
    case P2R_EPI_BF16:
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(cbase) + o) =
          zero ? make_uint2(0u, 0u) : pack4_bf16(v.x + b.x, v.y + b.y, v.z + b.z, v.w + b.w);
      break;
    case P2R_EPI_F32:
    case P2R_EPI_F32_BF16: {
      if (zero) {
        v = make_float4(0.f, 0.f, 0.f, 0.f);
      } else {
        v = make_float4(v.x + b.x, v.y + b.y, v.z + b.z, v.w + b.w);
        if (p.aux != nullptr) {
          const float4 a = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.aux) + row * p.ldaux + col);
          v = make_float4(v.x + a.x, v.y + a.y, v.z + a.z, v.w + a.w);
        }
      }
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(cbase) + o) = v;
      if (EPI == P2R_EPI_F32_BF16)
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.c2) + row * p.ldc2 + col) =
            pack4_bf16(v.x, v.y, v.z, v.w);
      break;
    }
    case P2R_EPI_ACC_F32: {
      if (zero) break;
      float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(cbase) + o);
      const float4 a = *d;
      *d = make_float4(a.x + v.x, a.y + v.y, a.z + v.z, a.w + v.w);
      break;
    }
    case P2R_EPI_BIAS_GELU: {
      const float4 pre = make_float4(v.x + b.x, v.y + b.y, v.z + b.z, v.w + b.w);
      float4 gd, g;
      g.x = gelu_pair_f(pre.x, gd.x);
      g.y = gelu_pair_f(pre.y, gd.y);
      g.z = gelu_pair_f(pre.z, gd.z);
      g.w = gelu_pair_f(pre.w, gd.w);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.c2) + row * p.ldc2 + col) =
          zero ? make_uint2(0u, 0u) : pack4_bf16(gd.x, gd.y, gd.z, gd.w);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(cbase) + o) =
          zero ? make_uint2(0u, 0u) : pack4_bf16(g.x, g.y, g.z, g.w);
      break;
    }
    case P2R_EPI_DGELU: {
      float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!zero) {
        const float4 gd = unpack4_bf16(
            *reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(p.aux) + row * p.ldaux + col));
        r = make_float4(v.x * gd.x, v.y * gd.y, v.z * gd.z, v.w * gd.w);
      }
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(cbase) + o) = pack4_bf16(r.x, r.y, r.z, r.w);
      return r;
    }
    default:
      break;
  }
  return make_float4(0.f, 0.f, 0.f, 0.f);
}

// Fast path (full 32x32 chunk, 16-byte aligned): the lane's global operand for
// each of its 8 row groups (GELU' pre-activation, fp32 residual, or the fp32
// accumulator being added into) is loaded while the TMEM load is in flight.
template <int EPI>
struct EpiOperand {
  static constexpr bool kHas = EPI == P2R_EPI_DGELU || EPI == P2R_EPI_ACC_F32 || EPI == P2R_EPI_F32 ||
                               EPI == P2R_EPI_F32_BF16;
  using T = typename std::conditional<EPI == P2R_EPI_DGELU, uint2, float4>::type;
};

template <int EPI>
P2R_DEVICE typename EpiOperand<EPI>::T epi_load(const GemmParams& p, long long row, int col, const char* cbase,
                                                int ldc) {
  if constexpr (EPI == P2R_EPI_DGELU) {
    return __ldg(reinterpret_cast<const uint2*>(reinterpret_cast<const __nv_bfloat16*>(p.aux) + row * p.ldaux + col));
  } else if constexpr (EPI == P2R_EPI_ACC_F32) {
    return *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(cbase) + row * ldc + col);
  } else {
    if (p.aux == nullptr) return make_float4(0.f, 0.f, 0.f, 0.f);
    return *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(p.aux) + row * p.ldaux + col);
  }
}

// Returns the 4 GELU' values (fp32, before bf16 rounding), else zeros.
template <int EPI>
P2R_DEVICE float4 epi_store_fast(const GemmParams& p, float4 v, typename EpiOperand<EPI>::T x, long long row,
                                 int col, float4 b, char* cbase, int ldc) {
  const long long o = row * ldc + col;
  if constexpr (EPI == P2R_EPI_BF16) {
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(cbase) + o) =
        pack4_bf16(v.x + b.x, v.y + b.y, v.z + b.z, v.w + b.w);
  } else if constexpr (EPI == P2R_EPI_F32 || EPI == P2R_EPI_F32_BF16) {
    v = make_float4(v.x + b.x + x.x, v.y + b.y + x.y, v.z + b.z + x.z, v.w + b.w + x.w);
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(cbase) + o) = v;
    if constexpr (EPI == P2R_EPI_F32_BF16)
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.c2) + row * p.ldc2 + col) =
          pack4_bf16(v.x, v.y, v.z, v.w);
  } else if constexpr (EPI == P2R_EPI_ACC_F32) {
    *reinterpret_cast<float4*>(reinterpret_cast<float*>(cbase) + o) =
        make_float4(x.x + v.x, x.y + v.y, x.z + v.z, x.w + v.w);
  } else if constexpr (EPI == P2R_EPI_BIAS_GELU) {
    const float2 p0 = __fadd2_rn(make_float2(v.x, v.y), make_float2(b.x, b.y));
    const float2 p1 = __fadd2_rn(make_float2(v.z, v.w), make_float2(b.z, b.w));
    float2 d0, d1;
    const float2 g0 = gelu_pair2(p0, d0), g1 = gelu_pair2(p1, d1);
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(p.c2) + row * p.ldc2 + col) =
        make_uint2(pack2_bf16(d0.x, d0.y), pack2_bf16(d1.x, d1.y));
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(cbase) + o) =
        make_uint2(pack2_bf16(g0.x, g0.y), pack2_bf16(g1.x, g1.y));
  } else if constexpr (EPI == P2R_EPI_DGELU) {
    const float4 gd = unpack4_bf16(x);  // the stored GELU derivative
    const float2 d0 = __fmul2_rn(make_float2(v.x, v.y), make_float2(gd.x, gd.y));
    const float2 d1 = __fmul2_rn(make_float2(v.z, v.w), make_float2(gd.z, gd.w));
    *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(cbase) + o) =
        make_uint2(pack2_bf16(d0.x, d0.y), pack2_bf16(d1.x, d1.y));
    return make_float4(d0.x, d0.y, d1.x, d1.y);
  }
  return make_float4(0.f, 0.f, 0.f, 0.f);
}


// EPI_ = epilogue kind | kEpiColsum (GELU' + bias-grad column partials).
constexpr int kEpiColsum = 0x100;

template <int BN, bool A_MN, bool B_MN, int EPI_, int CG>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmC2,
                const GemmParams p) {
  constexpr int EPI = EPI_ & 0xFF;
  constexpr bool kColsum = (EPI_ & kEpiColsum) != 0;
  using Cfg = GemmCfg<BN, CG>;
  constexpr int BNC = BN / CG;  // B rows (N) this CTA loads per stage
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* stg_all = smem + STAGES * Cfg::STAGE_BYTES;  // 1024-aligned (the TMA-store swizzle needs 512)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg_all + Cfg::STG_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // CTA pair: rank 0 (leader) issues the MMAs; tiles are indexed per pair.
  const int rank = CG == 2 ? static_cast<int>(cluster_ctarank()) : 0;
  const bool leader = rank == 0;
  const int tile0 = blockIdx.x / CG, tile_step = gridDim.x / CG;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar + s, 1);
      mbar_init(empty_bar + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull_bar + s, 1);
      // pair: one arrive per epilogue warp of both CTAs, on the leader's barrier
      mbar_init(tempty_bar + s, CG == 2 ? 2 * kEpiWarps : 32 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 2)
      tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
    else
      tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  }
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();  // both CTAs' barriers initialised before any cross-CTA signal
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  pdl_trigger();
  pdl_wait();  // operands / C / aux may come from the previous kernel

  if (warp == 0) {
    // ---------------- TMA producer (whole warp, one elected lane issues) ----------------
    int stage = 0;
    uint32_t phase = 0;
    const uint32_t s0 = smem_u32(smem);
    const uint32_t full0 = smem_u32(full_bar);
    for (int t = tile0; t < p.tiles_total; t += tile_step) {
      const Tile T = get_tile(p, t, BN, CG, rank);
      if (!T.valid) continue;
      for (int kb = T.kb0; kb < T.kb1; ++kb) {
        mbar_wait(empty_bar + stage, phase ^ 1);
        const uint32_t sa = s0 + stage * Cfg::STAGE_BYTES;
        const uint32_t sb = sa + Cfg::A_BYTES;
        const uint32_t fb = full0 + stage * 8;
        // pair: the leader expects both CTAs' bytes; each CTA's loads count on it
        if (leader) mbar_arrive_expect_tx_warp(fb, CG * Cfg::STAGE_BYTES);
        auto load = [&](uint32_t dst, const CUtensorMap* map, int c0, int c1) {
          if constexpr (CG == 2)
            tma_load_2d_pair_warp(dst, map, fb & 0xFEFFFFFFu, c0, c1);  // the leader's barrier
          else
            tma_load_2d_warp(dst, map, fb, c0, c1);
        };
        if (!A_MN) {
          load(sa, &tmA, kb * BK, T.a_row);
        } else {
#pragma unroll
          for (int j = 0; j < BM / 64; ++j) load(sa + j * 64 * BK * 2, &tmA, T.a_row + 64 * j, T.kbase + kb * BK);
        }
        if (!B_MN) {
          load(sb, &tmB, kb * BK, T.b_row);
        } else {
#pragma unroll
          for (int j = 0; j < BNC / 64; ++j) load(sb + j * 64 * BK * 2, &tmB, T.b_col + 64 * j, T.kbase + kb * BK);
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ---------------- MMA issuer (pair: leader only, M = 256) ----------------
      // Whole warp, one elected lane issues (uniform operands, no per-MMA
      // R2UR / elect loop): issue stays far below the tensor pipe's 128
      // cycles per MMA even when the epilogue warps saturate this SMSP.
      constexpr uint32_t idesc = make_idesc_bf16(BM * CG, BN, A_MN, B_MN);
      constexpr uint32_t kStep = A_MN ? 2048 : 32;   // 16 K-elements: 16 MN-major rows / 32 B in the row
      constexpr uint32_t kStepB = B_MN ? 2048 : 32;
      const uint32_t sa0 = smem_u32(smem);
      const uint64_t ad0 = A_MN ? make_sw128_desc(sa0, 64 * BK * 2, 1024) : make_sw128_desc(sa0, 16, 1024);
      const uint64_t bd0 = B_MN ? make_sw128_desc(sa0 + Cfg::A_BYTES, 64 * BK * 2, 1024)
                                : make_sw128_desc(sa0 + Cfg::A_BYTES, 16, 1024);
      static_assert(!B_MN || BNC >= 64, "MN-major B slice must hold whole 64-column atoms");
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = tile0; t < p.tiles_total; t += tile_step) {
        const Tile T = get_tile(p, t, BN, CG, rank);
        if (!T.valid) continue;
        mbar_wait(tempty_bar + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = T.kb0; kb < T.kb1; ++kb) {
          mbar_wait(full_bar + stage, phase);
          tc_fence_after();
          const uint32_t so = stage * Cfg::STAGE_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = desc_add(ad0, so + kk * kStep);
            const uint64_t bd = desc_add(bd0, so + kk * kStepB);
            const uint32_t accum = (kb > T.kb0 || kk > 0) ? 1u : 0u;
            if constexpr (CG == 2)
              umma_bf16_pair_warp(d_tmem, ad, bd, idesc, accum);
            else
              umma_bf16_warp(d_tmem, ad, bd, idesc, accum);
          }
          if constexpr (CG == 2)
            umma_commit_pair_warp(empty_bar + stage);
          else
            umma_commit_warp(empty_bar + stage);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CG == 2)
          umma_commit_pair_warp(tfull_bar + acc);
        else
          umma_commit_warp(tfull_bar + acc);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int ew = warp & 3;          // TMEM lanes [32*ew, 32*ew+32) (warp % 4 rule)
    const int cpart = (warp - 4) >> 2;  // which part of the BN columns this warp drains
    // per-warp 32x32 fp32 transpose tile, XOR-swizzled: (r, c) at r*32 + (c ^ r)
    // (shared-space address: a generic pointer here compiles to LD/ST on the long scoreboard)
    const uint32_t stg = smem_u32(stg_all) + (warp - 4) * 4096;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = tile0; t < p.tiles_total; t += tile_step) {
      const Tile T = get_tile(p, t, BN, CG, rank);
      if (!T.valid) continue;
      const int row0 = T.m_blk * BM * CG + rank * BM + ew * 32;  // first local row drained by this warp
      long long grow0 = row0;
      int row_lim, zero_from = 1 << 30;
      char* cbase = reinterpret_cast<char*>(p.c);
      const int ldc = p.ldc;
      const float* bias = p.bias;
      if (p.group_mode == P2R_GROUP_M) {
        grow0 = static_cast<long long>(T.g) * p.seg_rows + row0;
        row_lim = p.seg_rows;
        zero_from = __ldg(p.counts + T.g);
        if (bias != nullptr) bias += static_cast<long long>(T.g) * p.n;
      } else if (p.group_mode == P2R_GROUP_K) {
        row_lim = p.m;
        cbase += static_cast<long long>(T.g) * p.m * p.ldc * 4;  // fp32 grads
      } else {
        row_lim = p.m;
        if (p.split_k > 1 && !p.serial) cbase += static_cast<long long>(T.ks) * p.c_split_stride * 4;
      }
      const int nrows = min(32, row_lim - row0);
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN;
      // lane = (row group, 4-column group): a warp instruction covers 4 rows x 32 columns
      const int cg = lane & 7, rg = lane >> 3;
      // this warp's 32-column chunks (of BN / 32, split over the kEpiWarps / 4 warps of its quadrant)
      const int cb = cpart * (BN / 32) / (kEpiWarps / 4), ce = (cpart + 1) * (BN / 32) / (kEpiWarps / 4);
      auto is_fast = [&](int c) {
        const int c0 = T.n_blk * BN + c * 32;
        return p.vec4 && nrows == 32 && c0 + 32 <= p.n && row0 + 32 <= zero_from;
      };
      // GELU' reads a read-only operand: fetch it one chunk ahead, the first
      // chunk before the accumulator is even ready (DRAM latency off the chunk path)
      constexpr bool kPipe = EPI == P2R_EPI_DGELU;
      constexpr bool kTmaEpi = EPI == P2R_EPI_BF16 || EPI == P2R_EPI_BIAS_GELU;  // (host: p2r_gemm tma_c)
      const bool tma = kTmaEpi && p.tma_c;
      typename EpiOperand<EPI>::T xn[8];
      if constexpr (kPipe) {
        if (is_fast(cb) && !tma) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
            xn[i] = epi_load<EPI>(p, grow0 + 4 * i + rg, T.n_blk * BN + cb * 32 + 4 * cg, cbase, ldc);
        }
      }
      mbar_wait(tfull_bar + acc, acc_phase);
      tc_fence_after();
      int* ctr = nullptr;
      if (p.serial) {  // earlier splits of this tile must have added into C (ordered -> deterministic)
        ctr = p.counters + (T.r * CG + rank);
        if (lane == 0) {
          int v;
          do {
            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
          } while (v != T.ks);
        }
        __syncwarp();
      }
      if constexpr (kTmaEpi) {
        if (tma) {
          // lane = row: compute in the TMEM layout, pack bf16, write the 32x32 tile
          // once into a 64B-swizzled slot and TMA-store it (hardware clips ragged
          // edges). Slots alternate per chunk; BIAS_GELU fills both (out, pre).
          constexpr bool kTwo = EPI == P2R_EPI_BIAS_GELU;
          const bool zrow = row0 + lane >= zero_from;  // grouped padding rows are written as 0
#pragma unroll 1
          for (int c = cb; c < ce; ++c) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(taddr + c * 32, r);
            const int col0 = T.n_blk * BN + c * 32;
            const int nv = min(32, p.n - col0);  // valid columns of this chunk
            float4 b4[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) b4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (bias != nullptr) {
              if (nv == 32) {
#pragma unroll
                for (int i = 0; i < 8; ++i) b4[i] = __ldg(reinterpret_cast<const float4*>(bias + col0) + i);
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (j < nv) reinterpret_cast<float*>(b4)[j] = __ldg(bias + col0 + j);
              }
            }
            tmem_ld_wait();
            uint32_t o[16];
            uint32_t pr[kTwo ? 16 : 1];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const float2 x = __fadd2_rn(make_float2(__uint_as_float(r[2 * j]), __uint_as_float(r[2 * j + 1])),
                                          reinterpret_cast<const float2*>(b4)[j]);
              if constexpr (EPI == P2R_EPI_BF16) {
                o[j] = pack2_bf16(x.x, x.y);
              } else {  // BIAS_GELU: gelu and the stored derivative
                float2 gd;
                const float2 g = gelu_pair2(x, gd);
                pr[j] = pack2_bf16(gd.x, gd.y);
                o[j] = pack2_bf16(g.x, g.y);
              }
              if (zrow) {
                o[j] = 0u;
                if constexpr (kTwo) pr[j] = 0u;
              }
            }
            const uint32_t slot = stg + (kTwo ? 0u : static_cast<uint32_t>(c & 1) * 2048u);
            if (lane == 0) {
              if constexpr (kTwo)
                bulk_wait_read<0>();
              else
                bulk_wait_read<1>();
            }
            __syncwarp();
            const uint32_t rowa = slot + lane * 64;
            const uint32_t sw = (lane >> 1) & 3;  // SWIZZLE_64B: 16-byte chunk ^= address bits [7:8]
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              sts128(rowa + ((q ^ sw) << 4), make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]));
              if constexpr (kTwo)
                sts128(rowa + 2048 + ((q ^ sw) << 4), make_uint4(pr[4 * q], pr[4 * q + 1], pr[4 * q + 2], pr[4 * q + 3]));
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0 && nrows > 0 && nv > 0) {
              tma_store_2d(&tmC, slot, col0, static_cast<int>(grow0));
              if constexpr (kTwo) tma_store_2d(&tmC2, slot + 2048, col0, static_cast<int>(grow0));
              bulk_commit();
            }
          }
        }
      }
#pragma unroll 1
      for (int c = cb; c < (tma ? cb : ce); ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        const int col0 = T.n_blk * BN + c * 32;
        const int col = col0 + 4 * cg;
        const bool fast = is_fast(c);
        typename EpiOperand<EPI>::T x[8];
        if constexpr (kPipe) {
#pragma unroll
          for (int i = 0; i < 8; ++i) x[i] = xn[i];
          if (c + 1 < ce && is_fast(c + 1)) {
#pragma unroll
            for (int i = 0; i < 8; ++i) xn[i] = epi_load<EPI>(p, grow0 + 4 * i + rg, col + 32, cbase, ldc);
          }
        } else if constexpr (EpiOperand<EPI>::kHas) {
          if (fast) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = epi_load<EPI>(p, grow0 + 4 * i + rg, col, cbase, ldc);
          }
        }
        tmem_ld_wait();
        if (nrows <= 0 || col0 >= p.n) continue;  // warp-uniform
        // lane = row: 8 float4 stores into a float4-granular XOR swizzle
#pragma unroll
        for (int q = 0; q < 8; ++q)
          sts128(stg + 4 * (lane * 32 + ((q ^ (lane & 7)) << 2)), make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]));
        __syncwarp();
        const int nc = min(4, p.n - col);  // valid columns for this lane (<= 0: none)
        float4 b4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (bias != nullptr && nc > 0) {
          b4.x = __ldg(bias + col);
          if (nc > 1) b4.y = __ldg(bias + col + 1);
          if (nc > 2) b4.z = __ldg(bias + col + 2);
          if (nc > 3) b4.w = __ldg(bias + col + 3);
        }
        // GELU' bias grad (kColsum): this lane's fp32 column sums over its 8 rows, in row order
        float2 cs01 = make_float2(0.f, 0.f), cs23 = make_float2(0.f, 0.f);
        auto acc_cs = [&](float4 w) {
          if constexpr (kColsum) {
            cs01 = __fadd2_rn(cs01, make_float2(w.x, w.y));
            cs23 = __fadd2_rn(cs23, make_float2(w.z, w.w));
          }
        };
        if (fast) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = 4 * i + rg;
            const float4 v = lds128f(stg + 4 * (rr * 32 + ((cg ^ (rr & 7)) << 2)));
            acc_cs(epi_store_fast<EPI>(p, v, x[i], grow0 + rr, col, b4, cbase, ldc));
          }
        } else {
#pragma unroll 2
          for (int i = 0; i < 8; ++i) {
            const int rr = 4 * i + rg;
            if (rr >= nrows || nc <= 0) continue;
            const float4 v = lds128f(stg + 4 * (rr * 32 + ((cg ^ (rr & 7)) << 2)));
            acc_cs(epilogue_vec4<EPI>(p, v, grow0 + rr, col, nc, row0 + rr >= zero_from, b4, cbase, ldc));
          }
        }
        if constexpr (kColsum) {
          {  // fixed-order tree over the 4 row groups -> the warp's 32 rows
#pragma unroll
            for (int o = 8; o <= 16; o <<= 1) {
              cs01 = __fadd2_rn(cs01, make_float2(__shfl_xor_sync(0xffffffffu, cs01.x, o),
                                                  __shfl_xor_sync(0xffffffffu, cs01.y, o)));
              cs23 = __fadd2_rn(cs23, make_float2(__shfl_xor_sync(0xffffffffu, cs23.x, o),
                                                  __shfl_xor_sync(0xffffffffu, cs23.y, o)));
            }
            const float4 cs = make_float4(cs01.x, cs01.y, cs23.x, cs23.y);
            if (rg == 0 && nc > 0) {
              float* dst = p.colsum + (grow0 >> 5) * p.n + col;
              if (nc == 4 && (p.n & 3) == 0) {
                *reinterpret_cast<float4*>(dst) = cs;
              } else {
                dst[0] = cs.x;
                if (nc > 1) dst[1] = cs.y;
                if (nc > 2) dst[2] = cs.z;
                if (nc > 3) dst[3] = cs.w;
              }
            }
          }
        }
        __syncwarp();
      }
      if (p.serial) {  // publish this split's additions, then hand the tile to the next split
        __threadfence();
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kEpiWarps) : "memory");
        if (warp == 4 && lane == 0) {
          if (T.ks == p.split_k - 1)
            atomicExch(ctr, 0);  // last split: the counter is clean for the next launch
          else
            atomicAdd(ctr, 1);
        }
      }
      tc_fence_before();
      if constexpr (CG == 2) {
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty_bar + acc, 0);  // the leader's barrier
      } else {
        mbar_arrive(tempty_bar + acc);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  if (warp >= 4 && lane == 0) bulk_wait_all();  // TMA stores done before the staging smem goes away
  tc_fence_before();
  if constexpr (CG == 2)
    cluster_sync();  // no CTA leaves while its peer may still signal or read it
  else
    __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 2)
      tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
    else
      tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// Deterministic split-K reduction: c (+)= sum_s ws[s] in split order.
// One block row per output row, float4 along the row (n % 4 == 0 fast path).
__global__ void splitk_reduce_kernel(float* c, int ldc, const float* ws, int m, int n, int splits,
                                     int accumulate) {
  pdl_trigger();
  pdl_wait();
  const long long total = static_cast<long long>(m) * n;
  const int r = blockIdx.x;
  if ((n & 3) == 0 && (ldc & 3) == 0) {
    for (int c4 = threadIdx.x; c4 < n / 4; c4 += blockDim.x) {
      const long long i = static_cast<long long>(r) * n + 4 * c4;
      float4 s = *reinterpret_cast<const float4*>(ws + i);
      for (int k = 1; k < splits; ++k) {
        const float4 q = *reinterpret_cast<const float4*>(ws + k * total + i);
        s.x += q.x;
        s.y += q.y;
        s.z += q.z;
        s.w += q.w;
      }
      float4* dst = reinterpret_cast<float4*>(c + static_cast<long long>(r) * ldc + 4 * c4);
      if (accumulate) {
        const float4 o = *dst;
        s = make_float4(o.x + s.x, o.y + s.y, o.z + s.z, o.w + s.w);
      }
      *dst = s;
    }
  } else {
    for (int col = threadIdx.x; col < n; col += blockDim.x) {
      const long long i = static_cast<long long>(r) * n + col;
      float s = ws[i];
      for (int k = 1; k < splits; ++k) s += ws[k * total + i];
      float* dst = c + static_cast<long long>(r) * ldc + col;
      *dst = accumulate ? (*dst + s) : s;
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

bool make_map(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld,
              uint32_t box_cols, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// bf16 [rows, cols] output, 32x32 boxes, 64-byte swizzle (the epilogue's staging layout)
bool make_store_map(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

thread_local void* g_ws = nullptr;  // per calling thread: shards on several host threads each pass their own
thread_local size_t g_ws_bytes = 0;

// zero-initialised split-K tile counters, one buffer per stream (GEMMs on one
// stream are ordered; different streams must not share counters)
int* split_counters(cudaStream_t s, int n) {
  static std::mutex mu;
  static std::vector<std::pair<cudaStream_t, std::pair<int*, int>>> bufs;
  std::lock_guard<std::mutex> lk(mu);
  for (auto& b : bufs)
    if (b.first == s && b.second.second >= n) return b.second.first;
  int cap = 1 << 14;
  while (cap < n) cap *= 2;
  int* ptr = nullptr;
  if (cudaMalloc(&ptr, static_cast<size_t>(cap) * sizeof(int)) != cudaSuccess) return nullptr;
  if (cudaMemset(ptr, 0, static_cast<size_t>(cap) * sizeof(int)) != cudaSuccess) return nullptr;
  for (auto& b : bufs)
    if (b.first == s) {
      b.second = {ptr, cap};  // (the smaller buffer is not in flight: same-stream GEMMs are ordered)
      return ptr;
    }
  bufs.push_back({s, {ptr, cap}});
  return ptr;
}

template <int BN, bool AMN, bool BMN, int EPI, int CG>
cudaError_t launch(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const CUtensorMap& tc2,
                   const GemmParams& p, cudaStream_t s) {
  using Cfg = GemmCfg<BN, CG>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemm_kernel<BN, AMN, BMN, EPI, CG>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  });
  if (attr_err != cudaSuccess) return attr_err;
  // persistent: one CTA (pair) per SM (pair of SMs) of this device, so every CTA is
  // co-resident (serial split-K's ordered in-place accumulation waits on earlier CTAs)
  const int units = device_sms() / CG;
  const int grid = CG * (p.tiles_total < units ? p.tiles_total : units);
  if constexpr (CG == 1) {
    const cudaError_t e = launch_k(gemm_kernel<BN, AMN, BMN, EPI, 1>, dim3(grid), dim3(kGemmThreads),
                                   Cfg::SMEM_BYTES, s, 1, ta, tb, tc, tc2, p);
    if (e != cudaSuccess) return e;
  } else {
    const cudaError_t e = launch_k(gemm_kernel<BN, AMN, BMN, EPI, 2>, dim3(grid), dim3(kGemmThreads),
                                   Cfg::SMEM_BYTES, s, 2, ta, tb, tc, tc2, p);
    if (e != cudaSuccess) return e;
  }
  count_launch();
  return cudaGetLastError();
}

template <int BN, bool AMN, bool BMN, int CG>
cudaError_t dispatch_epi(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc, const CUtensorMap& tc2,
                         const GemmParams& p, cudaStream_t s) {
  switch (p.epi) {
    case P2R_EPI_BF16: return launch<BN, AMN, BMN, P2R_EPI_BF16, CG>(ta, tb, tc, tc2, p, s);
    case P2R_EPI_F32: return launch<BN, AMN, BMN, P2R_EPI_F32, CG>(ta, tb, tc, tc2, p, s);
    case P2R_EPI_ACC_F32: return launch<BN, AMN, BMN, P2R_EPI_ACC_F32, CG>(ta, tb, tc, tc2, p, s);
    case P2R_EPI_BIAS_GELU: return launch<BN, AMN, BMN, P2R_EPI_BIAS_GELU, CG>(ta, tb, tc, tc2, p, s);
    case P2R_EPI_DGELU:
      if (p.colsum != nullptr) return launch<BN, AMN, BMN, P2R_EPI_DGELU | kEpiColsum, CG>(ta, tb, tc, tc2, p, s);
      return launch<BN, AMN, BMN, P2R_EPI_DGELU, CG>(ta, tb, tc, tc2, p, s);
    default: return launch<BN, AMN, BMN, P2R_EPI_F32_BF16, CG>(ta, tb, tc, tc2, p, s);
  }
}

template <int BN, int CG>
cudaError_t dispatch_majors(bool amn, bool bmn, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tc,
                            const CUtensorMap& tc2, const GemmParams& p, cudaStream_t s) {
  if (!amn && !bmn) return dispatch_epi<BN, false, false, CG>(ta, tb, tc, tc2, p, s);
  if (!amn && bmn) return dispatch_epi<BN, false, true, CG>(ta, tb, tc, tc2, p, s);
  if (amn && !bmn) return dispatch_epi<BN, true, false, CG>(ta, tb, tc, tc2, p, s);
  return dispatch_epi<BN, true, true, CG>(ta, tb, tc, tc2, p, s);
}

// CTA pairs for ungrouped 256-wide tiles unless the caller or P2R_GEMM_CG=1 says otherwise.
int pick_cg(const p2r_gemm_args* a, int BN) {
  if (a->group_mode != P2R_GROUP_NONE || BN != 256) return 1;
  if (a->cta_group == 1 || a->cta_group == 2) return a->cta_group;
  static const bool force1 = [] {
    const char* e = std::getenv("P2R_GEMM_CG");
    return e != nullptr && e[0] == '1';
  }();
  return force1 ? 1 : 2;
}

int pick_bn(const p2r_gemm_args* a) { return a->n <= 128 ? 128 : 256; }

int pick_cg(const p2r_gemm_args* a, int BN);

// split_k <= 0: choose the split (1..4) that best fills the persistent grid's
// waves; a split must beat one pass by > 10 points of wave efficiency to pay
// for its fp32 partials and the reduction.
int auto_split(const p2r_gemm_args* a) {
  if (a->epi != P2R_EPI_ACC_F32 && a->epi != P2R_EPI_F32) return 1;
  if (a->bias != nullptr || a->aux != nullptr) return 1;
  const int BN = pick_bn(a), CG = pick_cg(a, BN);
  const long long tiles = 1LL * ((a->m + BM * CG - 1) / (BM * CG)) * ((a->n + BN - 1) / BN);
  const int units = device_sms() / CG;
  auto eff = [&](int s) {
    const long long t = tiles * s;
    return static_cast<double>(t) / (static_cast<double>(units) * ((t + units - 1) / units));
  };
  int best = 1;
  for (int s = 2; s <= 4; ++s)
    if ((a->k / BK) / s >= 8 && eff(s) > eff(best) + 0.10) best = s;
  return best;
}

// C += A.B splits accumulate in place, in split order, when every split spans
// enough tiles to keep its read-modify-write wide (measured on the C2 dW
// shapes: 1024x3072 split 3 in place 44.6 us vs 48.9 with partials + reduce;
// 1024x1024 split 4 in place 37.0 vs 21.7). P2R_GEMM_SERIAL=0 disables it.
bool serial_split_ok(const p2r_gemm_args* a, int split) {
  static const bool on = [] {
    const char* e = std::getenv("P2R_GEMM_SERIAL");
    return e == nullptr || std::atoi(e) != 0;
  }();
  if (!on || split <= 1 || a->epi != P2R_EPI_ACC_F32 || a->bias != nullptr || a->aux != nullptr) return false;
  const int BN = pick_bn(a), CG = pick_cg(a, BN);
  const long long tiles = 1LL * ((a->m + BM * CG - 1) / (BM * CG)) * ((a->n + BN - 1) / BN);
  return tiles >= 32;
}

int effective_split(const p2r_gemm_args* a) {
  if (a->group_mode != P2R_GROUP_NONE || a->split_k == 1) return 1;
  const int req = a->split_k <= 0 ? auto_split(a) : a->split_k;
  const int nkb = (a->k + BK - 1) / BK;
  int s = req < nkb ? req : nkb;
  return s < 1 ? 1 : s;
}

}  // namespace
}  // namespace p2r

using namespace p2r;

extern "C" size_t p2r_gemm_workspace_bytes(const p2r_gemm_args* a) {
  if (a->bias_grad != nullptr) return static_cast<size_t>((a->m + 31) / 32) * a->n * sizeof(float);
  const int s = effective_split(a);
  if (s <= 1) return 0;
  if (serial_split_ok(a, s)) return 0;  // serial split-K accumulates in place
  return static_cast<size_t>(s) * a->m * a->n * sizeof(float);
}

extern "C" p2r_status p2r_set_workspace(void* ptr, size_t bytes) {
  g_ws = ptr;
  g_ws_bytes = bytes;
  return P2R_OK;
}

extern "C" p2r_status p2r_gemm(const p2r_gemm_args* a, void* stream) {
  if (a == nullptr) return set_error(P2R_EINVAL, "gemm: null args");
  if (a->m <= 0 || a->n <= 0 || a->k <= 0) {
    if (a->m < 0 || a->n < 0 || a->k < 0) return set_error(P2R_EINVAL, "matmul: negative dimension");
    if (a->m == 0 || a->n == 0 || a->epi == P2R_EPI_ACC_F32) return P2R_OK;  // empty C, or C += 0
    // k == 0 with a writing epilogue would need C = epilogue(0); no caller does that
    return set_error(P2R_EINVAL, "gemm: k == 0 is only defined for EPI_ACC_F32 (C += 0)");
  }
  if ((a->lda % 8) || (a->ldb % 8))
    return set_error(P2R_EINVAL, "gemm: leading dimensions must be multiples of 8 elements");
  if ((reinterpret_cast<uintptr_t>(a->a) & 15) || (reinterpret_cast<uintptr_t>(a->b) & 15))
    return set_error(P2R_EINVAL, "gemm: operands must be 16-byte aligned");
  if (a->group_mode != P2R_GROUP_NONE && (a->counts == nullptr || a->groups <= 0 ||
                                          a->seg_rows <= 0 || (a->seg_rows % BM) != 0))
    return set_error(P2R_EINVAL, "gemm: grouped GEMM needs counts and seg_rows % 128 == 0");
  if (a->group_mode == P2R_GROUP_M && a->a_mn_major)
    return set_error(P2R_EINVAL, "gemm: GROUP_M needs a K-major A");
  if (a->group_mode == P2R_GROUP_M && a->b_mn_major && (a->k % BK) != 0)
    return set_error(P2R_EINVAL, "gemm: GROUP_M with MN-major B needs k % 64 == 0");
  if (a->group_mode == P2R_GROUP_K && !(a->a_mn_major && a->b_mn_major))
    return set_error(P2R_EINVAL, "gemm: GROUP_K needs MN-major operands");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int BN = pick_bn(a);
  const int split = effective_split(a);
  if (a->cta_group == 2 && (a->group_mode != P2R_GROUP_NONE || BN != 256))
    return set_error(P2R_EINVAL, "gemm: CTA pairs need an ungrouped GEMM with n > 128");
  const int CG = pick_cg(a, BN);

  GemmParams p{};
  p.m = a->m;
  p.n = a->n;
  p.k = a->k;
  p.num_m_blk = (a->m + BM * CG - 1) / (BM * CG);
  p.num_n_blk = (a->n + BN - 1) / BN;
  p.num_k_blk = (a->k + BK - 1) / BK;
  p.epi = a->epi;
  p.c = a->c;
  p.ldc = a->ldc;
  p.c2 = a->c2;
  p.ldc2 = a->c2 ? a->ldc2 : 8;
  p.bias = a->bias;
  p.aux = a->aux;
  p.ldaux = a->aux ? a->ldaux : 8;
  p.group_mode = a->group_mode;
  p.groups = a->groups;
  p.seg_rows = a->seg_rows;
  p.counts = a->counts;
  p.split_k = split;
  if (a->bias_grad != nullptr) {
    if (a->epi != P2R_EPI_DGELU || a->group_mode != P2R_GROUP_NONE || split != 1)
      return set_error(P2R_EINVAL, "gemm: bias_grad needs EPI_DGELU, ungrouped, no split");
    if (g_ws == nullptr || g_ws_bytes < p2r_gemm_workspace_bytes(a))
      return set_error(P2R_ERUNTIME, "gemm: bias_grad workspace too small (p2r_gemm_workspace_bytes)");
    p.colsum = static_cast<float*>(g_ws);
  }
  const bool serial = split > 1 && serial_split_ok(a, split);
  if (serial) {
    p.serial = 1;
    p.counters = split_counters(s, p.num_m_blk * p.num_n_blk * CG);
    if (p.counters == nullptr) return set_error(P2R_ECUDA, "gemm: split-K counters allocation failed");
  } else if (split > 1) {
    if (a->epi != P2R_EPI_ACC_F32 && a->epi != P2R_EPI_F32)
      return set_error(P2R_EINVAL, "gemm: split-K only for fp32 outputs");
    if (a->bias != nullptr || a->aux != nullptr)
      return set_error(P2R_EINVAL, "gemm: split-K does not support bias/aux");
    const size_t need = static_cast<size_t>(split) * a->m * a->n * sizeof(float);
    if (g_ws == nullptr || g_ws_bytes < need)
      return set_error(P2R_ERUNTIME, "gemm: split-K workspace too small");
    p.c = g_ws;
    p.ldc = a->n;
    p.epi = P2R_EPI_F32;
    p.c_split_stride = static_cast<long long>(a->m) * a->n;
  }
  {
    auto al = [](const void* q, uintptr_t b) { return (reinterpret_cast<uintptr_t>(q) % b) == 0; };
    p.vec4 = (p.ldc % 4 == 0) && (p.ldc2 % 4 == 0) && (p.ldaux % 4 == 0) && al(p.c, 16) && al(p.c2, 8) &&
             al(p.aux, 16);
  }
  {
    static const int raster = [] {
      const char* e = std::getenv("P2R_GEMM_RASTER");
      const int v = e ? std::atoi(e) : 0;
      return v > 0 ? v : 8;
    }();
    p.raster_g = raster < p.num_m_blk ? raster : p.num_m_blk;
  }
  if (a->group_mode == P2R_GROUP_M)
    p.tiles_total = a->groups * (a->seg_rows / BM) * p.num_n_blk;
  else if (a->group_mode == P2R_GROUP_K)
    p.tiles_total = a->groups * p.num_m_blk * p.num_n_blk;
  else
    p.tiles_total = p.num_m_blk * p.num_n_blk * split;

  // Tensor maps (rows x cols, row-major, ld in elements).
  CUtensorMap ta, tb;
  const long long a_rows_mn = a->group_mode == P2R_GROUP_K ? 1LL * a->groups * a->seg_rows : a->k;
  const long long a_rows_k = a->group_mode == P2R_GROUP_M ? 1LL * a->groups * a->seg_rows : a->m;
  const long long b_rows_k = a->group_mode == P2R_GROUP_M ? 1LL * a->groups * a->n : a->n;
  bool ok = a->a_mn_major ? make_map(&ta, a->a, a_rows_mn, a->m, a->lda, 64, 64)
                          : make_map(&ta, a->a, a_rows_k, a->k, a->lda, 64, BM);
  const long long b_rows_mn = a->group_mode == P2R_GROUP_M ? 1LL * a->groups * a->k : a_rows_mn;
  ok = ok && (a->b_mn_major ? make_map(&tb, a->b, b_rows_mn, a->n, a->ldb, 64, 64)
                            : make_map(&tb, a->b, b_rows_k, a->k, a->ldb, 64, BN / CG));
  if (!ok) return set_error(P2R_ECUDA, "gemm: cuTensorMapEncodeTiled failed");

  // bf16 epilogues store through TMA when the outputs are TMA-addressable
  CUtensorMap tc{}, tc2{};
  {
    static const bool tma_on = [] {
      const char* e = std::getenv("P2R_GEMM_TMA_STORE");
      return e == nullptr || std::atoi(e) != 0;
    }();
    auto a16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) % 16) == 0; };
    // (GELU' keeps the per-thread path: its operand prefetch one chunk ahead measured faster)
    const bool bf16_epi = a->epi == P2R_EPI_BF16 || a->epi == P2R_EPI_BIAS_GELU;
    bool t = tma_on && bf16_epi && split == 1 && a->group_mode != P2R_GROUP_K && a->ldc % 8 == 0 && a16(a->c) &&
             (a->bias == nullptr || a16(a->bias));
    if (a->epi == P2R_EPI_BIAS_GELU) t = t && a->ldc2 % 8 == 0 && a16(a->c2);
    if (a->epi == P2R_EPI_DGELU) t = t && a->ldaux % 8 == 0 && a16(a->aux);
    const long long out_rows = a->group_mode == P2R_GROUP_M ? 1LL * a->groups * a->seg_rows : a->m;
    if (t) t = make_store_map(&tc, a->c, out_rows, a->n, a->ldc);
    if (t && a->epi == P2R_EPI_BIAS_GELU) t = make_store_map(&tc2, a->c2, out_rows, a->n, a->ldc2);
    p.tma_c = t ? 1 : 0;
  }

  cudaError_t e = BN == 128 ? dispatch_majors<128, 1>(a->a_mn_major, a->b_mn_major, ta, tb, tc, tc2, p, s)
                 : CG == 2  ? dispatch_majors<256, 2>(a->a_mn_major, a->b_mn_major, ta, tb, tc, tc2, p, s)
                            : dispatch_majors<256, 1>(a->a_mn_major, a->b_mn_major, ta, tb, tc, tc2, p, s);
  if (e != cudaSuccess) return set_cuda_error(e, "gemm launch");
  if (a->bias_grad != nullptr) {  // bias_grad += sum of the per-32-row partials, in row-block order
    e = colsum_finish_launch(static_cast<const float*>(g_ws), (a->m + 31) / 32, a->n, 1, a->bias_grad, 0, s);
    count_launch();
    if (e != cudaSuccess) return set_cuda_error(e, "bias grad finish launch");
  }
  if (split > 1 && !serial) {
    e = launch_k(splitk_reduce_kernel, dim3(a->m), dim3(256), 0, s, 1, static_cast<float*>(a->c), a->ldc,
                 static_cast<const float*>(g_ws), a->m, a->n, split, a->epi == P2R_EPI_ACC_F32 ? 1 : 0);
    count_launch();
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "splitk reduce launch");
  }
  return P2R_OK;
}
