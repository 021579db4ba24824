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
#include <cstring>
#include <mutex>

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
};

struct Tile {
  bool valid;
  int m_blk, n_blk;
  int a_row;    // K-major A: first row (m)
  int b_row;    // K-major B: first row (n)
  int kbase;    // MN-major operands: first K row
  int kb0, kb1; // k-block range
  int g;
  int ks;
};

P2R_DEVICE Tile get_tile(const GemmParams& p, int t, int BN) {
  Tile T;
  T.valid = true;
  T.g = 0;
  T.ks = 0;
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
    T.kbase = T.g * p.seg_rows;
    T.kb0 = 0;
    T.kb1 = (cnt + BK - 1) / BK;
  } else {
    const int per_s = p.num_m_blk * p.num_n_blk;
    T.ks = t / per_s;
    const int r = t - T.ks * per_s;
    T.n_blk = r / p.num_m_blk;
    T.m_blk = r - T.n_blk * p.num_m_blk;
    T.a_row = T.m_blk * BM;
    T.b_row = T.n_blk * BN;
    T.kbase = 0;
    T.kb0 = static_cast<int>((static_cast<long long>(T.ks) * p.num_k_blk) / p.split_k);
    T.kb1 = static_cast<int>((static_cast<long long>(T.ks + 1) * p.num_k_blk) / p.split_k);
    T.valid = T.kb1 > T.kb0;
  }
  return T;
}

template <int BN>
struct GemmCfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (196608 / STAGE_BYTES) > 8 ? 8 : (196608 / STAGE_BYTES);
  static constexpr int TMEM_COLS = (2 * BN) < 32 ? 32 : (2 * BN);
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

P2R_DEVICE void store_bf16x32(__nv_bfloat16* dst, const float* v) {
  uint32_t w[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    w[j] = *reinterpret_cast<uint32_t*>(&h);
  }
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int j = 0; j < 4; ++j) d[j] = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
}
P2R_DEVICE void store_f32x32(float* dst, const float* v) {
  float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
  for (int j = 0; j < 8; ++j) d[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
}
P2R_DEVICE void load_f32x32(const float* src, float* v) {
  const float4* s = reinterpret_cast<const float4*>(src);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float4 q = s[j];
    v[4 * j] = q.x;
    v[4 * j + 1] = q.y;
    v[4 * j + 2] = q.z;
    v[4 * j + 3] = q.w;
  }
}
P2R_DEVICE void load_bf16x32(const __nv_bfloat16* src, float* v) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4 q = s[j];
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
      float2 f = __bfloat1622float2(h);
      v[8 * j + 2 * i] = f.x;
      v[8 * j + 2 * i + 1] = f.y;
    }
  }
}

// Epilogue for one 32-column chunk of one row. `zero_row` stores zeros (padding
// rows of a grouped segment) so later grouped-K GEMMs see clean padding.
P2R_DEVICE void epilogue_chunk(const GemmParams& p, float* v, long long row, int col0, int ncols,
                               bool vec_ok, char* cbase, int ldc, bool zero_row,
                               const float* bias) {
  const int epi = p.epi;
  if (zero_row) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = 0.0f;
  } else {
    if (bias != nullptr && (epi == P2R_EPI_BF16 || epi == P2R_EPI_F32 || epi == P2R_EPI_BIAS_GELU ||
                              epi == P2R_EPI_F32_BF16)) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] += (j < ncols) ? __ldg(bias + col0 + j) : 0.0f;
    }
  }
  if (epi == P2R_EPI_BF16) {
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(cbase) + row * ldc + col0;
    if (vec_ok) {
      store_bf16x32(dst, v);
    } else {
      for (int j = 0; j < ncols; ++j) dst[j] = __float2bfloat16_rn(v[j]);
    }
  } else if (epi == P2R_EPI_F32 || epi == P2R_EPI_F32_BF16) {
    float* dst = reinterpret_cast<float*>(cbase) + row * ldc + col0;
    if (p.aux != nullptr && !zero_row) {
      const float* src = reinterpret_cast<const float*>(p.aux) + row * p.ldaux + col0;
      if (vec_ok) {
        float a[32];
        load_f32x32(src, a);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += a[j];
      } else {
        for (int j = 0; j < ncols; ++j) v[j] += src[j];
      }
    }
    if (vec_ok) {
      store_f32x32(dst, v);
    } else {
      for (int j = 0; j < ncols; ++j) dst[j] = v[j];
    }
    if (epi == P2R_EPI_F32_BF16) {
      __nv_bfloat16* d2 = reinterpret_cast<__nv_bfloat16*>(p.c2) + row * p.ldc2 + col0;
      if (vec_ok) {
        store_bf16x32(d2, v);
      } else {
        for (int j = 0; j < ncols; ++j) d2[j] = __float2bfloat16_rn(v[j]);
      }
    }
  } else if (epi == P2R_EPI_ACC_F32) {
    float* dst = reinterpret_cast<float*>(cbase) + row * ldc + col0;
    if (vec_ok) {
      float a[32];
      load_f32x32(dst, a);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = a[j] + v[j];
      store_f32x32(dst, v);
    } else {
      for (int j = 0; j < ncols; ++j) dst[j] = dst[j] + v[j];
    }
  } else if (epi == P2R_EPI_BIAS_GELU) {
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(cbase) + row * ldc + col0;
    __nv_bfloat16* d2 = reinterpret_cast<__nv_bfloat16*>(p.c2) + row * p.ldc2 + col0;
    float gv[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) gv[j] = gelu_f(v[j]);
    if (vec_ok) {
      store_bf16x32(d2, v);
      store_bf16x32(dst, gv);
    } else {
      for (int j = 0; j < ncols; ++j) {
        d2[j] = __float2bfloat16_rn(v[j]);
        dst[j] = __float2bfloat16_rn(gv[j]);
      }
    }
  } else if (epi == P2R_EPI_DGELU) {
    __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(cbase) + row * ldc + col0;
    const __nv_bfloat16* pre = reinterpret_cast<const __nv_bfloat16*>(p.aux) + row * p.ldaux + col0;
    if (vec_ok) {
      float a[32];
      load_bf16x32(pre, a);
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = zero_row ? 0.0f : v[j] * gelu_grad_f(a[j]);
      store_bf16x32(dst, v);
    } else {
      for (int j = 0; j < ncols; ++j)
        dst[j] = __float2bfloat16_rn(zero_row ? 0.0f : v[j] * gelu_grad_f(__bfloat162float(pre[j])));
    }
  }
}

template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(256, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const GemmParams p) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar + s, 1);
      mbar_init(empty_bar + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(tfull_bar + s, 1);
      mbar_init(tempty_bar + s, 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.tiles_total; t += gridDim.x) {
        const Tile T = get_tile(p, t, BN);
        if (!T.valid) continue;
        for (int kb = T.kb0; kb < T.kb1; ++kb) {
          mbar_wait(empty_bar + stage, phase ^ 1);
          uint8_t* sa = smem + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          mbar_arrive_expect_tx(full_bar + stage, Cfg::STAGE_BYTES);
          if (!A_MN) {
            tma_load_2d(sa, &tmA, full_bar + stage, kb * BK, T.a_row);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_2d(sa + j * 64 * BK * 2, &tmA, full_bar + stage, T.m_blk * BM + 64 * j,
                          T.kbase + kb * BK);
          }
          if (!B_MN) {
            tma_load_2d(sb, &tmB, full_bar + stage, kb * BK, T.b_row);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_2d(sb + j * 64 * BK * 2, &tmB, full_bar + stage, T.n_blk * BN + 64 * j,
                          T.kbase + kb * BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idesc = make_idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < p.tiles_total; t += gridDim.x) {
        const Tile T = get_tile(p, t, BN);
        if (!T.valid) continue;
        mbar_wait(tempty_bar + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = T.kb0; kb < T.kb1; ++kb) {
          mbar_wait(full_bar + stage, phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // K-major: advance 16 elems = 32 B inside the swizzle row.
            // MN-major: advance 16 K-rows = 2048 B.
            const uint64_t ad = A_MN ? make_sw128_desc(sa + kk * 2048, 64 * BK * 2, 1024)
                                     : make_sw128_desc(sa + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_sw128_desc(sb + kk * 2048, 64 * BK * 2, 1024)
                                     : make_sw128_desc(sb + kk * 32, 16, 1024);
            umma_bf16(d_tmem, ad, bd, idesc, (kb > T.kb0 || kk > 0) ? 1u : 0u);
          }
          umma_commit(empty_bar + stage);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(tfull_bar + acc);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int ew = warp - 4;  // == warp % 4 -> TMEM lanes [32*ew, 32*ew+32)
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < p.tiles_total; t += gridDim.x) {
      const Tile T = get_tile(p, t, BN);
      if (!T.valid) continue;
      mbar_wait(tfull_bar + acc, acc_phase);
      tc_fence_after();
      const int local_row = T.m_blk * BM + ew * 32 + lane;
      long long row;
      bool row_ok, zero_row = false;
      char* cbase = reinterpret_cast<char*>(p.c);
      int ldc = p.ldc;
      const float* bias = p.bias;
      if (p.group_mode == P2R_GROUP_M) {
        row = static_cast<long long>(T.g) * p.seg_rows + local_row;
        row_ok = local_row < p.seg_rows;
        zero_row = local_row >= __ldg(p.counts + T.g);
        if (bias != nullptr) bias += static_cast<long long>(T.g) * p.n;
      } else if (p.group_mode == P2R_GROUP_K) {
        row = local_row;
        row_ok = local_row < p.m;
        cbase += static_cast<long long>(T.g) * p.m * p.ldc * 4;  // fp32 grads
      } else {
        row = local_row;
        row_ok = local_row < p.m;
        if (p.split_k > 1) cbase += static_cast<long long>(T.ks) * p.c_split_stride * 4;
      }
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        tmem_ld_wait();
        const int col0 = T.n_blk * BN + c * 32;
        if (row_ok && col0 < p.n) {
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          const int ncols = min(32, p.n - col0);
          const bool vec_ok = (ncols == 32) && ((ldc & 7) == 0) && ((p.ldc2 & 7) == 0) &&
                              ((p.ldaux & 7) == 0);
          epilogue_chunk(p, v, row, col0, ncols, vec_ok, cbase, ldc, zero_row, bias);
        }
      }
      tc_fence_before();
      mbar_arrive(tempty_bar + acc);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// Deterministic split-K reduction: c (+)= sum_s ws[s] in split order.
__global__ void splitk_reduce_kernel(float* c, int ldc, const float* ws, int m, int n, int splits,
                                     int accumulate) {
  const long long total = static_cast<long long>(m) * n;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / n), col = static_cast<int>(i % n);
    float s = ws[i];
    for (int k = 1; k < splits; ++k) s += ws[k * total + i];
    float* dst = c + static_cast<long long>(r) * ldc + col;
    *dst = accumulate ? (*dst + s) : s;
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

void* g_ws = nullptr;
size_t g_ws_bytes = 0;

template <int BN, bool AMN, bool BMN>
cudaError_t launch(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                   cudaStream_t s) {
  using Cfg = GemmCfg<BN>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemm_kernel<BN, AMN, BMN>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  });
  if (attr_err != cudaSuccess) return attr_err;
  const int grid = p.tiles_total < kNumSMs ? p.tiles_total : kNumSMs;
  gemm_kernel<BN, AMN, BMN><<<grid, 256, Cfg::SMEM_BYTES, s>>>(ta, tb, p);
  count_launch();
  return cudaGetLastError();
}

template <int BN>
cudaError_t dispatch_majors(bool amn, bool bmn, const CUtensorMap& ta, const CUtensorMap& tb,
                            const GemmParams& p, cudaStream_t s) {
  if (!amn && !bmn) return launch<BN, false, false>(ta, tb, p, s);
  if (!amn && bmn) return launch<BN, false, true>(ta, tb, p, s);
  if (amn && !bmn) return launch<BN, true, false>(ta, tb, p, s);
  return launch<BN, true, true>(ta, tb, p, s);
}

int pick_bn(const p2r_gemm_args* a) { return a->n <= 128 ? 128 : 256; }

int effective_split(const p2r_gemm_args* a) {
  if (a->group_mode != P2R_GROUP_NONE || a->split_k <= 1) return 1;
  const int nkb = (a->k + BK - 1) / BK;
  int s = a->split_k < nkb ? a->split_k : nkb;
  return s < 1 ? 1 : s;
}

}  // namespace
}  // namespace p2r

using namespace p2r;

extern "C" size_t p2r_gemm_workspace_bytes(const p2r_gemm_args* a) {
  const int s = effective_split(a);
  if (s <= 1) return 0;
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
    if (a->m >= 0 && a->n >= 0 && a->k >= 0) return P2R_OK;  // empty product: nothing to do
    return set_error(P2R_EINVAL, "matmul: negative dimension");
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

  GemmParams p{};
  p.m = a->m;
  p.n = a->n;
  p.k = a->k;
  p.num_m_blk = (a->m + BM - 1) / BM;
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
  if (split > 1) {
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
                            : make_map(&tb, a->b, b_rows_k, a->k, a->ldb, 64, BN));
  if (!ok) return set_error(P2R_ECUDA, "gemm: cuTensorMapEncodeTiled failed");

  cudaError_t e = BN == 128 ? dispatch_majors<128>(a->a_mn_major, a->b_mn_major, ta, tb, p, s)
                            : dispatch_majors<256>(a->a_mn_major, a->b_mn_major, ta, tb, p, s);
  if (e != cudaSuccess) return set_cuda_error(e, "gemm launch");
  if (split > 1) {
    const long long total = 1LL * a->m * a->n;
    int blocks = static_cast<int>((total + 255) / 256);
    if (blocks > 4 * kNumSMs) blocks = 4 * kNumSMs;
    splitk_reduce_kernel<<<blocks, 256, 0, s>>>(static_cast<float*>(a->c), a->ldc,
                                                  static_cast<const float*>(g_ws), a->m, a->n,
                                                  split, a->epi == P2R_EPI_ACC_F32 ? 1 : 0);
    count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) return set_cuda_error(e, "splitk reduce launch");
  }
  return P2R_OK;
}
