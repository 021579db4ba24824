// Microbenchmark: cycles per tcgen05.mma (kind::f16, cta_group::1, SS operands,
// SWIZZLE_128B K-major) vs N, one CTA per SM, back-to-back issue from one thread.
// Optional concurrent load: 8 warps doing tcgen05.ld of the accumulator region
// (models the attention softmax warps reading S/dP from TMEM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2110_03888_b200/csrc scripts/micro/mma_rate.cu -o build/mma_rate
#include <cstdio>
#include <cstdint>
#include "common.cuh"
using namespace p2r;

template <int N>
__global__ void __launch_bounds__(384, 1) k_mma(long long* out, int iters, int ldtm, int a_mn, int fresh = 0, int b_mn = 0) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 2) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // A: 128 rows x 64 K (16 KB), B: N rows x 64 K; `fresh` cycles through 4 distinct A/B slabs
  const uint32_t sa0 = smem_u32(smem), sbb0 = sa0 + 4 * 128 * 128;
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  if (warp == 1 && lane == 0) {
    const uint32_t idesc = make_idesc_bf16(128, N, a_mn != 0, b_mn != 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t sa = sa0 + (fresh ? (it & 3) * 128 * 128 : 0), sbb = sbb0 + (fresh ? (it & 3) * N * 128 : 0);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = a_mn ? make_sw128_desc(sa + k * 2048, 64 * 64 * 2, 1024) : make_sw128_desc(sa + k * 32, 16, 1024);
        const uint64_t bd = b_mn ? make_sw128_desc(sbb + k * 2048, 64 * 64 * 2, 1024) : make_sw128_desc(sbb + k * 32, 16, 1024);
        umma_bf16(tmem + (it & 1) * 256, ad, bd, idesc, k > 0 ? 1u : 0u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    done = 1;
  } else if (warp >= 4 && ldtm) {
    const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const int half = (warp - 4) >> 2;
    float acc = 0.f;
    while (!done) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + la + 256 + half * 32, r);
      tmem_ld_wait();
      acc += __uint_as_float(r[lane]);
    }
    if (acc == 12345.f) out[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N>
void run(long long* d, int ldtm, int a_mn, int fresh = 0, int b_mn = 0) {
  const int iters = 2000, smem = 4 * 128 * 128 + 4 * N * 128 + 2048;
  cudaFuncSetAttribute(k_mma<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_mma<N><<<148, 384, smem>>>(d, iters, ldtm, a_mn, fresh, b_mn);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double per = avg / (iters * 4.0);
  printf("M=128 N=%3d K=16 %s%s%s%s: %6.1f cyc/MMA (floor %d)  -> %.0f MAC/clk/SM\n", N, a_mn ? "A MN-major" : "A K-major ",
         b_mn ? " B MN-major" : "", fresh ? " fresh operands" : "", ldtm ? " + 8 warps tcgen05.ld" : "", per, 128 * N / 256,
         128.0 * N * 16 / per);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  for (int l = 0; l < 2; ++l) {
    run<64>(d, l, 0);
    run<128>(d, l, 0);
    run<256>(d, l, 0);
  }
  run<64>(d, 0, 1);
  run<128>(d, 0, 1);
  run<64>(d, 0, 0, 1);
  run<128>(d, 0, 0, 1);
  run<256>(d, 0, 0, 1);
  run<64>(d, 0, 0, 1, 1);
  run<64>(d, 1, 0, 1);
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
