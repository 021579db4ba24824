// tcgen05.mma (kind::f16, cta_group::1, SS) rate with FRESH operands per MMA and
// cheap issue: the whole warp runs the loop (uniform descriptors), one elected
// lane issues; 4 distinct A/B slabs with compile-time descriptor offsets.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2110_03888_b200/csrc scripts/micro/mma_rate2.cu -o build/mma_rate2
#include <cstdio>
#include <cstdint>
#include "common.cuh"
using namespace p2r;

template <int N, bool BMN>
__global__ void __launch_bounds__(128, 1) k_mma(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 2) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t sa = smem_u32(smem), sbb = sa + 4 * 16384;
  if (warp == 1) {
    const uint32_t idesc = make_idesc_bf16(128, N, false, BMN);
    const uint64_t a0 = make_sw128_desc(sa, 16, 1024);
    const uint64_t b0 = BMN ? make_sw128_desc(sbb, 64 * 64 * 2, 1024) : make_sw128_desc(sbb, 16, 1024);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int slab = 0; slab < 4; ++slab)
#pragma unroll
        for (int k = 0; k < 4; ++k)
          umma_bf16_warp(tmem + (slab & 1) * 256, a0 + ((slab * 16384 + k * 32) >> 4),
                         b0 + ((slab * N * 128 + k * (BMN ? 2048 : 32)) >> 4), idesc, k > 0 ? 1u : 0u);
    }
    umma_commit_warp(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool BMN>
void run(long long* d) {
  const int iters = 500, smem = 4 * 16384 + 4 * N * 128 + 2048;
  cudaFuncSetAttribute(k_mma<N, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_mma<N, BMN><<<148, 128, smem>>>(d, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += h[i];
  avg /= 148;
  const double per = avg / (iters * 16.0);
  printf("M=128 N=%3d K=16 fresh operands, warp-elect issue%s: %6.1f cyc/MMA (floor %d)\n", N, BMN ? ", B MN-major" : "",
         per, 128 * N / 256);
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  run<64, false>(d);
  run<64, true>(d);
  run<128, false>(d);
  run<256, false>(d);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
