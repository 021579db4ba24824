// Microbenchmark: aggregate tcgen05.ld throughput (bytes/cycle/SM) with W warps
// each loading 32 lanes x 32 columns (32x32b.x32, 4 KB per warp-instruction).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2110_03888_b200/csrc scripts/micro/tmem_ld_rate.cu -o build/tmem_ld_rate
#include <cstdio>
#include <cstdint>
#include "common.cuh"
using namespace p2r;

__global__ void __launch_bounds__(512, 1) k_ld(long long* out, int iters, int nwarps, int wait_each) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  float acc = 0.f;
  long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t la = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t col = (warp >> 2) * 32;
    for (int it = 0; it < iters; ++it) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + la + ((col + it * 64) & 511), r);
      if (wait_each || (it & 3) == 3) tmem_ld_wait();
      acc += __uint_as_float(r[it & 31]);
    }
    tmem_ld_wait();
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 1234.5f) out[1] = 0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int iters = 4096;
  for (int wait_each = 1; wait_each >= 0; --wait_each)
    for (int nw : {4, 8, 16}) {
      k_ld<<<148, 512>>>(d, iters, nw, wait_each);
      cudaDeviceSynchronize();
      long long h[148];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      const double bytes = 4096.0 * iters * nw;
      printf("warps=%2d wait_each=%d: %8.1f bytes/cycle/SM\n", nw, wait_each, bytes / avg);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
