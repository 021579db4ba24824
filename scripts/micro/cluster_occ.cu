// How many thread-block clusters of size 1/2/4/8 can be co-resident on this GPU
// with the GEMM's launch shape (384 threads, ~225 KB dynamic smem, 1 CTA/SM)?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/micro/cluster_occ.cu -o build/cluster_occ
#include <cstdio>
__global__ void k_dummy(int* p) { if (p && threadIdx.x == 0) p[blockIdx.x] = 1; }
int main() {
  const int smem = 230656;
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  printf("%s SMs=%d\n", prop.name, prop.multiProcessorCount);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cs;
    a[0].val.clusterDim.y = 1;
    a[0].val.clusterDim.z = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
    printf("cluster %2d: max active clusters %4d (%4d CTAs) %s\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  return 0;
}
