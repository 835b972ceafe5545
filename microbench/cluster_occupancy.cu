// How many 2-CTA clusters of the RNS kernel's shape (320 threads, ~193 KB of
// dynamic shared memory, one CTA per SM) can be co-resident on this GPU?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 cluster_occupancy.cu -o cluster_occupancy
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1) k_pair(int* out) {
  extern __shared__ unsigned char smem[];
  if (threadIdx.x == 0 && smem[0] == 123) out[blockIdx.x] = 1;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int smem : {192 * 1024 + 1024, 160 * 1024, 100 * 1024}) {
    cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(sms / 2 * 2);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2, attr.val.clusterDim.y = 1, attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int clusters = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&clusters, k_pair, &cfg);
    printf("SMs %d, smem %d B: max active 2-CTA clusters %d (%s)\n", sms, smem, clusters, cudaGetErrorString(e));
  }
  return 0;
}
