// Probe: how many 2-CTA clusters with the attention kernel's footprint can be co-resident on this
// GPU (cudaOccupancyMaxActiveClusters) -- the wave size the pair kernel's grid math assumes (SMs/2).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1) k(int* x) {
  extern __shared__ int s[];
  if (x) x[blockIdx.x] = s[threadIdx.x];
}
int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int smem : {100 * 1024, 180 * 1024, 200 * 1024, 220 * 1024}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * 148);
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("SMs %d  smem %d KB: max active 2-CTA clusters %d (%s)\n", sms, smem / 1024, n, cudaGetErrorString(e));
  }
  return 0;
}
