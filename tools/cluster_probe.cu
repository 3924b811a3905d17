// How many thread-block clusters of each size are co-resident on this GPU
// when every CTA needs a whole SM (K4's narrow variant: ~193 KiB of shared
// memory per CTA). Diagnostic for plan_attention's split/cluster choice.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/cluster_probe.cu -o build/cluster_probe
//   build/cluster_probe
#include <cstdio>

__global__ void probe_kernel(int* out) {
  extern __shared__ int smem[];
  smem[threadIdx.x] = threadIdx.x;
  if (threadIdx.x == 0 && out) out[blockIdx.x] = smem[0];
}

int main() {
  const int smem = 193 * 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"sms\": %d, \"max_active_clusters\": {", sms);
  for (int s = 1; s <= 16; ++s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(s * 16);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = s;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe_kernel, &cfg);
    printf("%s\"%d\": %d", s > 1 ? ", " : "", s, e == cudaSuccess ? n : -1);
  }
  printf("}}\n");
  return 0;
}
