// How many thread-block clusters of a given shape fit on this GPU at once
// (development aid for the 64-bit 2^15/2^16 cluster transforms):
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/co tools/cluster_occupancy.cu && /tmp/co
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dummy(int* p) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0];
}

int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = 139 * 1024 + 264;  // a 2^14-word 64-bit tile
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cl : {1, 2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl * 64);
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cl;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
    printf("SMs %d, cluster %d x 1024 threads, %zu B smem: max active clusters %d (%d SMs busy) %s\n",
           sms, cl, smem, n, n * cl, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
