// How many thread-block clusters of size CL can be co-resident on this GPU for
// a 1-CTA-per-SM kernel (256 threads, ~176 KB shared memory)?  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -o cluster_occupancy cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 1) dummy(float* p) {
  extern __shared__ float s[];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (p) p[threadIdx.x] = s[255 - threadIdx.x];
}

int main() {
  int smem = 176 * 1024;
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cl : {1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 12, 14, 16}) {
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.gridDim = dim3(cl * 1024);
    lc.blockDim = dim3(256);
    lc.dynamicSmemBytes = smem;
    lc.attrs = at;
    lc.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)dummy, &lc);
    printf("cluster %2d: max active clusters %d -> %d CTAs (%s)\n", cl, n, n * cl, cudaGetErrorString(e));
  }
  return 0;
}
