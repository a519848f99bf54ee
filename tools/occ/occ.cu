// Max co-resident clusters for a kernel shape (threads, dynamic smem, cluster size), via
// cudaOccupancyMaxActiveClusters.  usage: occ <threads> <smem_bytes> <cluster> [<cluster> ...]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void dummy(float* p) {
  extern __shared__ float s[];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (p) p[threadIdx.x] = s[(threadIdx.x + 1) % blockDim.x];
}

int main(int argc, char** argv) {
  const int threads = atoi(argv[1]), smem = atoi(argv[2]);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int i = 3; i < argc; ++i) {
    const int cl = atoi(argv[i]);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl, 1024, 1);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
    int blk = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blk, dummy, threads, smem);
    printf("threads %d smem %d cluster %2d: max active clusters %d (%d CTAs; %d CTAs/SM alone) %s\n", threads, smem,
           cl, n, n * cl, blk, cudaGetErrorString(e));
  }
  return 0;
}
