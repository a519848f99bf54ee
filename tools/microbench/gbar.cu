// Grid-barrier latency microbenchmark (design input for the persistent PCG kernel):
// P co-resident CTAs (cooperative launch) run `iters` barriers on one counter.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MODE>
__global__ void kbar(unsigned* ctr, int iters, double* partial, double* sink) {
  unsigned target = 0;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 1 && threadIdx.x == 0) partial[blockIdx.x] = it + blockIdx.x;
    __syncthreads();
    if (threadIdx.x == 0) {
      target += gridDim.x;
      if (MODE == 2) { __threadfence(); atomicAdd(ctr, 1u); } else red_rel(ctr, 1u);
      while (ld_acq(ctr) < target) {}
    }
    __syncthreads();
    if (MODE == 1 && threadIdx.x < 32) {  // every CTA sums all partials (fixed order)
      double s = 0;
      for (int i = threadIdx.x; i < gridDim.x; i += 32) s += __ldcg(partial + i);
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
      acc += s;
    }
    if (MODE == 1) __syncthreads();  // partial reuse next iteration
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = acc;
}

int main() {
  unsigned* ctr;
  double *part, *sink;
  cudaMalloc(&ctr, 4);
  cudaMalloc(&part, 8 * 1024);
  cudaMalloc(&sink, 8 * 1024);
  const int iters = 20000;
  for (int mode = 0; mode < 3; ++mode)
    for (int P : {128, 148, 256, 296}) {
      cudaMemset(ctr, 0, 4);
      void* args[] = {&ctr, (void*)&iters, &part, &sink};
      int it2 = iters;
      args[1] = &it2;
      void (*k)(unsigned*, int, double*, double*) = mode == 0 ? kbar<0> : (mode == 1 ? kbar<1> : kbar<2>);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaLaunchCooperativeKernel((void*)k, P, 192, args, 0, 0);  // warm
      cudaMemset(ctr, 0, 4);
      cudaEventRecord(e0);
      cudaError_t e = cudaLaunchCooperativeKernel((void*)k, P, 192, args, 0, 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("mode %d (%s) P=%d: %s  %.3f us per barrier\n", mode,
             mode == 0 ? "red.release/ld.acquire" : (mode == 1 ? "+partials sum" : "threadfence+atomicAdd"), P,
             cudaGetErrorString(e), 1e3 * ms / iters);
    }
  return 0;
}
