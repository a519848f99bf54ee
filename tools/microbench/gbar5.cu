// Grid barrier with the arrivals spread over NC counters (separate 128-byte lines): each CTA
// adds to counter (cta % NC); the poll loads all NC counters.  Fences as in k_persist.cu.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rlx(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

template <int NC, bool FENCE>
__global__ void kb(unsigned* ctr, int iters, double* sink) {
  unsigned gen = 0;
  const int P = gridDim.x;
  for (int it = 0; it < iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      ++gen;
      if (FENCE) fence();
      red_rlx(ctr + 32 * (blockIdx.x % NC), 1u);
      bool done;
      do {
        done = true;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const unsigned need = gen * (unsigned)((P - c + NC - 1) / NC);
          done &= ld_rlx(ctr + 32 * c) >= need;
        }
      } while (!done);
      if (FENCE) fence();
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = gen;
}

template <int NC, bool FENCE>
void run(unsigned* ctr, double* sink, int P) {
  const int iters = 20000;
  int it2 = iters;
  void* args[] = {&ctr, &it2, &sink};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  cudaError_t e = cudaSuccess;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(ctr, 0, 4 * 32 * 64);
    cudaEventRecord(e0);
    e = cudaLaunchCooperativeKernel((void*)kb<NC, FENCE>, P, 192, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("NC=%2d fence=%d P=%d: %-10s %.3f us/barrier\n", NC, (int)FENCE, P, cudaGetErrorString(e), 1e3 * best / iters);
}

int main() {
  unsigned* ctr;
  double* sink;
  cudaMalloc(&ctr, 4 * 32 * 64);
  cudaMalloc(&sink, 8 * 1024);
  for (int P : {256, 128}) {
    run<1, true>(ctr, sink, P);
    run<2, true>(ctr, sink, P);
    run<4, true>(ctr, sink, P);
    run<8, true>(ctr, sink, P);
    run<16, true>(ctr, sink, P);
    run<1, false>(ctr, sink, P);
    run<8, false>(ctr, sink, P);
  }
  return 0;
}
