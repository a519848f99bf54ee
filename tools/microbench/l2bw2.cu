// l2bw2.cu — L2 read+write bandwidth with the launch overhead amortised: one launch, every CTA
// streams its own slice of a working set of S bytes P times (ld.global.cg / st.global.cg, so
// L1 never serves the re-reads), i.e. the access pattern of an FFT pass pipeline whose
// intermediates stay in L2.  Prints bytes moved (read + write) per second per S.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw2 l2bw2.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void passes(float4* __restrict__ buf, size_t n_per_cta, int P) {
  float4* my = buf + blockIdx.x * n_per_cta;
  for (int p = 0; p < P; ++p) {
    for (size_t i = threadIdx.x; i < n_per_cta; i += blockDim.x) {
      float4 v = __ldcg(my + i);
      v.x += 1.f;
      __stcg(my + i, v);
    }
  }
}

int main() {
  const size_t sizes_mb[] = {16, 32, 48, 64, 80, 96, 112, 128, 256};
  const int ctas = 148 * 2, threads = 512, P = 20;
  for (size_t mb : sizes_mb) {
    const size_t bytes = mb << 20, n = bytes / 16, npc = n / ctas;
    float4* a;
    cudaMalloc(&a, bytes);
    cudaMemset(a, 0, bytes);
    passes<<<ctas, threads>>>(a, npc, 2);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    passes<<<ctas, threads>>>(a, npc, P);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("working set %4zu MB: %8.1f GB/s (read+write, %d passes in one launch, %.1f us)\n", mb,
           2.0 * npc * ctas * 16 * P / (ms * 1e-3) / 1e9, P, ms * 1e3);
    cudaFree(a);
  }
  return 0;
}
