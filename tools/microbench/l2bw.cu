// l2bw.cu — read+write streaming bandwidth vs working-set size (L2-resident vs HBM).
// Design input for staging FFT passes through L2.  Each launch copies a
// buffer of S bytes into a second one (16-byte loads/stores, grid = 148 x 8 CTAs, grid-stride);
// the pair is swapped between launches so the working set is 2 S.  Reports bytes moved
// (read + write) per second over 50 back-to-back launches after a warm-up.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2bw l2bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy4(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  const size_t sizes_mb[] = {8, 16, 24, 32, 48, 64, 96, 256, 1024};
  for (size_t mb : sizes_mb) {
    const size_t bytes = mb << 20, n = bytes / 16;
    float4 *a, *b;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMemset(a, 0, bytes);
    cudaMemset(b, 0, bytes);
    for (int i = 0; i < 5; ++i) copy4<<<148 * 8, 512>>>(i & 1 ? b : a, i & 1 ? a : b, n);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int R = 50;
    cudaEventRecord(e0);
    for (int i = 0; i < R; ++i) copy4<<<148 * 8, 512>>>(i & 1 ? b : a, i & 1 ? a : b, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("working set %5zu MB: %8.1f GB/s (read+write), %.2f us per launch\n", 2 * mb,
           2.0 * bytes * R / (ms * 1e-3) / 1e9, ms * 1e3 / R);
    cudaFree(a);
    cudaFree(b);
  }
  return 0;
}
