// Barrier + deterministic all-reduce without atomics ("LL" flags): every CTA publishes its
// fp64 partials as 32-bit halves tagged with a 32-bit generation (8-byte single-copy-atomic
// words); warp 0 of every CTA polls all P slots in parallel and sums them in a fixed order.
// Compared with the counter barrier + a separate partial read (k_persist.cu as of this test).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t ld_rlx64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acq64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rlx64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rlx(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// MODE 0: counter barrier (fence, red, relaxed poll, fence) + partial read (NS slots), as k_persist
// MODE 1: LL all-reduce, relaxed polls + one fence after
// MODE 2: LL all-reduce, acquire polls, no trailing fence
// MODE 3: LL all-reduce, relaxed polls, no trailing fence (ordering not guaranteed; floor)
template <int MODE, int P, int NS>
__global__ void __launch_bounds__(192) kll(unsigned* ctr, uint64_t* ll, double* part, int iters, double* sink) {
  __shared__ double bc[NS];
  double acc = 0;
  unsigned target = 0;
  constexpr int K = P / 32;
  for (int it = 0; it < iters; ++it) {
    double mine[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) mine[s] = it * 0.25 + blockIdx.x + s;
    if (MODE == 0) {
      if (threadIdx.x == 0)
        for (int s = 0; s < NS; ++s) part[(it & 1) * 4096 + s * P + blockIdx.x] = mine[s];
      __syncthreads();
      if (threadIdx.x == 0) {
        target += P;
        fence();
        red_rlx(ctr, 1u);
        while (ld_rlx(ctr) < target) {}
        fence();
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        double v[NS][K];
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
          for (int i = 0; i < K; ++i) v[s][i] = __ldcg(part + (it & 1) * 4096 + s * P + threadIdx.x + 32 * i);
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          double a = 0;
#pragma unroll
          for (int i = 0; i < K; ++i) a += v[s][i];
          for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(~0u, a, o);
          if (threadIdx.x == 0) bc[s] = a;
        }
      }
      __syncthreads();
    } else {
      const uint32_t gen = (uint32_t)(it + 1);
      uint64_t* slot = ll + (size_t)(it & 1) * 2 * NS * 1024;  // [NS][P][2] words
      __syncthreads();
      if (threadIdx.x < 2 * NS) {
        const int s = threadIdx.x >> 1, h = threadIdx.x & 1;
        const uint64_t bits = (uint64_t)__double_as_longlong(mine[s]);
        const uint32_t half = h ? (uint32_t)(bits & 0xffffffffu) : (uint32_t)(bits >> 32);
        fence();
        st_rlx64(slot + ((size_t)s * P + blockIdx.x) * 2 + h, ((uint64_t)gen << 32) | half);
      }
      if (threadIdx.x < 32) {
        uint64_t w[NS][K][2];
        bool done;
        do {
          done = true;
#pragma unroll
          for (int s = 0; s < NS; ++s)
#pragma unroll
            for (int i = 0; i < K; ++i)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const uint64_t* q = slot + ((size_t)s * P + threadIdx.x + 32 * i) * 2 + h;
                w[s][i][h] = MODE == 2 ? ld_acq64(q) : ld_rlx64(q);
                done &= (uint32_t)(w[s][i][h] >> 32) == gen;
              }
          done = __all_sync(~0u, done);
        } while (!done);
        if (MODE == 1) fence();
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          double a = 0;
#pragma unroll
          for (int i = 0; i < K; ++i)
            a += __longlong_as_double((long long)(((w[s][i][0] & 0xffffffffull) << 32) | (w[s][i][1] & 0xffffffffull)));
          for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(~0u, a, o);
          if (threadIdx.x == 0) bc[s] = a;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) acc += bc[s];
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = acc;
}

template <int MODE, int P, int NS>
void run(unsigned* ctr, uint64_t* ll, double* part, double* sink, const char* name) {
  const int iters = 20000;
  int it2 = iters;
  void* args[] = {&ctr, &ll, &part, &it2, &sink};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  cudaError_t e = cudaSuccess;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(ctr, 0, 4);
    cudaMemset(ll, 0, 8 * 2 * 2 * 2 * 1024);
    cudaEventRecord(e0);
    e = cudaLaunchCooperativeKernel((void*)kll<MODE, P, NS>, P, 192, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double h = 0;
  cudaMemcpy(&h, sink, 8, cudaMemcpyDeviceToHost);
  // expected: sum over it of sum_s sum_b (it*0.25 + b + s)
  double ex = 0;
  for (int it = 0; it < iters; ++it)
    for (int s = 0; s < NS; ++s) ex += P * (it * 0.25 + s) + P * (P - 1) / 2.0;
  printf("mode %d %-36s P=%d NS=%d: %-10s %.3f us  %s\n", MODE, name, P, NS, cudaGetErrorString(e), 1e3 * best / iters,
         h == ex ? "sum ok" : "SUM WRONG");
}

int main() {
  unsigned* ctr;
  uint64_t* ll;
  double *part, *sink;
  cudaMalloc(&ctr, 128);
  cudaMalloc(&ll, 8 * 2 * 2 * 2 * 1024);
  cudaMalloc(&part, 8 * 2 * 4096);
  cudaMalloc(&sink, 8 * 1024);
  run<0, 256, 1>(ctr, ll, part, sink, "counter barrier + partial read");
  run<1, 256, 1>(ctr, ll, part, sink, "LL, relaxed polls + fence");
  run<2, 256, 1>(ctr, ll, part, sink, "LL, acquire polls");
  run<3, 256, 1>(ctr, ll, part, sink, "LL, relaxed polls (no fence)");
  run<0, 256, 2>(ctr, ll, part, sink, "counter barrier + partial read");
  run<1, 256, 2>(ctr, ll, part, sink, "LL, relaxed polls + fence");
  run<2, 256, 2>(ctr, ll, part, sink, "LL, acquire polls");
  run<0, 64, 2>(ctr, ll, part, sink, "counter barrier + partial read");
  run<1, 64, 2>(ctr, ll, part, sink, "LL, relaxed polls + fence");
  return 0;
}
