// Grid-barrier latency: where does the time go? (fences vs signal latency vs syncthreads)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rlx(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acqrel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// MODE 0: relaxed red + relaxed poll, no fences
// MODE 1: fence before red only
// MODE 2: fence after poll only
// MODE 3: both fences (= the usual barrier)
// MODE 4: both fences, nanosleep(32) in the poll loop
// MODE 5: LL all-reduce of a double: {hi32|gen}, {lo32|gen} words per CTA, warp 0 polls all, no fence
// MODE 6: MODE 5 + fence before publish (release side)
template <int MODE>
__global__ void kbar(unsigned* ctr, uint64_t* ll, int iters, double* sink) {
  unsigned target = 0;
  double acc = 0;
  const int P = gridDim.x;
  for (int it = 0; it < iters; ++it) {
    if (MODE <= 4) {
      __syncthreads();
      if (threadIdx.x == 0) {
        target += P;
        if (MODE == 1 || MODE == 3 || MODE == 4) fence_acqrel();
        red_rlx(ctr, 1u);
        while (ld_rlx(ctr) < target) {
          if (MODE == 4) __nanosleep(32);
        }
        if (MODE >= 2) fence_acqrel();
      }
      __syncthreads();
    } else {
      const double part = it * 0.5 + blockIdx.x;
      const uint64_t gen = (uint64_t)(it + 1) << 32;
      const uint64_t bits = (uint64_t)__double_as_longlong(part);
      uint64_t* slot = ll + (size_t)(it & 1) * 2 * 1024;
      __syncthreads();
      if (threadIdx.x < 2) {
        if (MODE == 6) fence_acqrel();
        st_u64(slot + 2 * blockIdx.x + threadIdx.x, gen | (threadIdx.x == 0 ? (bits >> 32) : (bits & 0xffffffffull)));
      }
      if (threadIdx.x < 32) {
        double s = 0;
        for (int i = threadIdx.x; i < P; i += 32) {
          uint64_t hi, lo;
          do { hi = ld_u64(slot + 2 * i); } while ((hi >> 32) != (gen >> 32));
          do { lo = ld_u64(slot + 2 * i + 1); } while ((lo >> 32) != (gen >> 32));
          s += __longlong_as_double((long long)(((hi & 0xffffffffull) << 32) | (lo & 0xffffffffull)));
        }
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
        acc += s;
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = acc;
}

template <int MODE>
void run(unsigned* ctr, uint64_t* ll, double* sink, int P, int nt, const char* name) {
  const int iters = 20000;
  int it2 = iters;
  void* args[] = {&ctr, &ll, &it2, &sink};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  cudaError_t e = cudaSuccess;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(ctr, 0, 4);
    cudaMemset(ll, 0, 8 * 4096);
    cudaEventRecord(e0);
    e = cudaLaunchCooperativeKernel((void*)kbar<MODE>, P, nt, args, 0, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double h = 0;
  cudaMemcpy(&h, sink, 8, cudaMemcpyDeviceToHost);
  printf("mode %d %-40s P=%d nt=%d: %-10s %.3f us  (sink %.6g)\n", MODE, name, P, nt, cudaGetErrorString(e),
         1e3 * best / iters, h);
}

int main() {
  unsigned* ctr;
  uint64_t* ll;
  double* sink;
  cudaMalloc(&ctr, 128);
  cudaMalloc(&ll, 8 * 4096);
  cudaMalloc(&sink, 8 * 1024);
  for (int nt : {32, 192}) {
    run<0>(ctr, ll, sink, 256, nt, "no fences");
    run<1>(ctr, ll, sink, 256, nt, "release fence only");
    run<2>(ctr, ll, sink, 256, nt, "acquire fence only");
    run<3>(ctr, ll, sink, 256, nt, "both fences");
    run<4>(ctr, ll, sink, 256, nt, "both fences + nanosleep poll");
    run<5>(ctr, ll, sink, 256, nt, "LL allreduce (no fence)");
    run<6>(ctr, ll, sink, 256, nt, "LL allreduce + release fence");
  }
  run<3>(ctr, ll, sink, 16, 192, "both fences");
  run<0>(ctr, ll, sink, 16, 192, "no fences");
  run<5>(ctr, ll, sink, 16, 192, "LL allreduce (no fence)");
  return 0;
}
