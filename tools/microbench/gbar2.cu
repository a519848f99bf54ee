// Grid-barrier + all-reduce latency variants (design input for k_persist.cu).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_rlx(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
  unsigned o;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
  return o;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acqrel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// MODE 0: red.release + ld.acquire poll (baseline)
// MODE 1: fence + red.relaxed ; poll ld.relaxed ; fence after
// MODE 2: atom.acq_rel returns old ; last arriver st.release flag=gen ; others poll flag relaxed ; fence
// MODE 3: MODE 1 + per-CTA double partial, all CTAs read all partials unrolled (deterministic allreduce)
// MODE 4: MODE 2 + partial: last arriver sums partials (fixed order) and publishes result before the flag
// MODE 5: MODE 1 with 8-CTA cluster pre-barrier: only cluster rank 0 touches the global counter
template <int MODE, int P>
__global__ void kbar(unsigned* ctr, unsigned* flag, int iters, double* partial, double* res, double* sink) {
  unsigned target = 0;
  double acc = 0;
  __shared__ double bcast;
  for (int it = 0; it < iters; ++it) {
    if ((MODE == 3 || MODE == 4) && threadIdx.x == 0) partial[(it & 1) * 1024 + blockIdx.x] = it * 0.5 + blockIdx.x;
    __syncthreads();
    if (MODE == 5) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    if (threadIdx.x == 0) {
      if (MODE == 0) {
        target += gridDim.x;
        red_rel(ctr, 1u);
        while (ld_acq(ctr) < target) {}
      } else if (MODE == 1 || MODE == 3) {
        target += gridDim.x;
        fence_acqrel();
        red_rlx(ctr, 1u);
        while (ld_rlx(ctr) < target) {}
        fence_acqrel();
      } else if (MODE == 5) {
        unsigned cr;
        asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
        target += gridDim.x / 8;
        if (cr == 0) {
          fence_acqrel();
          red_rlx(ctr, 1u);
          while (ld_rlx(ctr) < target) {}
          fence_acqrel();
        }
      } else {  // 2, 4
        const unsigned gen = it + 1;
        unsigned old = atom_add_acqrel(ctr, 1u);
        if (old == gridDim.x * gen - 1) {
          if (MODE == 4) {
            double s = 0;
            for (int i = 0; i < (int)gridDim.x; ++i) s += __ldcg(partial + (it & 1) * 1024 + i);
            res[it & 1] = s;
          }
          st_rel(flag, gen);
        } else {
          while (ld_rlx(flag) < gen) {}
        }
        fence_acqrel();
        if (MODE == 4) bcast = __ldcg(res + (it & 1));
      }
    }
    if (MODE == 5) {
      asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else {
      __syncthreads();
    }
    if (MODE == 3 && threadIdx.x < 32) {
      constexpr int K = P / 32;
      double v[K];
#pragma unroll
      for (int k = 0; k < K; ++k) v[k] = __ldcg(partial + (it & 1) * 1024 + threadIdx.x + 32 * k);
      double s = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) s += v[k];
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
      acc += s;
    }
    if (MODE == 4 && threadIdx.x == 0) acc += bcast;
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = acc;
}

template <int MODE, int P>
void run(unsigned* ctr, unsigned* flag, double* part, double* res, double* sink, const char* name) {
  const int iters = 20000;
  int it2 = iters;
  void* args[] = {&ctr, &flag, &it2, &part, &res, &sink};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P);
  cfg.blockDim = dim3(192);
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  int na = 1;
  if (MODE == 5) {
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = 8;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    na = 2;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  cudaError_t e = cudaSuccess;
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(ctr, 0, 4);
    cudaMemset(flag, 0, 4);
    cudaEventRecord(e0);
    e = cudaLaunchKernelExC(&cfg, (void*)kbar<MODE, P>, args);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  double h[2] = {0, 0};
  cudaMemcpy(h, sink, 16, cudaMemcpyDeviceToHost);
  printf("mode %d %-44s P=%d: %-10s %.3f us/barrier  (sink %.6g)\n", MODE, name, P, cudaGetErrorString(e),
         1e3 * best / iters, h[0]);
}

int main() {
  unsigned *ctr, *flag;
  double *part, *sink, *res;
  cudaMalloc(&ctr, 128);
  cudaMalloc(&flag, 128);
  cudaMalloc(&part, 8 * 2048);
  cudaMalloc(&res, 64);
  cudaMalloc(&sink, 8 * 1024);
  run<0, 256>(ctr, flag, part, res, sink, "red.release + ld.acquire poll");
  run<1, 256>(ctr, flag, part, res, sink, "fence + red.relaxed, relaxed poll, fence");
  run<2, 256>(ctr, flag, part, res, sink, "atom.acq_rel, last arriver releases flag");
  run<3, 256>(ctr, flag, part, res, sink, "mode1 + all CTAs read 256 partials");
  run<4, 256>(ctr, flag, part, res, sink, "mode2 + last arriver reduces, bcast");
  run<5, 256>(ctr, flag, part, res, sink, "8-CTA cluster barrier + mode1 on rank 0");
  run<1, 128>(ctr, flag, part, res, sink, "fence + red.relaxed, relaxed poll, fence");
  run<5, 128>(ctr, flag, part, res, sink, "8-CTA cluster barrier + mode1 on rank 0");
  run<3, 128>(ctr, flag, part, res, sink, "mode1 + all CTAs read 128 partials");
  return 0;
}
