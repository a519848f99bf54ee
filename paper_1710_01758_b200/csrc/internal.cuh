// internal.cuh — device-side state shared by libsbpcg's kernels (not part of the ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "fft_core.cuh"

namespace sbk {

// Per-problem PCG scalars (fp64, device resident).  Written only by "last block"
// finalisers, read by the CTAs of the following kernels (see DESIGN.md "device-driven
// PCG").
struct Scal {
  double rho;     // <r_k, z_k>
  double alpha;   // alpha_k = rho_{k-1} / <p_k, A p_k>
  double beta;    // beta for the next p update
  double sigma;   // <p_k, A p_k>
  double nb2;     // ||b||^2
  double rr;      // ||r_k||^2
  int iter;       // completed iterations k
  int active;     // 1 while iterating
  int converged;
  int status;     // 0, SB_E_NONFINITE (6), SB_E_INDEFINITE (7)
  int zero_x;     // ||b|| = 0: x <- 0 at fixup
  int maxit;
  float eps;
  int log_slot;   // row of the recon log this solve writes
};

struct Ctl {
  unsigned int slices_done;  // last-slice detection for the graph condition
  int any_active;
  int solve_idx;
  int pad;
};

// Instrumentation not reset per call: problem-launches of K1 (for the roofline bytes).
struct Counters {
  unsigned long long k1_problems;
};

enum { ST_OK = 0, ST_NONFINITE = 6, ST_INDEFINITE = 7 };

// Per-kernel-family partial/counter slots.
struct Partials {
  double* p0;            // [B][cap] first partial
  double* p1;            // [B][cap] second partial (e.g. ||r||^2 with ||b||^2)
  unsigned int* cnt;     // [B] arrival counters
  int cap;
};

// PCG loop bookkeeping shared by the finalisers.
struct Loop {
  Scal* scal;            // [B]
  Ctl* ctl;
  float* hist;           // [B][hist_stride] relres history (nullable)
  int hist_stride;
  int32_t* log_iters;    // [slots][B] recon log (nullable)
  float* log_relres;     // [slots][B]
  int B;
  unsigned long long cond;  // cudaGraphConditionalHandle (0 = eager)
  Counters* cnt;            // nullable
};

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block sum (fixed shuffle tree, fixed warp order).  All threads call it;
// result valid in thread 0.  `red` must hold >= 32 doubles.  Blocks smaller than a warp
// (tiny images) take a serial shared-memory path: shuffles need every lane present.
__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (blockDim.x & 31) {
    __syncthreads();
    red[threadIdx.x] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0)
      for (int i = 0; i < (int)blockDim.x; ++i) s += red[i];
    return s;
  }
  const int nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (wid == 0) {
    s = lane < nw ? red[lane] : 0.0;
    s = warp_sum(s);
  }
  return s;
}

// Sum n partials in a fixed order using the first warp (lane i takes i, i+32, ...; then a
// fixed shuffle tree).  Call from threads 0..31 (or all threads of a sub-warp block);
// result valid in thread 0.
__device__ __forceinline__ double warp_sum_partials(const double* p, int n) {
  if (blockDim.x < 32) {
    double s = 0.0;
    if (threadIdx.x == 0)
      for (int i = 0; i < n; ++i) s += __ldcg(p + i);
    return s;
  }
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int i = lane; i < n; i += 32) s += __ldcg(p + i);
  return warp_sum(s);
}

// Publish a block partial and report whether this block is the last of `nblk` for the
// problem.  Call with all threads; returns the same flag in all threads.
__device__ __forceinline__ bool publish_and_check_last(double v0, double v1, const Partials& P,
                                                       int b, int slot, int nblk, int* flag) {
  if (threadIdx.x == 0) {
    P.p0[(size_t)b * P.cap + slot] = v0;
    if (P.p1) P.p1[(size_t)b * P.cap + slot] = v1;
    __threadfence();
    unsigned int t = atomicAdd(P.cnt + b, 1u);
    *flag = (t == (unsigned)(nblk - 1));
  }
  __syncthreads();
  bool last = *flag;
  if (last) __threadfence();
  return last;
}

// ------------------------------------------------------------------ programmatic dependent launch
// Every kernel of the PCG loop is launched with cudaLaunchAttributeProgrammaticStreamSerialization:
// it may start while its predecessor drains, does its constant setup (twiddles, masks, TMA of
// the constant coil maps), then waits for the predecessor grid (griddepcontrol.wait) before
// touching anything the predecessor produced.  Every CTA executes pdl_wait() before exiting,
// so completion stays transitive along the chain.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ------------------------------------------------------------------ mbarrier / TMA (sm_90+)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// distributed shared memory: the shared::cluster address of `addr` (a shared::cta address of
// this CTA's layout) in cluster CTA `rank`
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// asynchronous 8-byte store into a (possibly remote) CTA's shared memory; completion counts
// 8 bytes on that CTA's mbarrier `bar` (both shared::cluster addresses)
__device__ __forceinline__ void st_async_f2(uint32_t addr, float2 v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "f"(v.x), "f"(v.y), "r"(bar)
               : "memory");
}
// bulk copy (async proxy) of `bytes` (multiple of 16, 16-byte aligned) from this CTA's shared
// memory to a (possibly remote) CTA's shared memory, completion counted on that CTA's mbarrier
__device__ __forceinline__ void bulk_s2s(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(src_cta), "r"(bytes), "r"(bar_cluster)
               : "memory");
}
// split cluster barrier without memory ordering (the data exchanged by bulk copies is ordered by
// the mbarriers; mbarrier initialisation is released by fence.mbarrier_init): no GPU-scope
// fence, no L1 invalidate
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// 3D tiled TMA load into shared memory, completion on `bar`.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

}  // namespace sbk
