// k_coil.cu — kernels of the coil-sharded mode (BASELINE config 5 over 2/4/8 GPUs; DESIGN.md
// 8(e)).  Each rank holds C/G coils and full replicas of every vector.  Per matvec the plane
// kernel (k_plane.cu) writes the rank's partial coil sum
//     acc_r = sum_{c in rank r} conj(s_c) F^H R F (s_c p),
// one NCCL all-reduce forms acc = sum_r acc_r (the first term of A), and this
// epilogue applies  q = mu acc + lambda L p + gamma p  (W^H W = I) with the
// same PCG bookkeeping as the fused epilogue (sigma = Re<p, q>, last-block alpha), or the
// RESID form r0 = b - A x with the SB right-hand side / data feedback.  All ranks compute
// the same bits (the all-reduce result is identical on every rank), so the replicated
// vectors and scalars stay identical without a scalar all-reduce.
#include <algorithm>

#include "kernels.cuh"
#include "pcg_fin.cuh"

namespace sbk {

template <int MODE>
__global__ void __launch_bounds__(256) kc_epilogue(const KPArgs a) {
  __shared__ double red[32];
  __shared__ int lastflag;
  pdl_trigger();
  pdl_wait();
  const int b = blockIdx.y;
  const int planes = a.planes, NY = a.NY, NZ = a.NZ;
  const size_t pn = (size_t)NY * NZ, img = pn * planes, boff = (size_t)b * img;
  const float2* psrc = a.vin;
  if constexpr (MODE == KP_PCG) {
    const Scal& s = a.L.scal[b];
    if (!s.active) return;
    psrc = ((s.iter + 1) & 1) ? a.pbuf1 : a.pbuf0;  // p_k written by the plane kernel
  }
  const float cdeg = a.d3 ? 6.f : 4.f;
  double d0 = 0.0, d1 = 0.0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < img; i += (size_t)gridDim.x * blockDim.x) {
    const size_t xp = i / pn, yz = i % pn;
    const size_t y = yz / NZ, z = yz % NZ;
    const size_t gi = boff + i;
    const float2 p = psrc[gi];
    const float2 pl = psrc[boff + xp * pn + y * NZ + (z + NZ - 1) % NZ];
    const float2 pr = psrc[boff + xp * pn + y * NZ + (z + 1) % NZ];
    const float2 pu = psrc[boff + xp * pn + ((y + NY - 1) % NY) * NZ + z];
    const float2 pd = psrc[boff + xp * pn + ((y + 1) % NY) * NZ + z];
    float2 lp = make_float2(cdeg * p.x - pl.x - pr.x - pu.x - pd.x, cdeg * p.y - pl.y - pr.y - pu.y - pd.y);
    if (a.d3) {
      const float2 xm = psrc[boff + ((xp + planes - 1) % planes) * pn + yz];
      const float2 xq = psrc[boff + ((xp + 1) % planes) * pn + yz];
      lp.x -= xm.x + xq.x;
      lp.y -= xm.y + xq.y;
    }
    const float2 av = a.acc_in[gi];
    const float2 reg = make_float2(a.lam * lp.x + a.gam * p.x, a.lam * lp.y + a.gam * p.y);
    if constexpr (MODE == KP_RESID) {
      float2 bb;
      if (a.bvec != nullptr) {
        bb = a.bvec[gi];
      } else {
        float2 uu = a.u[gi];
        if (a.update_u) {
          const float2 u1 = a.u1[gi];
          uu = make_float2(uu.x + u1.x - av.x, uu.y + u1.y - av.y);
          a.u[gi] = uu;
        }
        const float2 rr = a.rhs_reg != nullptr ? a.rhs_reg[gi] : make_float2(0.f, 0.f);
        bb = make_float2(a.mu * uu.x + rr.x, a.mu * uu.y + rr.y);
        a.bout[gi] = bb;
      }
      const float2 rv = make_float2(bb.x - (a.mu * av.x + reg.x), bb.y - (a.mu * av.y + reg.y));
      a.out[gi] = rv;
      d0 += (double)bb.x * bb.x + (double)bb.y * bb.y;
      d1 += (double)rv.x * rv.x + (double)rv.y * rv.y;
    } else {
      const float2 q = make_float2(a.mu * av.x + reg.x, a.mu * av.y + reg.y);
      a.out[gi] = q;
      d0 += (double)p.x * q.x + (double)p.y * q.y;
    }
  }
  if constexpr (MODE == KP_APPLY) return;
  const double s0 = block_sum(d0, red);
  double s1 = 0.0;
  if constexpr (MODE == KP_RESID) s1 = block_sum(d1, red);
  const int nblk = gridDim.x;
  if (!publish_and_check_last(s0, s1, a.P, b, blockIdx.x, nblk, &lastflag)) return;
  if (threadIdx.x < 32) {
    const double t0 = warp_sum_partials(a.P.p0 + (size_t)b * a.P.cap, nblk);
    double t1 = 0.0;
    if constexpr (MODE == KP_RESID) t1 = warp_sum_partials(a.P.p1 + (size_t)b * a.P.cap, nblk);
    if (threadIdx.x == 0) {
      if constexpr (MODE == KP_PCG) fin_sigma(a.L, b, t0);
      else fin_init(a.L, b, t0, t1, a.eps, a.maxit);
      a.P.cnt[b] = 0;
    }
  }
}

cudaError_t launch_kc_epilogue(int mode, const KPArgs& a, cudaStream_t st) {
  const size_t img = (size_t)a.planes * a.NY * a.NZ;
  int nb = (int)std::min<size_t>(1024, (img + 1023) / 1024);
  const dim3 grid(nb, a.B);
  switch (mode) {
    case KP_APPLY: return launch_ex(kc_epilogue<KP_APPLY>, grid, dim3(256), 0, st, 0, a);
    case KP_PCG: return launch_ex(kc_epilogue<KP_PCG>, grid, dim3(256), 0, st, 0, a);
    case KP_RESID: return launch_ex(kc_epilogue<KP_RESID>, grid, dim3(256), 0, st, 0, a);
    default: return cudaErrorInvalidValue;
  }
}

// RSS init after the all-reduce of sum_c |F^H y_c|^2 (reading A12)
__global__ void __launch_bounds__(256) kc_sqrt_re(float2* v, size_t n) {
  pdl_trigger();
  pdl_wait();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    v[i] = make_float2(sqrtf(v[i].x), 0.f);
}

cudaError_t launch_kc_sqrt_re(float2* v, size_t n, cudaStream_t st) {
  const int nb = (int)std::min<size_t>(2048, (n + 255) / 256);
  return launch_ex(kc_sqrt_re, dim3(nb), dim3(256), 0, st, 0, v, n);
}

}  // namespace sbk
