// pcg_fin.cuh — "last block" finalisers of the device-driven PCG loop.
//
// PCG as in PAPER.md:234-238 (readings A15-A18):
//   init:  r0 = b - A x0 ; nb = ||b|| ; if nb == 0 -> x = 0 ; if eps>0, ||r0||/nb <= eps -> done
//          z0 = M^{-1} r0 ; p = z0 ; rho = Re<r0, z0>
//   iter k (K1): p_k = z_{k-1} + beta p_{k-1} (k>1), x += alpha_{k-1} p_{k-1} (deferred),
//                q = A p_k, sigma = Re<p_k, q>, alpha_k = rho / sigma           [fin_sigma]
//        (K2a):  r_k = r_{k-1} - alpha_k q, rel = ||r_k||/nb; stop if rel <= eps   [fin_rr]
//        (K2c):  z_k = M^{-1} r_k, rho' = Re<r_k, z_k>; stop if rho' == 0 or k == maxit;
//                beta = rho'/rho, rho = rho'                                      [fin_rho]
//   exit (fixup): x += alpha_k p_k for the last completed iteration.
#pragma once
#include "internal.cuh"

namespace sbk {

__device__ __forceinline__ void hist_put(const Loop& L, int b, int k, double rel) {
  if (L.hist != nullptr && k < L.hist_stride) L.hist[(size_t)b * L.hist_stride + k] = (float)rel;
}

// after the RESID kernel: ||b||^2, ||r0||^2
__device__ __forceinline__ void fin_init(const Loop& L, int b, double nb2, double rr, float eps,
                                         int maxit) {
  Scal& s = L.scal[b];
  s.nb2 = nb2;
  s.rr = rr;
  s.iter = 0;
  s.status = ST_OK;
  s.converged = 0;
  s.zero_x = 0;
  s.eps = eps;
  s.maxit = maxit;
  s.alpha = 0.0;
  s.beta = 0.0;
  s.rho = 0.0;
  s.active = 1;
  if (!(nb2 > 0.0)) {
    if (nb2 == 0.0) {
      s.zero_x = 1;
      s.converged = 1;
      hist_put(L, b, 0, 0.0);
    } else {
      s.status = ST_NONFINITE;
    }
    s.active = 0;
    return;
  }
  double rel = sqrt(rr / nb2);
  hist_put(L, b, 0, rel);
  if (!isfinite(rr)) {
    s.status = ST_NONFINITE;
    s.active = 0;
  } else if (eps > 0.f && rel <= (double)eps) {
    s.converged = 1;
    s.active = 0;
  }
}

__device__ __forceinline__ void fin_sigma(const Loop& L, int b, double sigma) {
  Scal& s = L.scal[b];
  s.sigma = sigma;
  if (!isfinite(sigma)) {
    s.status = ST_NONFINITE;
    s.active = 0;
  } else if (!(sigma > 0.0)) {
    s.status = ST_INDEFINITE;
    s.active = 0;
  } else {
    s.alpha = s.rho / sigma;
  }
}

__device__ __forceinline__ void fin_rr(const Loop& L, int b, double rr) {
  Scal& s = L.scal[b];
  s.rr = rr;
  const int k = ++s.iter;
  const double rel = sqrt(rr / s.nb2);
  hist_put(L, b, k, rel);
  if (!isfinite(rr)) {
    s.status = ST_NONFINITE;
    s.active = 0;
  } else if (s.eps > 0.f && rel <= (double)s.eps) {
    s.converged = 1;
    s.active = 0;
  }
}

// init = true: rho_0 after z_0 = M^{-1} r_0
__device__ __forceinline__ void fin_rho(const Loop& L, int b, double rz, bool init) {
  Scal& s = L.scal[b];
  if (!isfinite(rz)) {
    s.status = ST_NONFINITE;
    s.active = 0;
    return;
  }
  if (init) {
    s.rho = rz;
    return;
  }
  if (rz == 0.0) {
    s.converged = 1;
    s.active = 0;
  } else if (s.iter >= s.maxit) {
    s.converged = (s.eps == 0.f) ? 1 : 0;
    s.active = 0;
  } else {
    s.beta = rz / s.rho;
    s.rho = rz;
  }
}

// Called once per problem per iteration (by one thread): counts problems; the last one
// publishes "any problem still active" and sets the CUDA-graph while condition.
__device__ __forceinline__ void slice_arrive(const Loop& L) {
  __threadfence();
  unsigned int t = atomicAdd(&L.ctl->slices_done, 1u);
  if (t == (unsigned)(L.B - 1)) {
    __threadfence();
    int any = 0;
    for (int b = 0; b < L.B; ++b) any |= __ldcg(&L.scal[b].active);
    L.ctl->any_active = any;
    L.ctl->slices_done = 0;
    __threadfence();
    if (L.cond != 0ull) cudaGraphSetConditional((cudaGraphConditionalHandle)L.cond, any ? 1u : 0u);
  }
}

}  // namespace sbk
