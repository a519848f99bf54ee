// k_matvec.cu — K1: the fused system-matrix application q = A p,
//
//   A p = mu sum_c conj(s_c) . F^H( r . F(s_c . p) ) + lambda L p + gamma p,
//
// L = D_x^H D_x + D_y^H D_y (periodic 5-point Laplacian) and
// gamma W^H W = gamma I.  One CTA owns one column tile (all M = d0 rows x W
// columns) of one problem.
//
// Separable (line) masks (r depends on the d0 row only): with F = F_0 (x) F_1
// the data term is exactly  F_0^H R_0 F_0 (x) I  per coil, so each coil needs one length-M
// FFT pair down every column, scaled by r/M.  Other
// masks take the plane-cluster kernel K1P (k_plane.cu).
//
// Per coil: the s_c tile (M x W complex64) arrives by 3D TMA into a 2-stage ring (mbarrier
// complete_tx); the column FFT is register resident (four-step, fft_core.cuh); the coil
// sum accumulates in registers.  G CTAs of a thread-block cluster split the coils and
// reduce their partial sums through DSMEM in a fixed order (deterministic), then each
// finishes M/G rows of the epilogue.
#include <cooperative_groups.h>

#include "kernels.cuh"
#include "pcg_fin.cuh"

namespace cg = cooperative_groups;

namespace sbk {

template <int M, int W, int MODE>
__global__ void __launch_bounds__(Split<M>::N2* W)
    k1_matvec(const __grid_constant__ CUtensorMap tmap, const K1Args a) {
  constexpr int N1 = Split<M>::N1, N2 = Split<M>::N2;
  constexpr int NT = N2 * W;
  constexpr int TILE = M * W;          // complex elements per tile
  constexpr int PW = W + 2;            // p tile with +-1 column halo
  using Lay = typename ColLayout<M, W>::L;

  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* ring = reinterpret_cast<float2*>(smem_raw);                 // [2][TILE]
  float2* xch = ring + 2 * TILE;                                     // ColLayout size
  float2* pt = xch + ColLayout<M, W>::size;                          // [M][PW]
  float2* tw = pt + M * PW;                                          // [M]
  float* rm = reinterpret_cast<float*>(tw + M);                      // [M]
  uint64_t* bar = reinterpret_cast<uint64_t*>(rm + M + (M & 1));     // [2]
  __shared__ double red[32];
  __shared__ double cred[32];  // cluster pre-reduction slots (rank 0), 2 per CTA
  __shared__ int lastflag;

  const int G = gridDim.x;
  const int g = blockIdx.x;
  const int tile = blockIdx.y;
  const int b = blockIdx.z;
  const int tid = threadIdx.x;
  const int j = tid / W, l = tid % W;
  const int col0 = tile * W;
  const int N = a.N;
  const size_t img = (size_t)M * N;
  const size_t boff = (size_t)b * img;

  // ---- setup on constant data (overlaps the predecessor kernel under PDL): barriers,
  // twiddles, mask, and the TMA of the first two coil-map tiles (coil maps never change)
  const int ncoil = (a.C - g + G - 1) / G;  // coils g, g+G, ...
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < M; i += NT) {
    tw[i] = a.tw[i];
    rm[i] = a.rmask[(size_t)b * a.rmask_bstride + i];
  }
  __syncthreads();
  if (tid == 0) {
    for (int s = 0; s < 2 && s < ncoil; ++s) {
      const int c = g + s * G;
      mbar_expect_tx(&bar[s], TILE * 8);
      tma_load_3d(ring + s * TILE, &tmap, 2 * col0, 0, b * a.C + c, &bar[s]);
    }
  }
  pdl_trigger();
  pdl_wait();

  int pidx = 0;
  double beta = 0.0, alpha_prev = 0.0;
  bool first = true;
  if constexpr (MODE == K1_PCG) {
    const Scal& s = a.L.scal[b];
    if (!s.active) {  // uniform over the cluster (same problem): drain the TMAs, leave
      for (int st = 0; st < 2 && st < ncoil; ++st) mbar_wait(&bar[st], 0);
      return;
    }
    const int k = s.iter + 1;  // iteration being formed
    first = (k == 1);
    pidx = k & 1;
    beta = s.beta;
    alpha_prev = s.alpha;
  }

  if (g == 0 && tile == 0 && tid == 0 && a.L.cnt != nullptr) atomicAdd(&a.L.cnt->k1_problems, 1ull);

  // ---- prologue: the p tile (+halo) into shared memory, in batches of independent loads.
  // PCG forms p_k = z + beta p_{k-1} (standard PCG) and x += alpha p_{k-1}.
  // rows of the epilogue owned by this CTA (G need not divide M: the last CTAs take fewer)
  const int rows_ceil = (M + G - 1) / G;
  const int r0 = min(M, g * rows_ceil);
  const int rows_per = min(rows_ceil, M - r0);
  constexpr int PE = (M * PW + NT - 1) / NT;  // elements per thread
  constexpr int CH = PE < 10 ? PE : 10;
  const float2* pold = pidx ? a.pbuf0 : a.pbuf1;
  float2* pnew = pidx ? a.pbuf1 : a.pbuf0;
  const bool need_old = (MODE == K1_PCG) && !first;
  // one pass over the tile: p_k into shared memory, and for this CTA's own rows (non-halo
  // columns) also p_k -> pnew and the deferred x += alpha_{k-1} p_{k-1} (p_{k-1} is read once)
#pragma unroll 1
  for (int c0 = 0; c0 < PE; c0 += CH) {
    float2 zz[CH], po[CH], xv[CH];
    bool own[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int e = (c0 + i) * NT + tid;
      zz[i] = make_float2(0.f, 0.f);
      po[i] = make_float2(0.f, 0.f);
      own[i] = false;
      if (c0 + i < PE && e < M * PW) {
        const int row = e / PW, cc = e % PW;
        int gcol = col0 + cc - 1;
        gcol = gcol < 0 ? gcol + N : (gcol >= N ? gcol - N : gcol);
        const size_t gi = boff + (size_t)row * N + gcol;
        if constexpr (MODE == K1_PCG) {
          zz[i] = a.z[gi];
          if (need_old) po[i] = pold[gi];
          own[i] = cc >= 1 && cc <= W && row >= r0 && row < r0 + rows_per;
          if (own[i] && need_old) xv[i] = a.x[gi];
        } else {
          zz[i] = a.vin[gi];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      const int e = (c0 + i) * NT + tid;
      if (c0 + i < PE && e < M * PW) {
        const float2 p = need_old ? make_float2(zz[i].x + (float)beta * po[i].x, zz[i].y + (float)beta * po[i].y)
                                  : zz[i];
        pt[e] = p;
        if constexpr (MODE == K1_PCG) {
          if (own[i]) {
            const size_t gi = boff + (size_t)(e / PW) * N + col0 + (e % PW) - 1;
            pnew[gi] = p;
            if (need_old)
              a.x[gi] = make_float2(xv[i].x + (float)alpha_prev * po[i].x, xv[i].y + (float)alpha_prev * po[i].y);
          }
        }
      }
    }
  }
  __syncthreads();

  // ---- coil loop
  constexpr bool TWR = (N1 == N2);  // square split: twiddles in registers (fft_core.cuh)
  float2 twr[N1];
  if constexpr (TWR) load_twr<M>(twr, tw, j);
  float rmr[N1];  // this thread's spectral rows' mask factors r/M, fixed for the kernel
#pragma unroll
  for (int q = 0; q < N1; ++q) rmr[q] = rm[specidx<M>(j, q)];
  float2 acc[N1];
#pragma unroll
  for (int i = 0; i < N1; ++i) acc[i] = make_float2(0.f, 0.f);

  for (int ci = 0; ci < ncoil; ++ci) {
    const int stage = ci & 1;
    mbar_wait(&bar[stage], (ci >> 1) & 1);
    const float2* sc = ring + stage * TILE;
    float2 s[N1], v[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const int row = natidx<M>(j, n1);
      s[n1] = sc[row * W + l];
    }
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const int row = natidx<M>(j, n1);
      v[n1] = cmul(s[n1], pt[row * PW + l + 1]);
    }
    if constexpr (TWR) fft_fwd_r<M, Lay>(v, xch, twr, j, l);
    else fft_fwd<M, Lay>(v, xch, tw, j, l);
    // every thread has read ring[stage] before the barrier inside fft_fwd
    if (tid == 0 && ci + 2 < ncoil) {
      const int c = g + (ci + 2) * G;
      mbar_expect_tx(&bar[stage], TILE * 8);
      tma_load_3d(ring + stage * TILE, &tmap, 2 * col0, 0, b * a.C + c, &bar[stage]);
    }
#pragma unroll
    for (int q = 0; q < N1; ++q) v[q] = cscale(v[q], rmr[q]);
    if constexpr (TWR) fft_inv_r<M, Lay>(v, xch, twr, j, l);
    else fft_inv<M, Lay>(v, xch, tw, j, l);
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) acc[n1] = cfmac(s[n1], v[n1], acc[n1]);  // acc += conj(s_c) v
  }

  // ---- coil-group reduction (DSMEM) + epilogue
  __syncthreads();
  float2* accb = ring;  // TILE elements; the ring is drained
#pragma unroll
  for (int n1 = 0; n1 < N1; ++n1) accb[natidx<M>(j, n1) * W + l] = acc[n1];
  cg::cluster_group cluster = cg::this_cluster();
  if (G > 1) cluster.sync(); else __syncthreads();

  double d0 = 0.0, d1 = 0.0;
  constexpr int EE = (M * W + NT - 1) / NT;  // upper bound of epilogue elements per thread
  constexpr int CH3 = EE < 8 ? EE : 8;
  const int nep = rows_per * W;
#pragma unroll 1
  for (int c0 = 0; c0 < EE; c0 += CH3) {
    float2 lb[CH3], lu[CH3], lu1[CH3], lr[CH3];
    if constexpr (MODE == K1_RESID) {
#pragma unroll
      for (int i = 0; i < CH3; ++i) {
        const int e = (c0 + i) * NT + tid;
        if (c0 + i < EE && e < nep) {
          const size_t gi = boff + (size_t)(r0 + e / W) * N + col0 + e % W;
          if (a.bvec != nullptr) {
            lb[i] = a.bvec[gi];
          } else {
            lu[i] = a.u[gi];
            lu1[i] = a.update_u ? a.u1[gi] : make_float2(0.f, 0.f);
            lr[i] = a.rhs_reg != nullptr ? a.rhs_reg[gi] : make_float2(0.f, 0.f);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CH3; ++i) {
      const int e = (c0 + i) * NT + tid;
      if (!(c0 + i < EE && e < nep)) continue;
      const int row = r0 + e / W, cc = e % W;
      // fixed-order sum over the cluster's partials (rank 0 first), four DSMEM loads in flight
      float2 av = make_float2(0.f, 0.f);
#pragma unroll 1
      for (int g0 = 0; g0 < G; g0 += 4) {
        float2 t[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int gg = g0 + k;
          t[k] = make_float2(0.f, 0.f);
          if (gg < G) t[k] = ((gg == g) ? accb : cluster.map_shared_rank(accb, gg))[row * W + cc];
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (g0 + k < G) {
            av.x += t[k].x;
            av.y += t[k].y;
          }
        }
      }
      const float2 p = pt[row * PW + cc + 1];
      const float2 pu = pt[((row + M - 1) % M) * PW + cc + 1];
      const float2 pd = pt[((row + 1) % M) * PW + cc + 1];
      const float2 pl = pt[row * PW + cc];
      const float2 pr = pt[row * PW + cc + 2];
      const float2 lp = make_float2(4.f * p.x - pu.x - pd.x - pl.x - pr.x,
                                    4.f * p.y - pu.y - pd.y - pl.y - pr.y);
      const size_t gi = boff + (size_t)row * N + col0 + cc;
      const float2 reg = make_float2(a.lam * lp.x + a.gam * p.x, a.lam * lp.y + a.gam * p.y);
      if constexpr (MODE == K1_RESID) {
        float2 bb;
        if (a.bvec != nullptr) {
          bb = lb[i];
        } else {
          float2 uu = lu[i];
          if (a.update_u) {
            uu = make_float2(uu.x + lu1[i].x - av.x, uu.y + lu1[i].y - av.y);
            a.u[gi] = uu;
          }
          bb = make_float2(a.mu * uu.x + lr[i].x, a.mu * uu.y + lr[i].y);
          a.bout[gi] = bb;
        }
        const float2 r = make_float2(bb.x - (a.mu * av.x + reg.x), bb.y - (a.mu * av.y + reg.y));
        if (a.spec) accb[row * W + cc] = r;  // (G = 1) this thread's own accumulator cell
        else a.out[gi] = r;
        d0 += (double)bb.x * bb.x + (double)bb.y * bb.y;
        d1 += (double)r.x * r.x + (double)r.y * r.y;
      } else {
        const float2 q = make_float2(a.mu * av.x + reg.x, a.mu * av.y + reg.y);
        if (MODE != K1_APPLY && a.spec) accb[row * W + cc] = q;
        else a.out[gi] = q;
        d0 += (double)p.x * q.x + (double)p.y * q.y;
      }
    }
  }
  if (MODE != K1_APPLY && a.spec) {
    // spectral-residual preconditioner: the column spectrum
    // F_0 q (PCG) or F_0 r0 (RESID) of this tile, from the cells written above (G = 1: the
    // CTA holds every row of its columns), to `out` in spectral row order
    __syncthreads();
    float2 v[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) v[n1] = accb[natidx<M>(j, n1) * W + l];
    if constexpr (TWR) fft_fwd_r<M, Lay>(v, xch, twr, j, l);
    else fft_fwd<M, Lay>(v, xch, tw, j, l);
#pragma unroll
    for (int s = 0; s < N1; ++s) a.out[boff + (size_t)specidx<M>(j, s) * N + col0 + l] = v[s];
  }
  if constexpr (MODE == K1_APPLY) {
    if (G > 1) cluster.sync();  // peers finished reading this CTA's accb
    return;
  }
  // block sums, then a fixed-order pre-reduction over the cluster through DSMEM: one partial
  // (and one arrival atomic) per cluster instead of one per CTA
  double s0 = block_sum(d0, red);
  double s1 = 0.0;
  if constexpr (MODE == K1_RESID) s1 = block_sum(d1, red);
  if (G > 1) {
    if (tid == 0) {
      double* rk0 = cluster.map_shared_rank(cred, 0);
      rk0[2 * g] = s0;
      rk0[2 * g + 1] = s1;
    }
    cluster.sync();  // also: peers finished reading this CTA's accb
    if (g != 0) return;
    if (tid == 0) {
      s0 = 0.0;
      s1 = 0.0;
      for (int gg = 0; gg < G; ++gg) {
        s0 += cred[2 * gg];
        s1 += cred[2 * gg + 1];
      }
    }
  }
  const int nblk = gridDim.y;  // one publisher per cluster (tile)
  const bool last = publish_and_check_last(s0, s1, a.P, b, tile, nblk, &lastflag);
  if (!last) return;
  if (tid < 32) {
    const double t0 = warp_sum_partials(a.P.p0 + (size_t)b * a.P.cap, nblk);
    double t1 = 0.0;
    if constexpr (MODE == K1_RESID) t1 = warp_sum_partials(a.P.p1 + (size_t)b * a.P.cap, nblk);
    if (tid == 0) {
      if constexpr (MODE == K1_PCG) fin_sigma(a.L, b, t0);
      else fin_init(a.L, b, t0, t1, a.eps, a.maxit);
      a.P.cnt[b] = 0;
    }
  }
}

// ------------------------------------------------------------------ host launchers
template <int M, int W>
constexpr size_t k1_smem() {
  return (size_t)(2 * M * W + ColLayout<M, W>::size + M * (W + 2) + M) * sizeof(float2) +
         (M + (M & 1)) * sizeof(float) + 2 * sizeof(uint64_t);
}

template <int M, int W, int MODE>
static cudaError_t launch_k1_t(const K1Args& a, const CUtensorMap* tmap, int G, cudaStream_t st) {
  auto kern = k1_matvec<M, W, MODE>;
  constexpr size_t smem = k1_smem<M, W>();
  static bool attr_done = false;  // per instantiation
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess) return e;
    attr_done = true;
  }
  return launch_ex(kern, dim3(G, a.N / W, a.B), dim3(Split<M>::N2 * W), smem, st, G, *tmap, a);
}

template <int M, int W>
static cudaError_t launch_k1_mw(int mode, const K1Args& a, const CUtensorMap* tmap, int G, cudaStream_t st) {
  switch (mode) {
    case K1_APPLY: return launch_k1_t<M, W, K1_APPLY>(a, tmap, G, st);
    case K1_PCG: return launch_k1_t<M, W, K1_PCG>(a, tmap, G, st);
    default: return launch_k1_t<M, W, K1_RESID>(a, tmap, G, st);
  }
}

template <int M>
static cudaError_t launch_k1_m(int mode, const K1Args& a, const CUtensorMap* tmap, int W, int G,
                               cudaStream_t st) {
  switch (W) {
    case 4: return launch_k1_mw<M, 4>(mode, a, tmap, G, st);
    case 8: return launch_k1_mw<M, 8>(mode, a, tmap, G, st);
    default: return cudaErrorInvalidValue;
  }
}

bool k1_supported(int M, int N) {
  const bool m_ok = (M == 8 || M == 16 || M == 32 || M == 64 || M == 128 || M == 256);
  return m_ok && N >= 4 && N % 4 == 0 && N <= 65536;
}

int k1_default_W(int M, int N) { return (N % 8 == 0) ? 8 : 4; }

cudaError_t launch_k1(int mode, const K1Args& a, const CUtensorMap* tmap, int W, int G,
                      cudaStream_t st) {
  if (a.N % W != 0 || G > 16 || G < 1) return cudaErrorInvalidValue;
  switch (a.M) {
    case 8: return launch_k1_m<8>(mode, a, tmap, W, G, st);
    case 16: return launch_k1_m<16>(mode, a, tmap, W, G, st);
    case 32: return launch_k1_m<32>(mode, a, tmap, W, G, st);
    case 64: return launch_k1_m<64>(mode, a, tmap, W, G, st);
    case 128: return launch_k1_m<128>(mode, a, tmap, W, G, st);
    case 256: return launch_k1_m<256>(mode, a, tmap, W, G, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace sbk
