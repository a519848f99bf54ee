// k_pcgc.cu — KC: the whole PCG loop of one problem in ONE persistent 16-CTA cluster
// (line masks, 256 x 256; BASELINE configs 2 and 3).  PCG of PAPER.md:234-238 (readings
// A15-A18) with the circulant preconditioner M^{-1} = F^H diag(k)^{-1} F,
// exactly the iteration of the kernel sequence K1 -> K2a -> K2b -> K2c (pcg_fin.cuh), but:
//   * CTA g of the cluster owns columns [16g, 16g+16) of its problem for the matvec (the
//     line-mask identity: one 256-point FFT pair per column and coil, k_matvec.cu) and for
//     the column passes of the preconditioner, and rows [16g, 16g+16) for its row pass;
//   * the four global reductions per iteration (sigma, ||r||^2, <r,z>) are cluster
//     reductions: every CTA publishes its block sum in its own shared memory, one cluster
//     barrier, every CTA sums the 16 values through DSMEM in the same fixed order (so all
//     CTAs hold bit-identical scalars) — no kernel boundary, no grid-wide atomics;
//   * q = A p never leaves the registers (r -= alpha q uses the epilogue's values);
//   * the problem's coil maps and vectors stay L2-resident across its iterations, and the
//     next iteration's first two coil tiles are fetched (TMA) while the preconditioner runs.
// Cluster barriers per iteration: 4 (after sigma, after the column FFT + ||r||^2, after the
// row pass, after <r,z>).  Rank 0 mirrors the scalars into Scal (log, fixup, host); x is left
// with the deferred update of the last iteration for k_fixup, exactly as the kernel sequence.
#include <cooperative_groups.h>

#include "kernels.cuh"
#include "pcg_fin.cuh"

namespace cg = cooperative_groups;

namespace sbk {

constexpr int KC_M = 256, KC_W = 16, KC_G = 16;

template <int M, int W>
struct KcCfg {
  static constexpr int N1 = Split<M>::N1, N2 = Split<M>::N2;
  static_assert(N1 == N2, "square split");
  static constexpr int NT = N2 * W;           // 256 threads
  static constexpr int TILE = M * W;          // coil tile (complex)
  static constexpr int PW = W + 2;            // p tile with +-1 column halo
  using CLay = typename ColLayout<M, W>::L;
  using RLay = typename RowLayout<M, W>::L;  // W rows per CTA in the row pass
  static constexpr int XS = ColLayout<M, W>::size > RowLayout<M, W>::size ? ColLayout<M, W>::size
                                                                          : RowLayout<M, W>::size;
  static constexpr size_t smem = (size_t)(2 * TILE + XS + M * PW + M) * sizeof(float2) + M * sizeof(float) +
                                 2 * sizeof(uint64_t);
};

template <int M, int W>
__global__ void __launch_bounds__(KcCfg<M, W>::NT, 1)
    kc_pcg(const __grid_constant__ CUtensorMap tmap, const KcArgs a) {
  using K = KcCfg<M, W>;
  constexpr int N1 = K::N1, N2 = K::N2, NT = K::NT, TILE = K::TILE, PW = K::PW;
  constexpr int G = KC_G;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float2* ring = reinterpret_cast<float2*>(smem_raw);  // [2][TILE]
  float2* xch = ring + 2 * TILE;                        // K::XS
  float2* pt = xch + K::XS;                             // [M][PW]
  float2* tw = pt + M * PW;                             // [M]
  float* rm = reinterpret_cast<float*>(tw + M);         // [M]
  uint64_t* bar = reinterpret_cast<uint64_t*>(rm + M);  // [2]
  __shared__ double red[32];
  __shared__ double slot[4];                            // this CTA's published block sums

  cg::cluster_group cluster = cg::this_cluster();
  const int g = blockIdx.x;  // cluster rank
  const int b = blockIdx.y;
  const int tid = threadIdx.x, j = tid / W, l = tid % W;
  const int N = a.N;  // == M
  const int col0 = g * W;
  const size_t img = (size_t)M * N, boff = (size_t)b * img;
  const int C = a.C;

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
  float2 twr[N1];
  load_twr<M>(twr, tw, j);
  float rmr[N1];
#pragma unroll
  for (int q = 0; q < N1; ++q) rmr[q] = rm[specidx<M>(j, q)];

  // constant setup above overlaps the predecessor under programmatic dependent launch; every
  // read of solver state comes after the wait
  pdl_trigger();
  pdl_wait();
  // scalars (set by the init kernels); identical in every CTA of the cluster from here on
  Scal* S = a.L.scal + b;
  int active = __ldcg(&S->active);
  int k = __ldcg(&S->iter);
  double rho = __ldcg(&S->rho), beta = __ldcg(&S->beta), alpha = __ldcg(&S->alpha);
  const double nb2 = __ldcg(&S->nb2);
  const float eps = S->eps;
  const int maxit = S->maxit;
  const int k0 = k;
  if (!active) return;  // uniform over the cluster

  // coil tiles stream through a 2-stage ring in a running sequence (seq -> coil seq % C,
  // stage seq & 1) that continues across iterations, so the next iteration's first tiles load
  // while the preconditioner runs
  uint32_t seq_issue = 0, seq_use = 0;
  auto issue = [&]() {  // thread 0
    const int st = seq_issue & 1;
    mbar_expect_tx(&bar[st], TILE * 8);
    tma_load_3d(ring + st * TILE, &tmap, 2 * col0, 0, b * C + (int)(seq_issue % (uint32_t)C), &bar[st]);
  };
  for (int s = 0; s < 2; ++s) {
    if (tid == 0) issue();
    ++seq_issue;
  }

  // all CTAs of the cluster must have initialised their barriers/slots before DSMEM use
  cluster.sync();

  auto cluster_sum = [&](int which) -> double {  // fixed order, identical in every CTA
    double t = 0.0;
#pragma unroll 1
    for (int gg = 0; gg < G; ++gg) t += *cluster.map_shared_rank(slot + which, gg);
    return t;
  };

  int status = ST_OK;
  while (true) {
    const int kk = k + 1;  // iteration being formed
    const bool first = (kk == 1);
    const float2* pold = (kk & 1) ? a.pbuf0 : a.pbuf1;
    float2* pnew = (kk & 1) ? a.pbuf1 : a.pbuf0;

    // ---- (a) p_k = z + beta p_{k-1} on the tile (+halo); own columns: p_k -> pnew and the
    // deferred x += alpha_{k-1} p_{k-1}
    constexpr int PE = (M * PW + NT - 1) / NT;
    constexpr int CH = PE < 9 ? PE : 9;
    for (int c0 = 0; c0 < PE; c0 += CH) {
      float2 zz[CH], po[CH], xv[CH];
      bool own[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int e = (c0 + i) * NT + tid;
        own[i] = false;
        if (c0 + i < PE && e < M * PW) {
          const int row = e / PW, cc = e % PW;
          int gcol = col0 + cc - 1;
          gcol = gcol < 0 ? gcol + N : (gcol >= N ? gcol - N : gcol);
          const size_t gi = boff + (size_t)row * N + gcol;
          zz[i] = __ldcg(a.z + gi);
          if (!first) po[i] = __ldcg(pold + gi);
          own[i] = cc >= 1 && cc <= W;
          if (own[i] && !first) xv[i] = __ldcg(a.x + gi);
        }
      }
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int e = (c0 + i) * NT + tid;
        if (c0 + i < PE && e < M * PW) {
          const float2 p = first ? zz[i] : make_float2(zz[i].x + (float)beta * po[i].x, zz[i].y + (float)beta * po[i].y);
          pt[e] = p;
          if (own[i]) {
            const size_t gi = boff + (size_t)(e / PW) * N + col0 + (e % PW) - 1;
            pnew[gi] = p;
            if (!first)
              a.x[gi] = make_float2(xv[i].x + (float)alpha * po[i].x, xv[i].y + (float)alpha * po[i].y);
          }
        }
      }
    }
    __syncthreads();

    // ---- (b) coil loop: acc = sum_c conj(s_c) F0^H (r/M . F0 (s_c p))
    float2 acc[N1];
#pragma unroll
    for (int i = 0; i < N1; ++i) acc[i] = make_float2(0.f, 0.f);
    for (int ci = 0; ci < C; ++ci) {
      const int stage = seq_use & 1;
      mbar_wait(&bar[stage], (seq_use >> 1) & 1);
      ++seq_use;
      const float2* sc = ring + stage * TILE;
      float2 s[N1], v[N1];
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int row = natidx<M>(j, n1);
        s[n1] = sc[row * W + l];
        v[n1] = cmul(s[n1], pt[row * PW + l + 1]);
      }
      fft_fwd_r<M, typename K::CLay>(v, xch, twr, j, l);
      // ring[stage] has been read by every thread (barrier inside fft_fwd_r): refill it with
      // the tile two ahead in the sequence (possibly coil 0/1 of the next iteration)
      if (tid == 0) issue();
      ++seq_issue;
#pragma unroll
      for (int q = 0; q < N1; ++q) v[q] = cscale(v[q], rmr[q]);
      fft_inv_r<M, typename K::CLay>(v, xch, twr, j, l);
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) acc[n1] = cfmac(s[n1], v[n1], acc[n1]);
    }

    // ---- (c) epilogue: q = mu acc + lambda L p + gamma p ; sigma = Re<p, q>
    double d0 = 0.0;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const int row = natidx<M>(j, n1);
      const float2 p = pt[row * PW + l + 1];
      const float2 pu = pt[((row + M - 1) % M) * PW + l + 1], pd = pt[((row + 1) % M) * PW + l + 1];
      const float2 pl = pt[row * PW + l], pr = pt[row * PW + l + 2];
      const float2 lp = make_float2(4.f * p.x - pu.x - pd.x - pl.x - pr.x, 4.f * p.y - pu.y - pd.y - pl.y - pr.y);
      const float2 qv = make_float2(a.mu * acc[n1].x + a.lam * lp.x + a.gam * p.x,
                                    a.mu * acc[n1].y + a.lam * lp.y + a.gam * p.y);
      acc[n1] = qv;  // q stays in registers
      d0 += (double)p.x * qv.x + (double)p.y * qv.y;
    }
    {
      const double s0 = block_sum(d0, red);
      if (tid == 0) slot[0] = s0;
    }
    cluster.sync();  // #1: sigma partials
    const double sigma = cluster_sum(0);
    if (!isfinite(sigma)) status = ST_NONFINITE;
    else if (!(sigma > 0.0)) status = ST_INDEFINITE;
    if (status != ST_OK) break;
    alpha = rho / sigma;

    // ---- (d) r_k = r - alpha q ; ||r_k||^2 ; column FFT of r_k -> tmp (spectral rows)
    float2 v[N1];
    double d1 = 0.0;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const size_t gi = boff + (size_t)natidx<M>(j, n1) * N + col0 + l;
      const float2 rv = __ldcg(a.r + gi);
      v[n1] = make_float2(rv.x - (float)alpha * acc[n1].x, rv.y - (float)alpha * acc[n1].y);
      a.r[gi] = v[n1];
      d1 += (double)v[n1].x * v[n1].x + (double)v[n1].y * v[n1].y;
    }
    fft_fwd_r<M, typename K::CLay>(v, xch, twr, j, l);
#pragma unroll
    for (int s2 = 0; s2 < N1; ++s2) a.tmp[boff + (size_t)specidx<M>(j, s2) * N + col0 + l] = v[s2];
    {
      const double s1 = block_sum(d1, red);
      if (tid == 0) slot[1] = s1;
    }
    cluster.sync();  // #2: ||r||^2 partials; the column-FFT output is complete
    const double rr = cluster_sum(1);
    k = kk;
    const double rel = sqrt(rr / nb2);
    if (g == 0 && tid == 0) {
      S->alpha = alpha;
      S->sigma = sigma;
      S->rr = rr;
      S->iter = k;
      hist_put(a.L, b, k, rel);
    }
    if (!isfinite(rr)) {
      status = ST_NONFINITE;
      break;
    }
    if (eps > 0.f && rel <= (double)eps) {
      if (g == 0 && tid == 0) S->converged = 1;
      break;
    }

    // ---- (e) row pass: rows [16g, 16g+16): row FFT, x Lambda^{-1}, row IFFT (in place)
    {
      const int line = tid / N2, jj = tid % N2;
      const int row = g * W + line;
      float2* t = a.tmp + boff + (size_t)row * N;
      const float* li = a.lam_inv + boff + (size_t)row * N;
      float2 u[N1];
      float lv[N1];
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        u[n1] = __ldcg(t + natidx<M>(jj, n1));
        lv[n1] = li[specidx<M>(jj, n1)];
      }
      __syncthreads();  // xch reuse (the column FFT above)
      fft_fwd<M, typename K::RLay>(u, xch, tw, jj, line);
#pragma unroll
      for (int s2 = 0; s2 < N1; ++s2) u[s2] = cscale(u[s2], lv[s2]);
      fft_inv<M, typename K::RLay>(u, xch, tw, jj, line);
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) t[natidx<M>(jj, n1)] = u[n1];
    }
    cluster.sync();  // #3: row pass complete

    // ---- (f) column IFFT -> z_k ; rho' = <r_k, z_k>
    {
#pragma unroll
      for (int s2 = 0; s2 < N1; ++s2) v[s2] = __ldcg(a.tmp + boff + (size_t)specidx<M>(j, s2) * N + col0 + l);
      __syncthreads();  // xch reuse (row pass)
      fft_inv_r<M, typename K::CLay>(v, xch, twr, j, l);
      double d2 = 0.0;
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const size_t gi = boff + (size_t)natidx<M>(j, n1) * N + col0 + l;
        const float2 rv = __ldcg(a.r + gi);
        a.z[gi] = v[n1];
        d2 += (double)rv.x * v[n1].x + (double)rv.y * v[n1].y;
      }
      const double s2 = block_sum(d2, red);
      if (tid == 0) slot[2] = s2;
    }
    cluster.sync();  // #4: <r, z> partials
    const double rz = cluster_sum(2);
    if (!isfinite(rz)) {
      status = ST_NONFINITE;
      break;
    }
    bool stop = false;
    if (rz == 0.0) {
      if (g == 0 && tid == 0) S->converged = 1;
      stop = true;
    } else if (k >= maxit) {
      if (g == 0 && tid == 0) S->converged = (eps == 0.f) ? 1 : 0;
      stop = true;
    } else {
      beta = rz / rho;
      rho = rz;
      if (g == 0 && tid == 0) {
        S->beta = beta;
        S->rho = rho;
      }
    }
    if (stop) break;
    __syncthreads();  // xch reuse before the next coil loop
  }

  if (g == 0 && tid == 0) {
    if (status != ST_OK) S->status = status;
    S->active = 0;
  }
  // drain the prefetched coil tiles (issued for an iteration that will not run)
  while (seq_use < seq_issue) {
    mbar_wait(&bar[seq_use & 1], (seq_use >> 1) & 1);
    ++seq_use;
  }
  if (g == 0 && tid == 0 && a.L.cnt != nullptr) atomicAdd(&a.L.cnt->k1_problems, (unsigned long long)(k - k0));
  cluster.sync();  // no CTA leaves while peers may still read its slots
}

bool kc_supported(int M, int N) { return M == KC_M && N == KC_M; }

cudaError_t launch_kc(const KcArgs& a, const CUtensorMap* tmap, cudaStream_t st) {
  using K = KcCfg<KC_M, KC_W>;
  auto kern = kc_pcg<KC_M, KC_W>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K::smem);
    if (e != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess) return e;
    attr = true;
  }
  return launch_ex(kern, dim3(KC_G, a.B), dim3(K::NT), K::smem, st, KC_G, *tmap, a);
}

}  // namespace sbk
