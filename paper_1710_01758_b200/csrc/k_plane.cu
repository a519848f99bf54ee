// k_plane.cu — K1P: plane kernels for masks that are NOT constant along a plane axis.
//
// A plane is NY x NZ (row-major, NZ contiguous).  2D problems with a generic 2D mask (BASELINE
// config 4 after readout decoupling) are one plane per problem; 3D problems whose mask is
// constant along the readout d0 (BASELINE config 5, PAPER.md:265 Cartesian sampling with a
// fully sampled readout) are d0 planes per problem, because then
//     F_3^H R F_3 = I_0 (x) F_12^H R_12 F_12        (F_3 = F_0 (x) F_12, R = I_0 (x) R_12),
// so the data term of A is a 2D operation on every d0 plane (DESIGN.md a1).
//
// One thread-block cluster of G CTAs owns one plane.  CTA g holds the interleaved rows
// y = G*y' + g (y' < NYL = NY/G) in shared memory.  The 2D DFT of the plane is
//   (1) a length-NZ FFT along every local row (register four-step, fft_core.cuh);
//   (2) a length-NYL register DFT down every local column, times the twiddle W_NY^{g kb};
//   (3) a length-G DFT across the cluster: CTA h reads rows kb in [h*KB, (h+1)*KB) of every
//       CTA's tile through distributed shared memory (DSMEM), giving
//       X[kb + NYL*ka][kz] = sum_g W_G^{g ka} W_NY^{g kb} sum_y' x[G y' + g] W_NYL^{y' kb};
// the pointwise step (mask r/N, or Lambda^{-1}) is applied there, and the inverse runs the
// three stages backwards, writing the length-G inverse DFT back into the owners' tiles.
// No global-memory round trip for the spectra.  The exchange (XCH, the matvec and
// preconditioner modes) is push-based and runs on the bulk-copy (TMA) engine: after its column
// DFT, CTA g copies rows [h KB, (h+1) KB) of its tile into CTA h's receive buffer with one
// cp.async.bulk shared::cta -> shared::cluster per peer, completion counted in bytes on h's
// mbarrier; h waits for the full buffer, transforms in place, and bulk-copies each owner's rows
// back into the owner's tile against the owner's second mbarrier.  Every wait is a data
// dependency, so there is no cluster-wide barrier per coil (a cluster barrier costs ~0.4 us
// plus a GPU-scope fence and an L1 invalidate), and the threads issue no
// per-element remote stores.  ENCODE / ADJOINT keep the pull exchange between two cluster
// barriers.
//
// Modes:
//   KP_APPLY / KP_PCG / KP_RESID  q = mu sum_c conj(s_c) F^H(r F(s_c p))/.. + lambda L p + gamma p
//        with the same PCG fusion as K1 (k_matvec.cu): p_k = z + beta p_{k-1}, deferred
//        x += alpha p_{k-1}, sigma = Re<p,q> partials + last-block alpha,
//        or (RESID) r0 = b - A x with the SB right-hand side / data feedback epilogue.
//        L is the periodic 5-point (2D) or 7-point (3D) Laplacian sum_d D_d^H D_d.
//   KP_PRECOND   tmp plane <- F_12^{-1}( Lambda^{-1} . F_12 tmp ) (3D preconditioner middle
//                pass, between the d0 FFTs of k_passes.cu).
//   KP_ENCODE    out[c] = (R) F_12 (s_c . x) * scale
//   KP_ADJOINT   out = sum_c conj(s_c) F_12^{-1}(R tmp_c) * scale, out2 = RSS
#include <cooperative_groups.h>

#include "kernels.cuh"
#include "pcg_fin.cuh"

namespace cg = cooperative_groups;

namespace sbk {

template <int NY, int NZ, int G>
struct PlaneCfg {
  static constexpr int NYL = NY / G;
  static constexpr int KB = NYL / G;
  static constexpr int N1 = Split<NZ>::N1, N2 = Split<NZ>::N2;
  static constexpr int T = NYL * N2;  // row stage: one (row, j) slot per thread
  static_assert(NYL * G == NY && KB * G == NYL, "G must divide NY/G");
  static_assert(NZ <= T, "column stage needs one thread per column");
  static_assert(NYL <= 32, "column DFT is register resident");
  using RLay = typename RowLayout<NZ, NYL>::L;
  // row stride of the spectra tile in shared memory: == N2 (mod 32) elements, so the 32/N2 rows
  // a warp touches in the row stage fall on distinct banks (no conflicts for 8-byte elements)
  static constexpr int NZP = NZ + ((N2 - NZ) % 32 + 32) % 32;
  static constexpr int WBS = RowLayout<NZ, NYL>::size > NYL * NZP ? RowLayout<NZ, NYL>::size : NYL * NZP;
  // twiddles: forward table [k1][j] and inverse table [q][n2][j] (j fastest, conflict free) + NY
  static constexpr int TS = NYL * NZP;  // p tile / receive buffer slot
  static constexpr size_t smem0 = (size_t)(WBS + TS + 2 * NZ + NY) * sizeof(float2);
  // prefetch buffer for the next coil's s_c tile (cp.async), double-buffered (s_c stays in
  // shared memory for the conj multiply after the inverse).  Only where the kernel is already
  // at 1 CTA/SM: elsewhere occupancy wins (config 4's 256x128 planes: no prefetch + 4 CTAs/SM
  // at <= 128 registers is 915 us per K1P launch vs 1059 us with the prefetch at 3 CTAs/SM)
  static constexpr size_t sbytes = 2 * (size_t)NYL * NZ * sizeof(float2);
  static constexpr bool PREF = smem0 > 113 * 1024 && smem0 + sbytes <= 220 * 1024;
  static constexpr size_t smem = smem0 + (PREF ? sbytes : 0);
};

// bulk L2 prefetch (TMA engine) of `bytes` (multiple of 16) at a 16-byte aligned global address
__device__ __forceinline__ void l2_prefetch(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int G>
__device__ __forceinline__ void cl_sync() {
  if constexpr (G > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
}

template <int G>
__device__ __forceinline__ float2* peer(float2* p, int rank) {
  if constexpr (G > 1) {
    return cg::this_cluster().map_shared_rank(p, rank);
  } else {
    return p;
  }
}

template <int NY, int NZ, int G, int MODE>
__global__ void __launch_bounds__(PlaneCfg<NY, NZ, G>::T, PlaneCfg<NY, NZ, G>::T <= 128 ? 4 : (PlaneCfg<NY, NZ, G>::T <= 256 ? 2 : 1))
    kp_plane(const KPArgs a) {
  const bool D3 = a.d3 != 0;
  using P = PlaneCfg<NY, NZ, G>;
  constexpr int NYL = P::NYL, KB = P::KB, N1 = P::N1, N2 = P::N2, T = P::T, NZP = P::NZP;
  constexpr int PN = NY * NZ;
  constexpr bool MATVEC = (MODE == KP_APPLY || MODE == KP_PCG || MODE == KP_RESID);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* wb = reinterpret_cast<float2*>(smem_raw);  // P::WBS: row exchange / tile spectra
  // push exchange through bulk copies + mbarriers (see the header)
  constexpr bool XCH = (G > 1) && (MATVEC || MODE == KP_PRECOND || MODE == KP_PRE2D);
  // the p (or x) tile is kept in shared memory by the pull-exchange modes that multiply by it
  // (encode); with XCH its slot holds the receive buffer and p is re-read from global (L2)
  constexpr bool HAS_PT = !XCH && (MATVEC || MODE == KP_ENCODE);
  float2* pt = wb + P::WBS;                          // NYL x NZ: p (or x) tile, natural
  float2* recv = pt;                                 // XCH: NYL x NZ receive buffer
  float2* twz = pt + ((HAS_PT || XCH) ? P::TS : 0);  // 2 NZ: forward, inverse row twiddles
  float2* twy = twz + 2 * NZ;                        // NY
  float2* sbuf = twy + NY;                           // P::PREF: [2][NYL x NZ] s_c tiles
  __shared__ double red[32];
  __shared__ int lastflag;
  __shared__ __align__(8) uint64_t xbar[2];         // XCH: [0] receive buffer full, [1] tile returned
  constexpr uint32_t XBYTES = (uint32_t)(NYL * NZP * sizeof(float2));
  constexpr uint32_t XROWS = (uint32_t)(KB * NZP * sizeof(float2));  // one bulk copy: KB tile rows

  const int g = blockIdx.x;  // cluster rank (cluster dims = (G,1,1), grid.x = G)
  const int xpl = blockIdx.y + a.plane0;  // plane (launches may cover a chunk of planes)
  const int b = blockIdx.z;
  const int tid = threadIdx.x;
  const int r = tid / N2, j = tid % N2;  // row stage
  const int planes = a.planes;
  const size_t img = (size_t)planes * PN;
  const size_t boff = (size_t)b * img;
  const size_t poff = boff + (size_t)xpl * PN;

  for (int i = tid; i < NZ; i += T) {
    const int k1 = i / N2, jj = i % N2, q = i / (N2 * N2), n2 = (i / N2) % N2;
    twz[i] = a.tw_z[jj * k1];                 // W^{j k1}
    twz[NZ + i] = a.tw_z[n2 * (jj + q * N2)];  // W^{n2 k1}, k1 = j + q N2
  }
  for (int i = tid; i < NY; i += T) twy[i] = a.tw_y[i];
  pdl_trigger();
  pdl_wait();

  double beta = 0.0, alpha_prev = 0.0;
  bool first = true;
  int pidx = 0;
  if constexpr (MODE == KP_PCG) {
    const Scal& s = a.L.scal[b];
    if (!s.active) return;  // uniform over the cluster
    const int k = s.iter + 1;
    first = (k == 1);
    pidx = k & 1;
    beta = s.beta;
    alpha_prev = s.alpha;
  } else if constexpr (MODE == KP_PRECOND) {
    if (a.L.scal != nullptr && __ldcg(&a.L.scal[b].active) == 0) return;
  } else if constexpr (MODE == KP_PRE2D) {
    if (a.L.scal != nullptr && a.pmode >= 0 && __ldcg(&a.L.scal[b].active) == 0) {
      if (g == 0 && tid == 0) slice_arrive(a.L);  // uniform over the cluster
      return;
    }
  }
  if (MATVEC && g == 0 && xpl == 0 && tid == 0 && a.L.cnt != nullptr) atomicAdd(&a.L.cnt->k1_problems, 1ull);
  if constexpr (XCH) {
    // both barriers armed for coil 0 before any peer can copy: a split cluster barrier whose
    // wait sits just before the first copy, so its latency hides behind coil 0's row stage
    if (tid == 0) {
      mbar_init(&xbar[0], 1);
      mbar_init(&xbar[1], 1);
      fence_mbar_init();
      mbar_expect_tx(&xbar[0], XBYTES);
      mbar_expect_tx(&xbar[1], XBYTES);
    }
    __syncthreads();
    cluster_arrive_relaxed();
  } else {
    __syncthreads();
  }

  const float2* pold = pidx ? a.pbuf0 : a.pbuf1;
  float2* pnew = pidx ? a.pbuf1 : a.pbuf0;
  // global index of (local row rr, column z) of this plane
  auto gidx = [&](int rr, int z) { return poff + (size_t)(G * rr + g) * NZ + z; };
  // p (or x) at local row rr, column z: the shared tile, or (XCH) this CTA's rows from global
  auto pget = [&](int rr, int z) -> float2 {
    if constexpr (HAS_PT) return pt[rr * NZ + z];
    else if constexpr (MODE == KP_PCG) return pnew[gidx(rr, z)];
    else return a.vin[gidx(rr, z)];
  };

  // ---- prologue: p (or x / input) tile into shared memory; PCG p-update and deferred x
  if constexpr (HAS_PT || MODE == KP_PCG) {
    constexpr int E = (NYL * NZ + T - 1) / T;
    constexpr int CH = E < 8 ? E : 8;
    for (int c0 = 0; c0 < E; c0 += CH) {
      float2 zz[CH], po[CH], xv[CH];
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int e = (c0 + i) * T + tid;
        if (c0 + i < E && e < NYL * NZ) {
          const size_t gi = gidx(e / NZ, e % NZ);
          if constexpr (MODE == KP_PCG) {
            zz[i] = a.z[gi];
            if (!first) {
              po[i] = pold[gi];
              xv[i] = a.x[gi];
            }
          } else {
            zz[i] = a.vin[gi];
          }
        }
      }
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int e = (c0 + i) * T + tid;
        if (c0 + i < E && e < NYL * NZ) {
          float2 p = zz[i];
          if constexpr (MODE == KP_PCG) {
            const size_t gi = gidx(e / NZ, e % NZ);
            if (!first) {
              p = make_float2(zz[i].x + (float)beta * po[i].x, zz[i].y + (float)beta * po[i].y);
              a.x[gi] = make_float2(xv[i].x + (float)alpha_prev * po[i].x, xv[i].y + (float)alpha_prev * po[i].y);
            }
            pnew[gi] = p;
          }
          if constexpr (HAS_PT) pt[e] = p;
        }
      }
    }
    __syncthreads();
  }

  // ---- the per-coil transform pipeline
  float2 acc[N1];
  float rss[N1];
#pragma unroll
  for (int i = 0; i < N1; ++i) {
    acc[i] = make_float2(0.f, 0.f);
    rss[i] = 0.f;
  }
  const int ncoil = (MODE == KP_PRECOND || MODE == KP_PRE2D) ? 1 : a.C;
  // PRE2D: r_k = r_{k-1} - alpha_k q_k, kept in registers for <r, z>
  float2 rk[MODE == KP_PRE2D ? N1 : 1];
  double drr = 0.0, drz = 0.0;
  if constexpr (MODE == KP_PRE2D) {
    const double alpha = (a.pmode == 1) ? a.L.scal[b].alpha : 0.0;
    float2 qq[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const size_t gi = gidx(r, N2 * n1 + j);
      rk[n1] = a.vin[gi];
      qq[n1] = (a.pmode == 1) ? a.qv[gi] : make_float2(0.f, 0.f);
    }
    if (a.pmode == 1) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        rk[n1].x -= (float)alpha * qq[n1].x;
        rk[n1].y -= (float)alpha * qq[n1].y;
        a.rout[gidx(r, N2 * n1 + j)] = rk[n1];
        drr += (double)rk[n1].x * rk[n1].x + (double)rk[n1].y * rk[n1].y;
      }
    }
  }
  const uint8_t* mk = a.mask + (size_t)b * a.mask_bstride;
  float2 colv[NYL];
  // the mask values this thread applies in stage (3): rows kb + NYL*ka, kb in this CTA's
  // range, column kz = tid -> NYL <= 32 bits, loaded once
  uint32_t mbits = 0;
  if (tid < NZ) {
#pragma unroll
    for (int kbl = 0; kbl < KB; ++kbl)
#pragma unroll
      for (int ka = 0; ka < G; ++ka)
        if (mk[(size_t)(g * KB + kbl + NYL * ka) * NZ + tid]) mbits |= 1u << (kbl * G + ka);
  }
  constexpr bool PF = P::PREF && (MATVEC || MODE == KP_ENCODE);
  auto prefetch_s = [&](int cc) {  // s_cc tile (this CTA's rows) -> sbuf[cc & 1], 16-byte cp.async
    const size_t so = ((size_t)b * a.C + cc) * img + (size_t)xpl * PN;
    float2* dst = sbuf + (cc & 1) * NYL * NZ;
    for (int e = tid; e < NYL * NZ / 2; e += T) {
      const int row = e / (NZ / 2), c2 = e % (NZ / 2);
      cp_async16(dst + row * NZ + 2 * c2, a.sens + so + (size_t)(G * row + g) * NZ + 2 * c2);
    }
    cp_async_commit();
  };
  if constexpr (PF) prefetch_s(0);
  // without the shared-memory prefetch buffer: the next coil's s_c rows of this CTA are pulled
  // into L2 by the bulk-copy engine while this coil is transformed, so the loads that start the
  // next coil's row stage hit L2 instead of HBM (one elected thread, one 16-byte-multiple row
  // each; NZ * 8 bytes per row)
  constexpr bool L2PF = !PF && (MATVEC || MODE == KP_ENCODE) && (NZ * 8) % 16 == 0;
  auto l2_prefetch_s = [&](int cc) {
    if (tid < NYL) {
      const size_t so = ((size_t)b * a.C + cc) * img + (size_t)xpl * PN;
      l2_prefetch(a.sens + so + (size_t)(G * tid + g) * NZ, (uint32_t)(NZ * sizeof(float2)));
    }
  };
  if constexpr (L2PF) {
    l2_prefetch_s(0);
  }

  for (int c = 0; c < ncoil; ++c) {
    const size_t soff = ((size_t)b * a.C + c) * img + (size_t)xpl * PN;
    float2 v[N1];
    if constexpr (MODE != KP_ADJOINT) {
      // (1) row FFTs of s_c . p (or the preconditioner plane)
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const int z = N2 * n1 + j;
        if constexpr (MODE == KP_PRECOND) {
          v[n1] = a.tmp[gidx(r, z)];
        } else if constexpr (MODE == KP_PRE2D) {
          v[n1] = rk[n1];
        } else if constexpr (PF) {
          if (n1 == 0) {
            cp_async_wait_all();
            __syncthreads();
          }
          v[n1] = cmul(sbuf[(c & 1) * NYL * NZ + r * NZ + z], pget(r, z));
        } else {
          v[n1] = cmul(a.sens[soff + (size_t)(G * r + g) * NZ + z], pget(r, z));
        }
      }
      fft_fwd_t<NZ, typename P::RLay>(v, wb, twz, j, r);
      if constexpr (PF) {  // every thread read sbuf before the barrier inside fft_fwd
        if (c + 1 < ncoil) prefetch_s(c + 1);
      }
      if constexpr (L2PF) {
        if (c + 1 < ncoil) l2_prefetch_s(c + 1);
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < N1; ++q) wb[r * NZP + specidx<NZ>(j, q)] = v[q];
      __syncthreads();
      // (2) local column DFT over y', twiddle W_NY^{g kb}
      if (tid < NZ) {
#pragma unroll
        for (int y = 0; y < NYL; ++y) colv[y] = wb[y * NZP + tid];
        Dft<NYL, -1>::run(colv);
#pragma unroll
        for (int kb = 1; kb < NYL; ++kb)
          if (g > 0) colv[kb] = cmul(colv[kb], twy[g * kb]);
#pragma unroll
        for (int kb = 0; kb < NYL; ++kb) wb[kb * NZP + tid] = colv[kb];
      }
      if constexpr (XCH) {
        // rows [h KB, (h+1) KB) -> CTA h's receive buffer rows [g KB, (g+1) KB): G bulk copies
        fence_proxy_async();
        if (c == 0) cluster_wait();  // every peer's barriers are initialised
        __syncthreads();
        if (tid == 0) {
          const uint32_t dst = smem_u32(recv + g * KB * NZP), bar = smem_u32(&xbar[0]);
#pragma unroll 1
          for (int h = 0; h < G; ++h) bulk_s2s(mapa_u32(dst, h), smem_u32(wb + h * KB * NZP), XROWS, mapa_u32(bar, h));
        }
      }
    } else {
      // adjoint: the rows about to be overwritten by peers must be free (previous coil done)
    }
    // s_c for the conj multiply after the inverse: from the prefetch buffer, or loaded now so
    // the L2 latency hides behind the cluster exchange
    float2 sv[MATVEC && !PF ? N1 : 1];
    if constexpr (MATVEC && !PF) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) sv[n1] = a.sens[soff + (size_t)(G * r + g) * NZ + N2 * n1 + j];
    }
    // the preconditioner's Lambda^{-1} values of this CTA's spectral rows, loaded before the
    // exchange wait so their latency hides behind it
    constexpr bool LAMF = XCH && (MODE == KP_PRECOND || MODE == KP_PRE2D);
    float lf[LAMF ? KB : 1][LAMF ? G : 1];
    if constexpr (LAMF) {
      if (tid < NZ) {
#pragma unroll
        for (int kbl = 0; kbl < KB; ++kbl)
#pragma unroll
          for (int ka = 0; ka < G; ++ka)
            lf[kbl][ka] = a.lam_inv[boff + (size_t)xpl * PN + (size_t)(g * KB + kbl + NYL * ka) * NZ + tid];
      }
    }
    if constexpr (XCH) {
      mbar_wait(&xbar[0], c & 1);  // all G x KB rows of every peer arrived
      if (tid == 0 && c + 1 < ncoil) mbar_expect_tx(&xbar[0], XBYTES);
    } else {
      cl_sync<G>();
    }
    // (3) cross-cluster DFT, pointwise operator, inverse cross-cluster DFT
    if (XCH && tid < NZ) {
      const int kz = tid;
      float2 wa[KB][G];
#pragma unroll
      for (int kbl = 0; kbl < KB; ++kbl)
#pragma unroll
        for (int gg = 0; gg < G; ++gg) wa[kbl][gg] = recv[(gg * KB + kbl) * NZP + kz];
#pragma unroll
      for (int kbl = 0; kbl < KB; ++kbl) {
        const int kb = g * KB + kbl;
        float2* w = wa[kbl];
        Dft<G, -1>::run(w);
#pragma unroll
        for (int ka = 0; ka < G; ++ka) {
          const int ky = kb + NYL * ka;
          float f;
          if constexpr (LAMF) {
            f = lf[kbl][ka];
          } else {
            f = ((mbits >> (kbl * G + ka)) & 1u) ? a.scale : 0.f;
          }
          w[ka] = cscale(w[ka], f);
          (void)ky;
        }
        Dft<G, +1>::run(w);
      }
      // results in place: rows (gg KB + kbl) of the receive buffer belong to owner gg
#pragma unroll
      for (int kbl = 0; kbl < KB; ++kbl)
#pragma unroll
        for (int gg = 0; gg < G; ++gg) recv[(gg * KB + kbl) * NZP + kz] = wa[kbl][gg];
    }
    if constexpr (XCH) {
      // owner gg's rows [g KB, (g+1) KB) go back into its tile: G bulk copies
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        const uint32_t dst = smem_u32(wb + g * KB * NZP), bar = smem_u32(&xbar[1]);
#pragma unroll 1
        for (int gg = 0; gg < G; ++gg) bulk_s2s(mapa_u32(dst, gg), smem_u32(recv + gg * KB * NZP), XROWS, mapa_u32(bar, gg));
      }
    }
    if (!XCH && tid < NZ) {
      const int kz = tid;
#pragma unroll
      for (int kbl = 0; kbl < KB; ++kbl) {
        const int kb = g * KB + kbl;
        float2 w[G];
        if constexpr (MODE == KP_ADJOINT) {
#pragma unroll
          for (int ka = 0; ka < G; ++ka) {
            const int ky = kb + NYL * ka;
            const float2 yv = a.tmp[soff + (size_t)ky * NZ + kz];
            const float f = ((mbits >> (kbl * G + ka)) & 1u) ? a.scale : 0.f;
            w[ka] = make_float2(yv.x * f, yv.y * f);
          }
        } else {
#pragma unroll
          for (int gg = 0; gg < G; ++gg) w[gg] = peer<G>(wb, gg)[kb * NZP + kz];
          Dft<G, -1>::run(w);
#pragma unroll
          for (int ka = 0; ka < G; ++ka) {
            const int ky = kb + NYL * ka;
            float f;
            if constexpr (MODE == KP_PRECOND || MODE == KP_PRE2D) {
              f = a.lam_inv[boff + (size_t)xpl * PN + (size_t)ky * NZ + kz];
            } else if constexpr (MODE == KP_ENCODE) {
              f = (a.full || ((mbits >> (kbl * G + ka)) & 1u)) ? a.scale : 0.f;
            } else {
              f = ((mbits >> (kbl * G + ka)) & 1u) ? a.scale : 0.f;
            }
            w[ka] = cscale(w[ka], f);
          }
        }
        if constexpr (MODE == KP_ENCODE) {
          float2* o = a.out + soff;
#pragma unroll
          for (int ka = 0; ka < G; ++ka) o[(size_t)(kb + NYL * ka) * NZ + kz] = w[ka];
        } else {
          Dft<G, +1>::run(w);
#pragma unroll
          for (int gg = 0; gg < G; ++gg) peer<G>(wb, gg)[kb * NZP + kz] = w[gg];
        }
      }
    }
    if constexpr (MODE == KP_ENCODE) {
      cl_sync<G>();  // peers finished reading this tile before the next coil overwrites it
      continue;
    }
    if constexpr (XCH) {
      mbar_wait(&xbar[1], c & 1);  // every row of this tile is back from its transformer
      if (tid == 0 && c + 1 < ncoil) mbar_expect_tx(&xbar[1], XBYTES);
    } else {
      cl_sync<G>();
    }
    // (4) inverse local column DFT
    if (tid < NZ) {
#pragma unroll
      for (int kb = 0; kb < NYL; ++kb) {
        const float2 t = wb[kb * NZP + tid];
        colv[kb] = (g > 0 && kb > 0) ? cmul_conjb(t, twy[g * kb]) : t;
      }
      Dft<NYL, +1>::run(colv);
#pragma unroll
      for (int y = 0; y < NYL; ++y) wb[y * NZP + tid] = colv[y];
    }
    __syncthreads();
    // (5) inverse row FFTs
#pragma unroll
    for (int q = 0; q < N1; ++q) v[q] = wb[r * NZP + specidx<NZ>(j, q)];
    __syncthreads();
    fft_inv_t<NZ, typename P::RLay>(v, wb, twz + NZ, j, r);
    if constexpr (MODE == KP_PRECOND) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) a.tmp[gidx(r, N2 * n1 + j)] = v[n1];
    } else if constexpr (MODE == KP_PRE2D) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        a.zout[gidx(r, N2 * n1 + j)] = v[n1];
        drz += (double)rk[n1].x * v[n1].x + (double)rk[n1].y * v[n1].y;
      }
    } else if constexpr (MODE == KP_ADJOINT) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const float2 sv = a.sens[soff + (size_t)(G * r + g) * NZ + N2 * n1 + j];
        acc[n1] = cfmac(sv, v[n1], acc[n1]);
        rss[n1] += v[n1].x * v[n1].x + v[n1].y * v[n1].y;
      }
    } else {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        float2 s1;
        if constexpr (PF) s1 = sbuf[(c & 1) * NYL * NZ + r * NZ + N2 * n1 + j];
        else s1 = sv[n1];
        acc[n1] = cfmac(s1, v[n1], acc[n1]);  // acc += conj(s_c) v
      }
    }
    __syncthreads();  // exchange reads done before the next coil writes wb
  }
  if constexpr (XCH) {  // no CTA leaves while bulk copies may still read its tile
    cluster_arrive_relaxed();
    cluster_wait();
  }

  if constexpr (MODE == KP_ADJOINT) {
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const size_t gi = gidx(r, N2 * n1 + j);
      a.out[gi] = acc[n1];
      if (a.out2 != nullptr) a.out2[gi] = make_float2(a.rss_raw ? rss[n1] : sqrtf(rss[n1]), 0.f);
    }
  }
  if constexpr (MATVEC) {
    if (a.acc_out != nullptr) {  // coil-sharded: partial coil sum out, epilogue after the all-reduce
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) a.acc_out[gidx(r, N2 * n1 + j)] = acc[n1];
      return;
    }
  }
  if constexpr (MODE == KP_PRE2D) {
    if (a.L.scal == nullptr || a.pmode < 0) return;
    const double s0 = block_sum(drz, red);
    const double s1 = block_sum(drr, red);
    const bool last = publish_and_check_last(s0, s1, a.P, b, xpl * G + g, planes * G, &lastflag);
    if (!last) return;
    if (tid < 32 || T < 32) {
      const double trz = warp_sum_partials(a.P.p0 + (size_t)b * a.P.cap, planes * G);
      const double trr = warp_sum_partials(a.P.p1 + (size_t)b * a.P.cap, planes * G);
      if (tid == 0) {
        if (a.pmode == 1) {
          fin_rr(a.L, b, trr);                                   // ||r_k||/||b|| stop test
          if (a.L.scal[b].active) fin_rho(a.L, b, trz, false);  // rho', beta, max-iter stop
        } else {
          fin_rho(a.L, b, trz, true);                            // rho_0
        }
        a.P.cnt[b] = 0;
        slice_arrive(a.L);
      }
    }
    return;
  }
  if constexpr (!MATVEC) return;

  // ---- epilogue: q = mu acc + lambda L p + gamma p  (or the RESID form)
  // neighbour p values outside this CTA's rows come from stable buffers (z, p_{k-1}, vin)
  auto pval = [&](size_t gi) -> float2 {
    if constexpr (MODE == KP_PCG) {
      const float2 zz = a.z[gi];
      if (first) return zz;
      const float2 po = pold[gi];
      return make_float2(zz.x + (float)beta * po.x, zz.y + (float)beta * po.y);
    } else {
      return a.vin[gi];
    }
  };
  double d0 = 0.0, d1 = 0.0;
  const int yrow = G * r + g;
  const size_t rowbase = boff + (size_t)xpl * PN;
  const size_t up = rowbase + (size_t)((yrow + NY - 1) % NY) * NZ;
  const size_t dn = rowbase + (size_t)((yrow + 1) % NY) * NZ;
  size_t xm = 0, xp = 0;
  if (D3) {
    xm = boff + (size_t)((xpl + planes - 1) % planes) * PN + (size_t)yrow * NZ;
    xp = boff + (size_t)((xpl + 1) % planes) * PN + (size_t)yrow * NZ;
  }
  const float cdeg = D3 ? 6.f : 4.f;
  constexpr int CE = N1 < 4 ? N1 : 4;  // epilogue chunk: bounded registers, batched loads
#pragma unroll
  for (int c0 = 0; c0 < N1; c0 += CE) {
    float2 nb[CE][4];
    float2 lb[CE], lu[CE], lu1[CE], lr[CE];
#pragma unroll
    for (int i = 0; i < CE; ++i) {
      const int z = N2 * (c0 + i) + j;
      nb[i][0] = pval(up + z);
      nb[i][1] = pval(dn + z);
      if (D3) {
        nb[i][2] = pval(xm + z);
        nb[i][3] = pval(xp + z);
      }
      if constexpr (MODE == KP_RESID) {
        const size_t gi = gidx(r, z);
        if (a.bvec != nullptr) {
          lb[i] = a.bvec[gi];
        } else {
          lu[i] = a.u[gi];
          lu1[i] = a.update_u ? a.u1[gi] : make_float2(0.f, 0.f);
          lr[i] = a.rhs_reg != nullptr ? a.rhs_reg[gi] : make_float2(0.f, 0.f);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < CE; ++i) {
      const int z = N2 * (c0 + i) + j;
      const float2 p = pget(r, z);
      const float2 pl = pget(r, (z + NZ - 1) % NZ);
      const float2 pr = pget(r, (z + 1) % NZ);
      float2 lp = make_float2(cdeg * p.x - pl.x - pr.x - nb[i][0].x - nb[i][1].x,
                              cdeg * p.y - pl.y - pr.y - nb[i][0].y - nb[i][1].y);
      if (D3) {
        lp.x -= nb[i][2].x + nb[i][3].x;
        lp.y -= nb[i][2].y + nb[i][3].y;
      }
      const float2 av = acc[c0 + i];
      const float2 reg = make_float2(a.lam * lp.x + a.gam * p.x, a.lam * lp.y + a.gam * p.y);
      const size_t gi = gidx(r, z);
      if constexpr (MODE == KP_RESID) {
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
  }
  if constexpr (MODE == KP_APPLY) return;
  const double s0 = block_sum(d0, red);
  double s1 = 0.0;
  if constexpr (MODE == KP_RESID) s1 = block_sum(d1, red);
  const int nblk = planes * G;
  const bool last = publish_and_check_last(s0, s1, a.P, b, xpl * G + g, nblk, &lastflag);
  if (!last) return;
  if (tid < 32 || T < 32) {
    const double t0 = warp_sum_partials(a.P.p0 + (size_t)b * a.P.cap, nblk);
    double t1 = 0.0;
    if constexpr (MODE == KP_RESID) t1 = warp_sum_partials(a.P.p1 + (size_t)b * a.P.cap, nblk);
    if (tid == 0) {
      if constexpr (MODE == KP_PCG) fin_sigma(a.L, b, t0);
      else fin_init(a.L, b, t0, t1, a.eps, a.maxit);
      a.P.cnt[b] = 0;
    }
  }
}

// ------------------------------------------------------------------ host side
template <int NY, int NZ, int G, int MODE>
static cudaError_t kp_launch(const KPArgs& a, cudaStream_t st) {
  using P = PlaneCfg<NY, NZ, G>;
  auto kern = kp_plane<NY, NZ, G, MODE>;
  constexpr bool MATVEC = (MODE == KP_APPLY || MODE == KP_PCG || MODE == KP_RESID);
  constexpr bool XCH = (G > 1) && (MATVEC || MODE == KP_PRECOND || MODE == KP_PRE2D);
  constexpr bool HAS_PT = !XCH && (MATVEC || MODE == KP_ENCODE);
  constexpr bool PF = P::PREF && (MATVEC || MODE == KP_ENCODE);
  constexpr size_t smem = P::smem0 - ((HAS_PT || XCH) ? 0 : (size_t)P::TS * sizeof(float2)) + (PF ? P::sbytes : 0);
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (G > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
      return e;
    attr_done = true;
  }
  return launch_ex(kern, dim3(G, a.nplanes > 0 ? a.nplanes : a.planes, a.B), dim3(P::T), smem, st, G > 1 ? G : 0, a);
}

// cluster size per plane height: the column DFT holds NY/G <= 32 values and G | NY/G
// NY = 256 takes a 16-CTA (non-portable) cluster: 16 rows per CTA, every thread busy in
// both the row and the column stage, no register spills (G = 8 spilled at 128 registers)
template <int NY> struct PlaneG {
  static constexpr int value = NY <= 32 ? 1 : (NY <= 64 ? 2 : (NY <= 128 ? 4 : (NY == 256 ? 16 : 8)));
};

template <int NY, int NZ>
static cudaError_t kp_matvec_modes(int mode, const KPArgs& a, cudaStream_t st) {
  constexpr int G = PlaneG<NY>::value;
  switch (mode) {
    case KP_PRE2D: return kp_launch<NY, NZ, G, KP_PRE2D>(a, st);
    case KP_APPLY: return kp_launch<NY, NZ, G, KP_APPLY>(a, st);
    case KP_PCG: return kp_launch<NY, NZ, G, KP_PCG>(a, st);
    case KP_RESID: return kp_launch<NY, NZ, G, KP_RESID>(a, st);
    default: return cudaErrorInvalidValue;
  }
}
template <int NY, int NZ>
static cudaError_t kp_all_modes(int mode, const KPArgs& a, cudaStream_t st) {
  constexpr int G = PlaneG<NY>::value;
  switch (mode) {
    case KP_PRECOND: return kp_launch<NY, NZ, G, KP_PRECOND>(a, st);
    case KP_ENCODE: return kp_launch<NY, NZ, G, KP_ENCODE>(a, st);
    case KP_ADJOINT: return kp_launch<NY, NZ, G, KP_ADJOINT>(a, st);
    default: return kp_matvec_modes<NY, NZ>(mode, a, st);
  }
}

#ifdef SBK_PLANE_3D
// 3D problems: planes of a readout-constant mask (all six modes)
#define SBK_PLANE_SIZES(X) X(16, 16) X(32, 32) X(48, 48) X(64, 64) X(128, 128) X(192, 192) X(256, 256)
#define SBK_PLANE_FN kp_all_modes
#define SBK_PLANE_ENTRY launch_kp3
#define SBK_PLANE_SUPP kp3_supported
#else
// 2D problems with a non-separable mask (matvec modes; encode/adjoint/preconditioner use the
// column/row passes of k_passes.cu)
#define SBK_PLANE_SIZES(X)                                                                       \
  X(8, 8) X(8, 16) X(8, 32) X(8, 64) X(16, 8) X(16, 16) X(16, 32) X(16, 64) X(16, 128) X(16, 256)   \
  X(32, 8) X(32, 16) X(32, 32) X(32, 64) X(32, 128) X(32, 256) X(64, 8) X(64, 16) X(64, 32)         \
  X(64, 64) X(64, 128) X(64, 256) X(128, 8) X(128, 16) X(128, 32) X(128, 64) X(128, 128)             \
  X(128, 256) X(256, 8) X(256, 16) X(256, 32) X(256, 64) X(256, 128) X(256, 256)
#define SBK_PLANE_FN kp_matvec_modes
#define SBK_PLANE_ENTRY launch_kp2
#define SBK_PLANE_SUPP kp2_supported
#endif

bool SBK_PLANE_SUPP(int NY, int NZ) {
#define X(a_, b_) if (NY == a_ && NZ == b_) return true;
  SBK_PLANE_SIZES(X)
#undef X
  return false;
}

cudaError_t SBK_PLANE_ENTRY(int mode, const KPArgs& a, cudaStream_t st) {
#define X(a_, b_) if (a.NY == a_ && a.NZ == b_) return SBK_PLANE_FN<a_, b_>(mode, a, st);
  SBK_PLANE_SIZES(X)
#undef X
  return cudaErrorInvalidValue;
}

}  // namespace sbk
