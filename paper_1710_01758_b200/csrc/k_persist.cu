// k_persist.cu — KR: the whole Split Bregman reconstruction (Algorithm 1)
// or one PCG solve of a small batch of square line-mask problems in ONE
// cooperative launch that spans the GPU.
//
// Why: one 256^2 x 12-coil problem (BASELINE config 2) is ~10 MFLOP of FFT work per PCG
// iteration; as a kernel sequence each iteration is two latency chains of ~17 us on a
// fraction of the SMs.  Here every problem gets P = N CTAs that stay resident for the whole
// reconstruction, and the kernel boundaries become per-problem grid barriers (~1.3 us each,
// measured: tools/microbench/gbar*.cu).  Everything a CTA owns stays in shared memory, so a
// phase makes at most one dependent round trip to L2.
//
// Ownership.  CTA t of problem b owns
//   * image column t (all M rows): the data term of A (per coil one length-M FFT pair down the
//     column, the line-mask identity F^H R F = F_0^H R_0 F_0 (x) I of DESIGN.md a1), the
//     Laplacian epilogue, the column transforms F_0 of the preconditioner, and the PCG vectors
//     x, r, q of that column.  Its coil-map column lines are staged in shared memory once;
//   * spectral row t of the preconditioner's column spectrum S_r = F_0 r (kept in shared
//     memory), the row transforms F_1, the diagonal Lambda^{-1} = 1/(N k).
// The Laplacian needs p at the neighbouring columns t-1, t+1: each CTA recomputes z and p of
// those two columns itself (the column IFFT of T and z + beta p_old, the same instructions on
// the same inputs as their owners, so the values are bitwise the owners'), which removes every
// halo exchange from the loop.
//
// One PCG iteration (standard PCG; readings A15-A18) = three phases:
//   P1 (column t):  p = z + beta p (columns t-1, t, t+1; shared memory only);
//                   q = A p; Q = F_0 q (column spectrum, to L2); partial Re<p, q>      | barrier
//   P2 (row t):     alpha = rho / sigma (every CTA sums the same partials in the same order);
//                   S_r -= alpha Q (F_0 is linear: F_0 (r - alpha q) = F_0 r - alpha F_0 q);
//                   T = F_1^H Lambda^{-1} F_1 S_r (row t, to L2; T is stored column-major, so
//                   the strided side is the row owner's fire-and-forget stores)        | barrier
//   P3 (column t):  x += alpha p; r -= alpha q; z = F_0^H T (columns t-1, t, t+1);
//                   partials ||r||^2, Re<r, z>                                         | barrier
// then ||r||/||b|| <= eps stops, else beta = rho'/rho.  The solve prelude computes
// r0 = b - A x0 (recon: b = mu u + rhs_reg with the image-domain data feedback u += u1 - E^H E x,
// reading A28), S_r = F_0 r0 and z0 = M^{-1} r0; the SB phase (recon) is the K5 tile update
// (sb_tile.cuh) on 16 x 16 tiles.  All scalars are fp64 and identical in every CTA of a
// problem (fixed-order sums of the same partials), so control flow needs no broadcast.
#include "pcg_fin.cuh"
#include "sb_tile.cuh"

namespace sbk {

template <int M>
struct KrCfg {
  static constexpr int N1 = Split<M>::N1, N2 = Split<M>::N2;
  static_assert(N1 == N2, "square four-step split (register twiddles)");
  static constexpr int NT = 192;            // threads per CTA
  static constexpr int LPAR = NT / N2;      // column lines in flight (coils per round)
  static constexpr int XL = N1 * (N2 + 1);  // exchange cells per line
  static constexpr int TT = 16;             // SB tile edge
};

template <int M>
struct KrSmem {
  using C = KrCfg<M>;
  union {
    float2 xch[C::LPAR * C::XL];      // FFT exchange areas (one per line) / coil-sum buffer
    SbTile<C::TT> sb;
  } u;
  float2 pc[3][M];                    // p (x in the prelude) of columns t-1, t, t+1
  float2 zc[3][M];                    // z of columns t-1, t, t+1
  float2 xs[M];                       // x, own column
  float2 rs[M];                       // r, own column
  float2 qs[M];                       // q, own column (first the data-term accumulator)
  float2 srow[M];                     // row t of S_r = F_0 r
  float2 ss[M];                       // s = A p, own column (Chronopoulos-Gear loop)
  float2 ssrow[M];                    // row t of S_s = F_0 s (Chronopoulos-Gear loop)
  float2 wrow[M];                     // row t of W = F_0 w (cp.async prefetch after the barrier)
  float2 ub[M], u1b[M], rhb[M];       // prelude: u, u1, rhs_reg (or b) of the own column
  alignas(16) float2 sbpre[sb_pre_size<C::TT>()];  // recon: the SB tile's old b_x, b_y, b_w (cp.async in the prelude)
  float2 tw[M];
  float li[M];                        // Lambda^{-1} of spectral row t
  float rm[M];                        // r/M (row mask)
  double red[48];
  double bc[8];                       // broadcast of reduced scalars
  long long tclk, tclk0;              // stage timer state (one thread of one CTA)
  unsigned long long tgt0, tstage[4];  // rhs, pcg, shrink, init
  // followed (SMC) by the coil-map column lines [C][M]
};

template <int M>
constexpr size_t kr_smem_bytes(int C, bool smc) {
  return (sizeof(KrSmem<M>) + 15) / 16 * 16 + (smc ? (size_t)C * M * sizeof(float2) : 0);
}

// ------------------------------------------------------------------ primitives
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_relaxed(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void kr_cp16(void* dst, const void* src) {  // 16-byte global -> shared, L2 only
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void kr_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void kr_cp_wait() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// A barrier that has not completed after ~4 s traps (a bug must fail the launch, not hang it).
__device__ __noinline__ void pbar_stuck(const unsigned* ctr, unsigned target) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (ld_relaxed(ctr) < target) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 4000000000ull) __trap();
  }
}
// Barrier over the P CTAs of one problem.  The fences order every global write of the CTA
// before the arrival and every later read after the departure (cross-CTA reads also use
// ld.global.cg, so no stale L1 line is read).
__device__ __forceinline__ void pbar(unsigned* ctr, unsigned& target, unsigned P) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += P;
    fence_acq_rel();
    red_relaxed(ctr, 1u);
    int spins = 0;
    while (ld_relaxed(ctr) < target) {
      if (++spins == (1 << 20)) {
        pbar_stuck(ctr, target);
        break;
      }
    }
    fence_acq_rel();
  }
  __syncthreads();
}

// Sums of the P partials of NS consecutive slots (stride P) in a fixed order (16-byte loads,
// lane stride 32, then a fixed shuffle tree), identical in every CTA; one L2 round trip for all
// slots.  P is a multiple of 64.
template <int P, int NS>
__device__ __forceinline__ void psum(const double* part, double* bc) {
  static_assert(P % 64 == 0, "P multiple of 64");
  if (threadIdx.x < 32) {
    constexpr int K = P / 64;
    double2 v[NS][K];
#pragma unroll
    for (int s = 0; s < NS; ++s)
#pragma unroll
      for (int i = 0; i < K; ++i)
        v[s][i] = __ldcg(reinterpret_cast<const double2*>(part + s * P) + threadIdx.x + 32 * i);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) acc += v[s][i].x + v[s][i].y;
      acc = warp_sum(acc);
      if (threadIdx.x == 0) bc[s] = acc;
    }
  }
  __syncthreads();
}

// psum<P, 1> by the calling warp (any warp), result in *dst (lane 0); no block barrier.
template <int P>
__device__ __forceinline__ void psum1_warp(const double* part, double* dst) {
  constexpr int K = P / 64;
  const int lane = threadIdx.x & 31;
  double2 v[K];
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = __ldcg(reinterpret_cast<const double2*>(part) + lane + 32 * i);
  double acc = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) acc += v[i].x + v[i].y;
  acc = warp_sum(acc);
  if (lane == 0) *dst = acc;
}

// Two deterministic block sums at once (fixed shuffle tree, fixed warp order); thread 0.
__device__ __forceinline__ void block_sum2(double& a, double& b, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  a = warp_sum(a);
  b = warp_sum(b);
  __syncthreads();
  if (lane == 0) {
    red[wid] = a;
    red[16 + wid] = b;
  }
  __syncthreads();
  if (wid == 0) {
    a = warp_sum(lane < nw ? red[lane] : 0.0);
    b = warp_sum(lane < nw ? red[16 + lane] : 0.0);
  }
}

// Block reduction of NS partials (NS <= 6) in two halves so other work can sit between them:
// red_warps() leaves one fixed-tree warp sum per (slot, warp) in red[s * 8 + warp] and ends with
// __syncthreads; red_final() (lanes of one warp) adds the warp sums in warp order (lane 0 result).
template <int NS>
__device__ __forceinline__ void red_warps(double (&v)[NS], double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const double w = warp_sum(v[s]);
    if (lane == 0) red[s * 8 + wid] = w;
  }
  __syncthreads();
}
template <int NS>
__device__ __forceinline__ void red_final(const double* red, double (&out)[NS]) {
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll
  for (int s = 0; s < NS; ++s) out[s] = warp_sum(lane < nw ? red[s * 8 + lane] : 0.0);
}

// Line FFTs of the four-step split, one line per N2 consecutive lanes (a line never crosses a
// warp, so __syncwarp orders the exchange).  Forward: natural -> spectral layout; inverse:
// spectral -> natural (fft_core.cuh conventions; xl = this line's exchange area).
template <int M>
__device__ __forceinline__ void kr_fwd(float2 (&v)[KrCfg<M>::N1], float2* xl, const float2 (&twr)[KrCfg<M>::N1],
                                       int j) {
  constexpr int N1 = KrCfg<M>::N1, N2 = KrCfg<M>::N2;
  Dft<N1, -1>::run(v);
#pragma unroll
  for (int k1 = 1; k1 < N1; ++k1) v[k1] = cmul(v[k1], twr[k1]);
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) xl[k1 * (N2 + 1) + j] = v[k1];
  __syncwarp();
#pragma unroll
  for (int n2 = 0; n2 < N2; ++n2) v[n2] = xl[j * (N2 + 1) + n2];
  Dft<N2, -1>::run(v);
  __syncwarp();
}
template <int M>
__device__ __forceinline__ void kr_inv(float2 (&v)[KrCfg<M>::N1], float2* xl, const float2 (&twr)[KrCfg<M>::N1],
                                       int j) {
  constexpr int N1 = KrCfg<M>::N1, N2 = KrCfg<M>::N2;
  Dft<N2, +1>::run(v);
#pragma unroll
  for (int n2 = 0; n2 < N2; ++n2) xl[j * (N2 + 1) + n2] = (n2 == 0 || j == 0) ? v[n2] : cmul_conjb(v[n2], twr[n2]);
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) v[k1] = xl[k1 * (N2 + 1) + j];
  Dft<N1, +1>::run(v);
  __syncwarp();
}

// Per-problem PCG scalars, replicated in every CTA (same arithmetic as pcg_fin.cuh).
struct KrScal {
  double rho, alpha, beta, sigma, nb2, rr;
  int iter, active, converged, status, zero_x;
};

// Row t of the preconditioner: S_r -= alpha Q (upd), then T = F1^H Lambda^{-1} F1 S_r.  Warp 0,
// line 0; S_r's row lives in shared memory.
template <int M>
__device__ __forceinline__ void kr_row_pass(const KrArgs& a, KrSmem<M>& S, float2* xl,
                                            const float2 (&twr)[KrCfg<M>::N1], size_t boff, int t, float alpha,
                                            bool upd) {
  constexpr int N1 = KrCfg<M>::N1, N2 = KrCfg<M>::N2, N = M;
  const int tid = threadIdx.x, j = tid % N2, line = tid / N2;
  if (tid >= 32) return;
  float2 v[N1];
  if (upd) {
    const float2* qq = a.Qs + boff + (size_t)t * N;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) v[n1] = __ldcg(qq + N2 * n1 + j);
  }
#pragma unroll
  for (int n1 = 0; n1 < N1; ++n1) {
    const float2 sr = S.srow[N2 * n1 + j];
    if (upd) {
      v[n1] = make_float2(sr.x - alpha * v[n1].x, sr.y - alpha * v[n1].y);
      if (line == 0) S.srow[N2 * n1 + j] = v[n1];
    } else {
      v[n1] = sr;
    }
  }
  kr_fwd<M>(v, xl, twr, j);
#pragma unroll
  for (int s = 0; s < N1; ++s) v[s] = cscale(v[s], S.li[specidx<M>(j, s)]);
  kr_inv<M>(v, xl, twr, j);
  if (line == 0) {  // T is column-major: the column owners' reads are contiguous
    float2* tt = a.Tb + boff + t;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) tt[(size_t)(N2 * n1 + j) * M] = v[n1];
  }
}

// ---- per-CTA helpers (force-inlined free functions: captured arrays in lambdas that the
// compiler does not inline end up in local memory)

// data term for the own column vin (shared memory): S.qs = sum_c conj(s_c) F0^H R F0 (s_c vin)
template <int M, bool SMC>
__device__ __forceinline__ void kr_dataterm(KrSmem<M>& S, const float2* vin, const float2* coils, const float2* sTb,
                                            int C, float2* xl, const float2 (&twr)[KrCfg<M>::N1], uint32_t mbits,
                                            float minv) {
  // shared-memory bandwidth bounds this phase (12 coil lines x ~100 8-byte accesses per lane):
  // the mask is a bit per spectral slot in a register (mbits; r/M = minv where set), and the coil
  // sum first adds the lines of a warp with shuffles
  using Cf = KrCfg<M>;
  constexpr int N1 = Cf::N1, N2 = Cf::N2, NT = Cf::NT, LPAR = Cf::LPAR, N = M;
  constexpr int LW = 32 / N2, NW = NT / 32;  // lines per warp, warps
  const int tid = threadIdx.x, line = tid / N2, j = tid % N2;
  float2 acc[N1];
#pragma unroll
  for (int n1 = 0; n1 < N1; ++n1) acc[n1] = make_float2(0.f, 0.f);
  for (int c0 = 0; c0 < C; c0 += LPAR) {
    const int c = c0 + line;
    const bool act = c < C;
    const float2* sc = SMC ? coils + (act ? c : 0) * M + j : sTb + (size_t)(act ? c : 0) * N * M + j;
    float2 v[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) v[n1] = SMC ? sc[N2 * n1] : __ldg(sc + N2 * n1);
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) v[n1] = cmul(v[n1], vin[N2 * n1 + j]);
    kr_fwd<M>(v, xl, twr, j);
    const uint32_t mb = act ? mbits : 0u;
#pragma unroll
    for (int q = 0; q < N1; ++q) v[q] = cscale(v[q], ((mb >> q) & 1u) ? minv : 0.f);
    kr_inv<M>(v, xl, twr, j);
    // acc += conj(s_c) v: the coil line is re-read instead of held in registers
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) acc[n1] = cfmac(SMC ? sc[N2 * n1] : __ldg(sc + N2 * n1), v[n1], acc[n1]);
  }
  // lines of one warp: fixed shuffle tree (line l + line l + LW/2, ...) -> lanes of line 0
#pragma unroll
  for (int off = N2 * LW / 2; off >= N2; off >>= 1)
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      acc[n1].x += __shfl_xor_sync(0xffffffffu, acc[n1].x, off);
      acc[n1].y += __shfl_xor_sync(0xffffffffu, acc[n1].y, off);
    }
  __syncthreads();  // exchange areas -> coil-sum buffer
  float2* cs = S.u.xch;
  const int wid = tid >> 5;
  if ((tid & 31) < N2) {
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) cs[wid * M + N2 * n1 + j] = acc[n1];
  }
  __syncthreads();
  const int nw = (C < LPAR ? (C + LW - 1) / LW : NW);
  for (int i = tid; i < M; i += NT) {  // fixed order over the warps
    float2 sum = cs[i];
    for (int w = 1; w < nw; ++w) sum = cadd(sum, cs[w * M + i]);
    S.qs[i] = sum;
  }
  __syncthreads();
}

// column transform (warp 0, line 0): natural own-column vector in shared memory -> column
// spectrum dst[k][t] (strided store)
template <int M>
__device__ __forceinline__ void kr_col_fwd(const float2* src, float2* dst, float2* xl,
                                           const float2 (&twr)[KrCfg<M>::N1], size_t boff, int t) {
  constexpr int N1 = KrCfg<M>::N1, N2 = KrCfg<M>::N2, N = M;
  const int tid = threadIdx.x, line = tid / N2, j = tid % N2;
  if (tid < 32) {
    float2 v[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) v[n1] = src[N2 * n1 + j];
    kr_fwd<M>(v, xl, twr, j);
    if (line == 0) {
#pragma unroll
      for (int s = 0; s < N1; ++s) dst[boff + (size_t)specidx<M>(j, s) * N + t] = v[s];
    }
  }
}

// z of columns t-1, t, t+1 = F0^H T (lines 0, 1, 2); returns the partial Re<r, z> (own column)
template <int M>
__device__ __forceinline__ double kr_col_inv_z(KrSmem<M>& S, const float2* Tb, float2* xl,
                                               const float2 (&twr)[KrCfg<M>::N1], size_t boff, int t) {
  constexpr int N1 = KrCfg<M>::N1, N2 = KrCfg<M>::N2, N = M;
  const int tid = threadIdx.x, line = tid / N2, j = tid % N2;
  double rz = 0.0;
  constexpr int LW = 32 / N2;                 // lines per warp
  constexpr int LZ = (3 + LW - 1) / LW * LW;  // whole warps that hold the 3 lines
  if (line < LZ) {
    const bool real = line < 3;
    const int col = (t + (real ? line : 1) - 1 + N) % N;
    float2 v[N1];
#pragma unroll
    for (int s = 0; s < N1; ++s)
      v[s] = real ? __ldcg(Tb + boff + (size_t)col * M + specidx<M>(j, s)) : make_float2(0.f, 0.f);
    kr_inv<M>(v, xl, twr, j);
    if (real) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) S.zc[line][N2 * n1 + j] = v[n1];
    }
    if (line == 1) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) {
        const float2 r = S.rs[N2 * n1 + j];
        rz += (double)r.x * v[n1].x + (double)r.y * v[n1].y;
      }
    }
  }
  return rz;
}

// Alg. 1 step 1 inside the launch (recon, KrArgs::kinit): u1 = sum_c S_c^H F^H y_c and the
// root-sum-of-squares start x1 = sqrt(sum_c |F^H y_c|^2) (reading A12), with F the
// unitary 2D DFT and y zero-filled k-space masked by R (rows of a line mask).  Phase 1 (row t):
// the length-N inverse DFT of row t of every coil's k-space into Y1T (column-major, one line
// per coil, LPAR coils at a time).  Phase 2 (column t, after a barrier): the length-M inverse
// DFT of column t of every Y1T, the coil sums in a fixed order.  Results in shared memory
// (u1 -> S.u1b and S.ub, x1 -> S.xs) and x1 -> xT.
template <int M, bool SMC>
__device__ __forceinline__ void kr_init_rows(const KrArgs& a, KrSmem<M>& S, float2* xl,
                                             const float2 (&twr)[KrCfg<M>::N1], int b, int t) {
  using Cf = KrCfg<M>;
  constexpr int N1 = Cf::N1, N2 = Cf::N2, LPAR = Cf::LPAR, N = M;
  const int tid = threadIdx.x, line = tid / N2, j = tid % N2, C = a.C;
  const bool smp = S.rm[t] != 0.f;  // row t of the line mask
  for (int c0 = 0; c0 < C; c0 += LPAR) {
    const int c = c0 + line;
    const bool act = c < C;
    float2 v[N1];
    const float2* yr = a.y + (((size_t)b * C + (act ? c : 0)) * M + t) * N;
#pragma unroll
    for (int s = 0; s < N1; ++s) v[s] = (act && smp) ? __ldcg(yr + specidx<M>(j, s)) : make_float2(0.f, 0.f);
    kr_inv<M>(v, xl, twr, j);
    if (act) {
      float2* o = a.y1T + ((size_t)b * C + c) * N * M + t;
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) o[(size_t)(N2 * n1 + j) * M] = v[n1];
    }
  }
}
template <int M, bool SMC>
__device__ __forceinline__ void kr_init_cols(const KrArgs& a, KrSmem<M>& S, const float2* coils, const float2* sTb,
                                             float2* xl, const float2 (&twr)[KrCfg<M>::N1], size_t boff, int b,
                                             int t) {
  using Cf = KrCfg<M>;
  constexpr int N1 = Cf::N1, N2 = Cf::N2, NT = Cf::NT, LPAR = Cf::LPAR, N = M;
  constexpr int LW = 32 / N2, NW = NT / 32;
  const int tid = threadIdx.x, line = tid / N2, j = tid % N2, C = a.C;
  const float scale = rsqrtf((float)(M * N));
  float2 acc[N1];
  float rss[N1];
#pragma unroll
  for (int n1 = 0; n1 < N1; ++n1) {
    acc[n1] = make_float2(0.f, 0.f);
    rss[n1] = 0.f;
  }
  for (int c0 = 0; c0 < C; c0 += LPAR) {
    const int c = c0 + line;
    const bool act = c < C;
    float2 v[N1];
    const float2* col = a.y1T + ((size_t)b * C + (act ? c : 0)) * N * M + (size_t)t * M;
#pragma unroll
    for (int s = 0; s < N1; ++s) v[s] = act ? __ldcg(col + specidx<M>(j, s)) : make_float2(0.f, 0.f);
    kr_inv<M>(v, xl, twr, j);
    const float2* sc = SMC ? coils + (act ? c : 0) * M + j : sTb + (size_t)(act ? c : 0) * N * M + j;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const float2 vv = cscale(v[n1], act ? scale : 0.f);
      acc[n1] = cfmac(SMC ? sc[N2 * n1] : __ldg(sc + N2 * n1), vv, acc[n1]);  // acc += conj(s_c) v
      rss[n1] += vv.x * vv.x + vv.y * vv.y;
    }
  }
  // lines of one warp (fixed shuffle tree), then the warps in order (as kr_dataterm)
#pragma unroll
  for (int off = N2 * LW / 2; off >= N2; off >>= 1)
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      acc[n1].x += __shfl_xor_sync(0xffffffffu, acc[n1].x, off);
      acc[n1].y += __shfl_xor_sync(0xffffffffu, acc[n1].y, off);
      rss[n1] += __shfl_xor_sync(0xffffffffu, rss[n1], off);
    }
  __syncthreads();
  float2* cs = S.u.xch;  // [NW][M] coil-sum partials, then [NW][M] rss partials (real parts)
  const int wid = tid >> 5;
  if ((tid & 31) < N2) {
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      cs[wid * M + N2 * n1 + j] = acc[n1];
      cs[(NW + wid) * M + N2 * n1 + j] = make_float2(rss[n1], 0.f);
    }
  }
  __syncthreads();
  const int nw = (C < LPAR ? (C + LW - 1) / LW : NW);
  for (int i = tid; i < M; i += NT) {
    float2 u = cs[i];
    float r = cs[NW * M + i].x;
    for (int w = 1; w < nw; ++w) {
      u = cadd(u, cs[w * M + i]);
      r += cs[(NW + w) * M + i].x;
    }
    S.u1b[i] = u;
    S.ub[i] = u;
    const float2 x1 = make_float2(sqrtf(r), 0.f);
    S.xs[i] = x1;
    a.xT[boff + (size_t)t * M + i] = x1;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ the kernel
template <int M, bool SMC>
__global__ void __launch_bounds__(KrCfg<M>::NT, 2) k_persist(const __grid_constant__ KrArgs a) {
  using Cf = KrCfg<M>;
  constexpr int N1 = Cf::N1, N2 = Cf::N2, NT = Cf::NT, LPAR = Cf::LPAR, XL = Cf::XL;
  constexpr int N = M, P = M;  // square images; one CTA per column
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KrSmem<M>& S = *reinterpret_cast<KrSmem<M>*>(smem_raw);
  float2* coils = reinterpret_cast<float2*>(smem_raw + (sizeof(KrSmem<M>) + 15) / 16 * 16);  // SMC: [C][M]

  const int b = blockIdx.x / P;
  const int t = blockIdx.x % P;  // owned column and spectral row
  const int tid = threadIdx.x;
  const int line = tid / N2, j = tid % N2;
  const int C = a.C;
  const size_t img = (size_t)M * N, boff = (size_t)b * img;
  unsigned* barc = a.bar + b;
  unsigned target = 0;
  const bool lead = (t == 0);                 // writes the problem's Scal / hist / log
  const bool timer = lead && b == 0 && tid == 0 && a.stamp != nullptr;
  if (timer) {
    S.tclk = S.tclk0 = clock64();
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    S.tgt0 = g;
    S.tstage[0] = S.tstage[1] = S.tstage[2] = S.tstage[3] = 0;
  }
  long long pclk = 0;
  auto seg = [&](int k) {  // loop segment profile (SBPCG_KR_PROF=1)
    if (timer && a.prof) {
      const long long c = clock64();
      if (k >= 0) atomicAdd(a.stamp + 8 + k, (unsigned long long)(c - pclk));
      pclk = c;
    }
  };
  auto stamp = [&](int k) {
    if (timer) {
      const long long c = clock64();
      S.tstage[k] += (unsigned long long)(c - S.tclk);
      S.tclk = c;
    }
  };

  const float2* sTb = a.sT + (size_t)b * C * N * M + (size_t)t * M;  // + c * N * M: coil c, column t
  for (int i = tid; i < M; i += NT) {
    S.tw[i] = a.tw[i];
    S.li[i] = a.lam_inv[boff + (size_t)t * N + i];
    S.rm[i] = a.rmask[(size_t)b * a.rmask_bstride + i];
  }
  if constexpr (SMC) {  // this column of every coil map, once for the whole launch
    for (int e = tid; e < C * M; e += NT) coils[e] = __ldg(sTb + (size_t)(e / M) * N * M + e % M);
  }
  __syncthreads();
  float2 twr[N1];
  load_twr<M>(twr, S.tw, j);
  // the row mask at this lane's spectral slots as bits (r/M is either 0 or 1/M)
  // (the host stores r/M = 1.0f / M for sampled rows, sbpcg.cu)
  uint32_t mbits = 0;
#pragma unroll
  for (int q = 0; q < N1; ++q)
    if (S.rm[specidx<M>(j, q)] != 0.f) mbits |= 1u << q;
  const float minv = 1.0f / (float)M;

  double* part = a.part + (size_t)b * 8 * P;  // 6 slots used (Chronopoulos-Gear phase C)
  float2* xl = S.u.xch + line * XL;

  // A-product epilogue for row i: reg = lambda L v + gamma v from S.pc
  auto lap_reg3 = [&](const float2 (*v3)[M], int i, float2& vc) -> float2 {
    const float2 p = v3[1][i];
    const float2 pu = v3[1][(i + M - 1) % M];
    const float2 pd = v3[1][(i + 1) % M];
    const float2 pl = v3[0][i];
    const float2 pr = v3[2][i];
    const float2 lp = make_float2(4.f * p.x - pu.x - pd.x - pl.x - pr.x, 4.f * p.y - pu.y - pd.y - pl.y - pr.y);
    vc = p;
    return make_float2(a.lam * lp.x + a.gam * p.x, a.lam * lp.y + a.gam * p.y);
  };
  auto lap_reg = [&](int i, float2& vc) -> float2 { return lap_reg3(S.pc, i, vc); };
  auto hist_put = [&](int k, double rel) {
    if (lead && tid == 0 && a.L.hist != nullptr && k < a.L.hist_stride) a.L.hist[(size_t)b * a.L.hist_stride + k] = (float)rel;
  };

  const int n_solves = a.n_outer > 0 ? a.n_outer : 1;
  if (a.n_outer > 0 && a.kinit) {  // Alg. 1 step 1 (u1, x1 = RSS) in this launch
    kr_init_rows<M, SMC>(a, S, xl, twr, b, t);
    pbar(barc, target, P);
    kr_init_cols<M, SMC>(a, S, coils, sTb, xl, twr, boff, b, t);
    pbar(barc, target, P);  // x1 of every column (xT) visible to the first prelude
    stamp(3);
  }
  for (int js = 0; js < n_solves; ++js) {
    const bool recon = a.n_outer > 0;
    const bool update_u = recon && js > 0;
    KrScal sc;
    sc.rho = sc.alpha = sc.beta = sc.sigma = 0.0;
    sc.iter = 0;
    sc.status = ST_OK;
    sc.converged = 0;
    sc.zero_x = 0;
    sc.active = 1;

    // ================= prelude: r0 = b - A x0 (+ RHS and data feedback) ; S_r = F0 r0
    seg(-1);
    constexpr int TT = Cf::TT;
    const int ntj = N / TT, ntile = (M / TT) * ntj;
    const bool sbpre = recon && ntile <= P;  // one SB tile per CTA: stage its b_* now
    const int par = js & 1;
    if (sbpre && t < ntile && js == 0 && a.kinit) {  // fresh SB state (Alg. 1 step 1): b_* = 0
      for (int e = tid; e < sb_pre_size<TT>(); e += NT) S.sbpre[e] = make_float2(0.f, 0.f);
    } else if (sbpre && t < ntile) {
      SbArgs sa = a.sb;
      sa.bx_in = a.bxs[par];
      sa.by_in = a.bys[par];
      sb_tile_prefetch<TT, NT>(sa, S.sbpre, t / ntj, t % ntj, b);
    }
    const bool xt = recon && (js > 0 || a.kinit);
    if (xt) {
      // x of columns t-1, t, t+1 (column-major xT) and rhs_reg (column-major, written by the SB
      // step) are copied into shared memory asynchronously; the data term runs meanwhile on the
      // own column, already in shared memory (S.xs), and u, u1 stay in shared memory across the
      // solves (loaded from the image once when the launch did not compute them itself)
      for (int e = tid; e < 3 * (M / 2); e += NT) {
        const int c = e / (M / 2), i2 = 2 * (e % (M / 2));
        kr_cp16(&S.pc[c][i2], a.xT + boff + (size_t)((t + c - 1 + N) % N) * M + i2);
      }
      if (update_u)
        for (int e = tid; e < M / 2; e += NT) kr_cp16(S.rhb + 2 * e, a.rhs + boff + (size_t)t * M + 2 * e);
      kr_cp_commit();
      if (!a.kinit && js == 1)
        for (int i = tid; i < M; i += NT) S.u1b[i] = __ldcg(a.u1 + boff + (size_t)i * N + t);
      seg(10);
      kr_dataterm<M, SMC>(S, S.xs, coils, sTb, C, xl, twr, mbits, minv);
      kr_cp_wait();
      __syncthreads();
    } else {  // the first solve without kinit, or a single solve: one synchronous load batch of
      // x of columns t-1, t, t+1 (image layout) and u (recon) or b (solve) of column t
      constexpr int E = (3 * M + NT - 1) / NT, EO = (M + NT - 1) / NT;
      float2 xv[E], uv[EO], u1v[EO], rv[EO];
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int e = tid + k * NT;
        const int col = (t + e / M - 1 + N) % N;
        if (e < 3 * M)
          xv[k] = __ldcg(xt ? a.xT + boff + (size_t)col * M + e % M : a.x + boff + (size_t)(e % M) * N + col);
      }
#pragma unroll
      for (int k = 0; k < EO; ++k) {
        const int i = tid + k * NT;
        if (i < M) {
          const size_t gi = boff + (size_t)i * N + t;
          if (recon) {
            if (js == 0 && !a.kinit) uv[k] = __ldcg(a.u + gi);
            if (update_u) {
              if (js == 1 && !a.kinit) u1v[k] = __ldcg(a.u1 + gi);
              rv[k] = __ldcg(a.rhs + boff + (size_t)t * M + i);
            }
          } else {
            rv[k] = __ldcg(a.bvec + gi);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const int e = tid + k * NT;
        if (e < 3 * M) {
          S.pc[e / M][e % M] = xv[k];
          if (e / M == 1) {
            S.xs[e % M] = xv[k];
            if (!xt) a.xT[boff + (size_t)t * M + e % M] = xv[k];  // x0 -> xT (the SB step reads it)
          }
        }
      }
#pragma unroll
      for (int k = 0; k < EO; ++k) {
        const int i = tid + k * NT;
        if (i < M) {
          if (recon) {
            if (js == 0 && !a.kinit) S.ub[i] = uv[k];
            if (update_u) {
              if (js == 1 && !a.kinit) S.u1b[i] = u1v[k];
              S.rhb[i] = rv[k];
            }
          } else {
            S.rhb[i] = rv[k];
          }
        }
      }
      __syncthreads();
      seg(10);
      kr_dataterm<M, SMC>(S, S.pc[1], coils, sTb, C, xl, twr, mbits, minv);
    }
    seg(11);
    double d0 = 0.0, d1 = 0.0;
    for (int i = tid; i < M; i += NT) {
      const size_t gi = boff + (size_t)i * N + t;
      const float2 av = S.qs[i];
      float2 xc;
      const float2 reg = lap_reg(i, xc);
      float2 bb;
      if (recon) {
        float2 uu = S.ub[i];
        if (update_u) {  // u_{j+1} = u_j + u_1 - E^H E x (reading A28); kept in shared memory
          const float2 u1 = S.u1b[i];
          uu = make_float2(uu.x + u1.x - av.x, uu.y + u1.y - av.y);
          S.ub[i] = uu;
        }
        const float2 rr = update_u ? S.rhb[i] : make_float2(0.f, 0.f);
        bb = make_float2(a.mu * uu.x + rr.x, a.mu * uu.y + rr.y);
      } else {
        bb = S.rhb[i];
      }
      const float2 r = make_float2(bb.x - (a.mu * av.x + reg.x), bb.y - (a.mu * av.y + reg.y));
      S.rs[i] = r;
      d0 += (double)bb.x * bb.x + (double)bb.y * bb.y;
      d1 += (double)r.x * r.x + (double)r.y * r.y;
    }
    __syncthreads();
    kr_col_fwd<M>(S.rs, a.Sr, xl, twr, boff, t);
    block_sum2(d0, d1, S.red);
    if (tid == 0) {
      part[t] = d0;
      part[P + t] = d1;
    }
    seg(12);
    pbar(barc, target, P);
    seg(13);
    // row t of S_r for the solve's first row pass: its L2 round trip overlaps the all-reduce
    for (int e = tid; e < N / 2; e += NT) kr_cp16(S.srow + 2 * e, a.Sr + boff + (size_t)t * N + 2 * e);
    kr_cp_commit();
    psum<P, 2>(part, S.bc);
    {
      const double nb2 = S.bc[0], rr = S.bc[1];
      sc.nb2 = nb2;
      sc.rr = rr;
      if (!(nb2 > 0.0)) {
        if (nb2 == 0.0) {
          sc.zero_x = 1;
          sc.converged = 1;
          hist_put(0, 0.0);
        } else {
          sc.status = ST_NONFINITE;
        }
        sc.active = 0;
      } else {
        const double rel = sqrt(rr / nb2);
        hist_put(0, rel);
        if (!isfinite(rr)) {
          sc.status = ST_NONFINITE;
          sc.active = 0;
        } else if (a.eps > 0.f && rel <= (double)a.eps) {
          sc.converged = 1;
          sc.active = 0;
        }
      }
    }
    seg(14);
    stamp(0);
    if (!sc.active) kr_cp_wait();  // no row pass follows: retire the S_r row copy

    if (sc.active && a.cg) {
      // ================= Chronopoulos-Gear PCG: the same
      // iterates as the standard recurrences of PAPER.md:238 in exact arithmetic, with
      // s = A p carried by its own recurrence s_k = w_{k-1} + beta_k s_{k-1} (w = A z), so that
      // rho = Re<r, z>, delta = Re<w, z> and ||r||^2 of an iteration are reduced together and an
      // iteration needs two barriers:  [z = M^{-1} r (column IFFTs), w = A z, W = F0 w,
      // partials] | barrier | [p, s, x, r updates; S_s = W + beta S_s, S_r -= alpha S_s; row
      // FFTs of M^{-1}] | barrier.
      kr_cp_wait();  // row t of S_r (issued after the prelude barrier)
      __syncthreads();
      kr_row_pass<M>(a, S, xl, twr, boff, t, 0.f, false);
      pbar(barc, target, P);
      double rho_prev = 0.0;
      for (int kc = 0;; ++kc) {  // kc: index of the z_kc, w_kc formed in this pass
        seg(-1);
        // skew probe (SBPCG_KR_PROF=2): globaltimer at phase-C start / end / barrier exit of
        // every CTA of problem 0, pass 4 of the first solve -> stamp[32 + 4 t + {0, 1, 2}]
        const bool probe = a.prof == 2 && js == 0 && kc == 4 && tid == 0 && b == 0;
        auto gtime = []() {
          unsigned long long g;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
          return g;
        };
        if (probe) a.stamp[32 + 4 * t] = gtime();
        // ---- z_kc = F0^H T (columns t-1, t, t+1), w = A z, W = F0 w ; rho, delta, ||r||^2
        double rz = kr_col_inv_z<M>(S, a.Tb, xl, twr, boff, t);  // warps 0-1
        // ||r_kc||^2 (slot 6, published before the last barrier B), summed by the last warp
        // while the first ones transform T: the stop test on ||r_kc|| / ||b|| runs before the
        // data term, so the pass that would only confirm convergence is not computed
        if (kc > 0 && tid >= NT - 32) psum1_warp<P>(part + 6 * P, &S.bc[7]);
        __syncthreads();
        if (kc > 0) {  // checks of iteration kc on ||r_kc|| (fin_rr order)
          const double rr = S.bc[7];
          sc.rr = rr;
          sc.iter = kc;
          const double rel = sqrt(rr / sc.nb2);
          hist_put(kc, rel);
          if (!isfinite(rr)) {
            sc.status = ST_NONFINITE;
            break;
          }
          if (a.eps > 0.f && rel <= (double)a.eps) {
            sc.converged = 1;
            break;
          }
        }
        seg(0);
        kr_dataterm<M, SMC>(S, S.zc[1], coils, sTb, C, xl, twr, mbits, minv);
        seg(1);
        double dd = 0.0, drr = 0.0, de = 0.0, dq = 0.0, dp = 0.0;
        for (int i = tid; i < M; i += NT) {
          const float2 av = S.qs[i];
          float2 z;
          const float2 reg = lap_reg3(S.zc, i, z);
          const float2 w = make_float2(a.mu * av.x + reg.x, a.mu * av.y + reg.y);
          S.qs[i] = w;
          dd += (double)w.x * z.x + (double)w.y * z.y;
          const float2 r = S.rs[i];
          drr += (double)r.x * r.x + (double)r.y * r.y;
          if (kc > 0) {  // Re<z, s_kc>, Re<p_kc, w>, Re<p_kc, s_kc>: sigma of the next iteration
            const float2 so = S.ss[i], po = S.pc[1][i];
            de += (double)z.x * so.x + (double)z.y * so.y;
            dq += (double)po.x * w.x + (double)po.y * w.y;
            dp += (double)po.x * so.x + (double)po.y * so.y;
          }
        }
        {  // warp 0: W = F0 w ; warp 1: the block sums -> partials (concurrently)
          double v5[6] = {rz, dd, drr, de, dq, dp};
          red_warps<6>(v5, S.red);
          if (tid < 32) {
            kr_col_fwd<M>(S.qs, a.Qs, xl, twr, boff, t);
          } else if (tid < 64) {
            red_final<6>(S.red, v5);
            if (tid == 32) {
#pragma unroll
              for (int q = 0; q < 6; ++q) part[q * P + t] = v5[q];
            }
          }
        }
        seg(2);
        if (probe) a.stamp[32 + 4 * t + 1] = gtime();
        pbar(barc, target, P);
        if (probe) a.stamp[32 + 4 * t + 2] = gtime();
        seg(3);
        // row t of W: its L2 round trip overlaps the all-reduce read (cp.async, no registers)
        for (int e = tid; e < N / 2; e += NT) kr_cp16(S.wrow + 2 * e, a.Qs + boff + (size_t)t * N + 2 * e);
        kr_cp_commit();
        psum<P, 6>(part, S.bc);
        const double rho = S.bc[0], delta = S.bc[1], zs_ = S.bc[3], pw_ = S.bc[4], ps_ = S.bc[5];
        if (kc >= 1) {  // checks of iteration kc (fin_rho order; the ||r_kc|| ones ran above)
          if (!isfinite(rho)) {
            sc.status = ST_NONFINITE;
            break;
          }
          if (rho == 0.0) {
            sc.converged = 1;
            break;
          }
          if (kc >= a.maxit) {
            sc.converged = (a.eps == 0.f) ? 1 : 0;
            break;
          }
        } else if (!isfinite(rho)) {
          sc.status = ST_NONFINITE;
          break;
        }
        // ---- iteration k = kc + 1: beta_k, sigma_k = <p_k, A p_k>, alpha_k.  sigma is the
        // bilinear expansion of <z + beta p, w + beta s> (s = A p from its recurrence):
        // delta + beta (Re<z, s> + Re<p, w>) + beta^2 <p, s>, not the classical C-G identity
        // delta - beta rho / alpha, which assumes exact orthogonality and goes non-positive
        // once a fixed-count solve reaches the fp32 rounding floor.
        const double beta = kc == 0 ? 0.0 : rho / rho_prev;
        const double sigma = kc == 0 ? delta : delta + beta * (zs_ + pw_) + beta * beta * ps_;
        sc.sigma = sigma;
        if (!isfinite(sigma)) {
          sc.status = ST_NONFINITE;
          break;
        }
        if (!(sigma > 0.0)) {
          sc.status = ST_INDEFINITE;
          break;
        }
        sc.beta = beta;
        sc.rho = rho;
        sc.alpha = rho / sigma;
        rho_prev = rho;
        seg(4);
        const float fb = (float)beta, fa = (float)sc.alpha;
        const bool first = kc == 0;
        // column t: p = z + beta p ; s = w + beta s ; x += alpha p ; r -= alpha s ; ||r||^2
        double drn = 0.0;
        for (int i = tid; i < M; i += NT) {
          const float2 z = S.zc[1][i], w = S.qs[i];
          float2 pp = z, sv = w;
          if (!first) {
            const float2 po = S.pc[1][i], so = S.ss[i];
            pp = make_float2(z.x + fb * po.x, z.y + fb * po.y);
            sv = make_float2(w.x + fb * so.x, w.y + fb * so.y);
          }
          S.pc[1][i] = pp;
          S.ss[i] = sv;
          const float2 x = S.xs[i], r0 = S.rs[i];
          const float2 xn = make_float2(x.x + fa * pp.x, x.y + fa * pp.y);
          S.xs[i] = xn;
          // x_{k+1} to the image now (ordered by this pass's barrier B): a loop that stops at the
          // start of the next pass, or after its barrier A, needs no solve-exit store + barrier
          a.xT[boff + (size_t)t * M + i] = xn;
          const float2 rn = make_float2(r0.x - fa * sv.x, r0.y - fa * sv.y);
          S.rs[i] = rn;
          drn += (double)rn.x * rn.x + (double)rn.y * rn.y;
        }
        drn = warp_sum(drn);
        if ((tid & 31) == 0) S.red[40 + (tid >> 5)] = drn;  // (phase C's slot-5 sums are consumed)
        // row t: S_s = W + beta S_s ; S_r -= alpha S_s ; T = F1^H Lambda^{-1} F1 S_r
        kr_cp_wait();
        __syncthreads();  // every thread's part of the W row has landed
        if (tid < 32) {
          constexpr int N1_ = N1;
          float2 v[N1_];
#pragma unroll
          for (int n1 = 0; n1 < N1_; ++n1) v[n1] = S.wrow[N2 * n1 + j];
#pragma unroll
          for (int n1 = 0; n1 < N1_; ++n1) {
            const int i = N2 * n1 + j;
            float2 sv = v[n1];
            if (!first) {
              const float2 so = S.ssrow[i];
              sv = make_float2(sv.x + fb * so.x, sv.y + fb * so.y);
            }
            const float2 sr = S.srow[i];
            v[n1] = make_float2(sr.x - fa * sv.x, sr.y - fa * sv.y);
            if (line == 0) {
              S.ssrow[i] = sv;
              S.srow[i] = v[n1];
            }
          }
          kr_fwd<M>(v, xl, twr, j);
#pragma unroll
          for (int q = 0; q < N1_; ++q) v[q] = cscale(v[q], S.li[specidx<M>(j, q)]);
          kr_inv<M>(v, xl, twr, j);
          if (line == 0) {  // column-major T
            float2* tt = a.Tb + boff + t;
#pragma unroll
            for (int n1 = 0; n1 < N1_; ++n1) tt[(size_t)(N2 * n1 + j) * M] = v[n1];
          }
        } else if (tid == 32) {  // ||r_{k+1}||^2 partial of this column (slot 6), fixed warp order
          double sr = 0.0;
#pragma unroll
          for (int w = 0; w < NT / 32; ++w) sr += S.red[40 + w];
          part[6 * P + t] = sr;
        }
        seg(5);
        pbar(barc, target, P);
        seg(6);
      }
      sc.active = 0;
    } else if (sc.active) {
      // ================= z0 = M^{-1} r0 ; rho0 = Re<r0, z0>
      kr_cp_wait();  // row t of S_r (issued after the prelude barrier)
      __syncthreads();
      kr_row_pass<M>(a, S, xl, twr, boff, t, 0.f, false);
      pbar(barc, target, P);
      {
        double rz = kr_col_inv_z<M>(S, a.Tb, xl, twr, boff, t), dummy = 0.0;
        block_sum2(rz, dummy, S.red);
        if (tid == 0) part[2 * P + t] = rz;
      }
      pbar(barc, target, P);
      psum<P, 1>(part + 2 * P, S.bc);
      {
        const double rz = S.bc[0];
        if (!isfinite(rz)) {
          sc.status = ST_NONFINITE;
          sc.active = 0;
        } else {
          sc.rho = rz;
        }
      }
    }

    // ================= PCG iterations
    while (sc.active) {
      seg(-1);
      const int k = sc.iter + 1;
      const bool first = (k == 1);
      // ---- P1: p_k = z + beta p_{k-1} (columns t-1, t, t+1), q = A p_k, Q = F0 q, sigma partial
      const float beta = (float)sc.beta;
      for (int e = tid; e < 3 * M; e += NT) {
        const int cc = e / M, i = e % M;
        const float2 zz = S.zc[cc][i];
        float2 p = zz;
        if (!first) {
          const float2 po = S.pc[cc][i];
          p = make_float2(zz.x + beta * po.x, zz.y + beta * po.y);
        }
        S.pc[cc][i] = p;
      }
      __syncthreads();
      seg(0);
      kr_dataterm<M, SMC>(S, S.pc[1], coils, sTb, C, xl, twr, mbits, minv);
      seg(1);
      double ds = 0.0, dz = 0.0;
      for (int i = tid; i < M; i += NT) {
        const float2 av = S.qs[i];
        float2 p;
        const float2 reg = lap_reg(i, p);
        const float2 q = make_float2(a.mu * av.x + reg.x, a.mu * av.y + reg.y);
        S.qs[i] = q;
        ds += (double)p.x * q.x + (double)p.y * q.y;
      }
      {  // warp 0: Q = F0 q ; warp 1: sigma partial (concurrently)
        double v1[1] = {ds};
        red_warps<1>(v1, S.red);
        if (tid < 32) {
          kr_col_fwd<M>(S.qs, a.Qs, xl, twr, boff, t);
        } else if (tid < 64) {
          red_final<1>(S.red, v1);
          if (tid == 32) part[t] = v1[0];
        }
      }
      (void)dz;
      seg(2);
      pbar(barc, target, P);
      seg(3);
      // ---- alpha ; P2: S_r -= alpha Q ; T = F1^H Lambda^{-1} F1 S_r (row t)
      psum<P, 1>(part, S.bc);
      {
        const double sigma = S.bc[0];
        sc.sigma = sigma;
        if (!isfinite(sigma)) {
          sc.status = ST_NONFINITE;
          sc.active = 0;
        } else if (!(sigma > 0.0)) {
          sc.status = ST_INDEFINITE;
          sc.active = 0;
        } else {
          sc.alpha = sc.rho / sigma;
        }
      }
      if (!sc.active) break;
      seg(4);
      const float alpha = (float)sc.alpha;
      kr_row_pass<M>(a, S, xl, twr, boff, t, alpha, true);
      seg(5);
      pbar(barc, target, P);
      seg(6);
      // ---- P3: x += alpha p ; r -= alpha q ; z = F0^H T ; ||r||^2 , Re<r, z>
      double drr = 0.0;
      for (int i = tid; i < M; i += NT) {
        const float2 p = S.pc[1][i], q = S.qs[i], x = S.xs[i], r0 = S.rs[i];
        S.xs[i] = make_float2(x.x + alpha * p.x, x.y + alpha * p.y);
        const float2 r = make_float2(r0.x - alpha * q.x, r0.y - alpha * q.y);
        S.rs[i] = r;
        drr += (double)r.x * r.x + (double)r.y * r.y;
      }
      __syncthreads();
      {
        double rz = kr_col_inv_z<M>(S, a.Tb, xl, twr, boff, t);
        block_sum2(drr, rz, S.red);
        if (tid == 0) {
          part[P + t] = drr;
          part[2 * P + t] = rz;
        }
      }
      seg(7);
      pbar(barc, target, P);
      seg(8);
      psum<P, 2>(part + P, S.bc);
      {
        const double rr = S.bc[0], rz = S.bc[1];
        sc.rr = rr;
        sc.iter = k;
        const double rel = sqrt(rr / sc.nb2);
        hist_put(k, rel);
        if (!isfinite(rr)) {
          sc.status = ST_NONFINITE;
          sc.active = 0;
        } else if (a.eps > 0.f && rel <= (double)a.eps) {
          sc.converged = 1;
          sc.active = 0;
        } else if (!isfinite(rz)) {
          sc.status = ST_NONFINITE;
          sc.active = 0;
        } else if (rz == 0.0) {
          sc.converged = 1;
          sc.active = 0;
        } else if (k >= a.maxit) {
          sc.converged = (a.eps == 0.f) ? 1 : 0;
          sc.active = 0;
        } else {
          sc.beta = rz / sc.rho;
          sc.rho = rz;
        }
      }
      seg(9);
    }

    // ================= solve exit: x (own column) to the image, scalars and log.  The
    // Chronopoulos-Gear loop stored every x_k before the barrier B that ends its pass (it stops
    // after a barrier B or A), and a solve that stopped in the prelude left x0 unchanged, so there
    // only x = 0 (||b|| = 0) needs a store and the barrier before the SB step; the decision is
    // uniform over the problem's CTAs.
    // The image-layout x (the caller's output) is written by the last solve only.
    seg(-1);
    const bool xstore = !a.cg || sc.zero_x;
    const bool xout = !recon || js == n_solves - 1;
    if (xstore || xout)
      for (int i = tid; i < M; i += NT) {
        const float2 v = sc.zero_x ? make_float2(0.f, 0.f) : S.xs[i];
        if (sc.zero_x) S.xs[i] = v;  // the next prelude's data term reads the own column here
        if (xstore) a.xT[boff + (size_t)t * M + i] = v;
        if (xout) a.x[boff + (size_t)i * N + t] = v;
      }
    if (lead && tid == 0) {
      Scal& g = a.L.scal[b];
      g.rho = sc.rho;
      g.alpha = sc.alpha;
      g.beta = sc.beta;
      g.sigma = sc.sigma;
      g.nb2 = sc.nb2;
      g.rr = sc.rr;
      g.iter = sc.iter;
      g.active = 0;
      g.converged = sc.converged;
      g.status = sc.status;
      g.zero_x = sc.zero_x;
      g.maxit = a.maxit;
      g.eps = a.eps;
      if (a.L.log_iters) a.L.log_iters[(size_t)js * a.B + b] = sc.iter;
      if (a.L.log_relres) a.L.log_relres[(size_t)js * a.B + b] = (float)(sc.nb2 > 0 ? sqrt(sc.rr / sc.nb2) : 0.0);
    }
    stamp(1);
    if (!recon) break;

    // ================= SB step (Alg. 1 steps 6-11 and the regulariser RHS), 16 x 16 tiles
    seg(15);
    if (xstore) pbar(barc, target, P);  // x of every column visible (else ordered by barrier A)
    seg(16);
    {
      SbArgs sa = a.sb;
      sa.x = a.xT;  // column-major x in, column-major rhs_reg out (CM)
      sa.bx_in = a.bxs[par];
      sa.by_in = a.bys[par];
      sa.bx_out = a.bxs[1 - par];
      sa.by_out = a.bys[1 - par];
      for (int tile = t; tile < ntile; tile += P)
        sb_tile<TT, true, NT, true>(sa, S.u.sb, tile / ntj, tile % ntj, b, (timer && a.prof) ? a.stamp + 8 + 19 : nullptr,
                                    sbpre ? S.sbpre : nullptr);
    }
    seg(17);
    pbar(barc, target, P);  // rhs_reg, b_* visible to the next prelude
    seg(18);
    stamp(2);
  }
  if (timer) {
    unsigned long long gt1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
    a.stamp[0] += S.tstage[0];
    a.stamp[1] += S.tstage[1];
    a.stamp[2] += S.tstage[2];
    a.stamp[5] += S.tstage[3];
    a.stamp[3] += (unsigned long long)(clock64() - S.tclk0);
    a.stamp[4] += gt1 - S.tgt0;
  }
}

// ------------------------------------------------------------------ host side
bool kr_supported(int M, int N, int levels) {
  return M == N && (M == 64 || M == 256) && levels >= 0 && (16 % (1 << levels)) == 0;
}

int kr_ctas(int M, int N) { return N; }

// coil maps staged in shared memory when two CTAs per SM still fit
static bool kr_smc(int M, int C) {
  const size_t bytes = M == 64 ? kr_smem_bytes<64>(C, true) : kr_smem_bytes<256>(C, true);
  return bytes <= 110 * 1024;
}

template <int M, bool SMC>
static cudaError_t kr_attr(int C, int* per_sm) {
  auto kern = k_persist<M, SMC>;
  const size_t smem = kr_smem_bytes<M>(C, SMC);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (per_sm) return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kern, KrCfg<M>::NT, smem);
  return cudaSuccess;
}

int kr_max_problems(int M, int N, int C) {
  if (!kr_supported(M, N, 0)) return 0;
  int per_sm = 0, dev = 0, sms = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  const bool smc = kr_smc(M, C);
  cudaError_t e = (M == 64) ? (smc ? kr_attr<64, true>(C, &per_sm) : kr_attr<64, false>(C, &per_sm))
                            : (smc ? kr_attr<256, true>(C, &per_sm) : kr_attr<256, false>(C, &per_sm));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return per_sm * sms / kr_ctas(M, N);
}

template <int M, bool SMC>
static cudaError_t launch_kr_t(const KrArgs& a, cudaStream_t st) {
  cudaError_t e = kr_attr<M, SMC>(a.C, nullptr);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.B * kr_ctas(M, M));
  cfg.blockDim = dim3(KrCfg<M>::NT);
  cfg.dynamicSmemBytes = kr_smem_bytes<M>(a.C, SMC);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barriers)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_persist<M, SMC>, a);
}

cudaError_t launch_kr(const KrArgs& a, cudaStream_t st) {
  if (a.M != a.N) return cudaErrorInvalidValue;
  const bool smc = kr_smc(a.M, a.C);
  switch (a.M) {
    case 64: return smc ? launch_kr_t<64, true>(a, st) : launch_kr_t<64, false>(a, st);
    case 256: return smc ? launch_kr_t<256, true>(a, st) : launch_kr_t<256, false>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

// sT[bc][col][row] = s[bc][row][col] (32 x 32 tiles through shared memory)
__global__ void k_transpose_sens(const float2* __restrict__ s, float2* __restrict__ sT, int M, int N) {
  __shared__ float2 tile[32][33];
  const size_t off = (size_t)blockIdx.z * M * N;
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = r0 + k, c = c0 + threadIdx.x;
    if (r < M && c < N) tile[k][threadIdx.x] = s[off + (size_t)r * N + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k, r = r0 + threadIdx.x;
    if (r < M && c < N) sT[off + (size_t)c * M + r] = tile[threadIdx.x][k];
  }
}

cudaError_t launch_transpose_sens(const float2* s, float2* sT, int BC, int M, int N, cudaStream_t st) {
  k_transpose_sens<<<dim3((N + 31) / 32, (M + 31) / 32, BC), dim3(32, 8), 0, st>>>(s, sT, M, N);
  return cudaGetLastError();
}

}  // namespace sbk
