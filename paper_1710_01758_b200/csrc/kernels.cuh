// kernels.cuh — kernel argument structs and launcher declarations (internal).
#pragma once
#include "internal.cuh"

namespace sbk {

enum K1Mode { K1_APPLY = 0, K1_PCG = 1, K1_RESID = 2 };

// Fused matvec q = A p for one column tile (all d0 rows x W columns)
// of one problem; coil maps streamed by TMA; see k_matvec.cu.
struct K1Args {
  int B, C, M, N;
  float mu, lam, gam;
  const float* rmask;      // [B or 1][M] = r/M (line masks)
  int rmask_bstride;       // M or 0
  // APPLY: vin -> out = A vin.   RESID: vin = x, out = r.   PCG: out = q.
  const float2* vin;
  float2* out;
  // PCG
  const float2* z;
  float2* pbuf0;
  float2* pbuf1;
  float2* x;
  // RESID
  const float2* bvec;      // given b (solve); null in recon mode
  float2* u;               // recon: running u_j = sum_c E_c^H y_c^[j]
  const float2* u1;
  const float2* rhs_reg;   // nullable
  float2* bout;            // recon: b = mu u + rhs_reg
  int update_u;
  float eps;
  int maxit;
  int spec;                // 1: write the column spectrum F_0 q (PCG) / F_0 r0 (RESID) instead (G = 1)
  // bookkeeping
  Loop L;
  Partials P;
  const float2* tw;        // [M] twiddles W_M^m (float)
};

// Generic column/row FFT passes (k_passes.cu): preconditioner, RSS init, encode/adjoint,
// generic-mask matvec.
struct PassArgs {
  int B, C, M, N;
  float mu, lam, gam;
  const float2* tw_m;      // [M]
  const float2* tw_n;      // [N]
  const float* lam_inv;    // [B or 1][M][N] = 1/(N k)
  int lam_bstride;         // M*N or 0
  const uint8_t* mask;     // [B or 1][M][N]
  int mask_bstride;
  const float2* sens;      // [B][C][M][N]
  // vectors
  const float2* a0;
  const float2* a1;
  float2* o0;
  float2* o1;
  float2* tmp;             // [B][M][N] or [B][C][M][N]
  float scale;
  int mode;
  int full;
  Loop L;
  Partials P;
  // PCG p-update in the generic pass A
  const float2* z;
  float2* pbuf0;
  float2* pbuf1;
  float2* x;
  // Jacobi preconditioner: z = r . jinv, jinv = 1/diag(A) [B][N]
  const float* jinv;
};

// fp64 Lambda build (k_lambda.cu)
struct LamArgs {
  int B, C, M, N;
  double mu, lam, gam;
  const float2* sens;
  const uint8_t* mask;
  int mask_bstride;
  int nmask;               // number of distinct masks (B or 1)
  int nsens;               // number of distinct sens stacks (B)
  double2* tmp;            // [B][C][M][N] fp64 scratch
  double2* g;              // [B][M][N]
  double2* rhat;           // [nmask][M][N]
  double* k_out;           // [B][M][N]
  float* lam_inv;          // [B][M][N]
  const double2* tw_m;
  const double2* tw_n;
  int* bad;                // singular-k flag
  // 3D (readout-constant mask): the planes of every coil are fed
  // as extra "coils" of a 2D build in chunks; g accumulates over chunks.
  int accumulate;          // L_ROW_ACC: g += instead of g =
  int csplit;              // L_ROW_ACC: coils split over csplit CTA groups (partials in gpart)
  double* gpart;           // [B][csplit][M][N] partial coil sums (fixed-order reduction)
  int* nextra;             // host counter: +1 per extra (partial-sum) launch, may be null
  int d3;                  // final pass writes k_c (2D, fp64) to kc2 instead of k / Lambda^{-1}
  double* kc2;             // [B][D1*D2]
};

cudaError_t launch_lambda_sep(const LamArgs& a, cudaStream_t st);  // separable (line) masks, K4S
// 3D Lambda: k[x][y][z] = mu kc2[y][z] / D0 + lambda sum_d 4 sin^2(pi nu_d/n_d) + gamma,
// Lambda^{-1} = 1/(N k)
struct Lam3Args {
  int B, D0, D1, D2;
  double mu, lam, gam;
  const double* kc2;
  double* k_out;
  float* lam_inv;
  int* bad;
};

struct SbArgs {
  int B, M, N, levels;
  float lam, gam;
  const float2* x;
  const float2* bx_in;
  const float2* by_in;
  float2* bx_out;
  float2* by_out;
  float2* bw;              // in place (block-local)
  float2* rhs;             // rhs_reg out
  const Scal* scal;        // nullable
  // 3D (k_sb_update3): image [B][M][N][D2]
  int D2;
  const float2* bz_in;
  float2* bz_out;
};


// Persistent whole-GPU reconstruction / solve for small batches of square line-mask problems
// (k_persist.cu): one cooperative launch; CTA t of problem b owns image column
// t (the matvec, the preconditioner's column transforms) and spectral row t (its row
// transforms); the phases are separated by per-problem grid barriers.
struct KrArgs {
  int B, C, M, N, levels;
  float mu, lam, gam;
  const float2* sT;          // [B][C][N][M] coil maps, column-major per coil (transposed copy)
  const float* rmask;        // [B or 1][M] = r/M
  int rmask_bstride;
  const float* lam_inv;      // [B][M][N] = 1/(N k)
  const float2* tw;          // [M] forward twiddles
  // image-layout vectors [B][M][N]
  float2* x;                 // in: x0 (solve) / RSS init (recon); out: x
  const float2* bvec;        // solve mode: b
  float2* u;                 // recon: running u_j
  const float2* u1;
  float2* rhs;               // recon: rhs_reg (written by the SB phase, column-major [B][N][M])
  float2* xT;                // x, column-major [B][N][M] (internal; the image-layout x is the output)
  int kinit;                 // recon: Alg. 1 step 1 (u1, x1 = RSS) and the zero SB state in this launch
  const float2* y;           // kinit: zero-filled k-space [B][C][M][N]
  float2* y1T;               // kinit: scratch [B][C][N][M] (row-inverse-transformed k-space)
  SbArgs sb;                 // recon: SB state (bx/by double buffers, bw, rhs), parity 0 first
  float2* bxs[2];
  float2* bys[2];
  // internal state
  float2* Qs;                // [B][M][N] column spectrum of q (rows = spectral index)
  float2* Sr;                // [B][M][N] column spectrum of r
  float2* Tb;                // [B][N][M] row-phase output, column-major
  double* part;              // [B][8][P] block partials (B * 8 * P <= B * P.cap)
  unsigned* bar;             // [B] barrier counters (zero at launch)
  unsigned long long* stamp; // [32] stage cycle counters (nullable); [8, 20) loop segments
  int prof;                  // 1: also time the PCG loop's segments (SBPCG_KR_PROF=1)
  int cg;                    // 1: Chronopoulos-Gear recurrences (one reduction per iteration)
  Loop L;
  int n_outer;               // 0: one solve (b given) ; >= 1: SB reconstruction
  float eps;
  int maxit;
};
bool kr_supported(int M, int N, int levels);
// CTAs one problem needs, and how many problems fit one cooperative launch on this device
int kr_ctas(int M, int N);
int kr_max_problems(int M, int N, int C);
cudaError_t launch_kr(const KrArgs& a, cudaStream_t st);
cudaError_t launch_transpose_sens(const float2* s, float2* sT, int BC, int M, int N, cudaStream_t st);

// Plane kernels (k_plane*.cu): one G-CTA cluster per NY x NZ plane, DSMEM-exchanged 2D FFT.
enum KPMode { KP_APPLY = 0, KP_PCG = 1, KP_RESID = 2, KP_PRECOND = 3, KP_ENCODE = 4, KP_ADJOINT = 5,
              KP_PRE2D = 6 };
struct KPArgs {
  int B, C, planes, NY, NZ;  // image = planes x NY x NZ per problem (2D: planes = 1)
  int d3;                    // 1: 3D problem (7-point Laplacian across planes)
  float mu, lam, gam;
  const float2* sens;        // [B][C][planes][NY][NZ]
  const uint8_t* mask;       // [B or 1][NY][NZ] (plane mask; 3D masks are constant along d0)
  int mask_bstride;          // NY*NZ or 0
  const float* lam_inv;      // PRECOND: [B][planes][NY][NZ]
  const float2* tw_y;        // [NY]
  const float2* tw_z;        // [NZ]
  float scale;               // matvec: 1/(NY NZ); ENCODE/ADJOINT: 1/sqrt(N)
  int full;                  // ENCODE: R = I
  const float2* vin;         // APPLY/RESID: p or x ; ENCODE: x
  float2* out;               // q / r0 / encoded [B][C][img] / adjoint image
  float2* out2;              // ADJOINT: RSS image (nullable)
  float2* tmp;               // PRECOND in/out [B][img] ; ADJOINT input [B][C][img]
  // PCG
  const float2* z;
  float2* pbuf0;
  float2* pbuf1;
  float2* x;
  // RESID
  const float2* bvec;
  float2* u;
  const float2* u1;
  const float2* rhs_reg;
  float2* bout;
  int update_u;
  float eps;
  int maxit;
  // PRE2D (fused 2D preconditioner): r -= alpha q ; z = F^H Lambda^{-1} F r ; ||r||^2, <r, z>
  const float2* qv;
  float2* rout;
  float2* zout;
  int pmode;                 // -1 standalone apply, 0 PCG init, 1 PCG iteration
  // coil-sharded mode: the matvec kernel stops after the coil loop and
  // writes this rank's partial sum_c conj(s_c) F^H R F (s_c p) to acc_out; after the NCCL
  // all-reduce the epilogue kernel (k_coil.cu) reads the reduced sum from acc_in.
  float2* acc_out;
  const float2* acc_in;
  int plane0;                // first plane of this launch (coil mode: plane chunks overlap the
  int nplanes;               // all-reduce of the previous chunk); nplanes = 0: all planes
  int rss_raw;               // ADJOINT: out2 = sum_c |.|^2 (no sqrt; all-reduced first)
  Loop L;
  Partials P;
};
cudaError_t launch_kc_epilogue(int mode, const KPArgs& a, cudaStream_t st);  // k_coil.cu
cudaError_t launch_kc_sqrt_re(float2* v, size_t n, cudaStream_t st);

// Programmatic dependent launch on/off for subsequent launches (host-side switch; the
// graph builder turns it off while capturing unless SBPCG_GRAPH_PDL=1).
extern thread_local bool g_use_pdl;

// cudaLaunchKernelEx with programmatic dependent launch (+ optional cluster)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             int cluster, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (g_use_pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster > 0) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = cluster;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = 1;
    ++n;
  }
  cfg.attrs = attr;
  cfg.numAttrs = n;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// launchers (return cudaError_t of the launch)
cudaError_t launch_k1(int mode, const K1Args& a, const CUtensorMap* tmap, int W, int G,
                      cudaStream_t st);
bool k1_supported(int M, int N);
int k1_default_W(int M, int N);

enum PassKind {
  P_PRE_A_FWD_COL = 0,   // precond: r -= alpha q (PCG) ; col FFT fwd -> tmp
  P_PRE_B_ROW = 1,       // precond: row FFT, x Lambda^-1, row IFFT (tmp in place)
  P_PRE_C_INV_COL = 2,   // precond: col IFFT -> z ; <r, z>
  P_ENC_COL = 3,         // encode: t_c = s_c x ; col FFT fwd -> tmp[b][c]
  P_ENC_ROW = 4,         // encode: row FFT fwd, x mask / sqrt(N) -> y
  P_ADJ_ROW = 5,         // adjoint/init: y masked, row IFFT -> tmp[b][c]
  P_ADJ_COL = 6,         // adjoint/init: col IFFT, sum_c conj(s_c) . / sqrt(N) (+ RSS)
  // 7, 8: retired (non-separable masks use the plane kernel K1P)
  P_NOPRE = 9,           // no preconditioner: r -= alpha q ; z = r ; partials
  P_FIXUP = 10,          // x += alpha p (pending) / x = 0
  P_COL_FWD = 11,        // o0[b][c] = colFFT(a0[b][c]) * scale   (3D: the d0 transform of E)
  P_COL_INV = 12,        // o0[b][c] = colIFFT(a0[b][c]) * scale  (3D: the d0 transform of E^H)
  // spectral-residual preconditioner (2D line masks, circulant M):
  // K1 writes the column spectrum Q = F_0 q (RESID: S_r = F_0 r0), so one pass per direction:
  P_PRE_B_SPEC = 13,     // row k: S_r -= alpha Q (mode 1); T = F_1^H Lambda^-1 F_1 S_r -> tmp;
                         // ||r||^2 = sum|S_r|^2 / M and <r, z> = Re sum conj(S_r) T (fin_rr, fin_rho)
  P_PRE_C_SPEC = 14,     // z = F_0^H T (column IFFT), no reductions
  P_COL_DECOUPLE = 15,   // readout decoupling: o0[x][c] = colIFFT(a0[c])[x] * scale (B = 1)
};
cudaError_t launch_pass(int kind, const PassArgs& a, cudaStream_t st);
// jinv[b][i] = 1 / (mu f_b sum_c |s_c(i)|^2 + 2 nd lambda + gamma)
cudaError_t launch_jacobi_diag(const float2* sens, const float* frac, int B, int C, size_t img, int nd, float mu,
                               float lam, float gam, float* jinv, cudaStream_t st);
bool pass_supported(int M, int N);

cudaError_t launch_kp2(int mode, const KPArgs& a, cudaStream_t st);  // 2D, matvec modes
cudaError_t launch_kp3(int mode, const KPArgs& a, cudaStream_t st);  // 3D planes, all modes
bool kp2_supported(int NY, int NZ);
bool kp3_supported(int NY, int NZ);

// preprocessing (k_prep.cu)
cudaError_t launch_normalize_sens(const float2* s, const uint8_t* sup, size_t sup_bstride, int B, int C, size_t npix,
                                  float2* out, cudaStream_t st);
cudaError_t launch_normalize_images(const float2* m, const float2* sh, int B, int C, size_t npix, float2* out,
                                    cudaStream_t st);
cudaError_t launch_gram(const float2* d, int B, int C, size_t npix, double2* part, int nblk, double2* G,
                        cudaStream_t st);
cudaError_t launch_coil_apply(const float2* in, const float2* A, int B, int C, int K, size_t npix, float2* out,
                              cudaStream_t st);
}  // namespace sbk
#include <complex>
namespace sbk {
void hermitian_eig(int n, const std::complex<double>* G, double* w, std::complex<double>* U);

cudaError_t launch_lambda_build(const LamArgs& a, cudaStream_t st);
cudaError_t launch_lambda_chunk(const LamArgs& a, cudaStream_t st);  // L_COL_SENS + L_ROW_ACC only
cudaError_t launch_lambda_tail(const LamArgs& a, cudaStream_t st);   // from g to k (or kc2)
cudaError_t launch_lambda_expand3(const Lam3Args& a, cudaStream_t st);
cudaError_t launch_sb_update(const SbArgs& a, cudaStream_t st);
cudaError_t launch_sb_update3(const SbArgs& a, cudaStream_t st);
// Daubechies-4 wavelet part of the SB step (k_wav.cu): rhs += gamma W^H(d_w - b_w), b_w update
cudaError_t launch_d4_sb(const float2* x, float2* wbuf, float2* bw, float2* rhs, int B, int E0, int E1, int E2, int nd,
                         int levels, float gamma, cudaStream_t st, int* nlaunch);
cudaError_t launch_log(const Loop& L, cudaStream_t st);
cudaError_t launch_spin(cudaStream_t st, unsigned long long ns);

}  // namespace sbk
