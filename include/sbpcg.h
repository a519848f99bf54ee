/* sbpcg.h — C ABI of libsbpcg: circulant-preconditioned CG inside Split Bregman for
 * parallel-imaging + compressed-sensing MRI, B200 (sm_100a) native.
 *
 * Method: Koolstra, van Gemert, Boernert, Webb, Remis, "Accelerating CS in Parallel
 * Imaging Reconstructions Using an Efficient and Effective Circulant Preconditioner"
 * (arXiv 1710.01758).  "PAPER.md:n" below cites line n of that paper's LaTeX source.
 *
 * ------------------------------------------------------------------------------------
 * Data conventions (all entry points)
 *   * complex = interleaved (re, im) float32 pairs (sb_c64), i.e. torch.complex64;
 *   * images are row-major [B][d0][d1]; d0 is the phase-encode axis of line masks
 *     (a line mask samples whole rows: "random line pattern ... in the
 *     foot-head direction"), d1 is the readout;
 *   * coil stacks are [B][C][d0][d1]; k-space is unshifted (DC at index 0) and
 *     unitary-scaled: (F x)(nu) = N^{-1/2} sum_n x(n) exp(-2 pi i nu.n/n)  (reading A1);
 *   * mask is uint8 0/1 over the k-space grid, one per problem ([B][d0][d1]) or shared
 *     ([d0][d1], dims.mask_shared = 1);
 *   * every array pointer may be HOST or DEVICE memory (detected with
 *     cudaPointerGetAttributes).  Host arrays are staged through the context's device
 *     buffers inside the call; device arrays must live on the context's device, be
 *     16-byte aligned and C-contiguous.  Outputs must not alias inputs (SB_E_ARG).
 *   * B independent problems are solved together, each with its own PCG scalars and
 *     its own convergence (a converged problem is frozen; reading A26).
 * Ownership: the context copies sens and mask at create (the caller may free them
 * afterwards) and owns Lambda^{-1}, the workspace and the SB state; the caller owns
 * every I/O buffer.  One context must not be used by two host threads at once.
 * Streams: all work is enqueued on the CUDA stream given at create (NULL = legacy
 * default stream).  sb_pcg_apply_A / sb_pcg_apply_Pinv / sb_encode with device
 * pointers are asynchronous; every other call returns after the stream completed.
 * Errors: every call returns an sb_status and never throws across the ABI.  CUDA errors
 * are sticky (SB_E_CUDA): the context is then unusable; sb_last_error() explains.
 * ------------------------------------------------------------------------------------
 */
#ifndef SBPCG_H
#define SBPCG_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBPCG_ABI_VERSION 2

typedef struct sb_ctx sb_ctx;
typedef struct sb_comm sb_comm;  /* NCCL communicator of the coil-sharded mode (see below) */
typedef struct { float re, im; } sb_c64;

typedef enum {
  SB_OK = 0,
  SB_E_ARG = 1,              /* NULL/aliased/misaligned pointer, bad option value      */
  SB_E_DIM = 2,              /* shape/batch/coils/levels inconsistent, or batch*coils  */
                             /* > 65535 (launch-grid limit); levels must              */
                             /* divide the shape, PAPER.md:117 W unitary on the grid) */
  SB_E_UNSUPPORTED_SIZE = 3, /* an image axis is not in the FFT size set               */
  SB_E_PARAM = 4,            /* gamma <= 0, mu < 0 or lambda < 0 (k >= gamma > 0)      */
  SB_E_SINGULAR_K = 5,       /* min |k| <= 1e-14 or non-finite           */
  SB_E_NONFINITE = 6,        /* NaN/Inf in a PCG recurrence scalar                     */
  SB_E_INDEFINITE = 7,       /* <p, A p> <= 0 (A must be HPD)            */
  SB_E_CUDA = 8,             /* CUDA runtime error (sticky)                            */
  SB_E_NOMEM = 9,            /* device allocation failed                               */
  SB_E_COMM = 10             /* coil-sharded mode: NCCL could not be loaded, the        */
                             /* communicator could not be created, or an all-reduce    */
                             /* failed (sb_comm_*, sb_pcg_set_comm, solve/recon)       */
} sb_status;

/* Problem geometry.
 *   ndim = 2: images [d0][d1], shape = {d0, d1, 0}; d0, d1 in {8, 16, 32, 64, 128, 256}.
 *             Line masks (constant along d1) take the 1D-FFT matvec (K1); other masks the
 *             plane-cluster matvec (K1P) for the plane sizes k_plane.cu instantiates.
 *   ndim = 3: volumes [d0][d1][d2], shape = {d0, d1, d2}; d0 (the readout) in
 *             {8, ..., 256, 192}, (d1, d2) in {16^2, 32^2, 48^2, 64^2, 128^2, 192^2, 256^2}
 *             (radix-2/3, reading A23).  The mask must be constant along d0 (fully sampled
 *             readout; BASELINE config 5), else SB_E_UNSUPPORTED_SIZE.
 *             wavelet_levels <= 3 (8^3 Haar tiles); TV and Haar are 3D (readings A6, A10). */
typedef struct {
  int32_t ndim;
  int64_t shape[3];
  int32_t batch;           /* B >= 1 independent problems                              */
  int32_t wavelet_levels;  /* L-level orthonormal Haar W (reading A6), 2^L | d0, d1    */
  int32_t mask_shared;     /* 1: one mask for all problems                             */
} sb_dims;

/* Create a context for  A = mu sum_c (R F S_c)^H R F S_c + lambda sum_d D_d^H D_d
 * + gamma W^H W  (W^H W = I) and build the circulant
 * preconditioner  M^{-1} = F^H diag{k}^{-1} F,  k = mu k_c + lambda k_d + gamma
 * (PAPER.md:189-197), k_c by the circular-correlation form of PAPER.md:199-229 (reading
 * A2), k_d = sum_d 4 sin^2(pi nu_d/n_d), built once in fp64 on the
 * device ("constructed beforehand").
 *   out     receives the context (NULL on failure)
 *   dims    geometry, see sb_dims
 *   coils   C >= 1
 *   mask    uint8 [B or 1][d0][d1], values 0/1
 *   sens    complex [B][C][d0][d1] coil sensitivities S_c
 *   mu, lambda, gamma  weights of Eq. original; gamma > 0 required
 *   cuda_stream  cudaStream_t to enqueue on (NULL = default stream)
 *   comm    NULL (single GPU, or slice sharding: each rank its own context), or a coil-sharded
 *           communicator (sb_comm_init_nccl; ndim = 3 only): `coils` and `sens` are then this
 *           rank's coil shard and Lambda is built from the marginal over every rank's coils
 *           (a collective call: every rank of comm must create its context)
 * Errors: SB_E_ARG, SB_E_DIM, SB_E_UNSUPPORTED_SIZE, SB_E_PARAM, SB_E_SINGULAR_K,
 *         SB_E_NOMEM, SB_E_CUDA, SB_E_COMM.  Synchronises the stream before returning. */
sb_status sb_pcg_create(sb_ctx** out, const sb_dims* dims, int32_t coils, const uint8_t* mask,
                        const sb_c64* sens, float mu, float lambda, float gamma,
                        void* cuda_stream, sb_comm* comm);

/* Options (sb_set_option):
 *   SB_OPT_PERSISTENT  1 (default) / 0: solve and reconstruct small batches of square line-mask
 *                      problems (d0 = d1 in {64, 256}, Haar W, circulant M, single GPU, batch
 *                      * d1 CTAs co-resident) with the persistent whole-GPU kernel (k_persist.cu;
 *                      DESIGN.md "KR"); 0 forces the kernel sequence.  Results agree with the
 *                      sequence to rounding (both are checked against the oracle). */
#define SB_OPT_PERSISTENT 1
/*   SB_OPT_PCG_CG      1 (default) / 0: inside the persistent kernel, run PCG with the
 *                      Chronopoulos-Gear single-reduction recurrences (the iterates of
 *                      PAPER.md:238 in exact arithmetic; s = A p carried by a recurrence, the
 *                      two inner products of an iteration reduced together: two grid barriers
 *                      per iteration instead of three) or with the standard recurrences. */
#define SB_OPT_PCG_CG 2
sb_status sb_set_option(sb_ctx* ctx, int32_t option, int32_t value);

/* How the last sb_pcg_solve / sb_recon executed (for bench.py and tests). */
#define SB_PATH_NONE 0
#define SB_PATH_GRAPH 1          /* kernel sequence, device-driven loop in a CUDA graph       */
#define SB_PATH_EAGER 2          /* kernel sequence, host-checked loop                        */
#define SB_PATH_PERSISTENT 3     /* one cooperative launch of k_persist                       */
#define SB_PATH_COIL_SHARDED 4   /* coil-sharded kernel sequence with NCCL all-reduces        */
int32_t sb_last_path(const sb_ctx* ctx);

/* Wavelet family of W in the SB shrink step: 0 = orthonormal Haar (default; reading A6),
 * 1 = periodized Daubechies-4, the paper's W (reading A32), same Mallat layout
 * and levels (>= 1).  W^H W = I either way, so A and Lambda do not change. */
sb_status sb_set_wavelet(sb_ctx* ctx, int32_t family);

/* Replace the coil sensitivities (same shape; host or device pointer, copied) and rebuild
 * Lambda.  The mask, weights, buffers and captured CUDA graphs stay valid,
 * so a new acquisition with the same geometry reuses the context.  Asynchronous (a host `sens`
 * must stay valid until the next synchronising call); a singular k of the rebuilt Lambda is
 * reported as SB_E_SINGULAR_K by the next sb_pcg_solve / sb_recon / sb_pcg_get_k. */
sb_status sb_pcg_update_sens(sb_ctx* ctx, const sb_c64* sens);

/* Rebuild Lambda^{-1} from the context's sens/mask/weights (the preconditioner build of
 * PAPER.md:238 / Table 2, timed by bench.py as part of a step).  Asynchronous; a singular k
 * is reported by the next sb_pcg_solve / sb_recon / sb_pcg_get_k (SB_E_SINGULAR_K). */
sb_status sb_pcg_build_precond(sb_ctx* ctx);

/* y = A x for all B problems.  x, y: complex [B][d0][d1]. */
sb_status sb_pcg_apply_A(sb_ctx* ctx, const sb_c64* x, sb_c64* y);

/* z = M^{-1} r = F^H diag{k}^{-1} F r.  r, z: complex [B][d0][d1]. */
sb_status sb_pcg_apply_Pinv(sb_ctx* ctx, const sb_c64* r, sb_c64* z);

/* y_c = R F S_c x (Eq. ill0); full != 0 replaces R by I.
 * x: complex [B][d0][d1]; y: complex [B][C][d0][d1]. */
sb_status sb_encode(sb_ctx* ctx, const sb_c64* x, sb_c64* y, int32_t full);

/* x = sum_c S_c^H F^H R y_c (first term of b without mu).
 * y: complex [B][C][d0][d1]; x: complex [B][d0][d1]. */
sb_status sb_adjoint(sb_ctx* ctx, const sb_c64* y, sb_c64* x);

typedef struct {
  float eps;          /* stop when ||r_k||/||b|| <= eps; 0 => fixed count   */
  int32_t max_iters;  /* >= 1                                                              */
  int32_t precond;    /* 0 none, 1 circulant, 2 Jacobi z = r/diag(A) with  */
                      /* diag(A) = mu f sum_c |S_c|^2 + 2 nd lambda + gamma (PAPER.md:187;  */
                      /* f = sampled fraction; built on first use; not in coil-sharded mode)*/
  int32_t use_graph;  /* 1: device-driven loop in a CUDA graph (conditional while node)   */
} sb_pcg_opts;

typedef struct {      /* host arrays (NULL = not requested)                                */
  int32_t* iters;     /* [B] A p products in the loop (reading A16)                        */
  float* final_relres;/* [B] ||r_k|| / ||b|| (recurrence residual, reading A15)            */
  int8_t* converged;  /* [B]                                                               */
  float* relres_hist; /* [B][max_iters + 1]; entries past iters[b] are undefined           */
} sb_pcg_stats;

/* Solve A x = b by PCG for all B problems; x holds x0 on entry
 * and the solution on exit.  Reaching max_iters is not an error (converged = 0 when
 * eps > 0).  ||b|| = 0 returns x = 0, converged.  Errors: SB_E_INDEFINITE,
 * SB_E_NONFINITE (first failing problem's status), SB_E_ARG. */
sb_status sb_pcg_solve(sb_ctx* ctx, const sb_c64* b, sb_c64* x, const sb_pcg_opts* opts,
                       sb_pcg_stats* stats);

typedef struct {
  int32_t n_outer, n_inner;  /* Algorithm 1 loops; n_inner must be 1 */
  sb_pcg_opts pcg;
  int32_t stage_timers;      /* 1: fill the stage times of sb_recon_log on the kernel-   */
                             /* sequence path (runs it eagerly: CUDA-event pairs around  */
                             /* each stage).  The persistent path always fills them.     */
} sb_recon_opts;

/* Reconstruction log.  Stage times are device seconds summed over the call, split like the
 * paper's cost discussion: step 4 (RHS), the PCG solves, steps 6-11
 * (shrink/Bregman + regulariser RHS), steps 13-15 (data feedback).  Both paths form the RHS,
 * the data feedback u += u1 - E^H E x and r0 = b - A x in ONE coil pass (the feedback reuses
 * that pass's E^H E x), so its time is reported in rhs_s and feedback_s is 0.  init_s = step 1
 * (u1 = sum_c S_c^H F^H y_c, RSS); build_s = the last Lambda build of this context (PAPER.md
 * Table 2 analogue; create, sb_pcg_build_precond or sb_pcg_update_sens). */
typedef struct {             /* host outputs (NULL members = not requested)               */
  int32_t* pcg_iters;        /* [n_outer * n_inner][B]                                    */
  float* final_relres;       /* [n_outer * n_inner][B]                                    */
  double total_ms;           /* device time of the whole call (CUDA events)               */
  double rhs_s, pcg_s, shrink_s, feedback_s, build_s, init_s;
  int32_t stages_valid;      /* 1 when the stage times were measured                      */
} sb_recon_log;

/* Split Bregman reconstruction, Algorithm 1 with per-problem PCG.
 *   y      complex [B][C][d0][d1] zero-filled k-space
 *   x_out  complex [B][d0][d1] reconstruction
 * Step 1 x = RSS(F^H y_c) (reading A12); steps 6-11 with literal thresholds 1/lambda,
 * 1/gamma (reading A8); data feedback (steps 13-15) in the exact image-domain form
 * u_{j+1} = u_j + u_1 - E^H E x. */
sb_status sb_recon(sb_ctx* ctx, const sb_c64* y, const sb_recon_opts* opts, sb_c64* x_out,
                   sb_recon_log* log);

/* One SB shrink/Bregman step (Alg. 1 steps 6-11) plus the regulariser part of the next
 * RHS (step 4): given x and b_x, b_y, b_w (complex [B][d0][d1] each, b_w in the Haar
 * Mallat layout), writes the updated b_x, b_y, b_w and
 *   rhs_reg = lambda sum_d D_d^H (d_d - b_d) + gamma W^H (d_w - b_w).
 * In-place on b_* is allowed (the only aliasing allowed by the ABI). */
sb_status sb_sb_update(sb_ctx* ctx, const sb_c64* x, sb_c64* bx, sb_c64* by, sb_c64* bw,
                       sb_c64* rhs_reg);

/* 3D form of sb_sb_update (ndim = 3 contexts; b_z is the third TV auxiliary, 3D Mallat Haar
 * layout for b_w).  For ndim = 2 contexts bz is ignored and the call equals sb_sb_update. */
sb_status sb_sb_update3(sb_ctx* ctx, const sb_c64* x, sb_c64* bx, sb_c64* by, sb_c64* bz, sb_c64* bw,
                        sb_c64* rhs_reg);

/* Real k (not 1/(N k)) as built, fp64 [B or 1][d0][d1] — parity output. */
sb_status sb_pcg_get_k(sb_ctx* ctx, double* k_out);

/* Kernel timing for bench.py's roofline: when enabled, CUDA events bracket every launch of
 * the matvec kernel (K1 / K1P; which = 0) and of the persistent kernel (KR; which = 2) on the
 * context's stream (solves then run eagerly), and sb_get_kernel_time returns the accumulated
 * device ms, the launch count and the algorithmic bytes per launch. */
sb_status sb_set_kernel_timing(sb_ctx* ctx, int32_t enable);
sb_status sb_get_kernel_time(sb_ctx* ctx, int32_t which /*0 = matvec, 2 = persistent kernel*/,
                             double* ms, int64_t* launches, double* alg_bytes_per_launch);

/* ------------------------------------------------------------------------------------
 * Coil-sharded mode (BASELINE config 5 over G GPUs).  One process per GPU; rank
 * r creates its context with ITS coil shard (sens [B][C_r][...]) and the full mask, then
 * attaches a communicator.  Every vector is replicated; per matvec each rank computes its
 * partial coil sum sum_{c in r} S_c^H F^H R F S_c p and ONE NCCL all-reduce (sum, fp32) of
 * that image forms the data term of A; the preconditioner, the regulariser,
 * the dots and the SB steps then run identically on every rank (the all-reduce result is
 * bitwise identical across ranks, so no scalar all-reduce is needed).  Lambda's coil
 * marginal, u_1 and the RSS init are all-reduced as well.  NCCL is loaded at run time (the process's libnccl.so.2, or
 * SBPCG_NCCL_LIB).  For ndim = 3 contexts (2D batches shard by slice, with no collective).
 * ------------------------------------------------------------------------------------ */
/* rank 0: a 128-byte NCCL unique id to broadcast to the other ranks (out of band). */
sb_status sb_comm_unique_id(void* id_out);
/* Collective over the `world` ranks; binds to the current CUDA device.  SB_E_COMM on failure.
 * sb_comm_init_nccl is the name SURVEY 8(b) uses; sb_comm_init is the same call. */
sb_status sb_comm_init_nccl(const void* nccl_unique_id, int32_t rank, int32_t world, sb_comm** out);
sb_status sb_comm_init(const void* id, int32_t rank, int32_t world, sb_comm** out);
void sb_comm_destroy(sb_comm* comm);
/* Attach (comm != NULL) or detach the communicator; rebuilds Lambda (collective). */
sb_status sb_pcg_set_comm(sb_ctx* ctx, sb_comm* comm);

/* ------------------------------------------------------------------------------------
 * Data preprocessing of the paper's Methods (no context; DEVICE pointers only, SB_E_ARG
 * otherwise; enqueued on `stream`).  Arrays are [batch][coils][npix] complex, npix = the
 * pixels of one image (any dimensionality).
 * ------------------------------------------------------------------------------------ */
/* S_hat_i = [sum_j S_j^H S_j]^{-1/2} S_i, set to 0 outside the subject.
 * support: uint8 [batch or 1][npix] (support_shared = 1: one for all), NULL = everywhere.
 * Asynchronous. */
sb_status sb_normalize_sens(const sb_c64* sens, const uint8_t* support, int32_t batch, int32_t coils, int64_t npix,
                            int32_t support_shared, sb_c64* sens_out, void* stream);
/* m_i <- S_hat_i sum_j S_hat_j^H m_j.  Asynchronous; m_out may equal m. */
sb_status sb_normalize_coil_images(const sb_c64* m, const sb_c64* sens_hat, int32_t batch, int32_t coils, int64_t npix,
                                   sb_c64* m_out, void* stream);
/* SVD coil compression (Huang et al. 2008): per problem, the coil
 * covariance G = sum_n y(n) y(n)^H (fp64), its eigenvectors U (descending eigenvalues), and
 * A = U[:, :coils_out]^H applied to the data y and the maps: y_out = A y, sens_out = A sens
 * ([batch][coils_out][npix]).  coils <= 64.  eig_out: optional HOST float [batch][coils].
 * Synchronous (the C x C eigen-decomposition runs on the host).  Outputs must not alias. */
sb_status sb_coil_compress(const sb_c64* y, const sb_c64* sens, int32_t batch, int32_t coils, int64_t npix,
                           int32_t coils_out, sb_c64* y_out, sb_c64* sens_out, float* eig_out, void* stream);

/* Readout decoupling (BASELINE config 4; "fully sampled" readout):
 * for a 3D acquisition whose mask is constant along the readout d0, F_3 = F_0 (x) F_12 and
 * R = I_0 (x) R_12, so the unitary 1D IFFT along d0 of every coil's k-space splits the problem
 * into D0 independent 2D problems on the (d1, d2) planes:
 *   y2[x][c][k1][k2] = (F_0^H y3[c])(x, k1, k2),   s2[x][c][d1][d2] = s3[c][x][d1][d2]
 * (the maps are image-space: only their layout changes; the plane mask is the 3D mask's
 * d0 = 0 plane).  The y2 / s2 stacks are the [B][C][d1][d2] inputs of a 2D context with
 * B = D0 problems and mask_shared = 1.  shape = {D0, D1, D2}; D0 in the column-FFT size set
 * (8..256, 192); D1 * D2 a multiple of 8.  y3, s3: complex [C][D0][D1][D2]; y2, s2: complex
 * [D0][C][D1][D2]; s3 = s2 = NULL skips the maps.  DEVICE pointers only (SB_E_ARG otherwise);
 * outputs must not alias inputs.  Synchronous on `stream`. */
sb_status sb_readout_decouple(const sb_c64* y3, const sb_c64* s3, int32_t coils, const int64_t* shape, sb_c64* y2,
                              sb_c64* s2, void* stream);

/* Number of kernels launched by this context since creation (for bench.py). */
int64_t sb_kernel_launch_count(const sb_ctx* ctx);

void sb_pcg_destroy(sb_ctx* ctx);
const char* sb_status_str(sb_status s);
const char* sb_last_error(const sb_ctx* ctx);
int32_t sb_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SBPCG_H */
