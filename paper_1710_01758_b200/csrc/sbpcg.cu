// sbpcg.cu — libsbpcg host side: context, preconditioner build, device-driven PCG loop
// (CUDA graph with a conditional WHILE node), Split Bregman orchestration, C ABI.
//
// Method: PAPER.md:87-244 (see include/sbpcg.h for per-call citations).  PyTorch is not
// used here; the Python binding passes raw pointers and a cudaStream_t.
#include <cudaTypedefs.h>
#include <dlfcn.h>

#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sbpcg.h"
#include "kernels.cuh"

using namespace sbk;

namespace sbk {
thread_local bool g_use_pdl = true;
}

static bool env_flag(const char* name, bool dflt) {
  const char* v = getenv(name);
  if (!v) return dflt;
  return v[0] == '1';
}

// ------------------------------------------------------------------ NCCL (coil-sharded mode)
// NCCL is resolved at run time (dlopen of the libnccl.so.2 the process already uses — the one
// torch.distributed loaded — or SBPCG_NCCL_LIB), so the library has no link-time dependency.
typedef struct { char internal[128]; } nccl_uid_t;
typedef void* nccl_comm_t;
enum { NCCL_SUM = 0, NCCL_FLOAT32 = 7, NCCL_FLOAT64 = 8 };
struct NcclApi {
  void* h = nullptr;
  int (*getUniqueId)(nccl_uid_t*) = nullptr;
  int (*commInitRank)(nccl_comm_t*, int, nccl_uid_t, int) = nullptr;
  int (*commDestroy)(nccl_comm_t) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
  const char* (*getErrorString)(int) = nullptr;
};
static NcclApi g_nccl;
static bool nccl_load() {
  if (g_nccl.allReduce) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) {
    const char* e = getenv("SBPCG_NCCL_LIB");
    h = dlopen(e ? e : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  }
  if (!h) return false;
  g_nccl.h = h;
  g_nccl.getUniqueId = (int (*)(nccl_uid_t*))dlsym(h, "ncclGetUniqueId");
  g_nccl.commInitRank = (int (*)(nccl_comm_t*, int, nccl_uid_t, int))dlsym(h, "ncclCommInitRank");
  g_nccl.commDestroy = (int (*)(nccl_comm_t))dlsym(h, "ncclCommDestroy");
  g_nccl.allReduce =
      (int (*)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t))dlsym(h, "ncclAllReduce");
  g_nccl.getErrorString = (const char* (*)(int))dlsym(h, "ncclGetErrorString");
  return g_nccl.getUniqueId && g_nccl.commInitRank && g_nccl.commDestroy && g_nccl.allReduce;
}

struct sb_comm {
  nccl_comm_t comm = nullptr;
  int rank = 0, world = 1;
};

struct GraphSlot {
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  int nfixed = 0;      // kernels outside the loop
  int nbody = 0;       // kernels per while-body (unroll iterations)
  int unroll = 1;
  float eps = -1.f;
  int maxit = -1;
  int precond = -1;
};

struct sb_ctx {
  int dev = 0;
  cudaStream_t st = nullptr;
  cudaStream_t cap1 = nullptr;  // graph capture stream (the user stream may be the legacy NULL stream)
  cudaStream_t cap2 = nullptr;  // body capture stream
  int B = 0, C = 0, M = 0, N = 0, L = 0, mask_shared = 0;
  // geometry: 2D images are D0 x D1 (M = D0, N = D1); 3D volumes D0 x D1 x D2 with
  // M = D0 (the readout, column-pass length) and N = D1*D2 (column-pass columns)
  int ndim = 2, D0 = 0, D1 = 0, D2 = 1;
  bool plane = false;           // K1P plane kernels (2D non-separable masks, or 3D)
  bool pre2d = false;           // 2D preconditioner as one K1P cluster kernel (KP_PRE2D)
  bool spec_ok = false;         // spectral-residual preconditioner passes possible (2D lines, G = 1)
  bool spec_on = false;         // ... and selected for the solve being built / run (circulant M)
  uint8_t* pmask = nullptr;     // 3D: the plane mask [Bm][D1*D2] (mask constant along d0)
  float2 *tw_y = nullptr, *tw_z = nullptr;  // plane twiddles (3D: D1, D2)
  double2 *twd_y = nullptr, *twd_z = nullptr;
  float2* bz[2] = {nullptr, nullptr};       // 3D TV auxiliary b_z
  double k1_bytes = 0;          // algorithmic bytes per problem-launch of the matvec
  sb_comm* comm = nullptr;      // coil-sharded mode (this context holds a coil shard)
  float2* accbuf = nullptr;     // [B][img] partial / all-reduced coil sum
  cudaStream_t cst = nullptr;   // coil mode: the all-reduce stream (overlaps the plane kernel)
  int coil_chunks = 4;          // coil mode: plane chunks per matvec (SBPCG_COIL_CHUNKS)
  cudaEvent_t chunk_ev[16] = {};  // coil mode: chunk k's partial sums written / all-reduced
  cudaEvent_t red_done = nullptr;
  cudaGraphExec_t coil_exec[4][3] = {};  // coil mode [kind: solve, recon first, next par 0/1][0 pre, 1 body, 2 post]
  cudaGraph_t coil_graph[4][3] = {};
  int coil_unroll = 4;          // coil mode: PCG iterations per graph launch (host check between)
  float coil_eps = -1.f;
  int coil_maxit = -1, coil_pre = -1;
  float* jinv = nullptr;        // Jacobi: 1/diag(A) [B][img] (built on first use)
  int wavelet = 0;              // 0 Haar (reading A6), 1 Daubechies-4 (reading A32)
  float2* wbuf = nullptr;       // D4 coefficients [B][img]
  std::vector<float> samp_frac; // sampled fraction f of each problem's mask
  void* lscr[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // Lambda build scratch (kept)
  size_t lscr_bytes[6] = {0, 0, 0, 0, 0, 0};
  float mu = 0, lam = 0, gam = 0;
  bool separable = false;
  int W = 8, G = 1;
  size_t img = 0;
  // constant data
  float2* sens = nullptr;
  uint8_t* mask = nullptr;
  float* rowmask = nullptr;
  float* lam_inv = nullptr;
  double* kbuf = nullptr;
  float2 *tw_m = nullptr, *tw_n = nullptr;
  double2 *twd_m = nullptr, *twd_n = nullptr;
  // vectors [B][M][N]
  float2 *x = nullptr, *r = nullptr, *z = nullptr, *q = nullptr, *p0 = nullptr, *p1 = nullptr;
  float2 *tmp = nullptr, *bvec = nullptr, *u = nullptr, *u1 = nullptr, *rhs = nullptr;
  float2 *bx[2] = {nullptr, nullptr}, *by[2] = {nullptr, nullptr}, *bw = nullptr;
  float2* tmpc = nullptr;  // [B][C][M][N]
  float2* stage_in = nullptr;   // host staging [B][C][M][N]
  float2* stage_out = nullptr;  // host staging [B][C][M][N]
  // PCG bookkeeping
  Scal* scal = nullptr;
  Ctl* ctl = nullptr;
  Counters* counters = nullptr;
  Partials P{};
  float* hist = nullptr;
  int hist_stride = 0;
  int32_t* log_iters = nullptr;
  float* log_relres = nullptr;
  int log_cap = 0;
  CUtensorMap tmap;
  // graphs: 0 = solve, 1 = recon first, 2/3 = recon next (parity)
  GraphSlot gs[4];
  sb_status sticky = SB_OK;
  std::string err;
  int64_t launches = 0;
  // persistent reconstruction kernel (k_persist.cu): small batches of square line-mask problems
  bool kr_ok = false;           // geometry and batch fit one cooperative launch (decided at create)
  bool kr_on = true;            // sb_set_option(SB_OPT_PERSISTENT); env SBPCG_PERSIST=0 disables
  bool kr_cg = true;            // sb_set_option(SB_OPT_PCG_CG): single-reduction recurrences in KR
  float2* sT = nullptr;         // [B][C][N][M] column-major coil maps
  unsigned* kbar = nullptr;     // [B] barrier counters
  const float2* kr_y = nullptr;  // recon on the persistent path with kinit: the device k-space
  unsigned long long* kstamp = nullptr;  // [8] stage cycle counters
  double kr_alg_bytes = 0;      // algorithmic bytes of the timed persistent launches
  int last_path = 0;            // SB_PATH_* of the last solve / recon
  // stage timers (sb_recon_log) and the Lambda build time
  bool stage_timing = false;
  double stage_s[5] = {0, 0, 0, 0, 0};  // rhs, pcg, shrink, feedback, init (seconds)
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> stage_ev;
  std::vector<cudaEvent_t> stage_pool;
  size_t stage_next = 0;
  double build_s = 0;
  // the Lambda build is asynchronous: its singular-k flag (pinned host copy) and its event pair
  // are checked by the next call that completes the stream (build_checked)
  int* bad_host = nullptr;
  bool build_check = false;
  // pinned host copies of the per-call results (scalars, logs, stage counters), filled by async
  // copies enqueued before the call's final synchronisation (no blocking copies after it)
  unsigned char* hres = nullptr;
  size_t hres_bytes = 0;
  cudaEvent_t rev[2] = {nullptr, nullptr};  // sb_recon's total_ms event pair
  cudaEvent_t bev[2] = {nullptr, nullptr};
  // kernel timing (0 = matvec K1/K1P, 1 = unused, 2 = persistent kernel KR)
  bool timing = false;
  double t_ms[3] = {0, 0, 0};
  int64_t t_n[3] = {0, 0, 0};
  std::vector<cudaEvent_t> evpool;
  std::vector<std::pair<int, std::pair<int, int>>> evpend;  // (which, (ev0, ev1))
  size_t evnext = 0;
};

// ------------------------------------------------------------------ error helpers
static sb_status fail(sb_ctx* c, sb_status s, const std::string& msg) {
  if (c) {
    c->err = msg;
    if (s == SB_E_CUDA) c->sticky = SB_E_CUDA;
  }
  return s;
}
#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(c, SB_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

template <typename T>
static cudaError_t dalloc(T** p, size_t n) {
  return cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T));
}

static bool fft_len_ok(int64_t n) { return n == 8 || n == 16 || n == 32 || n == 64 || n == 128 || n == 256; }
static bool col3_len_ok(int64_t n) { return fft_len_ok(n) || n == 192; }

// ------------------------------------------------------------------ twiddles
template <typename V>
static std::vector<V> make_tw(int n) {
  std::vector<V> t(n);
  for (int m = 0; m < n; ++m) {
    const double a = -2.0 * M_PI * (double)m / (double)n;
    t[m].x = std::cos(a);
    t[m].y = std::sin(a);
  }
  return t;
}

// ------------------------------------------------------------------ TMA descriptor
static sb_status make_tmap_w(sb_ctx* c, CUtensorMap* out, int W);
static sb_status make_tmap(sb_ctx* c) { return make_tmap_w(c, &c->tmap, c->W); }
static sb_status make_tmap_w(sb_ctx* c, CUtensorMap* out, int W) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) return fail(c, SB_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  cuuint64_t gdim[3] = {(cuuint64_t)(2 * c->N), (cuuint64_t)c->M, (cuuint64_t)c->B * c->C};
  cuuint64_t gstride[2] = {(cuuint64_t)c->N * 8, (cuuint64_t)c->M * c->N * 8};
  cuuint32_t box[3] = {(cuuint32_t)(2 * W), (cuuint32_t)c->M, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)c->sens, gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(c, SB_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return SB_OK;
}

// ------------------------------------------------------------------ argument builders
static Loop make_loop(sb_ctx* c, unsigned long long cond) {
  Loop L;
  L.scal = c->scal;
  L.ctl = c->ctl;
  L.hist = c->hist;
  L.hist_stride = c->hist_stride;
  L.log_iters = c->log_iters;
  L.log_relres = c->log_relres;
  L.B = c->B;
  L.cond = cond;
  L.cnt = c->counters;
  return L;
}

static K1Args base_k1(sb_ctx* c) {
  K1Args a;
  memset(&a, 0, sizeof(a));
  a.B = c->B;
  a.C = c->C;
  a.M = c->M;
  a.N = c->N;
  a.mu = c->mu;
  a.lam = c->lam;
  a.gam = c->gam;
  a.rmask = c->rowmask;
  a.rmask_bstride = c->mask_shared ? 0 : c->M;
  a.P = c->P;
  a.tw = c->tw_m;
  return a;
}

static KPArgs base_kp(sb_ctx* c) {
  KPArgs a;
  memset(&a, 0, sizeof(a));
  a.B = c->B;
  a.C = c->C;
  a.planes = c->ndim == 3 ? c->D0 : 1;
  a.NY = c->ndim == 3 ? c->D1 : c->M;
  a.NZ = c->ndim == 3 ? c->D2 : c->N;
  a.d3 = c->ndim == 3;
  a.mu = c->mu;
  a.lam = c->lam;
  a.gam = c->gam;
  a.sens = c->sens;
  a.mask = c->ndim == 3 ? c->pmask : c->mask;
  a.mask_bstride = c->mask_shared ? 0 : a.NY * a.NZ;
  a.lam_inv = c->lam_inv;
  a.tw_y = c->ndim == 3 ? c->tw_y : c->tw_m;
  a.tw_z = c->ndim == 3 ? c->tw_z : c->tw_n;
  a.scale = 1.0f / (float)(a.NY * a.NZ);
  a.P = c->P;
  a.pbuf0 = c->p0;
  a.pbuf1 = c->p1;
  a.x = c->x;
  a.z = c->z;
  return a;
}

static PassArgs base_pass(sb_ctx* c) {
  PassArgs a;
  memset(&a, 0, sizeof(a));
  a.B = c->B;
  a.C = c->C;
  a.M = c->M;
  a.N = c->N;
  a.mu = c->mu;
  a.lam = c->lam;
  a.gam = c->gam;
  a.tw_m = c->tw_m;
  a.tw_n = c->tw_n;
  a.lam_inv = c->lam_inv;
  a.lam_bstride = (int)c->img;
  a.mask = c->mask;
  a.mask_bstride = c->mask_shared ? 0 : (int)c->img;
  a.sens = c->sens;
  a.P = c->P;
  a.pbuf0 = c->p0;
  a.pbuf1 = c->p1;
  a.x = c->x;
  a.z = c->z;
  return a;
}

// ------------------------------------------------------------------ timed launch wrappers
static cudaEvent_t ev_get(sb_ctx* c) {
  if (c->evnext >= c->evpool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->evpool.push_back(e);
  }
  return c->evpool[c->evnext++];
}

static sb_status run_k1(sb_ctx* c, int mode, const K1Args& a, cudaStream_t st) {
  int e0 = -1;
  if (c->timing) {
    CK(launch_spin(st, 20000));  // start event after the kernel is queued (no submission latency)
    e0 = (int)c->evnext;
    CK(cudaEventRecord(ev_get(c), st));
  }
  CK(launch_k1(mode, a, &c->tmap, c->W, c->G, st));
  if (c->timing) {
    int e1 = (int)c->evnext;
    CK(cudaEventRecord(ev_get(c), st));
    c->evpend.push_back({0, {e0, e1}});
  }
  c->launches++;
  return SB_OK;
}

static sb_status run_kp(sb_ctx* c, int mode, const KPArgs& a, cudaStream_t st) {
  const bool timed = c->timing && (mode == KP_APPLY || mode == KP_PCG || mode == KP_RESID);
  int e0 = -1;
  if (timed) {
    CK(launch_spin(st, 20000));  // start event after the kernel is queued (no submission latency)
    e0 = (int)c->evnext;
    CK(cudaEventRecord(ev_get(c), st));
  }
  CK(c->ndim == 3 ? launch_kp3(mode, a, st) : launch_kp2(mode, a, st));
  if (timed) {
    int e1 = (int)c->evnext;
    CK(cudaEventRecord(ev_get(c), st));
    c->evpend.push_back({0, {e0, e1}});
  }
  c->launches++;
  return SB_OK;
}

static sb_status run_pass(sb_ctx* c, int kind, const PassArgs& a, cudaStream_t st) {
  CK(launch_pass(kind, a, st));
  c->launches++;
  return SB_OK;
}

static void timing_collect(sb_ctx* c) {
  for (auto& pe : c->evpend) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->evpool[pe.second.first], c->evpool[pe.second.second]) == cudaSuccess) {
      c->t_ms[pe.first] += ms;
      c->t_n[pe.first] += 1;
    }
  }
  cudaGetLastError();
  c->evpend.clear();
  c->evnext = 0;
}

// Stage timers of sb_recon_log (SB_STAGE_*): an event pair around each stage on the context
// stream (eager execution only); summed after the call's final synchronisation.
enum { ST_RHS = 0, ST_PCG = 1, ST_SHRINK = 2, ST_FEEDBACK = 3, ST_INIT = 4 };
static cudaEvent_t stage_event(sb_ctx* c) {
  if (c->stage_next >= c->stage_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    c->stage_pool.push_back(e);
  }
  return c->stage_pool[c->stage_next++];
}
struct StageMark {  // records the start event; close() the end event
  sb_ctx* c;
  int stage;
  cudaEvent_t e0 = nullptr;
  cudaStream_t st;
  StageMark(sb_ctx* cc, int sg, cudaStream_t s_) : c(cc), stage(sg), st(s_) {
    if (c->stage_timing) {
      e0 = stage_event(c);
      cudaEventRecord(e0, st);
    }
  }
  void close() {
    if (e0) {
      cudaEvent_t e1 = stage_event(c);
      cudaEventRecord(e1, st);
      c->stage_ev.push_back({stage, {e0, e1}});
      e0 = nullptr;
    }
  }
};
static void stage_collect(sb_ctx* c) {
  for (auto& se : c->stage_ev) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, se.second.first, se.second.second) == cudaSuccess) c->stage_s[se.first] += 1e-3 * ms;
  }
  cudaGetLastError();
  c->stage_ev.clear();
  c->stage_next = 0;
}

static sb_status allreduce(sb_ctx* c, void* buf, size_t count, int dtype, cudaStream_t st) {
  const int r = g_nccl.allReduce(buf, buf, count, dtype, NCCL_SUM, c->comm->comm, st);
  if (r != 0)
    return fail(c, SB_E_COMM, std::string("ncclAllReduce: ") + (g_nccl.getErrorString ? g_nccl.getErrorString(r) : "?"));
  return SB_OK;
}

// Coil-sharded matvec: the plane kernel up to the partial coil sum, in plane chunks on the
// context stream; each chunk's NCCL all-reduce runs on the comm stream as soon as the chunk is
// written (event dependency), so the reduction of chunk k overlaps the transforms of chunk k+1;
// then the epilogue.  The fork/join through events also captures into CUDA graphs.
static sb_status run_kp_sharded(sb_ctx* c, int mode, KPArgs k, cudaStream_t st) {
  k.acc_out = c->accbuf;
  const int planes = k.planes;
  const int nch = std::max(1, std::min(std::min(c->coil_chunks, 16), planes));
  sb_status s;
  for (int ch = 0; ch < nch; ++ch) {
    const int p0 = (int)((int64_t)planes * ch / nch), p1 = (int)((int64_t)planes * (ch + 1) / nch);
    if (p1 <= p0) continue;
    KPArgs kc = k;
    kc.plane0 = p0;
    kc.nplanes = p1 - p0;
    if ((s = run_kp(c, mode, kc, st))) return s;
    CK(cudaEventRecord(c->chunk_ev[ch], st));
    CK(cudaStreamWaitEvent(c->cst, c->chunk_ev[ch], 0));
    const size_t pn = (size_t)k.NY * k.NZ;
    for (int b = 0; b < c->B; ++b) {
      float2* base = c->accbuf + (size_t)b * c->img + (size_t)p0 * pn;
      if ((s = allreduce(c, base, 2 * (size_t)(p1 - p0) * pn, NCCL_FLOAT32, c->cst))) return s;
    }
  }
  CK(cudaEventRecord(c->red_done, c->cst));
  CK(cudaStreamWaitEvent(st, c->red_done, 0));
  k.acc_out = nullptr;
  k.acc_in = c->accbuf;
  CK(launch_kc_epilogue(mode, k, st));
  c->launches++;
  return SB_OK;
}

// ------------------------------------------------------------------ kernel sequences
// q = A v (generic or separable)
static sb_status seq_apply(sb_ctx* c, const float2* v, float2* out, cudaStream_t st) {
  if (c->plane) {
    KPArgs k = base_kp(c);
    k.vin = v;
    k.out = out;
    return c->comm ? run_kp_sharded(c, KP_APPLY, k, st) : run_kp(c, KP_APPLY, k, st);
  }
  K1Args a = base_k1(c);
  a.vin = v;
  a.out = out;
  return run_k1(c, K1_APPLY, a, st);
}

// r0 = b - A x (+ recon RHS/feedback), fin_init
static sb_status seq_resid(sb_ctx* c, Loop L, const float2* bgiven, bool recon, bool update_u, bool use_rhs,
                           float eps, int maxit, cudaStream_t st) {
  if (c->plane) {
    KPArgs k = base_kp(c);
    k.vin = c->x;
    k.out = c->r;
    k.bvec = recon ? nullptr : bgiven;
    k.u = c->u;
    k.u1 = c->u1;
    k.rhs_reg = use_rhs ? c->rhs : nullptr;
    k.bout = c->bvec;
    k.update_u = update_u ? 1 : 0;
    k.eps = eps;
    k.maxit = maxit;
    k.L = L;
    return c->comm ? run_kp_sharded(c, KP_RESID, k, st) : run_kp(c, KP_RESID, k, st);
  }
  K1Args a = base_k1(c);
  a.vin = c->x;
  a.out = c->r;
  a.bvec = recon ? nullptr : bgiven;
  a.u = c->u;
  a.u1 = c->u1;
  a.rhs_reg = use_rhs ? c->rhs : nullptr;
  a.bout = c->bvec;
  a.update_u = update_u ? 1 : 0;
  a.eps = eps;
  a.maxit = maxit;
  a.L = L;
  a.spec = c->spec_on ? 1 : 0;  // r0 leaves as its column spectrum S_r = F_0 r0
  return run_k1(c, K1_RESID, a, st);
}

// z = M^{-1} r ; mode 0 = PCG init (rho_0), 1 = PCG iteration (r -= alpha q first),
// -1 = standalone apply (no scalars)
static sb_status seq_precond(sb_ctx* c, Loop L, int precond, int mode, const float2* rin, float2* zout,
                             cudaStream_t st) {
  PassArgs pa = base_pass(c);
  pa.L = L;
  pa.mode = mode;
  sb_status s;
  if (precond == 0 || precond == 2) {  // none, or Jacobi z = r / diag(A)
    pa.a0 = c->r;
    pa.a1 = c->q;
    pa.o0 = c->r;
    pa.o1 = c->z;
    pa.jinv = precond == 2 ? c->jinv : nullptr;
    return run_pass(c, P_NOPRE, pa, st);
  }
  if (c->spec_on && mode >= 0) {
    // spectral residual: K1 left S_r = F_0 r0 (RESID) / Q = F_0 q (PCG) in r / q;
    // one row pass (S_r -= alpha Q, F_1^H Lambda^{-1} F_1, ||r||^2 and <r, z> from the spectra)
    // and one column pass (z = F_0^H T)
    pa.a0 = c->r;
    pa.a1 = c->q;
    pa.o0 = c->r;
    pa.tmp = c->tmp;
    if ((s = run_pass(c, P_PRE_B_SPEC, pa, st))) return s;
    pa.o0 = zout;
    return run_pass(c, P_PRE_C_SPEC, pa, st);
  }
  if (c->pre2d) {  // one cluster kernel: r -= alpha q, ||r||^2, z = F^H Lambda^{-1} F r, <r, z>
    KPArgs k = base_kp(c);
    k.vin = rin;
    k.qv = c->q;
    k.rout = c->r;
    k.zout = zout;
    k.pmode = mode;
    k.L = L;
    return run_kp(c, KP_PRE2D, k, st);
  }
  pa.a0 = rin;
  pa.a1 = c->q;
  pa.o0 = c->r;
  pa.tmp = c->tmp;
  if ((s = run_pass(c, P_PRE_A_FWD_COL, pa, st))) return s;
  if (c->ndim == 3) {  // d0 FFT (pass A) -> plane FFT x Lambda^{-1} x plane IFFT -> d0 IFFT (pass C)
    KPArgs k = base_kp(c);
    k.tmp = c->tmp;
    k.L = L;
    if ((s = run_kp(c, KP_PRECOND, k, st))) return s;
  } else if ((s = run_pass(c, P_PRE_B_ROW, pa, st))) {
    return s;
  }
  pa.a0 = (mode >= 0) ? c->r : nullptr;
  pa.o0 = zout;
  return run_pass(c, P_PRE_C_INV_COL, pa, st);
}

static sb_status seq_body(sb_ctx* c, Loop L, int precond, cudaStream_t st, int* nk) {
  int n0 = (int)c->launches;
  sb_status s;
  if (c->plane) {
    KPArgs k = base_kp(c);
    k.out = c->q;
    k.L = L;
    if ((s = c->comm ? run_kp_sharded(c, KP_PCG, k, st) : run_kp(c, KP_PCG, k, st))) return s;
    if ((s = seq_precond(c, L, precond, 1, c->r, c->z, st))) return s;
    if (nk) *nk = (int)c->launches - n0;
    return SB_OK;
  }
  K1Args a = base_k1(c);
  a.z = c->z;
  a.pbuf0 = c->p0;
  a.pbuf1 = c->p1;
  a.x = c->x;
  a.out = c->q;
  a.L = L;
  a.spec = c->spec_on ? 1 : 0;  // q leaves as its column spectrum Q = F_0 q
  if ((s = run_k1(c, K1_PCG, a, st))) return s;
  if ((s = seq_precond(c, L, precond, 1, c->r, c->z, st))) return s;
  if (nk) *nk = (int)c->launches - n0;
  return SB_OK;
}

static sb_status seq_post(sb_ctx* c, Loop L, cudaStream_t st) {
  PassArgs pa = base_pass(c);
  pa.L = L;
  sb_status s;
  if ((s = run_pass(c, P_FIXUP, pa, st))) return s;
  CK(launch_log(L, st));
  c->launches++;
  return SB_OK;
}

static sb_status seq_shrink(sb_ctx* c, int par, cudaStream_t st) {
  SbArgs a;
  memset(&a, 0, sizeof(a));
  const bool d4 = c->wavelet == 1;
  a.B = c->B;
  a.M = c->M;
  a.N = c->N;
  a.levels = c->L;
  a.lam = c->lam;
  a.gam = d4 ? 0.f : c->gam;  // D4: the TV kernel writes the TV part only; k_wav.cu adds gamma W^H(.)
  a.x = c->x;
  a.bx_in = c->bx[par];
  a.by_in = c->by[par];
  a.bx_out = c->bx[1 - par];
  a.by_out = c->by[1 - par];
  a.bw = c->bw;
  a.rhs = c->rhs;
  if (c->ndim == 3) {
    a.M = c->D0;
    a.N = c->D1;
    a.D2 = c->D2;
    a.bz_in = c->bz[par];
    a.bz_out = c->bz[1 - par];
    CK(launch_sb_update3(a, st));
    c->launches++;
  } else {
    CK(launch_sb_update(a, st));
  }
  if (d4 && c->gam != 0.f) {
    int nl = 0;
    CK(launch_d4_sb(c->x, c->wbuf, c->bw, c->rhs, c->B, c->D0, c->ndim == 3 ? c->D1 : c->N, c->ndim == 3 ? c->D2 : 1,
                    c->ndim, c->L, c->gam, st, &nl));
    c->launches += nl;
  }
  if (c->ndim == 3 || d4) return SB_OK;
  c->launches++;
  return SB_OK;
}

// 3D adjoint: d0 IFFT of every coil's k-space (column pass), then per plane the masked plane
// IFFT, conj(s_c) combine and (optionally) the root sum of squares (K1P adjoint mode).
static sb_status seq_adjoint3(sb_ctx* c, const float2* ydev, float2* xout, float2* rssout, cudaStream_t st) {
  PassArgs pa = base_pass(c);
  pa.a0 = ydev;
  pa.o0 = c->tmpc;
  pa.scale = 1.0f;
  sb_status s;
  if ((s = run_pass(c, P_COL_INV, pa, st))) return s;
  KPArgs k = base_kp(c);
  k.tmp = c->tmpc;
  k.out = xout;
  k.out2 = rssout;
  k.rss_raw = c->comm ? 1 : 0;
  k.scale = 1.0f / std::sqrt((float)c->img);
  if ((s = run_kp(c, KP_ADJOINT, k, st))) return s;
  if (c->comm) {  // sum over all ranks' coils
    const size_t n = (size_t)c->B * c->img;
    if ((s = allreduce(c, xout, 2 * n, NCCL_FLOAT32, st))) return s;
    if (rssout) {
      if ((s = allreduce(c, rssout, 2 * n, NCCL_FLOAT32, st))) return s;
      CK(launch_kc_sqrt_re(rssout, n, st));
      c->launches++;
    }
  }
  return SB_OK;
}

static sb_status seq_init_recon(sb_ctx* c, const float2* ydev, cudaStream_t st) {
  if (c->ndim == 3) {
    sb_status s = seq_adjoint3(c, ydev, c->u1, c->x, st);
    if (s) return s;
    CK(cudaMemcpyAsync(c->u, c->u1, c->img * c->B * sizeof(float2), cudaMemcpyDeviceToDevice, st));
    return SB_OK;
  }
  PassArgs pa = base_pass(c);
  pa.a0 = ydev;
  pa.tmp = c->tmpc;
  pa.o0 = c->u1;
  pa.o1 = c->x;
  pa.scale = 1.0f / std::sqrt((float)c->img);
  pa.full = 0;
  sb_status s;
  if ((s = run_pass(c, P_ADJ_ROW, pa, st))) return s;
  if ((s = run_pass(c, P_ADJ_COL, pa, st))) return s;
  CK(cudaMemcpyAsync(c->u, c->u1, c->img * c->B * sizeof(float2), cudaMemcpyDeviceToDevice, st));
  return SB_OK;
}

// ------------------------------------------------------------------ graph building
// kind: 0 solve (b in c->bvec), 1 recon first outer, 2/3 recon next outer (b-parity 0/1)
static sb_status build_graph(sb_ctx* c, int kind, const sb_pcg_opts* o, const float2* ydev) {
  GraphSlot& g = c->gs[kind];
  if (g.exec && g.eps == o->eps && g.maxit == o->max_iters && g.precond == o->precond) return SB_OK;
  if (g.exec) {
    cudaGraphExecDestroy(g.exec);
    cudaGraphDestroy(g.graph);
    g.exec = nullptr;
  }
  cudaGraph_t G;
  CK(cudaGraphCreate(&G, 0));
  cudaGraphConditionalHandle h = 0;
  CK(cudaGraphConditionalHandleCreate(&h, G, 0, 0));
  Loop L = make_loop(c, (unsigned long long)h);
  cudaStream_t cs = c->cap1;
  int64_t l0 = c->launches;
  bool saved_timing = c->timing;
  c->timing = false;
  struct PdlGuard {
    bool old;
    PdlGuard(bool v) : old(g_use_pdl) { g_use_pdl = v; }
    ~PdlGuard() { g_use_pdl = old; }
  } pdl_guard(env_flag("SBPCG_GRAPH_PDL", false));
  CK(cudaStreamBeginCaptureToGraph(cs, G, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  sb_status s = SB_OK;
  if (kind == 0) {
    s = seq_resid(c, L, c->bvec, false, false, false, o->eps, o->max_iters, cs);
  } else if (kind == 1) {
    s = seq_init_recon(c, ydev, cs);
    if (!s) s = seq_resid(c, L, nullptr, true, false, false, o->eps, o->max_iters, cs);
  } else {
    const int par = kind - 2;
    s = seq_shrink(c, par, cs);
    if (!s) s = seq_resid(c, L, nullptr, true, true, true, o->eps, o->max_iters, cs);
  }
  if (!s) s = seq_precond(c, L, o->precond, 0, c->r, c->z, cs);
  if (s) {
    cudaGraph_t dummy;
    cudaStreamEndCapture(cs, &dummy);
    c->timing = saved_timing;
    return s;
  }
  cudaStreamCaptureStatus cst;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  CK(cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &deps, &ndeps));
  alignas(cudaGraphNodeParams) unsigned char cpbuf[sizeof(cudaGraphNodeParams)];
  memset(cpbuf, 0, sizeof(cpbuf));
  cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(cpbuf);
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode;
  CK(cudaGraphAddNode(&cnode, G, deps, ndeps, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies));
  const int64_t lb = c->launches;
  CK(cudaStreamBeginCaptureToGraph(c->cap2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  int nk = 0;
  // U iterations per evaluation of the while condition (SBPCG_UNROLL, default 1): a problem
  // that converges inside the group is frozen, so the extra kernels exit at once
  const int U = std::max(1, std::min(8, getenv("SBPCG_UNROLL") ? atoi(getenv("SBPCG_UNROLL")) : 1));
  for (int u = 0; u < U && !s; ++u) s = seq_body(c, L, o->precond, c->cap2, &nk);
  g.unroll = U;
  cudaGraph_t bodyout;
  cudaError_t e2 = cudaStreamEndCapture(c->cap2, &bodyout);
  if (s || e2 != cudaSuccess) {
    cudaGraph_t dummy;
    cudaStreamEndCapture(cs, &dummy);
    c->timing = saved_timing;
    if (s) return s;
    CK(e2);
  }
  const int64_t la = c->launches;
  s = seq_post(c, L, cs);
  cudaGraph_t Gout;
  cudaError_t e3 = cudaStreamEndCapture(cs, &Gout);
  c->timing = saved_timing;
  if (s) return s;
  CK(e3);
  CK(cudaGraphInstantiate(&g.exec, G, 0));
  g.graph = G;
  g.nbody = (int)(la - lb);
  g.nfixed = (int)((lb - l0) + (c->launches - la));
  c->launches = l0;  // capture does not launch
  g.eps = o->eps;
  g.maxit = o->max_iters;
  g.precond = o->precond;
  return SB_OK;
}

// eager (non-graph) execution of one solve whose prelude kind is given
static sb_status eager_solve(sb_ctx* c, int kind, const sb_pcg_opts* o, const float2* ydev) {
  Loop L = make_loop(c, 0ull);
  g_use_pdl = env_flag("SBPCG_EAGER_PDL", true);
  sb_status s;
  cudaStream_t st = c->st;
  // stage timers: the RESID kernel forms the RHS (step 4), the data feedback (steps 13-15) and
  // r0 in one pass, so its time is reported as rhs_s (feedback_s stays 0: fused)
  if (kind == 0) {
    StageMark m(c, ST_RHS, st);
    s = seq_resid(c, L, c->bvec, false, false, false, o->eps, o->max_iters, st);
    m.close();
  } else if (kind == 1) {
    StageMark m0(c, ST_INIT, st);
    s = seq_init_recon(c, ydev, st);
    m0.close();
    StageMark m1(c, ST_RHS, st);
    if (!s) s = seq_resid(c, L, nullptr, true, false, false, o->eps, o->max_iters, st);
    m1.close();
  } else {
    StageMark m0(c, ST_SHRINK, st);
    s = seq_shrink(c, kind - 2, st);
    m0.close();
    StageMark m1(c, ST_RHS, st);
    if (!s) s = seq_resid(c, L, nullptr, true, true, true, o->eps, o->max_iters, st);
    m1.close();
  }
  if (s) return s;
  StageMark mp(c, ST_PCG, st);
  struct Closer {
    StageMark& m;
    ~Closer() { m.close(); }
  } closer{mp};
  if ((s = seq_precond(c, L, o->precond, 0, c->r, c->z, st))) return s;
  int host_any = 1;
  CK(cudaMemcpyAsync(&host_any, &c->ctl->any_active, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  while (host_any) {
    if ((s = seq_body(c, L, o->precond, st, nullptr))) return s;
    CK(cudaMemcpyAsync(&host_any, &c->ctl->any_active, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  return seq_post(c, L, st);
}

// Coil-sharded mode in CUDA graphs (the NCCL all-reduces and the comm-stream fork/join are
// captured): [prelude] once, then [U PCG iterations] per launch with one host check of the
// "any problem active" flag between launches (a conditional node cannot hold the NCCL work),
// then [fixup + log].  Every rank sees the same flags (bitwise identical replicated scalars), so
// every rank launches the same collectives.
static void coil_graphs_drop(sb_ctx* c) {
  for (auto& row : c->coil_exec)
    for (auto& e : row)
      if (e) {
        cudaGraphExecDestroy(e);
        e = nullptr;
      }
  for (auto& row : c->coil_graph)
    for (auto& g : row)
      if (g) {
        cudaGraphDestroy(g);
        g = nullptr;
      }
  c->coil_maxit = -1;
}

template <typename F>
static sb_status capture(sb_ctx* c, F&& body, cudaGraph_t* g, cudaGraphExec_t* e) {
  cudaStream_t cs = c->cap1;
  CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  sb_status s = body(cs);
  cudaGraph_t gr = nullptr;
  cudaError_t ec = cudaStreamEndCapture(cs, &gr);
  if (s) {
    if (gr) cudaGraphDestroy(gr);
    return s;
  }
  CK(ec);
  CK(cudaGraphInstantiate(e, gr, 0));
  *g = gr;
  return SB_OK;
}

static sb_status coil_graph_solve(sb_ctx* c, int kind, const sb_pcg_opts* o, const float2* ydev) {
  if (c->coil_eps != o->eps || c->coil_maxit != o->max_iters || c->coil_pre != o->precond) {
    coil_graphs_drop(c);
    c->coil_eps = o->eps;
    c->coil_maxit = o->max_iters;
    c->coil_pre = o->precond;
  }
  const bool saved_timing = c->timing;
  c->timing = false;
  struct PdlGuard {
    bool old;
    PdlGuard() : old(g_use_pdl) { g_use_pdl = false; }
    ~PdlGuard() { g_use_pdl = old; }
  } pdl_guard;
  Loop L = make_loop(c, 0ull);
  sb_status s = SB_OK;
  const int64_t l0 = c->launches;
  int n_pre = 0, n_body = 0, n_post = 0;
  if (!c->coil_exec[kind][0]) {
    s = capture(c, [&](cudaStream_t cs) -> sb_status {
      sb_status r;
      if (kind == 0) {
        r = seq_resid(c, L, c->bvec, false, false, false, o->eps, o->max_iters, cs);
      } else if (kind == 1) {
        r = seq_init_recon(c, ydev, cs);
        if (!r) r = seq_resid(c, L, nullptr, true, false, false, o->eps, o->max_iters, cs);
      } else {
        r = seq_shrink(c, kind - 2, cs);
        if (!r) r = seq_resid(c, L, nullptr, true, true, true, o->eps, o->max_iters, cs);
      }
      if (!r) r = seq_precond(c, L, o->precond, 0, c->r, c->z, cs);
      return r;
    }, &c->coil_graph[kind][0], &c->coil_exec[kind][0]);
    if (!s)
      s = capture(c, [&](cudaStream_t cs) -> sb_status {
        for (int u = 0; u < c->coil_unroll; ++u) {
          sb_status r = seq_body(c, L, o->precond, cs, nullptr);
          if (r) return r;
        }
        return SB_OK;
      }, &c->coil_graph[kind][1], &c->coil_exec[kind][1]);
    if (!s)
      s = capture(c, [&](cudaStream_t cs) -> sb_status { return seq_post(c, L, cs); }, &c->coil_graph[kind][2],
                  &c->coil_exec[kind][2]);
  }
  (void)n_pre, (void)n_body, (void)n_post;
  c->launches = l0;  // capture does not launch
  c->timing = saved_timing;
  if (s) {
    coil_graphs_drop(c);
    return s;
  }
  auto kernel_nodes = [](cudaGraph_t g) -> int64_t {
    size_t n = 0;
    if (cudaGraphGetNodes(g, nullptr, &n) != cudaSuccess) return 0;
    std::vector<cudaGraphNode_t> nodes(n);
    if (n == 0 || cudaGraphGetNodes(g, nodes.data(), &n) != cudaSuccess) return 0;
    int64_t k = 0;
    for (auto nd : nodes) {
      cudaGraphNodeType t;
      if (cudaGraphNodeGetType(nd, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
    }
    return k;
  };
  int64_t nn = kernel_nodes(c->coil_graph[kind][0]);
  c->launches += nn;
  CK(cudaGraphLaunch(c->coil_exec[kind][0], c->st));
  int host_any = 1;
  CK(cudaMemcpyAsync(&host_any, &c->ctl->any_active, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  nn = kernel_nodes(c->coil_graph[kind][1]);
  while (host_any) {
    CK(cudaGraphLaunch(c->coil_exec[kind][1], c->st));
    c->launches += nn;
    CK(cudaMemcpyAsync(&host_any, &c->ctl->any_active, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
  }
  nn = kernel_nodes(c->coil_graph[kind][2]);
  c->launches += nn;
  CK(cudaGraphLaunch(c->coil_exec[kind][2], c->st));
  c->last_path = SB_PATH_COIL_SHARDED;
  return SB_OK;
}

static sb_status run_solve_kind(sb_ctx* c, int kind, const sb_pcg_opts* o, const float2* ydev) {
  c->spec_on = c->spec_ok && o->precond == 1;
  if (c->comm && o->use_graph && !c->timing && !c->stage_timing) return coil_graph_solve(c, kind, o, ydev);
  // coil-sharded mode runs the host-driven loop; stage timers need the eager sequence
  if (o->use_graph && !c->timing && !c->comm && !c->stage_timing) {
    sb_status s = build_graph(c, kind, o, ydev);
    if (s) return s;
    CK(cudaGraphLaunch(c->gs[kind].exec, c->st));
    c->last_path = SB_PATH_GRAPH;
    return SB_OK;
  }
  c->last_path = c->comm ? SB_PATH_COIL_SHARDED : SB_PATH_EAGER;
  return eager_solve(c, kind, o, ydev);
}

// ------------------------------------------------------------------ persistent kernel (KR)
static bool use_kr(sb_ctx* c, const sb_pcg_opts* o) {
  return c->kr_ok && c->kr_on && o->precond == 1 && c->wavelet == 0 && !c->comm;
}

// One cooperative launch: n_outer = 0 solves A x = b (b in c->bvec, x0 in c->x); n_outer >= 1
// runs the SB reconstruction after the init (u1, u, x = RSS already in place).
static sb_status run_kr(sb_ctx* c, int n_outer, const sb_pcg_opts* o, int par0) {
  KrArgs a;
  memset(&a, 0, sizeof(a));
  a.B = c->B;
  a.C = c->C;
  a.M = c->M;
  a.N = c->N;
  a.levels = c->L;
  a.mu = c->mu;
  a.lam = c->lam;
  a.gam = c->gam;
  a.sT = c->sT;
  a.rmask = c->rowmask;
  a.rmask_bstride = c->mask_shared ? 0 : c->M;
  a.lam_inv = c->lam_inv;
  a.tw = c->tw_m;
  a.x = c->x;
  a.bvec = c->bvec;
  a.u = c->u;
  a.u1 = c->u1;
  a.rhs = c->rhs;
  a.xT = c->z;  // free on the persistent path
  a.kinit = (n_outer > 0 && c->kr_y != nullptr) ? 1 : 0;
  a.y = c->kr_y;
  a.y1T = c->tmpc;
  a.sb.B = c->B;
  a.sb.M = c->M;
  a.sb.N = c->N;
  a.sb.levels = c->L;
  a.sb.lam = c->lam;
  a.sb.gam = c->gam;
  a.sb.x = c->x;
  a.sb.bw = c->bw;
  a.sb.rhs = c->rhs;
  for (int k = 0; k < 2; ++k) {
    a.bxs[k] = c->bx[(k + par0) & 1];
    a.bys[k] = c->by[(k + par0) & 1];
  }
  a.Qs = c->q;
  a.Sr = c->r;
  a.Tb = c->tmp;
  a.part = c->P.p0;
  a.bar = c->kbar;
  a.stamp = c->kstamp;
  a.prof = getenv("SBPCG_KR_PROF") ? atoi(getenv("SBPCG_KR_PROF")) : 0;
  a.cg = c->kr_cg ? 1 : 0;
  a.L = make_loop(c, 0ull);
  a.n_outer = n_outer;
  a.eps = o->eps;
  a.maxit = o->max_iters;
  CK(cudaMemsetAsync(c->kbar, 0, sizeof(unsigned) * c->B, c->st));
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->timing) {
    CK(launch_spin(c->st, 20000));
    e0 = ev_get(c);
    CK(cudaEventRecord(e0, c->st));
  }
  {
    const cudaError_t e = launch_kr(a, c->st);
    if (e == cudaErrorCooperativeLaunchTooLarge || e == cudaErrorLaunchOutOfResources) {
      // the problems do not fit one cooperative launch on this device after all (the limit was
      // estimated at create): drop the persistent path for this context; the caller re-runs the
      // call on the kernel sequence (no work of this launch has been enqueued)
      cudaGetLastError();
      c->kr_ok = false;
      c->err = std::string("persistent kernel not launchable, using the kernel sequence: ") + cudaGetErrorString(e);
      return SB_E_UNSUPPORTED_SIZE;
    }
    CK(e);
  }
  c->launches++;
  if (c->timing) {
    e1 = ev_get(c);
    CK(cudaEventRecord(e1, c->st));
    c->evpend.push_back({2, {(int)c->evnext - 2, (int)c->evnext - 1}});
  }
  c->last_path = SB_PATH_PERSISTENT;
  return SB_OK;
}

// algorithmic bytes of one persistent launch: B_iter per PCG
// iteration, plus the solve prelude and the SB step per problem and solve
static double kr_bytes(sb_ctx* c, const std::vector<int32_t>& iters, int n_solves, bool sb) {
  const double N = (double)c->img, C = (double)c->C, M = (double)c->M;
  const double b_iter = 8.0 * N * (C + 10.0) + 4.0 * N + 4.0 * M;
  const double b_pre = 8.0 * N * C + 84.0 * N + 4.0 * M;
  const double b_sb = 64.0 * N;
  double it = 0;
  for (int32_t v : iters) it += v;
  return it * b_iter + (double)n_solves * c->B * (b_pre + (sb ? b_sb : 0.0));
}

// ------------------------------------------------------------------ Lambda build
static sb_status build_lambda3(sb_ctx* c);
static sb_status finish_lambda(sb_ctx* c, void* tmp, void* g, void* rh, int* bad, void* kc2);

// Persistent Lambda-build scratch (allocated on the first build, reused by every rebuild so
// that sb_pcg_build_precond does no cudaMalloc/cudaFree: those block the host).
template <typename T>
static cudaError_t lscratch(sb_ctx* c, int slot, T** p, size_t n) {
  const size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
  if (c->lscr_bytes[slot] < bytes) {
    if (c->lscr[slot]) cudaFree(c->lscr[slot]);
    c->lscr[slot] = nullptr;
    c->lscr_bytes[slot] = 0;
    cudaError_t e = cudaMalloc(&c->lscr[slot], bytes);
    if (e != cudaSuccess) return e;
    c->lscr_bytes[slot] = bytes;
  }
  *p = (T*)c->lscr[slot];
  return cudaSuccess;
}

static sb_status build_lambda_impl(sb_ctx* c);
// Lambda build timed with an event pair (sb_recon_log.build_s; Table 2 analogue).
static sb_status build_lambda(sb_ctx* c) {
  if (!c->bev[0]) {
    CK(cudaEventCreate(&c->bev[0]));
    CK(cudaEventCreate(&c->bev[1]));
  }
  if (!c->bad_host) CK(cudaMallocHost(&c->bad_host, sizeof(int)));
  CK(cudaEventRecord(c->bev[0], c->st));
  sb_status s = build_lambda_impl(c);
  if (s) return s;
  CK(cudaEventRecord(c->bev[1], c->st));
  c->build_check = true;  // no host synchronisation: the next solve / recon overlaps its enqueue
  return SB_OK;
}

// After a stream synchronisation: the last Lambda build's time (sb_recon_log.build_s) and its
// singular-k flag (SB_E_SINGULAR_K is reported by the first synchronising call after the build).
static sb_status build_checked(sb_ctx* c) {
  if (!c->build_check) return SB_OK;
  c->build_check = false;
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, c->bev[0], c->bev[1]) == cudaSuccess) c->build_s = 1e-3 * ms;
  cudaGetLastError();
  if (*c->bad_host) return fail(c, SB_E_SINGULAR_K, "singular k (min |k| <= 1e-14 or non-finite)");
  return SB_OK;
}

static sb_status build_lambda_impl(sb_ctx* c) {
  if (c->ndim == 3) return build_lambda3(c);
  LamArgs a;
  memset(&a, 0, sizeof(a));
  a.B = c->B;
  a.C = c->C;
  a.M = c->M;
  a.N = c->N;
  a.mu = c->mu;
  a.lam = c->lam;
  a.gam = c->gam;
  a.sens = c->sens;
  a.mask = c->mask;
  a.mask_bstride = c->mask_shared ? 0 : (int)c->img;
  a.nmask = c->mask_shared ? 1 : c->B;
  a.nsens = c->B;
  a.k_out = c->kbuf;
  a.lam_inv = c->lam_inv;
  a.tw_m = c->twd_m;
  a.tw_n = c->twd_n;
  double2 *tmp = nullptr, *g = nullptr, *rh = nullptr;
  int* bad = nullptr;
  if (c->separable && env_flag("SBPCG_LSEP", true)) {
    // line masks: the one-dimensional form (k_lambda.cu K4S), three launches.  Coil groups
    // split the column pass when the batch alone leaves SMs idle.
    const int nct = c->N / 8;
    int S = std::max(1, std::min(c->C, (2 * 148 + c->B * nct - 1) / (c->B * nct)));
    const int per = (c->C + S - 1) / S;
    S = (c->C + per - 1) / per;
    double* gpart = nullptr;
    CK(lscratch(c, 3, &bad, 1));
    CK(lscratch(c, 1, &g, (size_t)c->B * c->M));
    CK(lscratch(c, 5, &gpart, (size_t)c->B * S * nct * c->M));
    CK(cudaMemsetAsync(bad, 0, sizeof(int), c->st));
    a.bad = bad;
    a.csplit = S;
    a.gpart = gpart;
    a.g = g;
    CK(launch_lambda_sep(a, c->st));
    c->launches += 3;
    return finish_lambda(c, nullptr, nullptr, nullptr, bad, nullptr);
  }
  CK(lscratch(c, 0, &tmp, (size_t)c->B * c->C * c->img));
  CK(lscratch(c, 1, &g, (size_t)c->B * c->img));
  CK(lscratch(c, 2, &rh, (size_t)a.nmask * c->img));
  CK(lscratch(c, 3, &bad, 1));
  double* gpart = nullptr;  // split the coil pass over coil groups only for small batches
  if (c->B * 32 < 2 * 148) CK(lscratch(c, 5, &gpart, (size_t)c->B * std::min(c->C, 16) * c->img));
  CK(cudaMemsetAsync(bad, 0, sizeof(int), c->st));
  a.tmp = tmp;
  a.g = g;
  a.rhat = rh;
  a.bad = bad;
  a.gpart = gpart;
  int extra = 0;
  a.nextra = &extra;
  CK(launch_lambda_build(a, c->st));
  c->launches += 8 + extra;
  return finish_lambda(c, tmp, g, rh, bad, nullptr);
}

// 3D (mask constant along d0): with F_3 = F_0 (x) F_12 and Parseval along d0,
//   sum_{q0} g(q0, q) = D0 sum_c sum_x |D_12 s_c(x)|^2 (q) / N^2,
// and k_c is constant along nu_0 and equals the 2D correlation of that marginal with the
// plane mask.  The planes of every coil are fed to the 2D build
// as extra "coils" in chunks (g accumulates), then k / Lambda^{-1} are expanded to 3D.
static sb_status build_lambda3(sb_ctx* c) {
  const size_t pn = (size_t)c->D1 * c->D2;
  const int nplanes = c->C * c->D0;  // per problem
  const int chunk = (int)std::max<size_t>(1, std::min<size_t>((size_t)nplanes, (size_t)(64u << 20) / (pn * 16)));
  LamArgs a;
  memset(&a, 0, sizeof(a));
  a.M = c->D1;
  a.N = c->D2;
  a.mu = c->mu;
  a.lam = c->lam;
  a.gam = c->gam;
  a.mask_bstride = c->mask_shared ? 0 : (int)pn;
  a.nmask = c->mask_shared ? 1 : c->B;
  a.tw_m = c->twd_y;
  a.tw_n = c->twd_z;
  double2 *tmp = nullptr, *g = nullptr, *rh = nullptr;
  double* kc2 = nullptr;
  int* bad = nullptr;
  CK(lscratch(c, 0, &tmp, (size_t)chunk * pn));
  CK(lscratch(c, 1, &g, (size_t)c->B * pn));
  CK(lscratch(c, 2, &rh, (size_t)a.nmask * pn));
  CK(lscratch(c, 4, &kc2, (size_t)c->B * pn));
  CK(lscratch(c, 3, &bad, 1));
  double* gpart = nullptr;
  CK(lscratch(c, 5, &gpart, (size_t)std::min(chunk, 16) * pn));
  CK(cudaMemsetAsync(bad, 0, sizeof(int), c->st));
  a.tmp = tmp;
  a.rhat = rh;
  a.bad = bad;
  a.gpart = gpart;
  int extra = 0;
  a.nextra = &extra;
  for (int b = 0; b < c->B; ++b) {
    for (int p0 = 0; p0 < nplanes; p0 += chunk) {
      a.B = 1;
      a.C = std::min(chunk, nplanes - p0);
      a.sens = c->sens + ((size_t)b * nplanes + p0) * pn;
      a.g = g + (size_t)b * pn;
      a.accumulate = p0 > 0;
      CK(launch_lambda_chunk(a, c->st));
      c->launches += 2;
    }
  }
  if (c->comm) {  // the marginal sums over ALL coils (every rank's shard)
    sb_status s = allreduce(c, g, 2 * (size_t)c->B * pn, NCCL_FLOAT64, c->st);
    if (s) return s;
  }
  a.B = c->B;
  a.C = 1;
  a.g = g;
  a.mask = c->pmask;
  a.d3 = 1;
  a.kc2 = kc2;
  a.gpart = nullptr;
  CK(launch_lambda_tail(a, c->st));
  c->launches += 6 + extra;
  Lam3Args e;
  e.B = c->B;
  e.D0 = c->D0;
  e.D1 = c->D1;
  e.D2 = c->D2;
  e.mu = c->mu;
  e.lam = c->lam;
  e.gam = c->gam;
  e.kc2 = kc2;
  e.k_out = c->kbuf;
  e.lam_inv = c->lam_inv;
  e.bad = bad;
  CK(launch_lambda_expand3(e, c->st));
  c->launches += 1;
  return finish_lambda(c, tmp, g, rh, bad, kc2);
}

static sb_status finish_lambda(sb_ctx* c, void* tmp, void* g, void* rh, int* bad, void* kc2) {
  CK(cudaMemcpyAsync(c->bad_host, bad, sizeof(int), cudaMemcpyDeviceToHost, c->st));
  (void)tmp, (void)g, (void)rh, (void)kc2;  // persistent scratch (lscratch)
  return SB_OK;
}

// ------------------------------------------------------------------ staging helpers
static sb_status stage_in(sb_ctx* c, const void* src, size_t bytes, const void** dev, void* scratch) {
  if (is_device_ptr(src)) {
    *dev = src;
    return SB_OK;
  }
  CK(cudaMemcpyAsync(scratch, src, bytes, cudaMemcpyHostToDevice, c->st));
  *dev = scratch;
  return SB_OK;
}

static sb_status check_ready(sb_ctx* c) {
  if (!c) return SB_E_ARG;
  if (c->sticky) return c->sticky;
  return SB_OK;
}

// Pinned results block: [Scal x B][log_iters][log_relres][kstamp x 32][hist]
struct HostRes {
  Scal* scal;
  int32_t* iters;
  float* relres;
  unsigned long long* stamp;
  float* hist;
};
static sb_status host_results(sb_ctx* c, int slots, HostRes* h) {
  const size_t nb = sizeof(Scal) * c->B, nl = (size_t)slots * c->B;
  const size_t need = nb + nl * 4 * 2 + 32 * 8 + (size_t)c->B * c->hist_stride * 4 + 64;
  if (c->hres_bytes < need) {
    if (c->hres) cudaFreeHost(c->hres);
    c->hres = nullptr;
    c->hres_bytes = 0;
    CK(cudaMallocHost(&c->hres, need));
    c->hres_bytes = need;
  }
  unsigned char* q = c->hres;
  h->scal = reinterpret_cast<Scal*>(q);
  q += (nb + 15) / 16 * 16;
  h->iters = reinterpret_cast<int32_t*>(q);
  q += (nl * 4 + 15) / 16 * 16;
  h->relres = reinterpret_cast<float*>(q);
  q += (nl * 4 + 15) / 16 * 16;
  h->stamp = reinterpret_cast<unsigned long long*>(q);
  q += 32 * 8;
  h->hist = reinterpret_cast<float*>(q);
  return SB_OK;
}

static sb_status status_of(sb_ctx* c, const Scal* hs) {
  for (int b = 0; b < c->B; ++b) {
    if (hs[b].status == ST_NONFINITE) return fail(c, SB_E_NONFINITE, "non-finite PCG scalar in problem " + std::to_string(b));
    if (hs[b].status == ST_INDEFINITE) return fail(c, SB_E_INDEFINITE, "<p, A p> <= 0 in problem " + std::to_string(b));
  }
  return SB_OK;
}


// ================================================================== C ABI
extern "C" {

int32_t sb_abi_version(void) { return SBPCG_ABI_VERSION; }

const char* sb_status_str(sb_status s) {
  switch (s) {
    case SB_OK: return "SB_OK";
    case SB_E_ARG: return "SB_E_ARG";
    case SB_E_DIM: return "SB_E_DIM";
    case SB_E_UNSUPPORTED_SIZE: return "SB_E_UNSUPPORTED_SIZE";
    case SB_E_PARAM: return "SB_E_PARAM";
    case SB_E_SINGULAR_K: return "SB_E_SINGULAR_K";
    case SB_E_NONFINITE: return "SB_E_NONFINITE";
    case SB_E_INDEFINITE: return "SB_E_INDEFINITE";
    case SB_E_CUDA: return "SB_E_CUDA";
    case SB_E_NOMEM: return "SB_E_NOMEM";
    case SB_E_COMM: return "SB_E_COMM";
  }
  return "SB_E_UNKNOWN";
}

const char* sb_last_error(const sb_ctx* c) { return c ? c->err.c_str() : "null context"; }

int64_t sb_kernel_launch_count(const sb_ctx* c) { return c ? c->launches : 0; }

void sb_pcg_destroy(sb_ctx* c) {
  if (!c) return;
  cudaStreamSynchronize(c->st);
  for (auto& g : c->gs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
  }
  for (auto e : c->evpool) cudaEventDestroy(e);
  for (auto e : c->stage_pool) cudaEventDestroy(e);
  for (auto e : c->chunk_ev)
    if (e) cudaEventDestroy(e);
  if (c->red_done) cudaEventDestroy(c->red_done);
  for (auto& row : c->coil_exec)
    for (auto& e : row)
      if (e) cudaGraphExecDestroy(e);
  for (auto& row : c->coil_graph)
    for (auto& g : row)
      if (g) cudaGraphDestroy(g);
  if (c->cst) cudaStreamDestroy(c->cst);
  if (c->bad_host) cudaFreeHost(c->bad_host);
  if (c->hres) cudaFreeHost(c->hres);
  for (auto e : c->rev)
    if (e) cudaEventDestroy(e);
  for (auto e : c->bev)
    if (e) cudaEventDestroy(e);
  void* bufs[] = {c->sens, c->mask, c->rowmask, c->lam_inv, c->kbuf, c->tw_m, c->tw_n, c->twd_m, c->twd_n,
                  c->x, c->r, c->z, c->q, c->p0, c->p1, c->tmp, c->bvec, c->u, c->u1, c->rhs,
                  c->bx[0], c->bx[1], c->by[0], c->by[1], c->bw, c->tmpc, c->stage_in, c->stage_out,
                  c->scal, c->ctl, c->counters, c->P.p0, c->P.p1, c->P.cnt, c->hist, c->log_iters, c->log_relres,
                  c->pmask, c->tw_y, c->tw_z, c->twd_y, c->twd_z, c->bz[0], c->bz[1], c->accbuf, c->jinv,
                  c->wbuf, c->sT, c->kbar, c->kstamp};
  for (void* p : bufs)
    if (p) cudaFree(p);
  for (void* p : c->lscr)
    if (p) cudaFree(p);
  if (c->cap1) cudaStreamDestroy(c->cap1);
  if (c->cap2) cudaStreamDestroy(c->cap2);
  delete c;
}

sb_status sb_pcg_create(sb_ctx** out, const sb_dims* dims, int32_t coils, const uint8_t* mask, const sb_c64* sens,
                        float mu, float lambda, float gamma, void* cuda_stream, sb_comm* comm) {
  if (!out) return SB_E_ARG;
  *out = nullptr;
  if (!dims || !mask || !sens) return SB_E_ARG;
  if (dims->ndim != 2 && dims->ndim != 3) return SB_E_DIM;
  if (dims->batch < 1 || coils < 1 || dims->wavelet_levels < 0) return SB_E_DIM;
  const bool d3 = dims->ndim == 3;
  const int64_t D0 = dims->shape[0], D1 = dims->shape[1], D2 = d3 ? dims->shape[2] : 1;
  const int64_t M = D0, N = D1 * D2;  // column-pass geometry
  const int Lv = dims->wavelet_levels;
  if (!d3) {
    if (!fft_len_ok(D0) || !fft_len_ok(D1)) return SB_E_UNSUPPORTED_SIZE;
    const int TH = M < 32 ? (int)M : 32, TW = N < 32 ? (int)N : 32;
    if (Lv > 5 || (TH % (1 << Lv)) || (TW % (1 << Lv))) return SB_E_DIM;
  } else {
    if (!col3_len_ok(D0) || !kp3_supported((int)D1, (int)D2)) return SB_E_UNSUPPORTED_SIZE;
    for (int64_t d : {D0, D1, D2}) {
      const int64_t T = d < 8 ? d : 8;
      if (Lv > 3 || d % T || T % (1 << Lv)) return SB_E_DIM;
    }
  }
  // launch-grid limits: coil passes put B*C images (and K1/K1P put B problems) on grid.y/z
  if ((int64_t)dims->batch * coils > 65535 || (d3 && D0 > 65535)) return SB_E_DIM;
  if (!(gamma > 0.f) || mu < 0.f || lambda < 0.f || !std::isfinite(mu) || !std::isfinite(lambda) ||
      !std::isfinite(gamma))
    return SB_E_PARAM;
  if (comm && !d3) return SB_E_UNSUPPORTED_SIZE;  // coil sharding is the 3D mode (2D batches shard by slice)

  sb_ctx* c = new sb_ctx();
  c->st = (cudaStream_t)cuda_stream;
  cudaGetDevice(&c->dev);
  c->B = dims->batch;
  c->C = coils;
  c->M = (int)M;
  c->N = (int)N;
  c->ndim = dims->ndim;
  c->D0 = (int)D0;
  c->D1 = (int)D1;
  c->D2 = (int)D2;
  c->L = Lv;
  c->mask_shared = dims->mask_shared ? 1 : 0;
  c->mu = mu;
  c->lam = lambda;
  c->gam = gamma;
  c->img = (size_t)M * N;
  const size_t img = c->img, BN = (size_t)c->B * img, BCN = BN * c->C;
  const size_t nmask = (c->mask_shared ? 1 : c->B) * img;

  auto bail = [&](sb_status s) {
    sb_pcg_destroy(c);
    return s;
  };
  if (cudaStreamCreateWithFlags(&c->cap1, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->cap2, cudaStreamNonBlocking) != cudaSuccess)
    return bail(SB_E_CUDA);
  bool ok = true;
  ok &= dalloc(&c->sens, BCN) == cudaSuccess;
  ok &= dalloc(&c->mask, nmask) == cudaSuccess;
  ok &= dalloc(&c->rowmask, (size_t)(c->mask_shared ? 1 : c->B) * M) == cudaSuccess;
  ok &= dalloc(&c->lam_inv, BN) == cudaSuccess;
  ok &= dalloc(&c->kbuf, BN) == cudaSuccess;
  ok &= dalloc(&c->tw_m, M) == cudaSuccess && dalloc(&c->tw_n, N) == cudaSuccess;
  ok &= dalloc(&c->twd_m, M) == cudaSuccess && dalloc(&c->twd_n, N) == cudaSuccess;
  float2** vecs[] = {&c->x, &c->r, &c->z, &c->q, &c->p0, &c->p1, &c->tmp, &c->bvec, &c->u, &c->u1, &c->rhs,
                     &c->bx[0], &c->bx[1], &c->by[0], &c->by[1], &c->bw};
  for (auto v : vecs) ok &= dalloc(v, BN) == cudaSuccess;
  ok &= dalloc(&c->tmpc, BCN) == cudaSuccess;
  if (d3) {
    ok &= dalloc(&c->pmask, (c->mask_shared ? 1 : c->B) * (size_t)D1 * D2) == cudaSuccess;
    ok &= dalloc(&c->bz[0], BN) == cudaSuccess && dalloc(&c->bz[1], BN) == cudaSuccess;
    ok &= dalloc(&c->tw_y, D1) == cudaSuccess && dalloc(&c->tw_z, D2) == cudaSuccess;
    ok &= dalloc(&c->twd_y, D1) == cudaSuccess && dalloc(&c->twd_z, D2) == cudaSuccess;
  }
  ok &= dalloc(&c->scal, c->B) == cudaSuccess && dalloc(&c->ctl, 1) == cudaSuccess;
  ok &= dalloc(&c->counters, 1) == cudaSuccess;
  c->P.cap = (int)std::max<int64_t>(4096, N / 2 + 64);  // column passes: N/W partials, W >= 2
  ok &= dalloc(&c->P.p0, (size_t)c->B * c->P.cap) == cudaSuccess;
  ok &= dalloc(&c->P.p1, (size_t)c->B * c->P.cap) == cudaSuccess;
  ok &= dalloc(&c->P.cnt, c->B) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    return bail(SB_E_NOMEM);
  }
  c->err.clear();
  // copy inputs (host or device)
  cudaMemcpyKind ks = is_device_ptr(sens) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  cudaMemcpyKind km = is_device_ptr(mask) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (cudaMemcpyAsync(c->sens, sens, BCN * sizeof(float2), ks, c->st) != cudaSuccess) return bail(SB_E_CUDA);
  if (cudaMemcpyAsync(c->mask, mask, nmask, km, c->st) != cudaSuccess) return bail(SB_E_CUDA);
  std::vector<uint8_t> hm(nmask);
  if (cudaMemcpyAsync(hm.data(), c->mask, nmask, cudaMemcpyDeviceToHost, c->st) != cudaSuccess ||
      cudaStreamSynchronize(c->st) != cudaSuccess)
    return bail(SB_E_CUDA);
  for (uint8_t v : hm)
    if (v > 1) return bail(SB_E_ARG);
  const int nm = c->mask_shared ? 1 : c->B;
  c->samp_frac.assign(c->B, 0.f);
  for (int b = 0; b < c->B; ++b) {
    const uint8_t* mb = hm.data() + (size_t)(c->mask_shared ? 0 : b) * img;
    size_t cnt = 0;
    for (size_t i = 0; i < img; ++i) cnt += mb[i];
    c->samp_frac[b] = (float)((double)cnt / (double)img);
  }
  if (!d3) {
    // separability (rows constant along d1): the line-mask identity of K1 (DESIGN.md a1)
    bool sep = true;
    std::vector<float> rm((size_t)nm * M);
    for (int b = 0; b < nm && sep; ++b)
      for (int64_t i = 0; i < M && sep; ++i) {
        const uint8_t* row = hm.data() + (size_t)b * img + (size_t)i * N;
        for (int64_t j = 0; j < N; ++j)
          if (row[j] != row[0]) {
            sep = false;
            break;
          }
        rm[(size_t)b * M + i] = row[0] ? 1.0f / (float)M : 0.f;
      }
    c->separable = sep;
    c->plane = !sep;
    if (!sep && !kp2_supported((int)M, (int)N)) {  // non-separable masks need the plane kernel
      c->err = "non-separable 2D mask: plane size not instantiated in k_plane.cu";
      sb_pcg_destroy(c);
      return SB_E_UNSUPPORTED_SIZE;
    }
    // the fused one-kernel preconditioner (KP_PRE2D) is slower than the three column/row
    // passes at the BASELINE sizes (measured: config 3 83k vs 135k it/s), so it is opt-in
    // ... except for small batches, where one cluster kernel per problem beats three
    // launches (config 2: 19.1k vs 17.8k it/s); SBPCG_PRE2D=0/1 forces either
    const int gpre = M <= 32 ? 1 : (M <= 64 ? 2 : (M <= 128 ? 4 : (M == 256 ? 16 : 8)));
    const bool small = (int64_t)c->B * gpre <= 2 * 148;
    const char* pe = getenv("SBPCG_PRE2D");
    c->pre2d = kp2_supported((int)M, (int)N) && (pe ? pe[0] == '1' : small);
    if (sep && (cudaMemcpyAsync(c->rowmask, rm.data(), rm.size() * sizeof(float), cudaMemcpyHostToDevice, c->st) !=
                    cudaSuccess ||
                cudaStreamSynchronize(c->st) != cudaSuccess))
      return bail(SB_E_CUDA);
  } else {
    // 3D: the mask must be constant along the readout d0 (BASELINE config 5):
    // then the data term factors per d0 plane (k_plane.cu)
    const size_t pn = (size_t)D1 * D2;
    for (int b = 0; b < nm; ++b)
      for (int64_t x = 1; x < D0; ++x)
        if (memcmp(hm.data() + (size_t)b * img + x * pn, hm.data() + (size_t)b * img, pn) != 0) {
          c->err = "3D mask must be constant along the readout axis d0";
          sb_pcg_destroy(c);
          return SB_E_UNSUPPORTED_SIZE;
        }
    for (int b = 0; b < nm; ++b)
      if (cudaMemcpyAsync(c->pmask + (size_t)b * pn, hm.data() + (size_t)b * img, pn, cudaMemcpyHostToDevice, c->st) !=
          cudaSuccess)
        return bail(SB_E_CUDA);
    if (cudaStreamSynchronize(c->st) != cudaSuccess) return bail(SB_E_CUDA);
    c->separable = false;
    c->plane = true;
  }
  // twiddles
  auto tm = make_tw<float2>((int)M), tn = make_tw<float2>((int)N);
  auto tdm = make_tw<double2>((int)M), tdn = make_tw<double2>((int)N);
  // twiddle uploads on the context stream; the host tables live until the synchronisation below
  if (cudaMemcpyAsync(c->tw_m, tm.data(), M * sizeof(float2), cudaMemcpyHostToDevice, c->st) ||
      cudaMemcpyAsync(c->tw_n, tn.data(), N * sizeof(float2), cudaMemcpyHostToDevice, c->st) ||
      cudaMemcpyAsync(c->twd_m, tdm.data(), M * sizeof(double2), cudaMemcpyHostToDevice, c->st) ||
      cudaMemcpyAsync(c->twd_n, tdn.data(), N * sizeof(double2), cudaMemcpyHostToDevice, c->st))
    return bail(SB_E_CUDA);
  std::vector<float2> ty, tz;
  std::vector<double2> tdy, tdz;
  if (d3) {
    ty = make_tw<float2>((int)D1);
    tz = make_tw<float2>((int)D2);
    tdy = make_tw<double2>((int)D1);
    tdz = make_tw<double2>((int)D2);
    if (cudaMemcpyAsync(c->tw_y, ty.data(), D1 * sizeof(float2), cudaMemcpyHostToDevice, c->st) ||
        cudaMemcpyAsync(c->tw_z, tz.data(), D2 * sizeof(float2), cudaMemcpyHostToDevice, c->st) ||
        cudaMemcpyAsync(c->twd_y, tdy.data(), D1 * sizeof(double2), cudaMemcpyHostToDevice, c->st) ||
        cudaMemcpyAsync(c->twd_z, tdz.data(), D2 * sizeof(double2), cudaMemcpyHostToDevice, c->st))
      return bail(SB_E_CUDA);
  }
  if (cudaStreamSynchronize(c->st) != cudaSuccess) return bail(SB_E_CUDA);
  // zero state
  for (auto v : vecs)
    if (cudaMemsetAsync(*v, 0, BN * sizeof(float2), c->st) != cudaSuccess) return bail(SB_E_CUDA);
  if (d3 && (cudaMemsetAsync(c->bz[0], 0, BN * sizeof(float2), c->st) ||
             cudaMemsetAsync(c->bz[1], 0, BN * sizeof(float2), c->st)))
    return bail(SB_E_CUDA);
  if (cudaMemsetAsync(c->P.cnt, 0, c->B * sizeof(unsigned int), c->st) ||
      cudaMemsetAsync(c->ctl, 0, sizeof(Ctl), c->st) || cudaMemsetAsync(c->scal, 0, sizeof(Scal) * c->B, c->st) ||
      cudaMemsetAsync(c->counters, 0, sizeof(Counters), c->st))
    return bail(SB_E_CUDA);
  // K1 configuration: W columns per tile; G-CTA clusters split the coils when the
  // problem alone would not fill the 148 SMs.
  c->W = k1_default_W(c->M, c->N);
  if (const char* we = getenv("SBPCG_K1_W")) {  // debugging override of the tile width (4 or 8)
    const int w = atoi(we);
    if ((w == 4 || w == 8) && c->N % w == 0) c->W = w;
  }
  c->G = 1;
  const int tiles = c->N / c->W;
  for (int g = 2; g <= 8; g *= 2)
    if (g <= c->C && c->M % g == 0 && (int64_t)c->B * tiles * g <= 2 * 148) c->G = g;
  if (const char* ge = getenv("SBPCG_K1_G")) {  // debugging override of the coil-group count
    const int g = atoi(ge);
    if (g >= 1 && g <= 16) c->G = g;  // G need not divide M (uneven rows); g > C leaves idle CTAs
  }
  // spectral-residual preconditioner passes: 2D line masks whose K1 CTAs hold whole columns
  // (G = 1) and that do not take the fused one-cluster preconditioner (SBPCG_SPEC=0 disables)
  c->spec_ok = !d3 && c->separable && c->G == 1 && !c->pre2d && env_flag("SBPCG_SPEC", true);
  // algorithmic bytes per problem-launch of the matvec: coil maps
  // 8NC + z, p_{k-1}, x read + p_k, x, q written (6 x 8N) + the mask (4M floats for line
  // masks, one byte per plane pixel otherwise)
  c->k1_bytes = 8.0 * (double)img * c->C + 48.0 * (double)img +
                (c->separable ? 4.0 * c->M : (double)(d3 ? (size_t)D1 * D2 : img));
  sb_status s = c->plane ? SB_OK : make_tmap(c);  // K1 streams the coil maps by TMA
  if (s) {
    sb_pcg_destroy(c);
    return s;
  }
  // the persistent whole-GPU kernel (k_persist.cu) for small batches of square line-mask
  // problems: a column-major copy of the coil maps, barrier counters, stage counters
  c->kr_on = env_flag("SBPCG_PERSIST", true);
  c->kr_cg = env_flag("SBPCG_CG", true);
  c->kr_ok = !d3 && c->separable && kr_supported(c->M, c->N, c->L) && c->B <= kr_max_problems(c->M, c->N, c->C);
  if (!s && c->kr_ok) {
    if (dalloc(&c->sT, BCN) != cudaSuccess || dalloc(&c->kbar, c->B) != cudaSuccess ||
        dalloc(&c->kstamp, 32 + 4 * 256) != cudaSuccess) {
      cudaGetLastError();
      sb_pcg_destroy(c);
      return SB_E_NOMEM;
    }
    if (launch_transpose_sens(c->sens, c->sT, c->B * c->C, c->M, c->N, c->st) != cudaSuccess) {
      sb_pcg_destroy(c);
      return SB_E_CUDA;
    }
  }
  if (!s && comm) {  // coil-sharded context (collective: Lambda from every rank's coils)
    if (dalloc(&c->accbuf, (size_t)c->B * c->img) != cudaSuccess) {
      sb_pcg_destroy(c);
      return SB_E_NOMEM;
    }
    c->comm = comm;
  }
  if (!s && d3) {  // the coil mode's comm stream and chunk events (also for sb_pcg_set_comm)
    if (cudaStreamCreateWithFlags(&c->cst, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->red_done, cudaEventDisableTiming) != cudaSuccess) {
      sb_pcg_destroy(c);
      return SB_E_CUDA;
    }
    for (auto& e : c->chunk_ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
        sb_pcg_destroy(c);
        return SB_E_CUDA;
      }
    if (const char* ce = getenv("SBPCG_COIL_CHUNKS")) c->coil_chunks = std::max(1, std::min(16, atoi(ce)));
    if (const char* cu = getenv("SBPCG_COIL_UNROLL")) c->coil_unroll = std::max(1, std::min(16, atoi(cu)));
  }
  s = build_lambda(c);
  if (!s) s = cudaStreamSynchronize(c->st) == cudaSuccess ? build_checked(c) : SB_E_CUDA;
  if (s) {
    sb_pcg_destroy(c);
    return s;
  }
  *out = c;
  return SB_OK;
}

sb_status sb_set_option(sb_ctx* c, int32_t option, int32_t value) {
  sb_status s = check_ready(c);
  if (s) return s;
  switch (option) {
    case SB_OPT_PERSISTENT:
      if (value != 0 && value != 1) return fail(c, SB_E_ARG, "SB_OPT_PERSISTENT takes 0 or 1");
      c->kr_on = value != 0;
      return SB_OK;
    case SB_OPT_PCG_CG:
      if (value != 0 && value != 1) return fail(c, SB_E_ARG, "SB_OPT_PCG_CG takes 0 or 1");
      c->kr_cg = value != 0;
      return SB_OK;
    default: return fail(c, SB_E_ARG, "unknown option");
  }
}

int32_t sb_last_path(const sb_ctx* c) { return c ? c->last_path : SB_PATH_NONE; }

sb_status sb_comm_unique_id(void* id_out) {
  if (!id_out) return SB_E_ARG;
  if (!nccl_load()) return SB_E_COMM;
  nccl_uid_t id;
  if (g_nccl.getUniqueId(&id) != 0) return SB_E_COMM;
  memcpy(id_out, &id, sizeof(id));
  return SB_OK;
}

sb_status sb_comm_init(const void* id, int32_t rank, int32_t world, sb_comm** out) {
  if (!out || !id || world < 1 || rank < 0 || rank >= world) return SB_E_ARG;
  *out = nullptr;
  // reading A24 (fixed reduction order): a pinned ring all-reduce reduces in the same order on
  // every call; NVLS / tree selection could change it.  The caller's settings win.
  setenv("NCCL_ALGO", "Ring", 0);
  setenv("NCCL_PROTO", "Simple", 0);
  if (!nccl_load()) return SB_E_COMM;
  nccl_uid_t uid;
  memcpy(&uid, id, sizeof(uid));
  sb_comm* cm = new sb_comm();
  if (g_nccl.commInitRank(&cm->comm, world, uid, rank) != 0) {
    delete cm;
    return SB_E_COMM;
  }
  cm->rank = rank;
  cm->world = world;
  *out = cm;
  return SB_OK;
}

sb_status sb_comm_init_nccl(const void* nccl_unique_id, int32_t rank, int32_t world, sb_comm** out) {
  return sb_comm_init(nccl_unique_id, rank, world, out);
}

void sb_comm_destroy(sb_comm* cm) {
  if (!cm) return;
  if (cm->comm && g_nccl.commDestroy) g_nccl.commDestroy(cm->comm);
  delete cm;
}

sb_status sb_pcg_set_comm(sb_ctx* c, sb_comm* cm) {
  sb_status s = check_ready(c);
  if (s) return s;
  // coil sharding is the 3D (BASELINE config 5) mode: its Lambda marginal, u_1 / RSS init and
  // adjoint all-reduce across ranks; the 2D paths are slice-sharded instead (no collective)
  if (c->ndim != 3) return fail(c, SB_E_UNSUPPORTED_SIZE, "coil sharding is for 3D contexts (slice-shard 2D batches)");
  if (cm && !c->accbuf) CK(dalloc(&c->accbuf, (size_t)c->B * c->img));
  c->comm = cm;
  for (auto& g : c->gs) g.maxit = -1;  // cached graphs do not apply
  coil_graphs_drop(c);
  return build_lambda(c);               // Lambda from the marginal over all ranks' coils
}

// ------------------------------------------------------------------ preprocessing (no context)
sb_status sb_normalize_sens(const sb_c64* sens, const uint8_t* support, int32_t batch, int32_t coils, int64_t npix,
                            int32_t support_shared, sb_c64* sens_out, void* stream) {
  if (!sens || !sens_out || batch < 1 || coils < 1 || npix < 1) return SB_E_ARG;
  if (!is_device_ptr(sens) || !is_device_ptr(sens_out) || (support && !is_device_ptr(support))) return SB_E_ARG;
  cudaError_t e = launch_normalize_sens((const float2*)sens, support, support_shared ? 0 : (size_t)npix, batch, coils,
                                        (size_t)npix, (float2*)sens_out, (cudaStream_t)stream);
  return e == cudaSuccess ? SB_OK : SB_E_CUDA;
}

sb_status sb_normalize_coil_images(const sb_c64* m, const sb_c64* sens_hat, int32_t batch, int32_t coils, int64_t npix,
                                   sb_c64* m_out, void* stream) {
  if (!m || !sens_hat || !m_out || batch < 1 || coils < 1 || npix < 1) return SB_E_ARG;
  if (!is_device_ptr(m) || !is_device_ptr(sens_hat) || !is_device_ptr(m_out)) return SB_E_ARG;
  cudaError_t e = launch_normalize_images((const float2*)m, (const float2*)sens_hat, batch, coils, (size_t)npix,
                                          (float2*)m_out, (cudaStream_t)stream);
  return e == cudaSuccess ? SB_OK : SB_E_CUDA;
}

sb_status sb_coil_compress(const sb_c64* y, const sb_c64* sens, int32_t batch, int32_t coils, int64_t npix,
                           int32_t coils_out, sb_c64* y_out, sb_c64* sens_out, float* eig_out, void* stream) {
  if (!y || !sens || !y_out || !sens_out || batch < 1 || coils < 1 || coils > 64 || npix < 1 || coils_out < 1 ||
      coils_out > coils)
    return SB_E_ARG;
  if (!is_device_ptr(y) || !is_device_ptr(sens) || !is_device_ptr(y_out) || !is_device_ptr(sens_out)) return SB_E_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int E = coils * coils;
  const int nblk = (int)std::max<int64_t>(1, std::min<int64_t>(256, npix / 256));
  double2 *part = nullptr, *G = nullptr;
  float2* A = nullptr;
  auto cleanup = [&]() {
    if (part) cudaFree(part);
    if (G) cudaFree(G);
    if (A) cudaFree(A);
  };
  if (cudaMalloc(&part, sizeof(double2) * (size_t)batch * nblk * E) != cudaSuccess ||
      cudaMalloc(&G, sizeof(double2) * (size_t)batch * E) != cudaSuccess ||
      cudaMalloc(&A, sizeof(float2) * (size_t)batch * coils_out * coils) != cudaSuccess) {
    cleanup();
    return SB_E_NOMEM;
  }
  // coil covariance of the data (k-space: equal to the image-domain one, F unitary)
  if (launch_gram((const float2*)y, batch, coils, (size_t)npix, part, nblk, G, st) != cudaSuccess) {
    cleanup();
    return SB_E_CUDA;
  }
  std::vector<std::complex<double>> hG((size_t)batch * E), U((size_t)E);
  std::vector<double> w(coils);
  std::vector<float2> hA((size_t)batch * coils_out * coils);
  if (cudaMemcpyAsync(hG.data(), G, sizeof(double2) * hG.size(), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    cleanup();
    return SB_E_CUDA;
  }
  for (int b = 0; b < batch; ++b) {
    hermitian_eig(coils, hG.data() + (size_t)b * E, w.data(), U.data());
    if (eig_out)
      for (int k = 0; k < coils; ++k) eig_out[(size_t)b * coils + k] = (float)w[k];
    for (int k = 0; k < coils_out; ++k)  // A = U[:, :K]^H
      for (int c = 0; c < coils; ++c) {
        const std::complex<double> u = std::conj(U[(size_t)c * coils + k]);
        hA[((size_t)b * coils_out + k) * coils + c] = make_float2((float)u.real(), (float)u.imag());
      }
  }
  if (cudaMemcpyAsync(A, hA.data(), sizeof(float2) * hA.size(), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      launch_coil_apply((const float2*)y, A, batch, coils, coils_out, (size_t)npix, (float2*)y_out, st) != cudaSuccess ||
      launch_coil_apply((const float2*)sens, A, batch, coils, coils_out, (size_t)npix, (float2*)sens_out, st) !=
          cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    cleanup();
    return SB_E_CUDA;
  }
  cleanup();
  return SB_OK;
}

sb_status sb_readout_decouple(const sb_c64* y3, const sb_c64* s3, int32_t coils, const int64_t* shape, sb_c64* y2,
                              sb_c64* s2, void* stream) {
  if (!y3 || !shape || !y2 || coils < 1 || (s3 == nullptr) != (s2 == nullptr)) return SB_E_ARG;
  if (!is_device_ptr(y3) || !is_device_ptr(y2) || (s3 && (!is_device_ptr(s3) || !is_device_ptr(s2)))) return SB_E_ARG;
  const int64_t D0 = shape[0], D1 = shape[1], D2 = shape[2];
  if (D1 < 1 || D2 < 1 || !col3_len_ok(D0) || (D1 * D2) % 8 != 0 || (int64_t)coils > 65535) return SB_E_UNSUPPORTED_SIZE;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t n12 = (size_t)D1 * D2;
  auto tw = make_tw<float2>((int)D0);
  float2* twd = nullptr;
  if (cudaMalloc(&twd, D0 * sizeof(float2)) != cudaSuccess) return SB_E_NOMEM;
  PassArgs a;
  memset(&a, 0, sizeof(a));
  a.B = 1;
  a.C = coils;
  a.M = (int)D0;
  a.N = (int)n12;
  a.tw_m = twd;
  a.a0 = (const float2*)y3;
  a.o0 = (float2*)y2;
  a.scale = 1.0f / std::sqrt((float)D0);
  sb_status rs = SB_OK;
  if (cudaMemcpyAsync(twd, tw.data(), D0 * sizeof(float2), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      launch_pass(P_COL_DECOUPLE, a, st) != cudaSuccess)
    rs = SB_E_CUDA;
  // image-space maps change layout only: s2[x][c] = s3[c][x] (one strided 2D copy per coil)
  for (int c = 0; s3 && rs == SB_OK && c < coils; ++c)
    if (cudaMemcpy2DAsync((float2*)s2 + (size_t)c * n12, (size_t)coils * n12 * sizeof(float2),
                          (const float2*)s3 + (size_t)c * D0 * n12, n12 * sizeof(float2), n12 * sizeof(float2),
                          (size_t)D0, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      rs = SB_E_CUDA;
  if (cudaStreamSynchronize(st) != cudaSuccess) rs = SB_E_CUDA;
  cudaFree(twd);
  return rs;
}

sb_status sb_set_wavelet(sb_ctx* c, int32_t family) {
  sb_status s = check_ready(c);
  if (s) return s;
  if (family != 0 && family != 1) return fail(c, SB_E_ARG, "wavelet family must be 0 (Haar) or 1 (D4)");
  if (family == 1 && c->L < 1) return fail(c, SB_E_DIM, "D4 needs wavelet_levels >= 1");
  if (family == 1 && !c->wbuf) CK(dalloc(&c->wbuf, (size_t)c->B * c->img));
  c->wavelet = family;
  for (auto& g : c->gs) g.maxit = -1;  // the captured shrink step changes
  coil_graphs_drop(c);
  return SB_OK;
}

sb_status sb_pcg_update_sens(sb_ctx* c, const sb_c64* sens) {
  sb_status s = check_ready(c);
  if (s) return s;
  if (!sens) return fail(c, SB_E_ARG, "update_sens: null");
  const size_t bytes = (size_t)c->B * c->C * c->img * sizeof(float2);
  CK(cudaMemcpyAsync(c->sens, sens, bytes, is_device_ptr(sens) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                     c->st));
  if (c->sT) CK(launch_transpose_sens(c->sens, c->sT, c->B * c->C, c->M, c->N, c->st));
  if (c->jinv) {  // Jacobi diagonal depends on the maps: rebuilt on next use
    cudaFree(c->jinv);
    c->jinv = nullptr;
  }
  return build_lambda(c);
}

sb_status sb_pcg_build_precond(sb_ctx* c) {
  sb_status s = check_ready(c);
  if (s) return s;
  return build_lambda(c);
}

sb_status sb_pcg_apply_A(sb_ctx* c, const sb_c64* x, sb_c64* y) {
  sb_status s = check_ready(c);
  if (s) return s;
  if (!x || !y || (const void*)x == (const void*)y) return fail(c, SB_E_ARG, "apply_A: bad pointers");
  const size_t bytes = c->B * c->img * sizeof(float2);
  const bool hy = !is_device_ptr(y);
  const void* xd;
  if ((s = stage_in(c, x, bytes, &xd, c->tmp))) return s;
  float2* yd = hy ? c->q : (float2*)y;
  if ((s = seq_apply(c, (const float2*)xd, yd, c->st))) return s;
  if (hy) {
    CK(cudaMemcpyAsync(y, yd, bytes, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
  }
  return SB_OK;
}

sb_status sb_pcg_apply_Pinv(sb_ctx* c, const sb_c64* r, sb_c64* z) {
  sb_status s = check_ready(c);
  if (s) return s;
  if (!r || !z || (const void*)r == (const void*)z) return fail(c, SB_E_ARG, "apply_Pinv: bad pointers");
  const size_t bytes = c->B * c->img * sizeof(float2);
  const bool hz = !is_device_ptr(z);
  const void* rd;
  if ((s = stage_in(c, r, bytes, &rd, c->q))) return s;
  float2* zd = hz ? c->z : (float2*)z;
  Loop L = make_loop(c, 0ull);
  L.scal = nullptr;
  if ((s = seq_precond(c, L, 1, -1, (const float2*)rd, zd, c->st))) return s;
  if (hz) {
    CK(cudaMemcpyAsync(z, zd, bytes, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
  }
  return SB_OK;
}

sb_status sb_encode(sb_ctx* c, const sb_c64* x, sb_c64* y, int32_t full) {
  sb_status s = check_ready(c);
  if (s) return s;
  if (!x || !y || (const void*)x == (const void*)y) return fail(c, SB_E_ARG, "encode: bad pointers");
  const size_t bytes = c->B * c->img * sizeof(float2), ybytes = bytes * c->C;
  const bool hy = !is_device_ptr(y);
  const void* xd;
  if ((s = stage_in(c, x, bytes, &xd, c->tmp))) return s;
  if (hy && !c->stage_out) CK(dalloc(&c->stage_out, c->B * c->C * c->img));
  float2* yd = hy ? c->stage_out : (float2*)y;
  if (c->ndim == 3) {  // per plane: (R) F_12 (s_c x) -> tmpc ; then the d0 FFT of every coil
    KPArgs k = base_kp(c);
    k.vin = (const float2*)xd;
    k.out = c->tmpc;
    k.full = full ? 1 : 0;
    k.scale = 1.0f / std::sqrt((float)c->img);
    if ((s = run_kp(c, KP_ENCODE, k, c->st))) return s;
    PassArgs pa = base_pass(c);
    pa.a0 = c->tmpc;
    pa.o0 = yd;
    pa.scale = 1.0f;
    if ((s = run_pass(c, P_COL_FWD, pa, c->st))) return s;
  } else {
    PassArgs pa = base_pass(c);
    pa.a0 = (const float2*)xd;
    pa.tmp = c->tmpc;
    pa.o0 = yd;
    pa.full = full ? 1 : 0;
    pa.scale = 1.0f / std::sqrt((float)c->img);
    if ((s = run_pass(c, P_ENC_COL, pa, c->st))) return s;
    if ((s = run_pass(c, P_ENC_ROW, pa, c->st))) return s;
  }
  if (hy) {
    CK(cudaMemcpyAsync(y, yd, ybytes, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
  }
  return SB_OK;
}

sb_status sb_adjoint(sb_ctx* c, const sb_c64* y, sb_c64* x) {
  sb_status s = check_ready(c);
  if (s) return s;
  if (!x || !y || (const void*)x == (const void*)y) return fail(c, SB_E_ARG, "adjoint: bad pointers");
  const size_t bytes = c->B * c->img * sizeof(float2), ybytes = bytes * c->C;
  const bool hx = !is_device_ptr(x);
  if (!is_device_ptr(y) && !c->stage_in) CK(dalloc(&c->stage_in, c->B * c->C * c->img));
  const void* yd;
  if ((s = stage_in(c, y, ybytes, &yd, c->stage_in))) return s;
  float2* xd = hx ? c->q : (float2*)x;
  if (c->ndim == 3) {
    if ((s = seq_adjoint3(c, (const float2*)yd, xd, nullptr, c->st))) return s;
  } else {
    PassArgs pa = base_pass(c);
    pa.a0 = (const float2*)yd;
    pa.tmp = c->tmpc;
    pa.o0 = xd;
    pa.o1 = nullptr;
    pa.scale = 1.0f / std::sqrt((float)c->img);
    if ((s = run_pass(c, P_ADJ_ROW, pa, c->st))) return s;
    if ((s = run_pass(c, P_ADJ_COL, pa, c->st))) return s;
  }
  if (hx) {
    CK(cudaMemcpyAsync(x, xd, bytes, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
  }
  return SB_OK;
}

static sb_status check_opts(sb_ctx* c, const sb_pcg_opts* o) {
  if (!o || o->max_iters < 1 || !(o->eps >= 0.f) || o->precond < 0 || o->precond > 2)
    return fail(c, SB_E_ARG, "bad pcg options");
  if (o->precond == 2 && c->comm)  // diag(A) needs sum_c |S_c|^2 over every rank's coils
    return fail(c, SB_E_UNSUPPORTED_SIZE, "Jacobi preconditioner is not available in the coil-sharded mode");
  if (o->precond == 2 && !c->jinv) {  // Jacobi diagonal, once
    CK(dalloc(&c->jinv, (size_t)c->B * c->img));
    float* fr = nullptr;
    CK(dalloc(&fr, c->B));
    // on the context stream (a non-blocking caller stream does not order after the legacy one);
    // samp_frac outlives the copy, and the stream is synchronised below
    CK(cudaMemcpyAsync(fr, c->samp_frac.data(), c->B * sizeof(float), cudaMemcpyHostToDevice, c->st));
    CK(launch_jacobi_diag(c->sens, fr, c->B, c->C, c->img, c->ndim, c->mu, c->lam, c->gam, c->jinv, c->st));
    CK(cudaStreamSynchronize(c->st));
    cudaFree(fr);
    c->launches++;
  }
  return SB_OK;
}

static sb_status ensure_hist(sb_ctx* c, int maxit, int slots) {
  if (c->hist_stride < maxit + 1) {
    if (c->hist) cudaFree(c->hist);
    c->hist = nullptr;
    CK(dalloc(&c->hist, (size_t)c->B * (maxit + 1)));
    c->hist_stride = maxit + 1;
    for (auto& g : c->gs) g.maxit = -1;  // graphs captured the old pointer
    coil_graphs_drop(c);
  }
  if (c->log_cap < slots) {
    if (c->log_iters) cudaFree(c->log_iters);
    if (c->log_relres) cudaFree(c->log_relres);
    CK(dalloc(&c->log_iters, (size_t)c->B * slots));
    CK(dalloc(&c->log_relres, (size_t)c->B * slots));
    c->log_cap = slots;
    for (auto& g : c->gs) g.maxit = -1;
    coil_graphs_drop(c);
  }
  return SB_OK;
}

sb_status sb_pcg_solve(sb_ctx* c, const sb_c64* b, sb_c64* x, const sb_pcg_opts* o, sb_pcg_stats* stats) {
  sb_status s = check_ready(c);
  if (s) return s;
  if (!b || !x || (const void*)b == (const void*)x) return fail(c, SB_E_ARG, "solve: bad pointers");
  if ((s = check_opts(c, o))) return s;
  if ((s = ensure_hist(c, o->max_iters, 1))) return s;
  const size_t bytes = c->B * c->img * sizeof(float2);
  const cudaMemcpyKind kb = is_device_ptr(b) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  const bool xdev = is_device_ptr(x);
  CK(cudaMemcpyAsync(c->bvec, b, bytes, kb, c->st));
  CK(cudaMemcpyAsync(c->x, x, bytes, xdev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->st));
  CK(cudaMemsetAsync(c->ctl, 0, sizeof(Ctl), c->st));
  if (c->timing) c->evnext = 0;
  bool kr = use_kr(c, o);
  s = kr ? run_kr(c, 0, o, 0) : run_solve_kind(c, 0, o, nullptr);
  if (s == SB_E_UNSUPPORTED_SIZE && kr && !c->kr_ok) {  // persistent launch refused: kernel sequence
    kr = false;
    s = run_solve_kind(c, 0, o, nullptr);
  }
  if (s) return s;
  CK(cudaMemcpyAsync(x, c->x, bytes, xdev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->st));
  HostRes hr;
  if ((s = host_results(c, 1, &hr))) return s;
  CK(cudaMemcpyAsync(hr.scal, c->scal, sizeof(Scal) * c->B, cudaMemcpyDeviceToHost, c->st));
  const bool want_hist = stats && stats->relres_hist;
  if (want_hist)
    CK(cudaMemcpyAsync(hr.hist, c->hist, (size_t)c->B * c->hist_stride * sizeof(float), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if ((s = build_checked(c))) return s;
  std::vector<Scal> hs(hr.scal, hr.scal + c->B);
  if (c->timing) {
    if (kr) {
      std::vector<int32_t> it(c->B);
      for (int i = 0; i < c->B; ++i) it[i] = hs[i].iter;
      c->kr_alg_bytes += kr_bytes(c, it, 1, false);
    }
    timing_collect(c);
  }
  if (c->last_path == SB_PATH_GRAPH && !c->timing) {
    int mx = 0;
    for (auto& h : hs) mx = std::max(mx, h.iter);
    const GraphSlot& g0 = c->gs[0];
    c->launches += g0.nfixed + (int64_t)g0.nbody * ((mx + g0.unroll - 1) / g0.unroll);
  }
  if (stats) {
    const float* hist = hr.hist;
    for (int i = 0; i < c->B; ++i) {
      if (stats->iters) stats->iters[i] = hs[i].iter;
      if (stats->converged) stats->converged[i] = (int8_t)hs[i].converged;
      if (stats->final_relres) stats->final_relres[i] = hs[i].nb2 > 0 ? (float)std::sqrt(hs[i].rr / hs[i].nb2) : 0.f;
      if (stats->relres_hist)
        for (int k = 0; k <= o->max_iters; ++k)
          stats->relres_hist[(size_t)i * (o->max_iters + 1) + k] = hist[(size_t)i * c->hist_stride + k];
    }
  }
  return status_of(c, hs.data());
}

sb_status sb_recon(sb_ctx* c, const sb_c64* y, const sb_recon_opts* ro, sb_c64* x_out, sb_recon_log* log) {
  sb_status s = check_ready(c);
  if (s) return s;
  if (!y || !x_out || !ro || (const void*)y == (const void*)x_out) return fail(c, SB_E_ARG, "recon: bad pointers");
  if (ro->n_outer < 1 || ro->n_inner != 1) return fail(c, SB_E_ARG, "recon: n_outer >= 1 and n_inner == 1 required");
  if ((s = check_opts(c, &ro->pcg))) return s;
  if ((s = ensure_hist(c, ro->pcg.max_iters, ro->n_outer))) return s;
  const size_t bytes = c->B * c->img * sizeof(float2), ybytes = bytes * c->C;
  if (!c->rev[0]) {
    CK(cudaEventCreate(&c->rev[0]));
    CK(cudaEventCreate(&c->rev[1]));
  }
  cudaEvent_t e0 = c->rev[0], e1 = c->rev[1];
  CK(cudaEventRecord(e0, c->st));
  const sb_pcg_opts* o = &ro->pcg;
  bool kr = use_kr(c, o);
  // the persistent kernel does Alg. 1 step 1 and starts from a zero SB state itself (kinit)
  const bool kinit = kr && env_flag("SBPCG_KR_INIT", true);
  // y is copied into the context's staging buffer so the cached graphs stay valid (the
  // persistent kernel reads a device y in place)
  const void* yd = y;
  if (!(kinit && is_device_ptr(y))) {
    if (!c->stage_in) CK(dalloc(&c->stage_in, c->B * c->C * c->img));
    CK(cudaMemcpyAsync(c->stage_in, y, ybytes, is_device_ptr(y) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                       c->st));
    yd = c->stage_in;
  }
  // fresh SB state (Alg. 1 step 1)
  auto zero_state = [&]() -> sb_status {
    float2* zs[] = {c->bx[0], c->bx[1], c->by[0], c->by[1], c->bw, c->rhs, c->bz[0], c->bz[1]};
    for (auto v : zs)
      if (v) CK(cudaMemsetAsync(v, 0, bytes, c->st));
    CK(cudaMemsetAsync(c->ctl, 0, sizeof(Ctl), c->st));
    return SB_OK;
  };
  if (!kinit && (s = zero_state())) return s;
  if (c->timing) c->evnext = 0;
  c->stage_timing = kr ? false : (ro->stage_timers != 0);
  for (double& v : c->stage_s) v = 0.0;
  c->stage_ev.clear();
  c->stage_next = 0;
  if (kr) {
    // Alg. 1 step 1 (u1, x = RSS) by the column/row passes, then the whole SB loop in one
    // cooperative launch (including the final shrink/Bregman step)
    if (!kinit) {
      cudaEvent_t ei0 = stage_event(c), ei1 = stage_event(c);
      CK(cudaEventRecord(ei0, c->st));
      if ((s = seq_init_recon(c, (const float2*)yd, c->st))) return s;
      CK(cudaEventRecord(ei1, c->st));
      c->stage_ev.push_back({ST_INIT, {ei0, ei1}});
    }
    CK(cudaMemsetAsync(c->kstamp, 0, 32 * sizeof(unsigned long long), c->st));
    c->kr_y = kinit ? (const float2*)yd : nullptr;
    s = run_kr(c, ro->n_outer, o, 0);
    c->kr_y = nullptr;
    if (s == SB_E_UNSUPPORTED_SIZE && !c->kr_ok) {  // persistent launch refused: kernel sequence
      kr = false;
      c->stage_timing = ro->stage_timers != 0;
      if (kinit) {
        if ((s = zero_state())) return s;
        if (yd != c->stage_in) {  // the sequence path's cached graphs read the staging buffer
          if (!c->stage_in) CK(dalloc(&c->stage_in, c->B * c->C * c->img));
          CK(cudaMemcpyAsync(c->stage_in, yd, ybytes, cudaMemcpyDeviceToDevice, c->st));
          yd = c->stage_in;
        }
      }
    } else if (s) {
      return s;
    }
  }
  if (!kr) {
    if ((s = run_solve_kind(c, 1, o, (const float2*)yd))) return s;
    for (int j = 1; j < ro->n_outer; ++j) {
      const int par = (j - 1) & 1;  // b_x/b_y buffer parity
      if ((s = run_solve_kind(c, 2 + par, o, nullptr))) return s;
    }
    // final shrink/Bregman step of the last inner iteration (Alg. 1 steps 6-11); the final
    // data feedback (steps 13-15) does not change x and is skipped.
    StageMark m(c, ST_SHRINK, c->st);
    if ((s = seq_shrink(c, (ro->n_outer - 1) & 1, c->st))) return s;
    m.close();
  }
  CK(cudaMemcpyAsync(x_out, c->x, bytes, is_device_ptr(x_out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaEventRecord(e1, c->st));
  HostRes hr;
  if ((s = host_results(c, ro->n_outer, &hr))) return s;
  const size_t nl = (size_t)ro->n_outer * c->B;
  CK(cudaMemcpyAsync(hr.scal, c->scal, sizeof(Scal) * c->B, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(hr.iters, c->log_iters, nl * sizeof(int32_t), cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(hr.relres, c->log_relres, nl * sizeof(float), cudaMemcpyDeviceToHost, c->st));
  if (kr) CK(cudaMemcpyAsync(hr.stamp, c->kstamp, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if ((s = build_checked(c))) return s;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const bool stages = kr || c->stage_timing;
  stage_collect(c);
  if (kr) {  // the kernel's stage cycle counters, converted with its own cycles -> ns ratio
    const unsigned long long* hst = hr.stamp;
    if (getenv("SBPCG_KR_PROF") && atoi(getenv("SBPCG_KR_PROF")) == 2 && c->N <= 256) {  // skew probe dump
      std::vector<unsigned long long> pr(4 * 256);
      CK(cudaMemcpy(pr.data(), c->kstamp + 32, pr.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      FILE* f = fopen("gpurun_out/kr_skew.txt", "w");
      if (f) {
        for (int t = 0; t < c->N; ++t) fprintf(f, "%d %llu %llu %llu\n", t, pr[4 * t], pr[4 * t + 1], pr[4 * t + 2]);
        fclose(f);
      }
    }
    if (getenv("SBPCG_KR_PROF") && atoi(getenv("SBPCG_KR_PROF")) > 0) {  // loop segment profile (stderr)
      fprintf(stderr, "KR segments (ns, all iterations):");
      for (int k = 0; k < 24; ++k) fprintf(stderr, " s%d=%.0f", k, hst[3] ? (double)hst[8 + k] * hst[4] / hst[3] : 0.0);
      fprintf(stderr, "\n");
    }
    const double s_per_cyc = hst[3] > 0 ? 1e-9 * (double)hst[4] / (double)hst[3] : 0.0;
    c->stage_s[ST_RHS] += s_per_cyc * (double)hst[0];
    c->stage_s[ST_PCG] += s_per_cyc * (double)hst[1];
    c->stage_s[ST_SHRINK] += s_per_cyc * (double)hst[2];
    c->stage_s[ST_INIT] += s_per_cyc * (double)hst[5];  // Alg. 1 step 1 inside the launch (kinit)
  }
  c->stage_timing = false;
  std::vector<int32_t> li(hr.iters, hr.iters + nl);
  std::vector<float> lr(hr.relres, hr.relres + nl);
  if (c->timing) {
    if (kr) c->kr_alg_bytes += kr_bytes(c, li, ro->n_outer, true);
    timing_collect(c);
  }
  if (c->last_path == SB_PATH_GRAPH && !c->timing) {
    for (int j = 0; j < ro->n_outer; ++j) {
      int mx = 0;
      for (int b = 0; b < c->B; ++b) mx = std::max(mx, li[(size_t)j * c->B + b]);
      const GraphSlot& g = c->gs[j == 0 ? 1 : 2 + ((j - 1) & 1)];
      c->launches += g.nfixed + (int64_t)g.nbody * ((mx + g.unroll - 1) / g.unroll);
    }
  }
  if (log) {
    if (log->pcg_iters) memcpy(log->pcg_iters, li.data(), li.size() * sizeof(int32_t));
    if (log->final_relres) memcpy(log->final_relres, lr.data(), lr.size() * sizeof(float));
    log->total_ms = ms;
    log->rhs_s = c->stage_s[ST_RHS];
    log->pcg_s = c->stage_s[ST_PCG];
    log->shrink_s = c->stage_s[ST_SHRINK];
    log->feedback_s = c->stage_s[ST_FEEDBACK];
    log->init_s = c->stage_s[ST_INIT];
    log->build_s = c->build_s;
    log->stages_valid = stages ? 1 : 0;
  }
  return status_of(c, hr.scal);
}

sb_status sb_sb_update3(sb_ctx* c, const sb_c64* x, sb_c64* bx, sb_c64* by, sb_c64* bz, sb_c64* bw,
                        sb_c64* rhs_reg) {
  sb_status s = check_ready(c);
  if (s) return s;
  if (!x || !bx || !by || !bw || !rhs_reg || (c->ndim == 3 && !bz)) return fail(c, SB_E_ARG, "sb_update: null pointer");
  const size_t bytes = c->B * c->img * sizeof(float2);
  auto kin = [&](const void* p) { return is_device_ptr(p) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice; };
  auto kout = [&](const void* p) { return is_device_ptr(p) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost; };
  CK(cudaMemcpyAsync(c->x, x, bytes, kin(x), c->st));
  CK(cudaMemcpyAsync(c->bx[0], bx, bytes, kin(bx), c->st));
  CK(cudaMemcpyAsync(c->by[0], by, bytes, kin(by), c->st));
  if (c->ndim == 3) CK(cudaMemcpyAsync(c->bz[0], bz, bytes, kin(bz), c->st));
  CK(cudaMemcpyAsync(c->bw, bw, bytes, kin(bw), c->st));
  if ((s = seq_shrink(c, 0, c->st))) return s;
  CK(cudaMemcpyAsync(bx, c->bx[1], bytes, kout(bx), c->st));
  CK(cudaMemcpyAsync(by, c->by[1], bytes, kout(by), c->st));
  if (c->ndim == 3) CK(cudaMemcpyAsync(bz, c->bz[1], bytes, kout(bz), c->st));
  CK(cudaMemcpyAsync(bw, c->bw, bytes, kout(bw), c->st));
  CK(cudaMemcpyAsync(rhs_reg, c->rhs, bytes, kout(rhs_reg), c->st));
  CK(cudaStreamSynchronize(c->st));
  return SB_OK;
}

sb_status sb_sb_update(sb_ctx* c, const sb_c64* x, sb_c64* bx, sb_c64* by, sb_c64* bw, sb_c64* rhs_reg) {
  sb_status s = check_ready(c);
  if (s) return s;
  if (c->ndim == 3) return fail(c, SB_E_DIM, "sb_sb_update is 2D; use sb_sb_update3");
  if (!x || !bx || !by || !bw || !rhs_reg) return fail(c, SB_E_ARG, "sb_update: null pointer");
  const size_t bytes = c->B * c->img * sizeof(float2);
  auto kin = [&](const void* p) { return is_device_ptr(p) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice; };
  auto kout = [&](const void* p) { return is_device_ptr(p) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost; };
  CK(cudaMemcpyAsync(c->x, x, bytes, kin(x), c->st));
  CK(cudaMemcpyAsync(c->bx[0], bx, bytes, kin(bx), c->st));
  CK(cudaMemcpyAsync(c->by[0], by, bytes, kin(by), c->st));
  CK(cudaMemcpyAsync(c->bw, bw, bytes, kin(bw), c->st));
  if ((s = seq_shrink(c, 0, c->st))) return s;
  CK(cudaMemcpyAsync(bx, c->bx[1], bytes, kout(bx), c->st));
  CK(cudaMemcpyAsync(by, c->by[1], bytes, kout(by), c->st));
  CK(cudaMemcpyAsync(bw, c->bw, bytes, kout(bw), c->st));
  CK(cudaMemcpyAsync(rhs_reg, c->rhs, bytes, kout(rhs_reg), c->st));
  CK(cudaStreamSynchronize(c->st));
  return SB_OK;
}

sb_status sb_pcg_get_k(sb_ctx* c, double* k_out) {
  sb_status s = check_ready(c);
  if (s) return s;
  if (!k_out) return fail(c, SB_E_ARG, "get_k: null");
  const size_t bytes = c->B * c->img * sizeof(double);
  CK(cudaMemcpyAsync(k_out, c->kbuf, bytes, is_device_ptr(k_out) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  return build_checked(c);
}

sb_status sb_set_kernel_timing(sb_ctx* c, int32_t enable) {
  if (!c) return SB_E_ARG;
  c->timing = enable != 0;
  for (int k = 0; k < 3; ++k) {
    c->t_ms[k] = 0;
    c->t_n[k] = 0;
  }
  c->kr_alg_bytes = 0;
  cudaStreamSynchronize(c->st);
  if (cudaMemset(c->counters, 0, sizeof(Counters)) != cudaSuccess) return fail(c, SB_E_CUDA, "memset counters");
  return SB_OK;
}

sb_status sb_get_kernel_time(sb_ctx* c, int32_t which, double* ms, int64_t* launches, double* alg_bytes) {
  if (!c || which < 0 || which > 2) return SB_E_ARG;
  if (ms) *ms = c->t_ms[which];
  if (launches) *launches = c->t_n[which];
  if (alg_bytes && which == 2) {
    *alg_bytes = c->t_n[2] > 0 ? c->kr_alg_bytes / (double)c->t_n[2] : 0.0;
    return SB_OK;
  }
  if (alg_bytes) {
    // K1 algorithmic bytes per problem-launch: coil maps 8NC
    // + z, p_{k-1} (and halo), x read + x, p_k, q written (6 x 8N) + row mask (4M);
    // averaged over the timed launches using the device count of active problems.
    const double N = (double)c->img;
    const double per = which == 0 ? c->k1_bytes : (4.0 * 8.0 * N + 4.0 * N);
    Counters h{};
    if (cudaMemcpy(&h, c->counters, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess) return fail(c, SB_E_CUDA, "counters");
    const double probs = (which == 0 && c->t_n[0] > 0) ? (double)h.k1_problems / (double)c->t_n[0] : (double)c->B;
    *alg_bytes = per * probs;
  }
  return SB_OK;
}

}  // extern "C"
