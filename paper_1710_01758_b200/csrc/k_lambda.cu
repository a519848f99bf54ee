// k_lambda.cu — K4: build of the circulant preconditioner's diagonal, in fp64 on the device
// (reading A5), once per context ("constructed beforehand").
//
//   k = mu k_c + lambda k_d + gamma k_w              (Eq. Kdiag)
//   k_c(nu) = sum_q g(q) r(nu + q),  g = sum_c |D s_c|^2 / N^2      (PAPER.md:199-229,
//             the circular correlation form of Eq. diagonalelements; reading A2)
//           = D^{-1}[ conj(D g) . D r ]            (D = unnormalised 2D DFT, g real)
//   k_d(nu) = sum_d 4 sin^2(pi nu_d / n_d)         (eigenvalues of t_1)
//   k_w = 1
// Outputs k (fp64, parity) and Lambda^{-1} = 1/(N k) (fp32; the 1/N of the unnormalised
// inverse FFT used by the preconditioner kernels is folded in).
// FLOPs (Table 1): C forward 2D FFTs of the coil maps plus 3 FFTs.
#include <algorithm>

#include "kernels.cuh"

namespace sbk {

enum LKind {
  L_COL_SENS = 0,   // tmp[b][c] = colFFT(sens[b][c])
  L_ROW_ACC = 1,    // g[b][k0][k1] = sum_c |rowFFT(tmp[b][c])|^2 / N^2
  L_COL_G = 2,      // g[b] = colFFT(g[b])           (in place)
  L_ROW_G = 3,      // g[b] = rowFFT(g[b])           (in place)
  L_COL_MASK = 4,   // rhat[m] = colFFT(mask[m])
  L_ROW_MASK = 5,   // rhat[m] = rowFFT(rhat[m])     (in place)
  L_ROW_PROD = 6,   // g[b] = rowIFFT(conj(g[b]) . rhat[mask(b)])
  L_COL_FINAL = 7,  // k_c = colIFFT(g[b]) / N ; k ; Lambda^{-1}
};

constexpr int LW = 8;  // columns per CTA

template <int M>
struct LCol {
  static constexpr int N1 = Split<M>::N1, N2 = Split<M>::N2, NT = N2 * LW;
  using Lay = typename ColLayout<M, LW>::L;
  static constexpr int XS = ColLayout<M, LW>::size;
};
template <int N>
struct LRow {
  static constexpr int N1 = Split<N>::N1, N2 = Split<N>::N2;
  static constexpr int L0 = (128 / N2) > 0 ? (128 / N2) : 1;
  static constexpr int LINES = (L0 * N1 * (N2 + 1) * 16 > 45000) ? L0 / 2 : L0;  // static smem <= 48 KB
  static constexpr int NT = LINES * N2;
  using Lay = typename RowLayout<N, LINES>::L;
  static constexpr int XS = RowLayout<N, LINES>::size;
};

template <int M, int KIND>
__global__ void __launch_bounds__(LCol<M>::NT) k_lcol(const LamArgs a) {
  using C = LCol<M>;
  constexpr int N1 = C::N1;
  __shared__ __align__(16) double2 xch[C::XS];
  __shared__ double2 tw[M];
  const int tid = threadIdx.x, j = tid / LW, l = tid % LW;
  const int N = a.N;
  const int col = blockIdx.x * LW + l;
  const size_t img = (size_t)M * N;
  for (int i = tid; i < M; i += C::NT) tw[i] = a.tw_m[i];
  __syncthreads();
  double2 v[N1];
  if constexpr (KIND == L_COL_SENS) {
    const int bc = blockIdx.y;  // b*C + c
    const float2* s = a.sens + (size_t)bc * img;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const float2 f = s[(size_t)natidx<M>(j, n1) * N + col];
      v[n1] = make_double2(f.x, f.y);
    }
    fft_fwd<M, typename C::Lay>(v, xch, tw, j, l);
    double2* t = a.tmp + (size_t)bc * img;
#pragma unroll
    for (int q = 0; q < N1; ++q) t[(size_t)specidx<M>(j, q) * N + col] = v[q];
  } else if constexpr (KIND == L_COL_G || KIND == L_COL_MASK) {
    const int bi = blockIdx.y;
    double2* t = (KIND == L_COL_G ? a.g : a.rhat) + (size_t)bi * img;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const size_t gi = (size_t)natidx<M>(j, n1) * N + col;
      if constexpr (KIND == L_COL_G) {
        v[n1] = t[gi];
      } else {
        v[n1] = make_double2(a.mask[(size_t)bi * a.mask_bstride + gi] ? 1.0 : 0.0, 0.0);
      }
    }
    __syncthreads();
    fft_fwd<M, typename C::Lay>(v, xch, tw, j, l);
#pragma unroll
    for (int q = 0; q < N1; ++q) t[(size_t)specidx<M>(j, q) * N + col] = v[q];
  } else if constexpr (KIND == L_COL_FINAL) {
    const int b = blockIdx.y;
    const double2* t = a.g + (size_t)b * img;
#pragma unroll
    for (int q = 0; q < N1; ++q) v[q] = t[(size_t)specidx<M>(j, q) * N + col];
    fft_inv<M, typename C::Lay>(v, xch, tw, j, l);
    const double invN = 1.0 / (double)img;
    if (a.d3) {  // 3D: the plane k_c only; k / Lambda^{-1} are expanded by k_lexpand3
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1)
        a.kc2[(size_t)b * img + (size_t)natidx<M>(j, n1) * N + col] = v[n1].x * invN;
      return;
    }
    const double PI = 3.14159265358979323846;
    const double sc = sin(PI * (double)col / (double)N);
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const int row = natidx<M>(j, n1);
      const double kc = v[n1].x * invN;  // k_c is real (Hermitian K)
      const double sr = sin(PI * (double)row / (double)M);
      const double kd = 4.0 * sr * sr + 4.0 * sc * sc;
      const double k = a.mu * kc + a.lam * kd + a.gam;
      const size_t gi = (size_t)b * img + (size_t)row * N + col;
      a.k_out[gi] = k;
      if (!(fabs(k) > 1e-14) || !isfinite(k)) atomicExch(a.bad, 1);
      a.lam_inv[gi] = (float)(1.0 / ((double)img * k));
    }
  }
}

template <int N, int KIND>
__global__ void __launch_bounds__(LRow<N>::NT) k_lrow(const LamArgs a) {
  using R = LRow<N>;
  constexpr int N1 = R::N1, N2 = R::N2, LINES = R::LINES;
  __shared__ __align__(16) double2 xch[R::XS];
  __shared__ double2 tw[N];
  const int tid = threadIdx.x, line = tid / N2, j = tid % N2;
  const int M = a.M;
  const int row0 = blockIdx.x * LINES + line;
  const bool in_range = row0 < M;
  const int row = in_range ? row0 : M - 1;
  const size_t img = (size_t)M * N;
  for (int i = tid; i < N; i += R::NT) tw[i] = a.tw_n[i];
  __syncthreads();
  double2 v[N1];
  if constexpr (KIND == L_ROW_ACC) {
    // coils [c0, c1) of problem b: all of them (csplit = 1), or one of csplit groups whose
    // partial sums are added in a fixed order by k_lacc_sum
    const int S = a.csplit > 1 ? a.csplit : 1;
    const int b = blockIdx.y / S, sg = blockIdx.y % S;
    const int per = (a.C + S - 1) / S;
    const int c0 = sg * per, c1 = min(a.C, c0 + per);
    double acc[N1];
#pragma unroll
    for (int s = 0; s < N1; ++s) acc[s] = 0.0;
    for (int c = c0; c < c1; ++c) {
      const double2* t = a.tmp + ((size_t)b * a.C + c) * img + (size_t)row * N;
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) v[n1] = t[natidx<N>(j, n1)];
      fft_fwd<N, typename R::Lay>(v, xch, tw, j, line);
#pragma unroll
      for (int s = 0; s < N1; ++s) acc[s] += v[s].x * v[s].x + v[s].y * v[s].y;
      __syncthreads();
    }
    const double inv = 1.0 / ((double)img * (double)img);
    if (in_range) {
      if (S > 1) {
        double* gp = a.gpart + ((size_t)b * S + sg) * img + (size_t)row * N;
#pragma unroll
        for (int s = 0; s < N1; ++s) gp[specidx<N>(j, s)] = acc[s] * inv;
      } else {
        double2* g = a.g + (size_t)b * img + (size_t)row * N;
#pragma unroll
        for (int s = 0; s < N1; ++s) {
          const int k = specidx<N>(j, s);
          const double prev = a.accumulate ? g[k].x : 0.0;
          g[k] = make_double2(prev + acc[s] * inv, 0.0);
        }
      }
    }
  } else if constexpr (KIND == L_ROW_G || KIND == L_ROW_MASK) {
    double2* t = (KIND == L_ROW_G ? a.g : a.rhat) + (size_t)blockIdx.y * img + (size_t)row * N;
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) v[n1] = t[natidx<N>(j, n1)];
    __syncthreads();
    fft_fwd<N, typename R::Lay>(v, xch, tw, j, line);
    if (in_range) {
#pragma unroll
      for (int s = 0; s < N1; ++s) t[specidx<N>(j, s)] = v[s];
    }
  } else if constexpr (KIND == L_ROW_PROD) {
    const int b = blockIdx.y;
    const int m = (a.nmask == 1) ? 0 : b;
    double2* t = a.g + (size_t)b * img + (size_t)row * N;
    const double2* rh = a.rhat + (size_t)m * img + (size_t)row * N;
#pragma unroll
    for (int s = 0; s < N1; ++s) {
      const int k = specidx<N>(j, s);
      v[s] = cmulc(t[k], rh[k]);  // conj(D g) . D r
    }
    __syncthreads();
    fft_inv<N, typename R::Lay>(v, xch, tw, j, line);
    if (in_range) {
#pragma unroll
      for (int n1 = 0; n1 < N1; ++n1) t[natidx<N>(j, n1)] = v[n1];
    }
  }
}

// g[b] (+)= sum over the csplit coil groups in fixed order
__global__ void __launch_bounds__(256) k_lacc_sum(const LamArgs a, size_t img) {
  const int b = blockIdx.y, S = a.csplit;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < img; i += (size_t)gridDim.x * blockDim.x) {
    double t = a.accumulate ? a.g[(size_t)b * img + i].x : 0.0;
    for (int sg = 0; sg < S; ++sg) t += a.gpart[((size_t)b * S + sg) * img + i];
    a.g[(size_t)b * img + i] = make_double2(t, 0.0);
  }
}

template <int M, int KIND>
static cudaError_t lcol(const LamArgs& a, int nimg, cudaStream_t st) {
  k_lcol<M, KIND><<<dim3(a.N / LW, nimg), LCol<M>::NT, 0, st>>>(a);
  return cudaGetLastError();
}
template <int N, int KIND>
static cudaError_t lrow(const LamArgs& a, int nimg, cudaStream_t st) {
  k_lrow<N, KIND><<<dim3((a.M + LRow<N>::LINES - 1) / LRow<N>::LINES, nimg), LRow<N>::NT, 0, st>>>(a);
  return cudaGetLastError();
}

// the coil accumulation pass, split over up to 16 coil groups (gpart holds B x 16 images) when
// B x rows alone would leave SMs idle
template <int N>
static cudaError_t row_acc(const LamArgs& a0, cudaStream_t st) {
  LamArgs a = a0;
  const int ctas = (a.M + LRow<N>::LINES - 1) / LRow<N>::LINES * a.B;
  a.csplit = (a.gpart != nullptr) ? std::max(1, std::min(std::min(a.C, 16), (2 * 148 + ctas - 1) / ctas)) : 1;
  cudaError_t e;
  if ((e = lrow<N, L_ROW_ACC>(a, a.B * a.csplit, st))) return e;
  if (a.csplit > 1) {
    const size_t img = (size_t)a.M * a.N;
    k_lacc_sum<<<dim3((unsigned)std::min<size_t>(1024, (img + 255) / 256), a.B), 256, 0, st>>>(a, img);
    e = cudaGetLastError();
    if (a.nextra) ++*a.nextra;
  }
  return e;
}

template <int M, int N>
static cudaError_t chunk_mn(const LamArgs& a, cudaStream_t st) {
  cudaError_t e;
  if ((e = lcol<M, L_COL_SENS>(a, a.B * a.C, st))) return e;
  return row_acc<N>(a, st);
}
template <int M, int N>
static cudaError_t tail_mn(const LamArgs& a, cudaStream_t st) {
  cudaError_t e;
  if ((e = lcol<M, L_COL_G>(a, a.B, st))) return e;
  if ((e = lrow<N, L_ROW_G>(a, a.B, st))) return e;
  if ((e = lcol<M, L_COL_MASK>(a, a.nmask, st))) return e;
  if ((e = lrow<N, L_ROW_MASK>(a, a.nmask, st))) return e;
  if ((e = lrow<N, L_ROW_PROD>(a, a.B, st))) return e;
  return lcol<M, L_COL_FINAL>(a, a.B, st);
}

template <int M, int N>
static cudaError_t build_mn(const LamArgs& a, cudaStream_t st) {
  cudaError_t e;
  if ((e = lcol<M, L_COL_SENS>(a, a.B * a.C, st))) return e;
  if ((e = row_acc<N>(a, st))) return e;
  if ((e = lcol<M, L_COL_G>(a, a.B, st))) return e;
  if ((e = lrow<N, L_ROW_G>(a, a.B, st))) return e;
  if ((e = lcol<M, L_COL_MASK>(a, a.nmask, st))) return e;
  if ((e = lrow<N, L_ROW_MASK>(a, a.nmask, st))) return e;
  if ((e = lrow<N, L_ROW_PROD>(a, a.B, st))) return e;
  return lcol<M, L_COL_FINAL>(a, a.B, st);
}

#define SBK_LAM_SIZES(X) X(8) X(16) X(32) X(48) X(64) X(128) X(192) X(256)

template <int M, int WHICH>
static cudaError_t lam_n(const LamArgs& a, cudaStream_t st) {
#define X(n_) \
  if (a.N == n_) return WHICH == 0 ? build_mn<M, n_>(a, st) : (WHICH == 1 ? chunk_mn<M, n_>(a, st) : tail_mn<M, n_>(a, st));
  SBK_LAM_SIZES(X)
#undef X
  return cudaErrorInvalidValue;
}

template <int WHICH>
static cudaError_t lam_mn(const LamArgs& a, cudaStream_t st) {
#define X(m_) \
  if (a.M == m_) return lam_n<m_, WHICH>(a, st);
  SBK_LAM_SIZES(X)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_lambda_build(const LamArgs& a, cudaStream_t st) { return lam_mn<0>(a, st); }
cudaError_t launch_lambda_chunk(const LamArgs& a, cudaStream_t st) { return lam_mn<1>(a, st); }
cudaError_t launch_lambda_tail(const LamArgs& a, cudaStream_t st) { return lam_mn<2>(a, st); }

// ------------------------------------------------------------------ separable (line) masks
// K4S: for a mask constant along d1 (r(nu0, nu1) = r0(nu0), the Cartesian lines of PAPER.md:265)
// the correlation collapses to one dimension:
//   k_c(nu0, nu1) = sum_{q0} r0(nu0 + q0) g0(q0),   g0(q0) = sum_{q1} g(q0, q1)
//                 = (N1 / N^2) sum_c sum_{x1} |(D_0 s_c)(q0, x1)|^2      (Parseval along d1),
// with D_0 the unnormalised length-M DFT down every column and N1 the row length, so the
// build needs one fp64 column FFT per coil column (instead of C + 3 2D FFTs) and k_c depends on
// nu0 only.  Exact (up to rounding) for separable masks; pinned by the same get_k parity tests.
template <int M>
__global__ void __launch_bounds__(LCol<M>::NT) k_lsep_col(const LamArgs a) {
  using Cf = LCol<M>;
  constexpr int N1 = Cf::N1;
  __shared__ __align__(16) double2 xch[Cf::XS];
  __shared__ double2 tw[M];
  static_assert(M * (LW + 1) <= 2 * Cf::XS, "column partials fit the exchange buffer");
  double (*red)[LW + 1] = reinterpret_cast<double (*)[LW + 1]>(xch);  // after the coil loop
  const int tid = threadIdx.x, j = tid / LW, l = tid % LW;
  const int N = a.N, S = a.csplit;
  const int cta = blockIdx.x, sg = blockIdx.y, b = blockIdx.z;
  const int col = cta * LW + l;
  const size_t img = (size_t)M * N;
  for (int i = tid; i < M; i += Cf::NT) tw[i] = a.tw_m[i];
  __syncthreads();
  const int per = (a.C + S - 1) / S, c0 = sg * per, c1 = min(a.C, c0 + per);
  double acc[N1];
#pragma unroll
  for (int q = 0; q < N1; ++q) acc[q] = 0.0;
  for (int c = c0; c < c1; ++c) {
    const float2* sc = a.sens + ((size_t)b * a.C + c) * img;
    double2 v[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) {
      const float2 f = sc[(size_t)natidx<M>(j, n1) * N + col];
      v[n1] = make_double2(f.x, f.y);
    }
    fft_fwd<M, typename Cf::Lay>(v, xch, tw, j, l);
#pragma unroll
    for (int q = 0; q < N1; ++q) acc[q] += v[q].x * v[q].x + v[q].y * v[q].y;
    __syncthreads();  // xch reused by the next coil
  }
#pragma unroll
  for (int q = 0; q < N1; ++q) red[specidx<M>(j, q)][l] = acc[q];
  __syncthreads();
  // this CTA's LW columns summed in a fixed order -> gpart[b][sg][cta][q0]
  const int nct = gridDim.x;
  for (int q0 = tid; q0 < M; q0 += Cf::NT) {
    double t = 0.0;
#pragma unroll
    for (int ll = 0; ll < LW; ++ll) t += red[q0][ll];
    a.gpart[(((size_t)b * S + sg) * nct + cta) * M + q0] = t;
  }
}

// g0(q0) for 32 consecutive q0 per CTA: thread (p, qq) sums partial rows p, p + 8, ... of the
// (coil group, column tile) list for q0 = base + qq (coalesced loads, independent of each other),
// then the 8 chains are added in a fixed order
__global__ void __launch_bounds__(256) k_lsep_g0(const LamArgs a, int nrow) {
  __shared__ double part[8][33];
  const int M = a.M, N = a.N, b = blockIdx.y;
  const int qq = threadIdx.x & 31, p = threadIdx.x >> 5, q0 = blockIdx.x * 32 + qq;
  double t = 0.0;
  if (q0 < M)
    for (int r = p; r < nrow; r += 8) t += a.gpart[((size_t)b * nrow + r) * M + q0];
  part[p][qq] = t;
  __syncthreads();
  if (p == 0 && q0 < M) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += part[k][qq];
    const double img = (double)M * (double)N;
    a.g[(size_t)b * M + q0].x = s * ((double)N / (img * img));
  }
}

// one row nu0 per CTA: k_c(nu0) = sum_q g0(q) r0(nu0 + q) (fixed-order block sum), then
// k = mu k_c + lambda (4 sin^2(pi nu0/M) + 4 sin^2(pi nu1/N)) + gamma and Lambda^{-1} = 1/(N k)
// along the row
__global__ void __launch_bounds__(256) k_lsep_expand(const LamArgs a) {
  __shared__ double red[32];
  const int M = a.M, N = a.N, row = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const int m = (a.nmask == 1) ? 0 : b;
  double v = 0.0;
  for (int q = tid; q < M; q += blockDim.x)
    if (a.mask[(size_t)m * a.mask_bstride + (size_t)((row + q) % M) * N]) v += a.g[(size_t)b * M + q].x;
  const double kc = block_sum(v, red);
  if (tid == 0) red[0] = kc;
  __syncthreads();
  const double kcr = red[0];
  const size_t img = (size_t)M * N;
  const double PI = 3.14159265358979323846;
  const double sr = sin(PI * (double)row / (double)M);
  for (int col = tid; col < N; col += blockDim.x) {
    const double sc = sin(PI * (double)col / (double)N);
    const double k = a.mu * kcr + a.lam * (4.0 * sr * sr + 4.0 * sc * sc) + a.gam;
    const size_t gi = (size_t)b * img + (size_t)row * N + col;
    a.k_out[gi] = k;
    if (!(fabs(k) > 1e-14) || !isfinite(k)) atomicExch(a.bad, 1);
    a.lam_inv[gi] = (float)(1.0 / ((double)img * k));
  }
}

template <int M>
static cudaError_t lsep_m(const LamArgs& a, cudaStream_t st) {
  const int nct = a.N / LW;
  k_lsep_col<M><<<dim3(nct, a.csplit, a.B), LCol<M>::NT, 0, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_lsep_g0<<<dim3((M + 31) / 32, a.B), 256, 0, st>>>(a, a.csplit * nct);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  k_lsep_expand<<<dim3(M, a.B), 256, 0, st>>>(a);
  return cudaGetLastError();
}

// csplit coil groups, gpart >= B * csplit * (N / 8) * M doubles, g >= B * M (g0 in .x)
cudaError_t launch_lambda_sep(const LamArgs& a, cudaStream_t st) {
  if (a.N % LW != 0) return cudaErrorInvalidValue;
  switch (a.M) {
#define X(m_) \
  case m_: return lsep_m<m_>(a, st);
    SBK_LAM_SIZES(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

__global__ void __launch_bounds__(256) k_lexpand3(const Lam3Args a) {
  const size_t pn = (size_t)a.D1 * a.D2, img = pn * a.D0;
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= img) return;
  const int x = (int)(i / pn);
  const size_t yz = i % pn;
  const int y = (int)(yz / a.D2), z = (int)(yz % a.D2);
  const double PI = 3.14159265358979323846;
  const double s0 = sin(PI * x / (double)a.D0), s1 = sin(PI * y / (double)a.D1), s2 = sin(PI * z / (double)a.D2);
  const double kd = 4.0 * (s0 * s0 + s1 * s1 + s2 * s2);
  const double kc = a.kc2[(size_t)b * pn + yz] / (double)a.D0;
  const double k = a.mu * kc + a.lam * kd + a.gam;
  const size_t gi = (size_t)b * img + i;
  a.k_out[gi] = k;
  if (!(fabs(k) > 1e-14) || !isfinite(k)) atomicExch(a.bad, 1);
  a.lam_inv[gi] = (float)(1.0 / ((double)img * k));
}

cudaError_t launch_lambda_expand3(const Lam3Args& a, cudaStream_t st) {
  const size_t img = (size_t)a.D0 * a.D1 * a.D2;
  k_lexpand3<<<dim3((unsigned)((img + 255) / 256), a.B), 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace sbk
