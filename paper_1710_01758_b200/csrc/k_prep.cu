// k_prep.cu — data preprocessing of the paper's Methods:
//   * sensitivity normalisation with support masking
//       S_hat_i = [sum_j S_j^H S_j]^{-1/2} S_i  inside the subject, 0 outside;
//   * coil-image normalisation   m_i <- S_hat_i sum_j S_hat_j^H m_j;
//   * SVD coil compression (Huang et al. 2008): coil covariance
//       G = sum_n d(n) d(n)^H (deterministic fp64 block reduction on the device), Hermitian
//       eigen-decomposition on the host (cyclic complex Jacobi, C <= 64), A = U[:, :C']^H,
//       virtual coils out_k = sum_c A_kc in_c for the data and the maps.
// All HBM-bound elementwise/reduction passes; coil vectors are read once per pixel.
#include <algorithm>
#include <cmath>
#include <complex>
#include <vector>

#include "kernels.cuh"

namespace sbk {

__global__ void __launch_bounds__(256) kpp_normalize_sens(const float2* __restrict__ s, const uint8_t* support,
                                                          size_t sup_bstride, int C, size_t npix, float2* out) {
  const int b = blockIdx.y;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < npix; i += (size_t)gridDim.x * blockDim.x) {
    float r2 = 0.f;
    for (int c = 0; c < C; ++c) {
      const float2 v = s[((size_t)b * C + c) * npix + i];
      r2 += v.x * v.x + v.y * v.y;
    }
    const bool keep = r2 > 0.f && (support == nullptr || support[(size_t)b * sup_bstride + i] != 0);
    const float f = keep ? rsqrtf(r2) : 0.f;
    for (int c = 0; c < C; ++c) {
      const size_t gi = ((size_t)b * C + c) * npix + i;
      const float2 v = s[gi];
      out[gi] = make_float2(v.x * f, v.y * f);
    }
  }
}

__global__ void __launch_bounds__(256) kpp_normalize_images(const float2* __restrict__ m, const float2* __restrict__ sh,
                                                            int C, size_t npix, float2* out) {
  const int b = blockIdx.y;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < npix; i += (size_t)gridDim.x * blockDim.x) {
    float2 x = make_float2(0.f, 0.f);
    for (int c = 0; c < C; ++c) {
      const size_t gi = ((size_t)b * C + c) * npix + i;
      const float2 t = cmulc(sh[gi], m[gi]);
      x.x += t.x;
      x.y += t.y;
    }
    for (int c = 0; c < C; ++c) {
      const size_t gi = ((size_t)b * C + c) * npix + i;
      out[gi] = cmul(sh[gi], x);
    }
  }
}

// Block partials of G[c][c'] = sum_n d_c(n) conj(d_c'(n)) over a pixel range (fp64, fixed
// order): pixels staged in shared memory in chunks of 64, entries (c, c') spread over threads.
constexpr int GP = 64;
__global__ void __launch_bounds__(256) kpp_gram_partial(const float2* __restrict__ d, int C, size_t npix,
                                                        size_t per_block, double2* part) {
  extern __shared__ float2 tile[];  // [C][GP]
  const int b = blockIdx.y, blk = blockIdx.x;
  const size_t p0 = (size_t)blk * per_block, p1 = std::min(npix, p0 + per_block);
  const int E = C * C;
  double2 acc[4] = {};
  for (size_t q = p0; q < p1; q += GP) {
    const int n = (int)std::min<size_t>(GP, p1 - q);
    __syncthreads();
    for (int e = threadIdx.x; e < C * GP; e += blockDim.x) {
      const int c = e / GP, k = e % GP;
      tile[e] = k < n ? d[((size_t)b * C + c) * npix + q + k] : make_float2(0.f, 0.f);
    }
    __syncthreads();
    for (int r = 0; r < 4; ++r) {
      const int e = threadIdx.x + r * blockDim.x;
      if (e >= E) break;
      const int c = e / C, c2 = e % C;
      double sx = 0.0, sy = 0.0;
      for (int k = 0; k < n; ++k) {
        const float2 u = tile[c * GP + k], v = tile[c2 * GP + k];
        sx += (double)u.x * v.x + (double)u.y * v.y;  // u conj(v)
        sy += (double)u.y * v.x - (double)u.x * v.y;
      }
      acc[r].x += sx;
      acc[r].y += sy;
    }
  }
  for (int r = 0; r < 4; ++r) {
    const int e = threadIdx.x + r * blockDim.x;
    if (e < E) part[((size_t)b * gridDim.x + blk) * E + e] = acc[r];
  }
}

__global__ void kpp_gram_sum(const double2* part, int nblk, int E, double2* G) {
  const int b = blockIdx.y;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < E; e += gridDim.x * blockDim.x) {
    double2 s = make_double2(0.0, 0.0);
    for (int k = 0; k < nblk; ++k) {
      const double2 v = part[((size_t)b * nblk + k) * E + e];
      s.x += v.x;
      s.y += v.y;
    }
    G[(size_t)b * E + e] = s;
  }
}

// out[b][k][i] = sum_c A[b][k][c] in[b][c][i]
__global__ void __launch_bounds__(256) kpp_apply(const float2* __restrict__ in, const float2* __restrict__ A, int C,
                                                 int K, size_t npix, float2* out) {
  extern __shared__ float2 As[];  // [K][C]
  const int b = blockIdx.y;
  for (int e = threadIdx.x; e < K * C; e += blockDim.x) As[e] = A[(size_t)b * K * C + e];
  __syncthreads();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < npix; i += (size_t)gridDim.x * blockDim.x) {
    float2 v[64];
    for (int c = 0; c < C; ++c) v[c] = in[((size_t)b * C + c) * npix + i];
    for (int k = 0; k < K; ++k) {
      float2 o = make_float2(0.f, 0.f);
      for (int c = 0; c < C; ++c) {
        const float2 t = cmul(As[k * C + c], v[c]);
        o.x += t.x;
        o.y += t.y;
      }
      out[((size_t)b * K + k) * npix + i] = o;
    }
  }
}

static int grid_for(size_t n) { return (int)std::min<size_t>(2048, (n + 255) / 256); }

cudaError_t launch_normalize_sens(const float2* s, const uint8_t* sup, size_t sup_bstride, int B, int C, size_t npix,
                                  float2* out, cudaStream_t st) {
  kpp_normalize_sens<<<dim3(grid_for(npix), B), 256, 0, st>>>(s, sup, sup_bstride, C, npix, out);
  return cudaGetLastError();
}

cudaError_t launch_normalize_images(const float2* m, const float2* sh, int B, int C, size_t npix, float2* out,
                                    cudaStream_t st) {
  kpp_normalize_images<<<dim3(grid_for(npix), B), 256, 0, st>>>(m, sh, C, npix, out);
  return cudaGetLastError();
}

cudaError_t launch_gram(const float2* d, int B, int C, size_t npix, double2* part, int nblk, double2* G,
                        cudaStream_t st) {
  const size_t per = (npix + nblk - 1) / nblk;
  kpp_gram_partial<<<dim3(nblk, B), 256, C * GP * sizeof(float2), st>>>(d, C, npix, per, part);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  kpp_gram_sum<<<dim3(4, B), 256, 0, st>>>(part, nblk, C * C, G);
  return cudaGetLastError();
}

cudaError_t launch_coil_apply(const float2* in, const float2* A, int B, int C, int K, size_t npix, float2* out,
                              cudaStream_t st) {
  kpp_apply<<<dim3(grid_for(npix), B), 256, K * C * sizeof(float2), st>>>(in, A, C, K, npix, out);
  return cudaGetLastError();
}

// Hermitian eigen-decomposition by cyclic complex Jacobi rotations (host, fp64, n <= 64):
// G (row-major n x n) -> eigenvalues w (descending) and eigenvectors U (columns).
void hermitian_eig(int n, const std::complex<double>* G, double* w, std::complex<double>* U) {
  using cd = std::complex<double>;
  std::vector<cd> a(G, G + (size_t)n * n);
  std::vector<cd> v((size_t)n * n, cd(0.0));
  for (int i = 0; i < n; ++i) v[(size_t)i * n + i] = 1.0;
  auto A = [&](int i, int j) -> cd& { return a[(size_t)i * n + j]; };
  auto V = [&](int i, int j) -> cd& { return v[(size_t)i * n + j]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) (i == j ? tot : off) += std::norm(A(i, j));
    if (off <= 1e-30 * (tot + off) || off == 0.0) break;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const cd apq = A(p, q);
        const double mag = std::abs(apq);
        if (mag == 0.0) continue;
        // 2x2 Hermitian block [[app, apq],[conj(apq), aqq]]: rotation zeroing apq
        const double app = A(p, p).real(), aqq = A(q, q).real();
        const cd ph = apq / mag;  // e^{i phi}
        const double theta = 0.5 * std::atan2(2.0 * mag, aqq - app);
        const double c = std::cos(theta), s = std::sin(theta);
        // J: columns p, q  ->  p' = c p - s conj(ph) q ,  q' = s ph p + c q   (unitary)
        for (int k = 0; k < n; ++k) {  // A <- A J
          const cd akp = A(k, p), akq = A(k, q);
          A(k, p) = c * akp - s * std::conj(ph) * akq;
          A(k, q) = s * ph * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {  // A <- J^H A
          const cd apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * ph * aqk;
          A(q, k) = s * std::conj(ph) * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {  // V <- V J
          const cd vkp = V(k, p), vkq = V(k, q);
          V(k, p) = c * vkp - s * std::conj(ph) * vkq;
          V(k, q) = s * ph * vkp + c * vkq;
        }
      }
  }
  std::vector<int> idx(n);
  for (int i = 0; i < n; ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](int x, int y) { return A(x, x).real() > A(y, y).real(); });
  for (int k = 0; k < n; ++k) {
    w[k] = A(idx[k], idx[k]).real();
    for (int i = 0; i < n; ++i) U[(size_t)i * n + k] = V(i, idx[k]);
  }
}

}  // namespace sbk
