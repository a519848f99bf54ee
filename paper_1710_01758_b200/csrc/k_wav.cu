// k_wav.cu — the paper's Daubechies-4 wavelet W (reading A32; SURVEY 8(f)
// NEXT-2) for the SB shrink step (Algorithm 1 steps 8, 11 and the gamma W^H(d_w - b_w) part
// of step 4).  W^H W = I, so A and Lambda are unchanged.
//
// Periodized D4 (h = [1+r3, 3+r3, 3-r3, 1-r3]/(4 sqrt2), g_m = (-1)^m h_{3-m}):
//   analysis  a_k = sum_m h_m x_{(2k+m) mod n},  d_k = sum_m g_m x_{(2k+m) mod n}
//   synthesis x_j = sum_{m = j mod 2, +2} h_m a_k + g_m d_k,  k = ((j - m) mod n) / 2
// in the Mallat layout of the Haar path: per level, along d0, d1[, d2] on the approximation
// block.  Unlike Haar, D4 is not local to 2^L blocks, so each (level, axis) is one pass: a CTA
// stages LW whole lines of the block in shared memory and writes the transformed lines back.
#include <algorithm>

#include "kernels.cuh"

namespace sbk {

__constant__ float c_d4h[4] = {0.48296291314453414f, 0.83651630373780790f, 0.22414386804201339f,
                               -0.12940952255126037f};
__constant__ float c_d4g[4] = {-0.12940952255126037f, -0.22414386804201339f, 0.83651630373780790f,
                               -0.48296291314453414f};

constexpr int LW = 32;  // lines per CTA

// One (level, axis) pass over the block n[0] x n[1] x n[2] (top-left corner of the image
// E0 x E1 x E2) along `axis`.  in may equal out.  acc != 0 (inverse only): out += scale * x.
template <bool FWD>
__global__ void __launch_bounds__(256) kw_d4_pass(const float2* in, float2* out, int E1, int E2, int n0, int n1,
                                                  int n2, int axis, size_t img, float scale, int acc) {
  extern __shared__ float2 ln[];  // [LW][na]
  const int b = blockIdx.y;
  const int nb[3] = {n0, n1, n2};
  const size_t S[3] = {(size_t)E1 * E2, (size_t)E2, 1};
  const int na = nb[axis];
  // the two other axes: o1 (slower), o2 (faster, the contiguous one when axis != 2)
  const int o1 = axis == 0 ? 1 : 0, o2 = axis == 2 ? 1 : 2;
  const int nlines = nb[o1] * nb[o2];
  const int l0 = blockIdx.x * LW;
  const int nl = min(LW, nlines - l0);
  const size_t boff = (size_t)b * img;
  auto base = [&](int l) {
    const int li = l0 + l;
    return boff + (size_t)(li / nb[o2]) * S[o1] + (size_t)(li % nb[o2]) * S[o2];
  };
  const bool contig = axis == 2 || (axis == 1 && E2 == 1);
  for (int e = threadIdx.x; e < nl * na; e += blockDim.x) {
    int l, j;
    if (contig) { l = e / na; j = e % na; } else { l = e % nl; j = e / nl; }
    ln[l * na + j] = in[base(l) + (size_t)j * S[axis]];
  }
  __syncthreads();
  const int h = na / 2;
  if constexpr (FWD) {
    for (int e = threadIdx.x; e < nl * h; e += blockDim.x) {
      int l, k;
      if (contig) { l = e / h; k = e % h; } else { l = e % nl; k = e / nl; }
      float2 a = make_float2(0.f, 0.f), d = a;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const float2 v = ln[l * na + (2 * k + m) % na];
        a.x += c_d4h[m] * v.x;
        a.y += c_d4h[m] * v.y;
        d.x += c_d4g[m] * v.x;
        d.y += c_d4g[m] * v.y;
      }
      const size_t bl = base(l);
      out[bl + (size_t)k * S[axis]] = a;
      out[bl + (size_t)(h + k) * S[axis]] = d;
    }
  } else {
    for (int e = threadIdx.x; e < nl * na; e += blockDim.x) {
      int l, j;
      if (contig) { l = e / na; j = e % na; } else { l = e % nl; j = e / nl; }
      float2 x = make_float2(0.f, 0.f);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int m = (j & 1) + 2 * t;
        const int k = (((j - m) % na + na) % na) / 2;
        const float2 a = ln[l * na + k], d = ln[l * na + h + k];
        x.x += c_d4h[m] * a.x + c_d4g[m] * d.x;
        x.y += c_d4h[m] * a.y + c_d4g[m] * d.y;
      }
      const size_t gi = base(l) + (size_t)j * S[axis];
      if (acc) {
        const float2 o = out[gi];
        out[gi] = make_float2(o.x + scale * x.x, o.y + scale * x.y);
      } else {
        out[gi] = x;
      }
    }
  }
}

// z = w + b_w ; d = shrink(z, t) ; b_w <- z - d ; w <- d - b_w
__global__ void __launch_bounds__(256) kw_shrink(float2* w, float2* bw, size_t n, float t) {
  const size_t off = (size_t)blockIdx.y * n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const size_t gi = off + i;
    const float2 z = make_float2(w[gi].x + bw[gi].x, w[gi].y + bw[gi].y);
    const float a = sqrtf(z.x * z.x + z.y * z.y);
    const float s = (a > t) ? (a - t) / a : 0.f;
    const float2 d = make_float2(z.x * s, z.y * s);
    const float2 bn = make_float2(z.x - d.x, z.y - d.y);
    bw[gi] = bn;
    w[gi] = make_float2(d.x - bn.x, d.y - bn.y);
  }
}

// Full D4 wavelet part of the SB step for B problems of E0 x E1 x E2 (nd = 2: E2 = 1):
//   wbuf = W x ; shrink/Bregman with b_w ; rhs += gamma W^H (d_w - b_w)
cudaError_t launch_d4_sb(const float2* x, float2* wbuf, float2* bw, float2* rhs, int B, int E0, int E1, int E2, int nd,
                         int levels, float gamma, cudaStream_t st, int* nlaunch) {
  const size_t img = (size_t)E0 * E1 * E2;
  int n[3] = {E0, E1, E2};
  int cnt = 0;
  auto pass = [&](bool fwd, const float2* in, float2* out, int lvl, int axis, int acc) -> cudaError_t {
    int nb[3] = {n[0] >> lvl, n[1] >> lvl, nd == 3 ? (n[2] >> lvl) : 1};
    const int o1 = axis == 0 ? 1 : 0, o2 = axis == 2 ? 1 : 2;
    const int nlines = nb[o1] * nb[o2];
    const dim3 grid((nlines + LW - 1) / LW, B);
    const size_t sm = (size_t)LW * nb[axis] * sizeof(float2);
    if (fwd)
      kw_d4_pass<true><<<grid, 256, sm, st>>>(in, out, E1, E2, nb[0], nb[1], nb[2], axis, img, 1.f, 0);
    else
      kw_d4_pass<false><<<grid, 256, sm, st>>>(in, out, E1, E2, nb[0], nb[1], nb[2], axis, img, gamma, acc);
    ++cnt;
    return cudaGetLastError();
  };
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(kw_d4_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(kw_d4_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr = true;
  }
  cudaError_t e;
  const float2* src = x;
  for (int lvl = 0; lvl < levels; ++lvl)
    for (int axis = 0; axis < nd; ++axis) {
      if ((e = pass(true, src, wbuf, lvl, axis, 0))) return e;
      src = wbuf;
    }
  if (levels < 1) return cudaErrorInvalidValue;  // D4 needs >= 1 level (checked at sb_set_wavelet)
  kw_shrink<<<dim3((unsigned)std::min<size_t>(1024, (img + 255) / 256), B), 256, 0, st>>>(wbuf, bw, img, 1.f / gamma);
  ++cnt;
  if ((e = cudaGetLastError())) return e;
  for (int lvl = levels - 1; lvl >= 0; --lvl)
    for (int axis = nd - 1; axis >= 0; --axis) {
      const bool last = (lvl == 0 && axis == 0);
      if ((e = pass(false, wbuf, last ? rhs : wbuf, lvl, axis, last ? 1 : 0))) return e;
    }
  if (nlaunch) *nlaunch += cnt;
  return cudaSuccess;
}

}  // namespace sbk
