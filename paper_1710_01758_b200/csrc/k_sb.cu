// k_sb.cu — K5: Split Bregman shrink + Bregman update + regulariser RHS, one pass
// (Algorithm 1 steps 6-11 and the lambda/gamma part of step 4):
//
//   z_d = D_d x + b_d ; d_d = shrink(z_d, 1/lambda) ; b_d <- z_d - d_d      (d = x, y)
//   z_w = W x + b_w   ; d_w = shrink(z_w, 1/gamma)  ; b_w <- z_w - d_w
//   rhs_reg = lambda sum_d D_d^H (d_d - b_d) + gamma W^H (d_w - b_w)
//
// shrink(z, t) = z max(|z| - t, 0)/|z| (reading A9), literal thresholds (reading A8).
// D_d periodic first differences.  W = L-level orthonormal Haar in the
// Mallat layout (reading A6); Haar with L levels is local to 2^L x 2^L blocks, so one CTA
// tile (TH x TW, multiples of 2^L) computes W, W^H locally and addresses b_w at the global
// Mallat positions.  D_d^H needs (d - b) at i+1 / j+1: recomputed from a one-pixel halo, so
// b_x, b_y are double-buffered (read old, write new).
#include "sb_tile.cuh"

namespace sbk {

template <int TT, bool FIX>
__global__ void __launch_bounds__(256) k_sb_update(const SbArgs a) {
  __shared__ SbTile<TT> S;
  pdl_trigger();
  pdl_wait();
  sb_tile<TT, FIX, 256>(a, S, blockIdx.x, blockIdx.y, blockIdx.z);
}

cudaError_t launch_sb_update(const SbArgs& a, cudaStream_t st) {
  const int TH = a.M < SBT ? a.M : SBT, TW = a.N < SBT ? a.N : SBT;
  if (a.M % TH || a.N % TW || (TH % (1 << a.levels)) || (TW % (1 << a.levels))) return cudaErrorInvalidValue;
  const bool small = (int64_t)(a.M / TH) * (a.N / TW) * a.B < 2 * 148;
  if (small && a.M >= 16 && a.N >= 16 && a.M % 16 == 0 && a.N % 16 == 0 && (16 % (1 << a.levels)) == 0)
    return launch_ex(k_sb_update<16, true>, dim3(a.M / 16, a.N / 16, a.B), dim3(256), 0, st, 0, a);
  if (a.M % SBT == 0 && a.N % SBT == 0)
    return launch_ex(k_sb_update<SBT, true>, dim3(a.M / SBT, a.N / SBT, a.B), dim3(256), 0, st, 0, a);
  return launch_ex(k_sb_update<SBT, false>, dim3(a.M / TH, a.N / TW, a.B), dim3(256), 0, st, 0, a);
}

}  // namespace sbk

// ------------------------------------------------------------------ 3D (BASELINE config 5)
// Same step in 3D: anisotropic TV with d_x, d_y, d_z (reading A10) and the 3D Mallat Haar
// (per level, along d0 then d1 then d2: 8 subbands, reading A6), on 8x8x8 tiles (L <= 3).
namespace sbk {

constexpr int S3 = 8;

// FIX: every edge is a multiple of S3, so the tile is S3^3 at compile time (index math as shifts)
template <bool FIX>
__global__ void __launch_bounds__(256) k_sb_update3(const SbArgs a) {
  __shared__ float2 xs[S3 + 2][S3 + 2][S3 + 2];
  __shared__ float2 v0[S3 + 1][S3][S3];
  __shared__ float2 v1[S3][S3 + 1][S3];
  __shared__ float2 v2[S3][S3][S3 + 1];
  __shared__ float2 wa[S3][S3][S3];
  __shared__ float2 wv[S3][S3][S3];
  const int D0 = a.M, D1 = a.N, D2 = a.D2, L = a.levels;
  const int T0 = FIX ? S3 : (D0 < S3 ? D0 : S3), T1 = FIX ? S3 : (D1 < S3 ? D1 : S3),
            T2 = FIX ? S3 : (D2 < S3 ? D2 : S3);
  const int n1t = D1 / T1, n2t = D2 / T2;
  const int t = blockIdx.x;
  const int i0 = (t / (n1t * n2t)) * T0, j0 = ((t / n2t) % n1t) * T1, k0 = (t % n2t) * T2;
  const int b = blockIdx.y;
  const size_t img = (size_t)D0 * D1 * D2, boff = (size_t)b * img;
  auto G = [&](int i, int j, int k) { return boff + ((size_t)i * D1 + j) * D2 + k; };
  const int tid = threadIdx.x;
  constexpr int nt = 256;  // launch_sb_update3's block size
  const bool do_tv = a.lam != 0.f, do_w = a.gam != 0.f;
  const float tl = do_tv ? 1.f / a.lam : 0.f, tg = do_w ? 1.f / a.gam : 0.f;
  pdl_trigger();
  pdl_wait();

  const int X0 = T0 + 2, X1 = T1 + 2, X2 = T2 + 2;
  // x / d, x % d for the Haar pair indices (d a power of two when FIX)
  auto dv = [&](int x, int d) { return FIX ? (x >> (31 - __clz(d))) : x / d; };
  auto md = [&](int x, int d) { return FIX ? (x & (d - 1)) : x % d; };
  for (int e = tid; e < X0 * X1 * X2; e += nt) {
    const int u = e / (X1 * X2), v = (e / X2) % X1, w = e % X2;
    xs[u][v][w] = a.x[G((i0 + u - 1 + D0) % D0, (j0 + v - 1 + D1) % D1, (k0 + w - 1 + D2) % D2)];
  }
  if (do_tv) {
    for (int e = tid; e < (T0 + 1) * T1 * T2; e += nt) {
      const int u = e / (T1 * T2), v = (e / T2) % T1, w = e % T2;
      v0[u][v][w] = a.bx_in[G((i0 + u) % D0, j0 + v, k0 + w)];
    }
    for (int e = tid; e < T0 * (T1 + 1) * T2; e += nt) {
      const int u = e / ((T1 + 1) * T2), v = (e / T2) % (T1 + 1), w = e % T2;
      v1[u][v][w] = a.by_in[G(i0 + u, (j0 + v) % D1, k0 + w)];
    }
    for (int e = tid; e < T0 * T1 * (T2 + 1); e += nt) {
      const int u = e / (T1 * (T2 + 1)), v = (e / (T2 + 1)) % T1, w = e % (T2 + 1);
      v2[u][v][w] = a.bz_in[G(i0 + u, j0 + v, (k0 + w) % D2)];
    }
  }
  __syncthreads();

  if (do_tv) {
    // z_d = D_d x + b_d ; d_d = shrink(z_d, 1/lambda) ; b_d <- z_d - d_d ; keep d_d - b_d
    for (int e = tid; e < (T0 + 1) * T1 * T2; e += nt) {
      const int u = e / (T1 * T2), v = (e / T2) % T1, w = e % T2;
      const float2 xc = xs[u + 1][v + 1][w + 1], xm = xs[u][v + 1][w + 1], bo = v0[u][v][w];
      const float2 z = make_float2(xc.x - xm.x + bo.x, xc.y - xm.y + bo.y);
      const float2 d = shrinkc(z, tl);
      const float2 bn = make_float2(z.x - d.x, z.y - d.y);
      v0[u][v][w] = make_float2(d.x - bn.x, d.y - bn.y);
      if (u < T0) a.bx_out[G(i0 + u, j0 + v, k0 + w)] = bn;
    }
    for (int e = tid; e < T0 * (T1 + 1) * T2; e += nt) {
      const int u = e / ((T1 + 1) * T2), v = (e / T2) % (T1 + 1), w = e % T2;
      const float2 xc = xs[u + 1][v + 1][w + 1], xm = xs[u + 1][v][w + 1], bo = v1[u][v][w];
      const float2 z = make_float2(xc.x - xm.x + bo.x, xc.y - xm.y + bo.y);
      const float2 d = shrinkc(z, tl);
      const float2 bn = make_float2(z.x - d.x, z.y - d.y);
      v1[u][v][w] = make_float2(d.x - bn.x, d.y - bn.y);
      if (v < T1) a.by_out[G(i0 + u, j0 + v, k0 + w)] = bn;
    }
    for (int e = tid; e < T0 * T1 * (T2 + 1); e += nt) {
      const int u = e / (T1 * (T2 + 1)), v = (e / (T2 + 1)) % T1, w = e % (T2 + 1);
      const float2 xc = xs[u + 1][v + 1][w + 1], xm = xs[u + 1][v + 1][w], bo = v2[u][v][w];
      const float2 z = make_float2(xc.x - xm.x + bo.x, xc.y - xm.y + bo.y);
      const float2 d = shrinkc(z, tl);
      const float2 bn = make_float2(z.x - d.x, z.y - d.y);
      v2[u][v][w] = make_float2(d.x - bn.x, d.y - bn.y);
      if (w < T2) a.bz_out[G(i0 + u, j0 + v, k0 + w)] = bn;
    }
  }

  if (do_w) {
    for (int e = tid; e < T0 * T1 * T2; e += nt) {
      const int u = e / (T1 * T2), v = (e / T2) % T1, w = e % T2;
      wa[u][v][w] = xs[u + 1][v + 1][w + 1];
    }
    __syncthreads();
    const float h = 0.70710678118654752440f;
    // forward: per level, Haar along d0, then d1, then d2 on the current approximation block
    for (int lv = 1; lv <= L; ++lv) {
      const int e0 = T0 >> (lv - 1), e1 = T1 >> (lv - 1), e2 = T2 >> (lv - 1);
      for (int ax = 0; ax < 3; ++ax) {
        const int n = e0 * e1 * e2 / 2;  // pairs along axis ax
        float2 lo = make_float2(0.f, 0.f), hi = lo;
        int p0 = 0, p1 = 0, p2 = 0;
        const bool act = tid < n;  // <= 256 pairs at an 8^3 tile
        if (act) {
          if (ax == 0) { p0 = dv(tid, e1 * e2); p1 = md(dv(tid, e2), e1); p2 = md(tid, e2); }
          else if (ax == 1) { p0 = dv(tid, (e1 / 2) * e2); p1 = md(dv(tid, e2), e1 / 2); p2 = md(tid, e2); }
          else { p0 = dv(tid, e1 * (e2 / 2)); p1 = md(dv(tid, e2 / 2), e1); p2 = md(tid, e2 / 2); }
          float2 ev, od;
          if (ax == 0) { ev = wa[2 * p0][p1][p2]; od = wa[2 * p0 + 1][p1][p2]; }
          else if (ax == 1) { ev = wa[p0][2 * p1][p2]; od = wa[p0][2 * p1 + 1][p2]; }
          else { ev = wa[p0][p1][2 * p2]; od = wa[p0][p1][2 * p2 + 1]; }
          lo = make_float2(h * (ev.x + od.x), h * (ev.y + od.y));
          hi = make_float2(h * (ev.x - od.x), h * (ev.y - od.y));
        }
        __syncthreads();
        if (act) {
          if (ax == 0) { wa[p0][p1][p2] = lo; wa[e0 / 2 + p0][p1][p2] = hi; }
          else if (ax == 1) { wa[p0][p1][p2] = lo; wa[p0][e1 / 2 + p1][p2] = hi; }
          else { wa[p0][p1][p2] = lo; wa[p0][p1][e2 / 2 + p2] = hi; }
        }
        __syncthreads();
      }
    }
    // shrink in the coefficient domain; b_w at the global Mallat positions
    for (int e = tid; e < T0 * T1 * T2; e += nt) {
      const int u = e / (T1 * T2), v = (e / T2) % T1, w = e % T2;
      int lv = 1, hi0 = 0, hi1 = 0, hi2 = 0, ca = u, cb = v, cc = w;
      bool ll = true;
      for (; lv <= L; ++lv) {
        const int h0 = T0 >> lv, h1 = T1 >> lv, h2 = T2 >> lv;
        if (u < h0 && v < h1 && w < h2) continue;
        hi0 = u >= h0;
        hi1 = v >= h1;
        hi2 = w >= h2;
        ca = u - hi0 * h0;
        cb = v - hi1 * h1;
        cc = w - hi2 * h2;
        ll = false;
        break;
      }
      int gu, gv, gw;
      if (ll) {
        gu = (i0 >> L) + u;
        gv = (j0 >> L) + v;
        gw = (k0 >> L) + w;
      } else {
        gu = (hi0 ? (D0 >> lv) : 0) + (i0 >> lv) + ca;
        gv = (hi1 ? (D1 >> lv) : 0) + (j0 >> lv) + cb;
        gw = (hi2 ? (D2 >> lv) : 0) + (k0 >> lv) + cc;
      }
      const size_t gi = G(gu, gv, gw);
      const float2 wc = wa[u][v][w], bo = a.bw[gi];
      const float2 z = make_float2(wc.x + bo.x, wc.y + bo.y);
      const float2 d = shrinkc(z, tg);
      const float2 bn = make_float2(z.x - d.x, z.y - d.y);
      a.bw[gi] = bn;
      wv[u][v][w] = make_float2(d.x - bn.x, d.y - bn.y);
    }
    __syncthreads();
    // inverse: coarsest level first, axes in reverse order
    for (int lv = L; lv >= 1; --lv) {
      const int e0 = T0 >> (lv - 1), e1 = T1 >> (lv - 1), e2 = T2 >> (lv - 1);
      for (int ax = 2; ax >= 0; --ax) {
        const int n = e0 * e1 * e2 / 2;
        float2 ev = make_float2(0.f, 0.f), od = ev;
        int p0 = 0, p1 = 0, p2 = 0;
        const bool act = tid < n;
        if (act) {
          float2 lo, hi;
          if (ax == 0) { p0 = dv(tid, e1 * e2); p1 = md(dv(tid, e2), e1); p2 = md(tid, e2); lo = wv[p0][p1][p2]; hi = wv[e0 / 2 + p0][p1][p2]; }
          else if (ax == 1) { p0 = dv(tid, (e1 / 2) * e2); p1 = md(dv(tid, e2), e1 / 2); p2 = md(tid, e2); lo = wv[p0][p1][p2]; hi = wv[p0][e1 / 2 + p1][p2]; }
          else { p0 = dv(tid, e1 * (e2 / 2)); p1 = md(dv(tid, e2 / 2), e1); p2 = md(tid, e2 / 2); lo = wv[p0][p1][p2]; hi = wv[p0][p1][e2 / 2 + p2]; }
          ev = make_float2(h * (lo.x + hi.x), h * (lo.y + hi.y));
          od = make_float2(h * (lo.x - hi.x), h * (lo.y - hi.y));
        }
        __syncthreads();
        if (act) {
          if (ax == 0) { wv[2 * p0][p1][p2] = ev; wv[2 * p0 + 1][p1][p2] = od; }
          else if (ax == 1) { wv[p0][2 * p1][p2] = ev; wv[p0][2 * p1 + 1][p2] = od; }
          else { wv[p0][p1][2 * p2] = ev; wv[p0][p1][2 * p2 + 1] = od; }
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();
  for (int e = tid; e < T0 * T1 * T2; e += nt) {
    const int u = e / (T1 * T2), v = (e / T2) % T1, w = e % T2;
    float2 out = make_float2(0.f, 0.f);
    if (do_tv) {
      const float2 a0 = v0[u][v][w], a1 = v0[u + 1][v][w];
      const float2 b0 = v1[u][v][w], b1 = v1[u][v + 1][w];
      const float2 c0 = v2[u][v][w], c1 = v2[u][v][w + 1];
      out.x = a.lam * ((a0.x - a1.x) + (b0.x - b1.x) + (c0.x - c1.x));
      out.y = a.lam * ((a0.y - a1.y) + (b0.y - b1.y) + (c0.y - c1.y));
    }
    if (do_w) {
      out.x += a.gam * wv[u][v][w].x;
      out.y += a.gam * wv[u][v][w].y;
    }
    a.rhs[G(i0 + u, j0 + v, k0 + w)] = out;
  }
}

cudaError_t launch_sb_update3(const SbArgs& a, cudaStream_t st) {
  const int T0 = a.M < S3 ? a.M : S3, T1 = a.N < S3 ? a.N : S3, T2 = a.D2 < S3 ? a.D2 : S3;
  const int q = 1 << a.levels;
  if (a.M % T0 || a.N % T1 || a.D2 % T2 || T0 % q || T1 % q || T2 % q) return cudaErrorInvalidValue;
  const int tiles = (a.M / T0) * (a.N / T1) * (a.D2 / T2);
  if (a.M % S3 == 0 && a.N % S3 == 0 && a.D2 % S3 == 0)
    return launch_ex(k_sb_update3<true>, dim3(tiles, a.B), dim3(256), 0, st, 0, a);
  return launch_ex(k_sb_update3<false>, dim3(tiles, a.B), dim3(256), 0, st, 0, a);
}

}  // namespace sbk
