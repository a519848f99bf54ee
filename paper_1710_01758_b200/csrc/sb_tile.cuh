// sb_tile.cuh — one tile of the 2D Split Bregman shrink/Bregman/RHS step (K5), shared by the
// standalone kernel k_sb_update (k_sb.cu) and the SB phase of the persistent reconstruction
// kernel (k_persist.cu).  See k_sb.cu for the method.
#pragma once
#include "kernels.cuh"

namespace sbk {

constexpr int SBT = 32;  // max tile edge

// rows padded to an odd number of 8-byte cells: the column-order loops of the CM variant read
// vx, wv down columns without bank conflicts
template <int TT>
struct SbTile {
  float2 xs[TT + 2][TT + 2];
  float2 vx[TT + 1][TT + 1];
  float2 vy[TT][TT + 1];
  float2 wa[TT][TT + 1];
  float2 wv[TT][TT + 1];
};

__device__ __forceinline__ float2 shrinkc(float2 z, float t) {
  const float a = sqrtf(z.x * z.x + z.y * z.y);
  const float s = (a > t) ? (a - t) / a : 0.f;
  return make_float2(z.x * s, z.y * s);
}

// TT = max tile edge: 32, or 16 when a 32-tile grid would leave SMs idle (one 256^2 slice).
// FIX: both image edges are multiples of TT, so the tile is TT x TT at compile time and every
// index division below is a shift or a constant-divisor multiply (the kernel is issue bound).
// One TT x TT tile (tile row ti, tile column tj) of problem b, with `nt` threads (all of the
// CTA); also the SB phase of the persistent reconstruction kernel (k_persist.cu).
// prof (nullable): phase cycle counters of the KR segment profile (SBPCG_KR_PROF=1), added by
// thread 0 of the caller's profiled CTA: [0] load batch, [1] TV, [2] forward Haar, [3] shrink,
// [4] inverse Haar + rhs
// CM: x is read from, and rhs written to, column-major images [B][N][M] (the persistent kernel's
// layout, whose column owners then read them contiguously); the element loops of those two run
// rows fastest so the accesses stay coalesced.  b_x, b_y, b_w keep the image layout.
// pre (nullable, with CM): the tile's old b_x, b_y, b_w already staged in shared memory by
// sb_tile_prefetch (cp.async issued earlier by the same threads), so the load batch is x only.
template <int TT>
constexpr int sb_pre_size() { return (TT + 1) * TT + TT * (TT + 2) + TT * TT; }  // b_y rows padded to even

template <int TT, bool FIX, int nt, bool CM = false>
__device__ __forceinline__ void sb_tile(const SbArgs& a, SbTile<TT>& S, int ti, int tj, int b,
                                        unsigned long long* prof = nullptr, const float2* pre = nullptr) {
  long long pc = prof ? clock64() : 0;
  auto ph = [&](int k) {
    if (prof) {
      const long long c = clock64();
      atomicAdd(prof + k, (unsigned long long)(c - pc));
      pc = c;
    }
  };
  auto& xs = S.xs;
  auto& vx = S.vx;
  auto& vy = S.vy;
  auto& wa = S.wa;
  auto& wv = S.wv;
  const int M = a.M, N = a.N, L = a.levels;
  const int TH = FIX ? TT : (M < TT ? M : TT), TW = FIX ? TT : (N < TT ? N : TT);
  constexpr int LTT = TT == 32 ? 5 : 4;  // log2(TT)
  // e / (TW >> lv) and e % (TW >> lv) for the Haar groups (TW a power of two when FIX)
  auto gdiv = [&](int e, int lv) { return FIX ? (e >> (LTT - lv)) : e / (TW >> lv); };
  auto gmod = [&](int e, int lv) { return FIX ? (e & ((TT >> lv) - 1)) : e % (TW >> lv); };
  const int i0 = ti * TH, j0 = tj * TW;
  const size_t img = (size_t)M * N, boff = (size_t)b * img;
  const int tid = threadIdx.x;
  const bool do_tv = a.lam != 0.f, do_w = a.gam != 0.f;
  const float tl = do_tv ? 1.f / a.lam : 0.f, tg = do_w ? 1.f / a.gam : 0.f;

  // Mallat position (in the image) of the tile's coefficient (u, v) after L levels
  auto mallat_gi = [&](int u, int v) -> size_t {
    int lv = 1, hi0 = 0, hi1 = 0, ca = u, cb = v;
    bool ll = true;
    for (; lv <= L; ++lv) {
      const int h0 = TH >> lv, h1 = TW >> lv;
      if (u < h0 && v < h1) continue;
      hi0 = u >= h0;
      hi1 = v >= h1;
      ca = u - hi0 * h0;
      cb = v - hi1 * h1;
      ll = false;
      break;
    }
    int gu, gv;
    if (ll) {
      gu = (i0 >> L) + u;
      gv = (j0 >> L) + v;
    } else {
      gu = (hi0 ? (M >> lv) : 0) + (i0 >> lv) + ca;
      gv = (hi1 ? (N >> lv) : 0) + (j0 >> lv) + cb;
    }
    return boff + (size_t)gu * N + gv;
  };

  // every global load of the tile issued in one batch (x with a one-pixel halo, the old b_x /
  // b_y with their halo row / column, b_w at the tile's Mallat positions), then staged: one L2
  // round trip instead of three
  constexpr int KX = ((TT + 2) * (TT + 2) + nt - 1) / nt, KV = ((TT + 1) * TT + nt - 1) / nt;
  constexpr int KB = (TT * TT + nt - 1) / nt;
  float2 rx[KX], rvx[KV], rvy[KV], rbw[KB];
#pragma unroll
  for (int k = 0; k < KX; ++k) {
    const int e = tid + k * nt;
    if (e < (TH + 2) * (TW + 2)) {
      const int u = CM ? e % (TH + 2) : e / (TW + 2), v = CM ? e / (TH + 2) : e % (TW + 2);
      const int gi = (i0 + u - 1 + M) % M, gj = (j0 + v - 1 + N) % N;
      rx[k] = __ldcg(a.x + boff + (CM ? (size_t)gj * M + gi : (size_t)gi * N + gj));
    }
  }
  if (do_tv && pre == nullptr) {
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int e = tid + k * nt;
      if (e < (TH + 1) * TW) {
        const int u = e / TW, v = e % TW;
        rvx[k] = __ldcg(a.bx_in + boff + (size_t)((i0 + u) % M) * N + j0 + v);
      }
      if (e < TH * (TW + 1)) {
        const int u = e / (TW + 1), v = e % (TW + 1);
        rvy[k] = __ldcg(a.by_in + boff + (size_t)(i0 + u) * N + (j0 + v) % N);
      }
    }
  }
  if (do_w && pre == nullptr) {
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      const int e = tid + k * nt;
      if (e < TH * TW) rbw[k] = __ldcg(a.bw + mallat_gi(e / TW, e % TW));
    }
  }
  if (pre != nullptr) {  // every thread's staged copies have landed, then visible to all
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int e = tid + k * nt;
      if (e < (TH + 1) * TW) rvx[k] = pre[e];
      if (e < TH * (TW + 1)) rvy[k] = pre[(TT + 1) * TT + (e / (TT + 1)) * (TT + 2) + e % (TT + 1)];
    }
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      const int e = tid + k * nt;
      if (e < TH * TW) rbw[k] = pre[(TT + 1) * TT + TT * (TT + 2) + e];
    }
  }
#pragma unroll
  for (int k = 0; k < KX; ++k) {
    const int e = tid + k * nt;
    if (e < (TH + 2) * (TW + 2)) {
      if constexpr (CM) xs[e % (TH + 2)][e / (TH + 2)] = rx[k];
      else xs[e / (TW + 2)][e % (TW + 2)] = rx[k];
    }
  }
  if (do_tv) {
#pragma unroll
    for (int k = 0; k < KV; ++k) {
      const int e = tid + k * nt;
      if (e < (TH + 1) * TW) vx[e / TW][e % TW] = rvx[k];
      if (e < TH * (TW + 1)) vy[e / (TW + 1)][e % (TW + 1)] = rvy[k];
    }
  }
  if (do_w) {  // the old b_w, coefficient order, parked in wv until the shrink
#pragma unroll
    for (int k = 0; k < KB; ++k) {
      const int e = tid + k * nt;
      if (e < TH * TW) wv[e / TW][e % TW] = rbw[k];
    }
  }
  __syncthreads();
  ph(0);

  if (do_tv) {
    // v_x at rows i0..i0+TH (TH+1), cols j0..j0+TW-1 ; v_y at rows i0..i0+TH-1, cols j0..j0+TW
    for (int e = tid; e < (TH + 1) * TW; e += nt) {
      const int u = e / TW, v = e % TW;
      const int gi = (i0 + u) % M, gj = j0 + v;
      const float2 xc = xs[u + 1][v + 1], xm = xs[u][v + 1];
      const float2 bo = vx[u][v];
      const float2 z = make_float2(xc.x - xm.x + bo.x, xc.y - xm.y + bo.y);
      const float2 d = shrinkc(z, tl);
      const float2 bn = make_float2(z.x - d.x, z.y - d.y);
      vx[u][v] = make_float2(d.x - bn.x, d.y - bn.y);
      if (u < TH) a.bx_out[boff + (size_t)gi * N + gj] = bn;
    }
    for (int e = tid; e < TH * (TW + 1); e += nt) {
      const int u = e / (TW + 1), v = e % (TW + 1);
      const int gi = i0 + u, gj = (j0 + v) % N;
      const float2 xc = xs[u + 1][v + 1], xm = xs[u + 1][v];
      const float2 bo = vy[u][v];
      const float2 z = make_float2(xc.x - xm.x + bo.x, xc.y - xm.y + bo.y);
      const float2 d = shrinkc(z, tl);
      const float2 bn = make_float2(z.x - d.x, z.y - d.y);
      vy[u][v] = make_float2(d.x - bn.x, d.y - bn.y);
      if (v < TW) a.by_out[boff + (size_t)gi * N + gj] = bn;
    }
  }

  ph(1);
  if (do_w) {
    // forward Haar, tile-local Mallat layout in wa
    for (int e = tid; e < TH * TW; e += nt) wa[e / TW][e % TW] = xs[e / TW + 1][e % TW + 1];
    __syncthreads();
    for (int lv = 1; lv <= L; ++lv) {
      const int h0 = TH >> lv, h1 = TW >> lv;  // output quadrant sizes
      float2 o[4];
      int ga = -1, gb = -1;
      // at most 256 groups at level 1 for a 32x32 tile: one group per thread per round
      for (int base = 0; base < h0 * h1; base += nt) {
        const int e = base + tid;
        const bool act = e < h0 * h1;
        if (act) {
          ga = gdiv(e, lv);
          gb = gmod(e, lv);
          const float2 p = wa[2 * ga][2 * gb], q = wa[2 * ga][2 * gb + 1];
          const float2 r = wa[2 * ga + 1][2 * gb], s = wa[2 * ga + 1][2 * gb + 1];
          const float2 pr = make_float2(p.x + r.x, p.y + r.y), mr = make_float2(p.x - r.x, p.y - r.y);
          const float2 qs = make_float2(q.x + s.x, q.y + s.y), ms = make_float2(q.x - s.x, q.y - s.y);
          o[0] = make_float2(0.5f * (pr.x + qs.x), 0.5f * (pr.y + qs.y));  // LL
          o[1] = make_float2(0.5f * (pr.x - qs.x), 0.5f * (pr.y - qs.y));  // low d0, high d1
          o[2] = make_float2(0.5f * (mr.x + ms.x), 0.5f * (mr.y + ms.y));  // high d0, low d1
          o[3] = make_float2(0.5f * (mr.x - ms.x), 0.5f * (mr.y - ms.y));  // HH
        }
        __syncthreads();
        if (act) {
          wa[ga][gb] = o[0];
          wa[ga][h1 + gb] = o[1];
          wa[h0 + ga][gb] = o[2];
          wa[h0 + ga][h1 + gb] = o[3];
        }
        __syncthreads();
      }
    }
    ph(2);
    // shrink in the coefficient domain, b_w update at global Mallat positions (the old b_w was
    // parked in wv by the load batch; each thread reads and overwrites only its own cells)
    for (int e = tid; e < TH * TW; e += nt) {
      const int u = e / TW, v = e % TW;
      const size_t gi = mallat_gi(u, v);
      const float2 w = wa[u][v], bo = wv[u][v];
      const float2 z = make_float2(w.x + bo.x, w.y + bo.y);
      const float2 d = shrinkc(z, tg);
      const float2 bn = make_float2(z.x - d.x, z.y - d.y);
      a.bw[gi] = bn;
      wv[u][v] = make_float2(d.x - bn.x, d.y - bn.y);
    }
    __syncthreads();
    ph(3);
    // inverse Haar of wv (coarsest level first)
    for (int lv = L; lv >= 1; --lv) {
      const int h0 = TH >> lv, h1 = TW >> lv;
      for (int base = 0; base < h0 * h1; base += nt) {
        const int e = base + tid;
        const bool act = e < h0 * h1;
        float2 p, q, r, s;
        int ga = 0, gb = 0;
        if (act) {
          ga = gdiv(e, lv);
          gb = gmod(e, lv);
          const float2 LL = wv[ga][gb], LH = wv[ga][h1 + gb], HL = wv[h0 + ga][gb],
                       HH = wv[h0 + ga][h1 + gb];
          p = make_float2(0.5f * (LL.x + LH.x + HL.x + HH.x), 0.5f * (LL.y + LH.y + HL.y + HH.y));
          q = make_float2(0.5f * (LL.x - LH.x + HL.x - HH.x), 0.5f * (LL.y - LH.y + HL.y - HH.y));
          r = make_float2(0.5f * (LL.x + LH.x - HL.x - HH.x), 0.5f * (LL.y + LH.y - HL.y - HH.y));
          s = make_float2(0.5f * (LL.x - LH.x - HL.x + HH.x), 0.5f * (LL.y - LH.y - HL.y + HH.y));
        }
        __syncthreads();
        if (act) {
          wv[2 * ga][2 * gb] = p;
          wv[2 * ga][2 * gb + 1] = q;
          wv[2 * ga + 1][2 * gb] = r;
          wv[2 * ga + 1][2 * gb + 1] = s;
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();

  for (int e = tid; e < TH * TW; e += nt) {
    const int u = CM ? e % TH : e / TW, v = CM ? e / TH : e % TW;
    float2 out = make_float2(0.f, 0.f);
    if (do_tv) {
      const float2 a0 = vx[u][v], a1 = vx[u + 1][v], c0 = vy[u][v], c1 = vy[u][v + 1];
      out.x = a.lam * ((a0.x - a1.x) + (c0.x - c1.x));
      out.y = a.lam * ((a0.y - a1.y) + (c0.y - c1.y));
    }
    if (do_w) {
      out.x += a.gam * wv[u][v].x;
      out.y += a.gam * wv[u][v].y;
    }
    a.rhs[boff + (CM ? (size_t)(j0 + v) * M + (i0 + u) : (size_t)(i0 + u) * N + (j0 + v))] = out;
  }
  __syncthreads();  // the tile's shared memory may be reused at once
  ph(4);
}

// Stage the old b_x, b_y (with their halo row / column) and b_w (Mallat positions) of tile
// (ti, tj) into pre[sb_pre_size<TT>()] (FIX tiles only; pre 16-byte aligned): layout b_x
// [TT+1][TT], b_y [TT][TT+2] (TT+1 used), b_w [TT][TT] in the order sb_tile's load batch uses.
template <int TT, int nt>
__device__ __forceinline__ void sb_tile_prefetch(const SbArgs& a, float2* pre, int ti, int tj, int b) {
  // 16-byte copies of aligned element pairs (tile columns start at multiples of TT, and every
  // Mallat run of a tile starts at an even column); b_y's halo column is one 8-byte copy per row
  const int M = a.M, N = a.N, L = a.levels;
  const int i0 = ti * TT, j0 = tj * TT;
  const size_t boff = (size_t)b * M * N;
  constexpr int H = TT / 2;                        // pairs per tile row
  constexpr int NX = (TT + 1) * H, NY = TT * H, NW = TT * H;
  for (int e = threadIdx.x; e < NX + NY + TT + NW; e += nt) {
    const float2* src;
    float2* dst;
    bool pair = true;
    if (e < NX) {
      const int u = e / H, v = 2 * (e % H);
      src = a.bx_in + boff + (size_t)((i0 + u) % M) * N + j0 + v;
      dst = pre + u * TT + v;
    } else if (e < NX + NY) {
      const int f = e - NX, u = f / H, v = 2 * (f % H);
      src = a.by_in + boff + (size_t)(i0 + u) * N + j0 + v;
      dst = pre + (TT + 1) * TT + u * (TT + 2) + v;
    } else if (e < NX + NY + TT) {  // b_y halo column j0 + TT (periodic)
      const int u = e - NX - NY;
      src = a.by_in + boff + (size_t)(i0 + u) * N + (j0 + TT) % N;
      dst = pre + (TT + 1) * TT + u * (TT + 2) + TT;
      pair = false;
    } else {
      const int f = e - NX - NY - TT, u = f / H, v = 2 * (f % H);
      int lv = 1, hi0 = 0, hi1 = 0, ca = u, cb = v;
      bool ll = true;
      for (; lv <= L; ++lv) {
        const int h0 = TT >> lv, h1 = TT >> lv;
        if (u < h0 && v < h1) continue;
        hi0 = u >= h0;
        hi1 = v >= h1;
        ca = u - hi0 * h0;
        cb = v - hi1 * h1;
        ll = false;
        break;
      }
      const int gu = ll ? (i0 >> L) + u : (hi0 ? (M >> lv) : 0) + (i0 >> lv) + ca;
      const int gv = ll ? (j0 >> L) + v : (hi1 ? (N >> lv) : 0) + (j0 >> lv) + cb;
      src = a.bw + boff + (size_t)gu * N + gv;
      dst = pre + (TT + 1) * TT + TT * (TT + 2) + u * TT + v;
    }
    if (pair) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
    } else {
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

}  // namespace sbk
