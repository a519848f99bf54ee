// fft_core.cuh — register-resident DFT building blocks and the four-step line transform
// used by every FFT in libsbpcg (sm_100a).  No cuFFT on the hot path (BASELINE.json
// north_star item (1)).
//
// Conventions: unnormalised transforms, W_N = exp(S * 2*pi*i / N); S = -1 forward,
// S = +1 inverse.  Scaling (1/N, 1/sqrt(N)) is folded by the callers into the mask
// (R/M) and into Lambda^{-1} = 1/(N k).
//
// Four-step layout for a line of length N = N1 * N2 handled by N2 threads that each hold
// N1 values in registers:
//   layout A ("natural"):  thread j holds x[N2*n1 + j],          n1 in [0, N1)
//   layout B ("spectral"): thread j holds X[(j + q*N2) + N1*k2]  at slot q*N2 + k2
// fwd(A -> B) and inv(B -> A) each do two register DFTs and ONE shared-memory exchange.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>

namespace sbk {

// ------------------------------------------------------------------ complex helpers
template <typename T> struct V2;
template <> struct V2<float>  { using type = float2; };
template <> struct V2<double> { using type = double2; };
template <typename T> using vec2 = typename V2<T>::type;

template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return {a.x + b.x, a.y + b.y}; }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return {a.x - b.x, a.y - b.y}; }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
// conj(a) * b
template <typename V> __device__ __forceinline__ V cmulc(V a, V b) {
  return {a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x};
}
// a * conj(b)
template <typename V> __device__ __forceinline__ V cmul_conjb(V a, V b) {
  return {a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y};
}
template <typename V, typename T> __device__ __forceinline__ V cscale(V a, T s) { return {a.x * s, a.y * s}; }
// multiply by S*i (S = +-1):  i*(a+ib) = -b + ia
template <int S, typename V> __device__ __forceinline__ V mul_si(V a) {
  if constexpr (S > 0) return {-a.y, a.x};
  else return {a.y, -a.x};
}

// fp32 complex arithmetic on the packed f32x2 pipe (sm_100: FADD2 / FMUL2 / FFMA2 process the
// (re, im) pair in one instruction; swaps and half negations fold into operand modifiers).
// Scalar FP32 instructions issue at half the FP32 lane rate on this architecture, and the FFT
// kernels are FP32-issue bound, so every hot complex operation goes through these overloads
// (the templates above remain for double2).  Rounding per lane is that of the scalar ops.
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
// Operand placement matters: the swapped / half-negated vector goes in operand A (folded as
// .LO_HI.NP) and the real factor in operand B as a scalar broadcast (.F32), so a complex
// multiply is exactly FMUL2 + FFMA2 with no register moves.
__device__ __forceinline__ float2 bc(float s) { return make_float2(s, s); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {  // a * b
  const float2 t = __fmul2_rn(b, bc(a.x));
  return __ffma2_rn(make_float2(-b.y, b.x), bc(a.y), t);
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {  // conj(a) * b
  const float2 t = __fmul2_rn(b, bc(a.x));
  return __ffma2_rn(make_float2(b.y, -b.x), bc(a.y), t);
}
__device__ __forceinline__ float2 cmul_conjb(float2 a, float2 b) {  // a * conj(b)
  const float2 t = __fmul2_rn(a, bc(b.x));
  return __ffma2_rn(make_float2(a.y, -a.x), bc(b.y), t);
}
__device__ __forceinline__ float2 cscale(float2 a, float s) { return __fmul2_rn(a, bc(s)); }
// acc + a * b
__device__ __forceinline__ float2 cfma(float2 a, float2 b, float2 acc) {
  const float2 t = __ffma2_rn(b, bc(a.x), acc);
  return __ffma2_rn(make_float2(-b.y, b.x), bc(a.y), t);
}
// acc + conj(a) * b
__device__ __forceinline__ float2 cfmac(float2 a, float2 b, float2 acc) {
  const float2 t = __ffma2_rn(b, bc(a.x), acc);
  return __ffma2_rn(make_float2(b.y, -b.x), bc(a.y), t);
}
#else
__host__ __device__ inline float2 cfma(float2 a, float2 b, float2 acc) {
  return {acc.x + a.x * b.x - a.y * b.y, acc.y + a.x * b.y + a.y * b.x};
}
__host__ __device__ inline float2 cfmac(float2 a, float2 b, float2 acc) {
  return {acc.x + a.x * b.x + a.y * b.y, acc.y + a.x * b.y - a.y * b.x};
}
#endif

// ------------------------------------------------------------------ compile-time trig
// cos/sin of 2*pi*e/n evaluated in constexpr double (octant reduction + Taylor series),
// so register-DFT twiddles become instruction immediates.
__host__ __device__ constexpr double kpi() { return 3.14159265358979323846264338327950288; }
__host__ __device__ constexpr double ktaylor_sin(double x) {
  double term = x, sum = x;
  for (int k = 1; k < 14; ++k) { term *= -x * x / ((2 * k) * (2 * k + 1)); sum += term; }
  return sum;
}
__host__ __device__ constexpr double ktaylor_cos(double x) {
  double term = 1.0, sum = 1.0;
  for (int k = 1; k < 14; ++k) { term *= -x * x / ((2 * k - 1) * (2 * k)); sum += term; }
  return sum;
}
// cos(2*pi*e/n), sin(2*pi*e/n) for integer e (any sign), n > 0
__host__ __device__ constexpr double kcos2pi(long e, long n) {
  long m = ((e % n) + n) % n;        // angle = 2*pi*m/n in [0, 2pi)
  // reduce by octants: 8m/n
  long e8 = 8 * m;                    // angle = (pi/4) * e8/n
  long oct = e8 / n;                  // 0..7
  double frac = double(e8 - oct * n) / double(n);  // in [0,1): angle = pi/4*(oct + frac)
  double a = kpi() / 4 * frac;
  double c = ktaylor_cos(a), s = ktaylor_sin(a);
  double c2 = 0.70710678118654752440 * (c - s), s2 = 0.70710678118654752440 * (c + s);
  // rotate (c,s) by oct * pi/4
  switch (oct) {
    case 0: return c;
    case 1: return c2;
    case 2: return -s;
    case 3: return -s2;
    case 4: return -c;
    case 5: return -c2;
    case 6: return s;
    default: return s2;
  }
}
__host__ __device__ constexpr double ksin2pi(long e, long n) { return kcos2pi(4 * e - n, 4 * n); }

// v * W_N^E, W_N = exp(S*2*pi*i/N), E a compile-time integer
template <int N, int E, int S, typename V>
__device__ __forceinline__ V twc(V v) {
  using T = decltype(v.x);
  constexpr int e = ((E % N) + N) % N;
  if constexpr (e == 0) {
    return v;
  } else if constexpr (2 * e == N) {
    return {-v.x, -v.y};
  } else if constexpr (4 * e == N) {
    return mul_si<S>(v);
  } else if constexpr (4 * e == 3 * N) {
    return mul_si<-S>(v);
  } else if constexpr ((8 * e) % N == 0) {
    // (+-1 +- i)/sqrt2
    constexpr T h = T(0.70710678118654752440);
    constexpr T c = T(kcos2pi(e, N) > 0 ? 1 : -1);
    constexpr T s = T((ksin2pi(e, N) > 0 ? 1 : -1) * S);
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
    if constexpr (std::is_same<T, float>::value) {  // (c h + i s h)(v): packed constant multiply
      const float2 t = __fmul2_rn(v, bc(c * h));
      return __ffma2_rn(make_float2(-v.y, v.x), bc(s * h), t);
    }
#endif
    // (a+ib)(c + i s) * h
    return {h * (c * v.x - s * v.y), h * (s * v.x + c * v.y)};
  } else {
    constexpr T c = T(kcos2pi(e, N));
    constexpr T s = T(S * ksin2pi(e, N));
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
    if constexpr (std::is_same<T, float>::value) {
      const float2 t = __fmul2_rn(v, bc(c));
      return __ffma2_rn(make_float2(-v.y, v.x), bc(s), t);
    }
#endif
    return {v.x * c - v.y * s, v.x * s + v.y * c};
  }
}

template <int B, int E, typename F>
__device__ __forceinline__ void sfor(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    sfor<B + 1, E>(f);
  }
}

// ------------------------------------------------------------------ register DFTs
// In-place, natural order in and out, unnormalised.
template <int N, int S> struct Dft;

template <int S> struct Dft<1, S> {
  template <typename V> __device__ __forceinline__ static void run(V*) {}
};
template <int S> struct Dft<2, S> {
  template <typename V> __device__ __forceinline__ static void run(V* x) {
    V a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
  }
};
template <int S> struct Dft<3, S> {
  template <typename V> __device__ __forceinline__ static void run(V* x) {
    using T = decltype(x[0].x);
    constexpr T h = T(0.86602540378443864676);  // sqrt(3)/2
    V a = x[0], b = x[1], c = x[2];
    V s = cadd(b, c), d = csub(b, c);
    V m = csub(a, cscale(s, T(0.5)));
    V t = mul_si<S>(cscale(d, h));
    x[0] = cadd(a, s);
    x[1] = cadd(m, t);
    x[2] = csub(m, t);
  }
};
template <int S> struct Dft<4, S> {
  template <typename V> __device__ __forceinline__ static void run(V* x) {
    V a = x[0], b = x[1], c = x[2], d = x[3];
    V s0 = cadd(a, c), d0 = csub(a, c), s1 = cadd(b, d), d1 = mul_si<S>(csub(b, d));
    x[0] = cadd(s0, s1);
    x[2] = csub(s0, s1);
    x[1] = cadd(d0, d1);
    x[3] = csub(d0, d1);
  }
};

// Generic mixed radix (decimation in time): N = R * M
//   X[k + M*s] = sum_r W_R^{r s} (W_N^{r k} * DFT_M(x[R*m + r])[k])
template <int N> struct Radix {
  static constexpr int value = (N % 4 == 0 && N > 4) ? 4 : ((N % 2 == 0) ? 2 : 3);
};
template <int N, int S> struct Dft {
  static_assert(N % 2 == 0 || N % 3 == 0, "DFT length must be 2^a 3^b");
  template <typename V> __device__ __forceinline__ static void run(V* x) {
    constexpr int R = Radix<N>::value;
    constexpr int M = N / R;
    V sub[R][M];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int m = 0; m < M; ++m) sub[r][m] = x[R * m + r];
#pragma unroll
    for (int r = 0; r < R; ++r) Dft<M, S>::run(sub[r]);
    sfor<0, M>([&](auto kc) {
      constexpr int k = decltype(kc)::value;
      V t[R];
      sfor<0, R>([&](auto rc) {
        constexpr int r = decltype(rc)::value;
        t[r] = twc<N, r * k, S>(sub[r][k]);
      });
      Dft<R, S>::run(t);
#pragma unroll
      for (int s = 0; s < R; ++s) x[k + M * s] = t[s];
    });
  }
};

// ------------------------------------------------------------------ four-step line FFT
// Factorisation N = N1 * N2 (N1 registers per thread, N2 threads per line, N1 % N2 == 0).
template <int N> struct Split;
template <> struct Split<2>    { static constexpr int N1 = 2,  N2 = 1; };
template <> struct Split<4>    { static constexpr int N1 = 2,  N2 = 2; };
template <> struct Split<8>    { static constexpr int N1 = 4,  N2 = 2; };
template <> struct Split<12>   { static constexpr int N1 = 6,  N2 = 2; };
template <> struct Split<16>   { static constexpr int N1 = 4,  N2 = 4; };
template <> struct Split<24>   { static constexpr int N1 = 12, N2 = 2; };
template <> struct Split<32>   { static constexpr int N1 = 8,  N2 = 4; };
template <> struct Split<48>   { static constexpr int N1 = 12, N2 = 4; };
template <> struct Split<64>   { static constexpr int N1 = 8,  N2 = 8; };
template <> struct Split<96>   { static constexpr int N1 = 24, N2 = 4; };
template <> struct Split<128>  { static constexpr int N1 = 16, N2 = 8; };
template <> struct Split<192>  { static constexpr int N1 = 24, N2 = 8; };
template <> struct Split<256>  { static constexpr int N1 = 16, N2 = 16; };
template <> struct Split<384>  { static constexpr int N1 = 48, N2 = 8; };
template <> struct Split<512>  { static constexpr int N1 = 32, N2 = 16; };
template <> struct Split<1024> { static constexpr int N1 = 32, N2 = 32; };

// Shared-memory exchange layout: offset(k1, n2, line) = k1*SK1 + n2*SN2 + line*SL.
//  * column tiles (threads (j, col), col fastest, W columns): SL = 1, SN2 = W, SK1 = (N2+1)*W
//  * row groups (threads (line, j), j fastest):               SN2 = 1, SK1 = N2+1, SL = N1*(N2+1)
template <int SK1, int SN2, int SL> struct XLayout {
  __device__ __forceinline__ static int off(int k1, int n2, int l) { return k1 * SK1 + n2 * SN2 + l * SL; }
};
template <int N, int W> struct ColLayout {
  static constexpr int N1 = Split<N>::N1, N2 = Split<N>::N2;
  using L = XLayout<(N2 + 1) * W, W, 1>;
  static constexpr int size = N1 * (N2 + 1) * W;  // elements
};
template <int N, int LINES> struct RowLayout {
  static constexpr int N1 = Split<N>::N1, N2 = Split<N>::N2;
  using L = XLayout<N2 + 1, 1, N1 * (N2 + 1)>;
  static constexpr int size = LINES * N1 * (N2 + 1);
};

// tw[m] = W_N^m = exp(-2*pi*i*m/N) (forward table; the inverse uses its conjugate).
// Forward: layout A (v[n1] = x[N2*n1 + j]) -> layout B.  Barrier between the halves is
// the caller's choice: BAR = __syncthreads() for cross-warp lines.
template <int N, typename Lay, typename V>
__device__ __forceinline__ void fft_fwd(V (&v)[Split<N>::N1], V* xch, const V* __restrict__ tw,
                                        int j, int line) {
  constexpr int N1 = Split<N>::N1, N2 = Split<N>::N2;
  Dft<N1, -1>::run(v);
#pragma unroll
  for (int k1 = 1; k1 < N1; ++k1) v[k1] = cmul(v[k1], tw[j * k1]);
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) xch[Lay::off(k1, j, line)] = v[k1];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < N1 / N2; ++q) {
    V u[N2];
    const int k1 = j + q * N2;
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) u[n2] = xch[Lay::off(k1, n2, line)];
    Dft<N2, -1>::run(u);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) v[q * N2 + k2] = u[k2];
  }
}

// Inverse (unnormalised, S = +1): layout B -> layout A.  The exchange buffer may be the
// one fft_fwd used: each thread overwrites only the cells it read in fft_fwd's second half.
template <int N, typename Lay, typename V>
__device__ __forceinline__ void fft_inv(V (&v)[Split<N>::N1], V* xch, const V* __restrict__ tw,
                                        int j, int line) {
  constexpr int N1 = Split<N>::N1, N2 = Split<N>::N2;
#pragma unroll
  for (int q = 0; q < N1 / N2; ++q) {
    V u[N2];
    const int k1 = j + q * N2;
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) u[k2] = v[q * N2 + k2];
    Dft<N2, +1>::run(u);
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) {
      V w = (n2 == 0 || k1 == 0) ? u[n2] : cmul_conjb(u[n2], tw[n2 * k1]);
      xch[Lay::off(k1, n2, line)] = w;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) v[k1] = xch[Lay::off(k1, j, line)];
  Dft<N1, +1>::run(v);
}

// Transposed-table variants (row groups, j fastest across lanes): the forward twiddles come
// from tf[k1 * N2 + j] = W_N^{j k1} and the inverse ones from ti[(q N2 + n2) N2 + j] =
// W_N^{n2 (j + q N2)}, so the lanes of a warp read consecutive entries (the natural table
// tw[j k1] is a strided gather with up to N2-way bank conflicts).
template <int N, typename Lay, typename V>
__device__ __forceinline__ void fft_fwd_t(V (&v)[Split<N>::N1], V* xch, const V* __restrict__ tf, int j, int line) {
  constexpr int N1 = Split<N>::N1, N2 = Split<N>::N2;
  Dft<N1, -1>::run(v);
#pragma unroll
  for (int k1 = 1; k1 < N1; ++k1) v[k1] = cmul(v[k1], tf[k1 * N2 + j]);
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) xch[Lay::off(k1, j, line)] = v[k1];
  __syncthreads();
#pragma unroll
  for (int q = 0; q < N1 / N2; ++q) {
    V u[N2];
    const int k1 = j + q * N2;
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) u[n2] = xch[Lay::off(k1, n2, line)];
    Dft<N2, -1>::run(u);
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) v[q * N2 + k2] = u[k2];
  }
}
template <int N, typename Lay, typename V>
__device__ __forceinline__ void fft_inv_t(V (&v)[Split<N>::N1], V* xch, const V* __restrict__ ti, int j, int line) {
  constexpr int N1 = Split<N>::N1, N2 = Split<N>::N2;
#pragma unroll
  for (int q = 0; q < N1 / N2; ++q) {
    V u[N2];
#pragma unroll
    for (int k2 = 0; k2 < N2; ++k2) u[k2] = v[q * N2 + k2];
    Dft<N2, +1>::run(u);
    const int k1 = j + q * N2;
#pragma unroll
    for (int n2 = 0; n2 < N2; ++n2) {
      const V w = (n2 == 0) ? u[n2] : cmul_conjb(u[n2], ti[(q * N2 + n2) * N2 + j]);
      xch[Lay::off(k1, n2, line)] = w;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) v[k1] = xch[Lay::off(k1, j, line)];
  Dft<N1, +1>::run(v);
}

// Register-twiddle variants for square splits (N1 == N2): thread j's forward twiddles
// W_N^{j k1} (k1 < N1) and inverse twiddles conj(W_N^{n2 j}) (n2 < N2) are the same N1 values,
// loaded once per kernel into twr[m] = W_N^{j m} instead of from shared memory per transform.
template <int N, typename V>
__device__ __forceinline__ void load_twr(V (&twr)[Split<N>::N1], const V* __restrict__ tw, int j) {
  static_assert(Split<N>::N1 == Split<N>::N2, "square split only");
#pragma unroll
  for (int m = 0; m < Split<N>::N1; ++m) twr[m] = tw[j * m];
}
template <int N, typename Lay, typename V>
__device__ __forceinline__ void fft_fwd_r(V (&v)[Split<N>::N1], V* xch, const V (&twr)[Split<N>::N1], int j,
                                          int line) {
  constexpr int N1 = Split<N>::N1, N2 = Split<N>::N2;
  static_assert(N1 == N2, "square split only");
  Dft<N1, -1>::run(v);
#pragma unroll
  for (int k1 = 1; k1 < N1; ++k1) v[k1] = cmul(v[k1], twr[k1]);
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) xch[Lay::off(k1, j, line)] = v[k1];
  __syncthreads();
  V u[N2];
#pragma unroll
  for (int n2 = 0; n2 < N2; ++n2) u[n2] = xch[Lay::off(j, n2, line)];
  Dft<N2, -1>::run(u);
#pragma unroll
  for (int k2 = 0; k2 < N2; ++k2) v[k2] = u[k2];
}
template <int N, typename Lay, typename V>
__device__ __forceinline__ void fft_inv_r(V (&v)[Split<N>::N1], V* xch, const V (&twr)[Split<N>::N1], int j,
                                          int line) {
  constexpr int N1 = Split<N>::N1, N2 = Split<N>::N2;
  static_assert(N1 == N2, "square split only");
  V u[N2];
#pragma unroll
  for (int k2 = 0; k2 < N2; ++k2) u[k2] = v[k2];
  Dft<N2, +1>::run(u);
#pragma unroll
  for (int n2 = 0; n2 < N2; ++n2) xch[Lay::off(j, n2, line)] = (n2 == 0 || j == 0) ? u[n2] : cmul_conjb(u[n2], twr[n2]);
  __syncthreads();
#pragma unroll
  for (int k1 = 0; k1 < N1; ++k1) v[k1] = xch[Lay::off(k1, j, line)];
  Dft<N1, +1>::run(v);
}

// spectral index held in slot s of thread j (layout B)
template <int N> __device__ __forceinline__ int specidx(int j, int s) {
  constexpr int N1 = Split<N>::N1, N2 = Split<N>::N2;
  return (j + (s / N2) * N2) + N1 * (s % N2);
}
// natural index held in slot n1 of thread j (layout A)
template <int N> __device__ __forceinline__ int natidx(int j, int n1) { return Split<N>::N2 * n1 + j; }

}  // namespace sbk
