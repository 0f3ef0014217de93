// fhtb_core.cuh -- device building blocks shared by every kernel of libfhtb200.
//
//  * complex helpers on double2
//  * exact-phase unit roots  e^{i pi P / D}  for integer P, D
//  * register/shared-memory Stockham FFT (radix 16/8/4/2, fp64) used by the
//    DCT-I/DST-I far-field kernels (reference: trig.py:59-77 rfft embeddings,
//    schlomilch.py:301-329 block application)
//
// Everything here is header-only and compiled for sm_100a.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fhtb {

// ---------------------------------------------------------------- complex
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * (S*i), S = +1 or -1
template <int S> __device__ __forceinline__ double2 cmul_i(double2 a) {
  return S > 0 ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// e^{i pi P / D} for integer P (any sign) and D > 0, with the argument reduced
// in exact integer arithmetic to [0, 1/2) before sincospi, so the phase
// error stays below one ulp even for D that is not a power of two.
__device__ __forceinline__ double2 expi_pi_frac(long long P, long long D) {
  long long m = P % (2 * D);
  if (m < 0) m += 2 * D;
  double sgn = 1.0;
  if (m >= D) { m -= D; sgn = -1.0; }
  // angle pi*m/D in [0, pi)
  double s, c;
  if (2 * m >= D) {
    // pi*m/D = pi/2 + pi*(2m-D)/(2D);  e^{i(pi/2+x)} = i e^{ix}
    sincospi((double)(2 * m - D) / (double)(2 * D), &s, &c);
    return make_double2(-s * sgn, c * sgn);
  }
  sincospi((double)m / (double)D, &s, &c);
  return make_double2(c * sgn, s * sgn);
}

// ------------------------------------------------------------ small DFTs
// In-place DFT of R consecutive registers, X_k = sum_n a_n w^{nk},
// w = e^{S 2 pi i / R}.
template <int R, int S> struct Dft;

template <int S> struct Dft<1, S> {
  static __device__ __forceinline__ void run(double2*) {}
};

template <int S> struct Dft<2, S> {
  static __device__ __forceinline__ void run(double2* v) {
    double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <int S> struct Dft<4, S> {
  static __device__ __forceinline__ void run(double2* v) {
    double2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    double2 t2 = cadd(v[1], v[3]), t3 = cmul_i<S>(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  }
};

#define FHTB_SQRT1_2 0.70710678118654752440
#define FHTB_COS_PI8 0.92387953251128675613
#define FHTB_SIN_PI8 0.38268343236508977173

// w8 = (1 + S i)/sqrt2,  w8^3 = (-1 + S i)/sqrt2
template <int S> __device__ __forceinline__ double2 mul_w8(double2 a) {
  return make_double2((a.x - S * a.y) * FHTB_SQRT1_2, (a.y + S * a.x) * FHTB_SQRT1_2);
}
template <int S> __device__ __forceinline__ double2 mul_w8_3(double2 a) {
  return make_double2((-a.x - S * a.y) * FHTB_SQRT1_2, (-a.y + S * a.x) * FHTB_SQRT1_2);
}

template <int S> struct Dft<8, S> {
  static __device__ __forceinline__ void run(double2* v) {
    double2 e[4] = {v[0], v[2], v[4], v[6]};
    double2 o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4, S>::run(e);
    Dft<4, S>::run(o);
    o[1] = mul_w8<S>(o[1]);
    o[2] = cmul_i<S>(o[2]);
    o[3] = mul_w8_3<S>(o[3]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = cadd(e[k], o[k]);
      v[k + 4] = csub(e[k], o[k]);
    }
  }
};

template <int S> struct Dft<16, S> {
  static __device__ __forceinline__ void run(double2* v) {
    double2 e[8], o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) { e[k] = v[2 * k]; o[k] = v[2 * k + 1]; }
    Dft<8, S>::run(e);
    Dft<8, S>::run(o);
    const double c1 = FHTB_COS_PI8, s1 = FHTB_SIN_PI8;
    o[1] = cmul(o[1], make_double2(c1, S * s1));
    o[2] = mul_w8<S>(o[2]);
    o[3] = cmul(o[3], make_double2(s1, S * c1));
    o[4] = cmul_i<S>(o[4]);
    o[5] = cmul(o[5], make_double2(-s1, S * c1));
    o[6] = mul_w8_3<S>(o[6]);
    o[7] = cmul(o[7], make_double2(-c1, S * s1));
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = cadd(e[k], o[k]);
      v[k + 8] = csub(e[k], o[k]);
    }
  }
};

// DFT of R points whose upper half is zero (a zero-padded R/2-point input):
// X_2m = DFT_{R/2}(a)_m, X_{2m+1} = DFT_{R/2}(a_n w_R^n)_m.  Used by the
// far-field pass 1, whose input n2 >= L2/2 lies beyond the grid (n > L).
template <int R, int S> struct DftHalfZero {
  static __device__ __forceinline__ void run(double2* v) { Dft<R, S>::run(v); }
};

template <int S> struct DftHalfZero<16, S> {
  static __device__ __forceinline__ void run(double2* v) {
    double2 e[8], o[8];
    const double c1 = FHTB_COS_PI8, s1 = FHTB_SIN_PI8;
#pragma unroll
    for (int n = 0; n < 8; ++n) e[n] = v[n];
    o[0] = v[0];
    o[1] = cmul(v[1], make_double2(c1, S * s1));
    o[2] = mul_w8<S>(v[2]);
    o[3] = cmul(v[3], make_double2(s1, S * c1));
    o[4] = cmul_i<S>(v[4]);
    o[5] = cmul(v[5], make_double2(-s1, S * c1));
    o[6] = mul_w8_3<S>(v[6]);
    o[7] = cmul(v[7], make_double2(-c1, S * s1));
    Dft<8, S>::run(e);
    Dft<8, S>::run(o);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      v[2 * m] = e[m];
      v[2 * m + 1] = o[m];
    }
  }
};

template <int S> struct DftHalfZero<8, S> {
  static __device__ __forceinline__ void run(double2* v) {
    double2 e[4], o[4];
#pragma unroll
    for (int n = 0; n < 4; ++n) e[n] = v[n];
    o[0] = v[0];
    o[1] = mul_w8<S>(v[1]);
    o[2] = cmul_i<S>(v[2]);
    o[3] = mul_w8_3<S>(v[3]);
    Dft<4, S>::run(e);
    Dft<4, S>::run(o);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      v[2 * m] = e[m];
      v[2 * m + 1] = o[m];
    }
  }
};

// ----------------------------------------------------- block Stockham FFT
//
// An N-point FFT executed by T threads, each holding E = N/T points in
// registers.  Input layout: thread t holds x[t + T*e], e < E.  Output
// layout: slot s = b*RL + r holds X[t + T*b + r*(N/RL)], RL = last radix.
// Radices: E first, then E repeatedly, last radix = N / E^p.  Shared
// memory holds N double2 (swizzled, no padding) and is used between passes.
//
// tw: table of e^{+2 pi i m / N}, m < N (global, read through L1).

constexpr __host__ __device__ int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n >> 1); }

template <int N, int E> struct FftShape {
  static constexpr int LOGN = ilog2c(N);
  static constexpr int LOGE = ilog2c(E);
  static constexpr int T = N / E;
  static constexpr int NPASS = (LOGN + LOGE - 1) / LOGE;        // ceil
  static constexpr int LOGRL = LOGN - (NPASS - 1) * LOGE;         // last radix log
  static constexpr int RL = 1 << LOGRL;
};

// XOR swizzle: conflict-free for both unit-stride and stride-E 16-byte accesses.
template <int LOGE> __device__ __forceinline__ int swz(int i) {
  return LOGE >= 3 ? (i ^ ((i >> LOGE) & 7)) : i;
}

template <int S> __device__ __forceinline__ double2 twid(const double2* __restrict__ tw, int m) {
  double2 w = __ldg(tw + m);
  return S > 0 ? w : cconj(w);
}

// Twiddles w^r, r < R, of one radix-R butterfly, w = e^{S 2 pi i m / N}.
// Three table reads (w, w^4, w^8) and products of depth <= 3 instead of
// R-1 table reads: the passes are L1/shared-bandwidth bound, the fp64 pipe
// is not (fftmicro: 63% of L1 bandwidth, 34% of fp64 peak).
#ifndef FHTB_TW_COMPUTE
#define FHTB_TW_COMPUTE 1
#endif
// tw is the size-N table inside the twiddle pool (pool + N - 2; the pool holds
// the table of every power of two n at offset n - 2).  The butterflies of a
// pass with span Ns need e^{S 2 pi i k r / n}, n = Ns R, k < Ns: w comes from
// the size-n table, w^4 and w^8 from the size-n/4 and size-n/8 tables, all
// indexed by k itself (same bits as tw[k N/n], tw[4 k N/n], tw[8 k N/n]), so
// that a warp's gather touches consecutive entries instead of entries N/n,
// 4 N/n and 8 N/n apart (up to 32 cache lines per request in the last pass).
template <int N, int R, int S>
__device__ __forceinline__ void butterfly_twiddles(const double2* __restrict__ tw, int n, int k, double2 (&w)[R]) {
  w[0] = make_double2(1.0, 0.0);
  if (R == 1) return;
  if (!FHTB_TW_COMPUTE) {
    const int m = k * (N / n);
#pragma unroll
    for (int r = 1; r < R; ++r) w[r] = twid<S>(tw, r * m);
    return;
  }
  const double2* pool = tw - (N - 2);
  w[1] = twid<S>(pool + (n - 2), k);
  if (R >= 4) {
    w[2] = cmul(w[1], w[1]);
    w[3] = cmul(w[2], w[1]);
  }
  if (R >= 8) {
    w[4] = twid<S>(pool + (n / 4 - 2), k);
    w[5] = cmul(w[4], w[1]);
    w[6] = cmul(w[4], w[2]);
    w[7] = cmul(w[4], w[3]);
  }
  if (R >= 16) {
    w[8] = twid<S>(pool + (n / 8 - 2), k);
#pragma unroll
    for (int r = 9; r < 12; ++r) w[r] = cmul(w[8], w[r - 8]);
    w[12] = cmul(w[8], w[4]);
#pragma unroll
    for (int r = 13; r < 16; ++r) w[r] = cmul(w[12], w[r - 12]);
  }
}

// One Stockham pass with radix R over the registers of thread t.
template <int N, int E, int R, int S>
__device__ __forceinline__ void stockham_mid(double2 (&v)[E], double2* sm, int t, int Ns,
                                             const double2* __restrict__ tw, bool last) {
  constexpr int T = N / E;
  constexpr int NB = E / R;
  constexpr int STR = N / R;
  constexpr int LOGE = ilog2c(E);
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + T * b;
#pragma unroll
    for (int r = 0; r < R; ++r) v[b * R + r] = sm[swz<LOGE>(j + r * STR)];
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int j = t + T * b;
    const int k = j % Ns;
    double2 w[R];
    butterfly_twiddles<N, R, S>(tw, Ns * R, k, w);
#pragma unroll
    for (int r = 1; r < R; ++r) v[b * R + r] = cmul(v[b * R + r], w[r]);
    Dft<R, S>::run(v + b * R);
  }
  if (!last) {
    __syncthreads();
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      const int j = t + T * b;
      const int k = j % Ns;
      const int d = (j / Ns) * Ns * R + k;
#pragma unroll
      for (int r = 0; r < R; ++r) sm[swz<LOGE>(d + r * Ns)] = v[b * R + r];
    }
    __syncthreads();
  }
}

// Full FFT.  Caller guarantees that no other thread of the CTA still reads
// `sm` from a previous use (a __syncthreads before the call).
// HZ: the upper half of the thread's first-pass inputs (slots e >= E/2) is
// zero, except `extra` added to slot E/2 (a single element, 0 elsewhere).
// SYNC0: the caller has NOT synchronised; the CTA barrier (preceded, in
// thread t == 0, by the wait for the reads of the previous TMA store from
// `sm`) is taken after the register-only first pass, so that pass overlaps
// the barrier wait and the bulk copy still reading shared memory.
template <int N, int E, int S, bool HZ = false, bool SYNC0 = false>
__device__ __forceinline__ void block_fft(double2 (&v)[E], double2* sm, int t,
                                          const double2* __restrict__ tw,
                                          double2 extra = make_double2(0.0, 0.0)) {
  using Sh = FftShape<N, E>;
  constexpr int LOGE = Sh::LOGE;
  // pass 0: radix E, Ns = 1, inputs already in place, no twiddles
  if (HZ) {
    DftHalfZero<E, S>::run(v);
    if (extra.x != 0.0 || extra.y != 0.0) {
#pragma unroll
      for (int r = 0; r < E; ++r) v[r] = (r & 1) ? csub(v[r], extra) : cadd(v[r], extra);
    }
  } else {
    Dft<E, S>::run(v);
  }
  if (SYNC0) {
    if (t == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
  }
  if (Sh::NPASS == 1) return;
#pragma unroll
  for (int r = 0; r < E; ++r) sm[swz<LOGE>(t * E + r)] = v[r];
  __syncthreads();
  int Ns = E;
#pragma unroll
  for (int p = 1; p < Sh::NPASS - 1; ++p) {
    stockham_mid<N, E, E, S>(v, sm, t, Ns, tw, false);
    Ns *= E;
  }
  stockham_mid<N, E, Sh::RL, S>(v, sm, t, Ns, tw, true);
}

// Output index held by slot s of thread t after block_fft.
template <int N, int E>
__device__ __forceinline__ int fft_out_index(int t, int s) {
  using Sh = FftShape<N, E>;
  constexpr int RL = Sh::RL;
  return t + Sh::T * (s / RL) + (s % RL) * (N / RL);
}

}  // namespace fhtb
