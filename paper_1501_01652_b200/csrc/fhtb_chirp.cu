// fhtb_chirp.cu -- far field on grids that are not a power of two, or whose
// output rows are a strided subset (the DHT's padded grid 4N+3 with rows
// 4k-1, dht.py:158-174), by chirp-z convolution on power-of-two FFTs.
//
// For block rows k_j = k0 + s j (j < J; k0 = the grid's first output row so
// that output ownership is block independent) and block columns
// n_m = n0 + m (m < Mn), with E(P) = e^{i pi P / (2L)} and all phases reduced
// in exact integer arithmetic:
//
//   sum_m x_m e^{i pi k_j n_m / L}
//     = E(2 k0 n0 + 2 s j n0 + s j^2) * sum_m [x_m E(2 k0 m + s m^2)] E(-s (j-m)^2)
//
// i.e. a linear convolution of length Mn + J - 1 <= Q = 2^logQ computed as
// IFFT_Q(FFT_Q(a) * H), H = FFT_Q(h) precomputed per block.  Each of the 2M
// asymptotic terms of a request is one convolution; the column weights,
// pre-multipliers and in-chirp are applied while loading, the out-chirp, the
// row weights, order combination and post-multipliers in the epilogue.
//
//   pass 1: per column n1 of a = (n1 + Q1 n2), Q2-point FFT over n2, twiddle
//   pass 2: per column k2, Q1-point FFT over n1, * H, inverse Q1-point FFT,
//           twiddle, in place
//   pass 3: per column n1', inverse Q2-point FFT over k2, epilogue
#include "fhtb_core.cuh"
#include "fhtb_launch.h"

namespace fhtb {

int g_chirp_variant = 0;   // tuning bits (performance only): 1 = pass 3 unbounded regs

// x^p by binary powering (pre/post multipliers reach p = 10 per element)
__device__ __forceinline__ double ipow_c(double x, int p) {
  double r = 1.0;
  for (; p; p >>= 1) {
    if (p & 1) r *= x;
    x *= x;
  }
  return r;
}

__device__ __forceinline__ long long mod4(long long P, long long L4) {
  long long m = P % L4;
  return m < 0 ? m + L4 : m;
}

// e^{i pi P / (2L)}
__device__ __forceinline__ double2 chirpE(long long P, long long L) { return expi_pi_frac(mod4(P, 4 * L), 2 * L); }

__device__ __forceinline__ double2 qtw_s(const FarArgs& a, long long m, int sign) {
  const int lo = (int)(m & ((1LL << a.qbits) - 1));
  const long long hi = m >> a.qbits;
  double2 w = __ldg(a.qlo + lo);
  if (hi) w = cmul(w, __ldg(a.qhi + hi));
  return sign > 0 ? w : cconj(w);
}

// ------------------------------------------------------------------ pass 1
// HZ: the block's columns m < Mn <= Q/2 lie in the lower half of every
// column (n2 < N2/2), so the upper half of each thread's slots is zero and
// the first radix pass is the half-zero DFT.  The four-step twiddles
// e^{-2 pi i n1 k2/Q} of the thread's outputs are the same for every term:
// built once into shared memory (thread-private slot-major slots).
// QT = false (8192-point columns): the four-step twiddles are formed per
// use, the table would not fit beside the FFT buffer.
template <int N2, int E, int W, int MINB, bool HZ, bool QT = true>
__global__ void __launch_bounds__(W * (N2 / E), MINB)
chirp_pass1_kernel(FarArgs a) {
  constexpr int T = N2 / E;
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  constexpr int NP = N2 + PAD;
  constexpr int EH = HZ ? E / 2 : E;
  constexpr int NTH = W * T;
  extern __shared__ double2 sm2[];
  const int tid = threadIdx.x, w = tid % W, tt = tid / W;
  const int Q1 = a.L1;
  const long long Q = (long long)Q1 * N2;
  const long long n1 = (long long)blockIdx.x * W + w;
  const int ul = blockIdx.y;
  const UnitDesc U = a.units[a.u0 + ul];
  const ReqDesc& R = a.reqs[U.req];
  const BlockDesc& B = a.blocks[U.block];
  const long long cA = max(max(B.c0, R.col_lo), 1LL);
  const long long cB = min(B.c1, min(a.n_data_cols + 1, a.L + 1));
  const long long k0 = a.first, s = a.stride, n0 = B.c0, L = a.L;
  double br[EH], bi[EH], iw[EH];
#pragma unroll
  for (int e = 0; e < EH; ++e) {
    const long long m = n1 + (long long)Q1 * (tt + T * e);
    const long long n = n0 + m;
    br[e] = bi[e] = iw[e] = 0.0;
    if (n >= cA && n < cB) {
      double x = a.C[(long long)R.vec * a.ldc + (n - 1)];
      if (R.preA) x *= ipow_c(R.preA[n - 1], R.pa);
      if (R.preB) x *= ipow_c(R.preB[n - 1], R.pb);
      const double om = ((double)n + a.gamma) * 3.141592653589793;
      iw[e] = 1.0 / om;
      const double v = x * (1.0 / sqrt(om));
      const double2 c = chirpE(2 * k0 * m + s * ((m * m) % (4 * L)), L);
      br[e] = v * c.x;
      bi[e] = v * c.y;
    }
  }
  double2* sm = sm2 + w * NP;
  double2* qt = sm2 + W * NP + tid;
#pragma unroll
  for (int q = 0; q < E; ++q)
    if (QT) qt[q * NTH] = qtw_s(a, n1 * fft_out_index<N2, E>(tt, q), -1);
  const double2* tw = a.tw + (N2 - 2);
  const int nterm = 2 * a.M;
  const int t0 = 2 * a.p0, t1 = 2 * a.p1;     // this shard's terms
  for (int i = 0; i < t0; ++i) {
#pragma unroll
    for (int e = 0; e < EH; ++e) {
      br[e] *= iw[e];
      bi[e] *= iw[e];
    }
  }
  for (int i = t0; i < t1; ++i) {
    double2 z[E];
#pragma unroll
    for (int e = 0; e < EH; ++e) {
      z[e] = make_double2(br[e], bi[e]);
      br[e] *= iw[e];
      bi[e] *= iw[e];
    }
#pragma unroll
    for (int e = EH; e < E; ++e) z[e] = make_double2(0.0, 0.0);
    __syncthreads();
    block_fft<N2, E, -1, HZ>(z, sm, tt, tw);
    double2* G = a.G + (long long)(ul * nterm + i) * Q;
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int k2 = fft_out_index<N2, E>(tt, q);
      G[(long long)k2 * Q1 + n1] = cmul(z[q], QT ? qt[q * NTH] : qtw_s(a, n1 * k2, -1));
    }
  }
}

// ------------------------------------------------------------------ pass 2
// One CTA per (row k2, unit).  The filter row H_t[k2][.] and the four-step
// twiddles e^{2 pi i n1 k2/Q} are the same for all 2M terms of the unit:
// staged once in shared memory.  The next term's row is loaded while the
// current one is transformed (the kernel is otherwise latency bound).
template <int N1, int E, int MINB>
__global__ void __launch_bounds__(N1 / E, MINB)
chirp_pass2_kernel(FarArgs a) {
  constexpr int T = N1 / E;
  using Sh = FftShape<N1, E>;
  constexpr int RL = Sh::RL;
  extern __shared__ double2 sm2[];
  double2* shH = sm2 + N1;
  double2* shT = sm2 + 2 * N1;
  const int tt = threadIdx.x;
  const int k2 = blockIdx.x;
  const int ul = blockIdx.y;
  const long long Q = (long long)N1 * a.L2;
  const UnitDesc U = a.units[a.u0 + ul];
  const BlockDesc& B = a.blocks[U.block];
  const double2* __restrict__ H = B.H + (long long)k2 * N1;   // transposed spectrum row
  for (int x = tt; x < N1; x += T) {
    shH[x] = __ldg(H + x);
    shT[x] = qtw_s(a, (long long)x * k2, 1);
  }
  const double2* tw = a.tw + (N1 - 2);
  const int nterm = 2 * a.M;
  const int t0 = 2 * a.p0, t1 = 2 * a.p1;     // this shard's terms
  double2* row = a.G + (long long)(ul * nterm + t0) * Q + (long long)k2 * N1;
  double2 zn[E];
#pragma unroll
  for (int e = 0; e < E; ++e) zn[e] = row[tt + T * e];
  for (int i = t0; i < t1; ++i, row += Q) {
    double2 z[E];
#pragma unroll
    for (int e = 0; e < E; ++e) z[e] = zn[e];
    if (i + 1 < t1) {
#pragma unroll
      for (int e = 0; e < E; ++e) zn[e] = row[Q + tt + T * e];
    }
    __syncthreads();
    block_fft<N1, E, -1>(z, sm2, tt, tw);
    double2 y[E];
#pragma unroll
    for (int q = 0; q < E; ++q) y[(q / RL) + (q % RL) * (E / RL)] = cmul(z[q], shH[fft_out_index<N1, E>(tt, q)]);
    __syncthreads();
    block_fft<N1, E, 1>(y, sm2, tt, tw);
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const int n1 = fft_out_index<N1, E>(tt, q);
      row[n1] = cmul(y[q], shT[n1]);
    }
  }
}

// ------------------------------------------------------------------ pass 3
// One CTA per (column group, unit): all 2M terms of the unit are reduced in
// registers and written as a per-unit partial row part[unit][j]; the
// partials of one vector are summed in unit order by chirp_reduce_kernel.
//
// Row j (k = k0 + s j) of term i contributes
//   rp0 (L/k)^i [cos(th) Re((a_i - i b_i) w_i) + sin(th) Re((as_i - i bs_i) w_i)]
// with w_i = Y_i * oc (oc = out-chirp / Q) and th = -gamma pi k/L.  The
// per-term scalars satisfy as_i = -b_i, bs_i = a_i (pack_requests), so the
// second sum is Im of the first: one complex accumulator S, folded by
// Horner's rule in 1/k from the last term down, S <- S (L/k) + (a_i - i b_i) Y_i;
// oc, rp0 and the rotation are applied once at the end.  The next term's
// column is loaded while the current one is transformed.
template <int N2, int E, int W, int MINB>
__global__ void __launch_bounds__(W * (N2 / E), MINB)
chirp_pass3_kernel(FarArgs a) {
  constexpr int T = N2 / E;
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  constexpr int NP = N2 + PAD;
  extern __shared__ double2 sm2[];
  const int tid = threadIdx.x, w = tid % W, tt = tid / W;
  const int Q1 = a.L1;
  const long long Q = (long long)Q1 * N2;
  const long long n1 = (long long)blockIdx.x * W + w;
  const int ul = blockIdx.y;
  const long long L = a.L, k0 = a.first, s = a.stride;
  const UnitDesc U = a.units[a.u0 + ul];
  const ReqDesc& R = a.reqs[U.req];
  const BlockDesc& B = a.blocks[U.block];
  double ir[E];
  double2 SC[E];
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const long long j = n1 + (long long)Q1 * fft_out_index<N2, E>(tt, q);
    const long long k = k0 + s * j;
    ir[q] = (j < B.J && k >= B.r0 && k < B.r1 && k <= L) ? a.Ld / (double)k : 0.0;
    SC[q] = make_double2(0.0, 0.0);
  }
  double2* sm = sm2 + w * NP;
  const double2* tw = a.tw + (N2 - 2);
  const int nterm = 2 * a.M;
  const int t0 = 2 * a.p0, t1 = 2 * a.p1;     // this shard's terms
  const double2* G = a.G + (long long)(ul * nterm + t1 - 1) * Q + n1;
  double2 zn[E];
#pragma unroll
  for (int e = 0; e < E; ++e) zn[e] = G[(long long)(tt + T * e) * Q1];
  for (int i = t1 - 1; i >= t0; --i, G -= Q) {
    double2 z[E];
#pragma unroll
    for (int e = 0; e < E; ++e) z[e] = zn[e];
    if (i > t0) {
#pragma unroll
      for (int e = 0; e < E; ++e) zn[e] = G[(long long)(tt + T * e) * Q1 - Q];
    }
    __syncthreads();
    block_fft<N2, E, 1>(z, sm, tt, tw);
    const double ac = R.ac[i], bc = R.bc[i];
#pragma unroll
    for (int q = 0; q < E; ++q) {
      // S = S * ir + (ac - i bc) z
      SC[q].x = fma(SC[q].x, ir[q], fma(ac, z[q].x, bc * z[q].y));
      SC[q].y = fma(SC[q].y, ir[q], fma(ac, z[q].y, -bc * z[q].x));
    }
  }
  const double invQ = 1.0 / (double)Q;
  const long long n0 = B.c0;
  double* part = a.part + (long long)ul * a.part_stride;
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const long long j = n1 + (long long)Q1 * fft_out_index<N2, E>(tt, q);
    if (j < a.n_out && ir[q] != 0.0) {
      const long long k = k0 + s * j;
      double post = 1.0;
      if (R.pr) post = ipow_c((double)k / a.Ld, R.pr);
      if (R.post_e && R.pe) post *= ipow_c(R.post_e[j], R.pe);
      double rp0 = post * sqrt(ir[q]) * invQ;
      for (int i = 0; i < t0; ++i) rp0 *= ir[q];                  // (L/k)^{t0}
      const long long P = 2 * k0 * n0 + 2 * s * j * n0 + s * ((j * j) % (4 * L));
      const double2 oc = chirpE(P, L);
      const double2 wv = cmul(oc, SC[q]);
      double v = wv.x;
      if (a.gamma != 0.0) {
        double th, tc;
        sincos(-a.gamma * (double)k * a.pi_over_L, &th, &tc);
        v = tc * wv.x + th * wv.y;
      }
      part[j] = rp0 * v;
    }
  }
}

// F[vec][j] += sum over the chunk's units of that vector (unit order).
__global__ void chirp_reduce_kernel(FarArgs a, int n_units) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= a.n_out) return;
  int u = 0;
  while (u < n_units) {
    const int vec = a.units[a.u0 + u].vec;
    // unit by unit into F: independent of chunk boundaries (far_reduce_kernel)
    double* f = a.F + (long long)vec * a.ldf + j;
    double s = *f;
    while (u < n_units && a.units[a.u0 + u].vec == vec) {
      s += a.part[(long long)u * a.part_stride + j];
      ++u;
    }
    *f = s;
    if (!isfinite(s)) *a.nf = 1;
  }
}

cudaError_t launch_chirp_reduce(const FarArgs& a, int n_units, cudaStream_t st) {
  const long long b = (a.n_out + 255) / 256;
  note_launch(), chirp_reduce_kernel<<<(unsigned)b, 256, 0, st>>>(a, n_units);
  return cudaGetLastError();
}

// ----------------------------------------------- plain FFT passes (filters)
// out[k2*Q1 + n1] = e^{S 2 pi i n1 k2/Q} * FFT_{N2}(in[n1 + Q1 n2])
template <int N2, int E, int W, int S>
__global__ void __launch_bounds__(W * (N2 / E))
plain_pass1_kernel(const double2* __restrict__ in, double2* __restrict__ out, FarArgs a) {
  constexpr int T = N2 / E;
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  constexpr int NP = N2 + PAD;
  extern __shared__ double2 sm2[];
  const int tid = threadIdx.x, w = tid % W, tt = tid / W;
  const int Q1 = a.L1;
  const long long n1 = (long long)blockIdx.x * W + w;
  double2 z[E];
#pragma unroll
  for (int e = 0; e < E; ++e) z[e] = in[n1 + (long long)Q1 * (tt + T * e)];
  block_fft<N2, E, S>(z, sm2 + w * NP, tt, a.tw + (N2 - 2));
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int k2 = fft_out_index<N2, E>(tt, q);
    out[(long long)k2 * Q1 + n1] = cmul(z[q], qtw_s(a, n1 * k2, S));
  }
}

// out[k2 + Q2 k1] = FFT_{N1}(in[k2*N1 + n1]); tr: out[k2*N1 + k1] (the
// transposed spectrum layout chirp_pass2 reads row by row)
template <int N1, int E, int S>
__global__ void __launch_bounds__(N1 / E)
plain_pass2_kernel(const double2* __restrict__ in, double2* __restrict__ out, FarArgs a, int tr) {
  constexpr int T = N1 / E;
  extern __shared__ double2 sm2[];
  const int tt = threadIdx.x, k2 = blockIdx.x, Q2 = a.L2;
  double2 z[E];
#pragma unroll
  for (int e = 0; e < E; ++e) z[e] = in[(long long)k2 * N1 + tt + T * e];
  block_fft<N1, E, S>(z, sm2, tt, a.tw + (N1 - 2));
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const int k1 = fft_out_index<N1, E>(tt, q);
    out[tr ? (long long)k2 * N1 + k1 : k2 + (long long)Q2 * k1] = z[q];
  }
}

// h[d mod Q] = E(-s d^2) for d in [-(Mn-1), J-1], else 0
__global__ void chirp_filter_kernel(double2* h, long long Q, long long Mn, long long J, long long s, long long L) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < Q; i += (long long)gridDim.x * blockDim.x) {
    long long d = i <= J - 1 ? i : i - Q;   // i in [0, J) -> d = i ; i in [Q-(Mn-1), Q) -> d = i - Q
    double2 v = make_double2(0.0, 0.0);
    if (i < J || (i >= Q - (Mn - 1))) {
      const long long d2 = (d * d) % (4 * L);
      v = chirpE(-s * d2, L);
    }
    h[i] = v;
  }
}

// ------------------------------------------------------------ DCT-I/DST-I
// One CTA per row, Q <= 8192: out[k] = Re/Im sum_{m<n} v_m e^{i pi (k0+k)(n0+m)/L}
template <int N, int E>
__global__ void __launch_bounds__(N / E)
trig_kernel(int kind, long long n, long long L, long long k0, long long n0, const double* __restrict__ v,
            double* __restrict__ out, const double2* __restrict__ H, const double2* __restrict__ tw_pool) {
  constexpr int T = N / E;
  using Sh = FftShape<N, E>;
  constexpr int RL = Sh::RL;
  extern __shared__ double2 sm2[];
  const int tt = threadIdx.x;
  const double* x = v + (long long)blockIdx.x * n;
  double2 z[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const long long m = tt + T * e;
    z[e] = make_double2(0.0, 0.0);
    if (m < n) {
      const double2 c = chirpE(2 * k0 * m + ((m * m) % (4 * L)), L);
      z[e] = make_double2(x[m] * c.x, x[m] * c.y);
    }
  }
  const double2* tw = tw_pool + (N - 2);
  block_fft<N, E, -1>(z, sm2, tt, tw);
  double2 y[E];
#pragma unroll
  for (int q = 0; q < E; ++q) y[(q / RL) + (q % RL) * (E / RL)] = cmul(z[q], __ldg(H + fft_out_index<N, E>(tt, q)));
  __syncthreads();
  block_fft<N, E, 1>(y, sm2, tt, tw);
  double* o = out + (long long)blockIdx.x * n;
#pragma unroll
  for (int q = 0; q < E; ++q) {
    const long long j = fft_out_index<N, E>(tt, q);
    if (j < n) {
      const long long P = 2 * k0 * n0 + 2 * j * n0 + ((j * j) % (4 * L));
      const double2 c = chirpE(P, L);
      const double2 Y = cmul(y[q], c);
      o[j] = (kind == 0 ? Y.x : Y.y) / (double)N;
    }
  }
}

// Lengths with Q > 8192 (any length, trig.py:80-92 has no cap): the same
// chirp-z convolution on the multi-pass power-of-two FFT (plain_fft), per row:
//   A = v * in-chirp (zero padded to Q);  A2 = FFT(A);  A = conj(A2 * H);
//   A2 = FFT(A)  (= conj of the unnormalised inverse FFT of A2 * H);
//   out = Re/Im(conj(A2) * out-chirp) / Q.
__global__ void trig_pre_kernel(const double* __restrict__ x, long long n, long long L, long long k0,
                                long long Q, double2* __restrict__ A) {
  for (long long m = blockIdx.x * (long long)blockDim.x + threadIdx.x; m < Q; m += (long long)gridDim.x * blockDim.x) {
    double2 z = make_double2(0.0, 0.0);
    if (m < n) {
      const double2 c = chirpE(2 * k0 * m + ((m * m) % (4 * L)), L);
      const double xv = x[m];
      z = make_double2(xv * c.x, xv * c.y);
    }
    A[m] = z;
  }
}

__global__ void trig_mid_kernel(const double2* __restrict__ A2, const double2* __restrict__ H, long long Q,
                                double2* __restrict__ A) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < Q; i += (long long)gridDim.x * blockDim.x)
    A[i] = cconj(cmul(A2[i], __ldg(H + i)));
}

__global__ void trig_post_kernel(int kind, const double2* __restrict__ A2, long long n, long long L, long long k0,
                                 long long n0, long long Q, double* __restrict__ o) {
  const double inv = 1.0 / (double)Q;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < n; j += (long long)gridDim.x * blockDim.x) {
    const long long P = 2 * k0 * n0 + 2 * j * n0 + ((j * j) % (4 * L));
    const double2 Y = cmul(cconj(A2[j]), chirpE(P, L));
    o[j] = (kind == 0 ? Y.x : Y.y) * inv;
  }
}

static unsigned ew_blocks(long long n) {
  long long b = (n + 255) / 256;
  return (unsigned)(b > 148 * 32 ? 148 * 32 : (b < 1 ? 1 : b));
}

cudaError_t launch_trig_pre(const double* x, long long n, long long L, long long k0, long long Q, double2* A,
                            cudaStream_t st) {
  note_launch(), trig_pre_kernel<<<ew_blocks(Q), 256, 0, st>>>(x, n, L, k0, Q, A);
  return cudaGetLastError();
}

cudaError_t launch_trig_mid(const double2* A2, const double2* H, long long Q, double2* A, cudaStream_t st) {
  note_launch(), trig_mid_kernel<<<ew_blocks(Q), 256, 0, st>>>(A2, H, Q, A);
  return cudaGetLastError();
}

cudaError_t launch_trig_post(int kind, const double2* A2, long long n, long long L, long long k0, long long n0,
                             long long Q, double* out, cudaStream_t st) {
  note_launch(), trig_post_kernel<<<ew_blocks(n), 256, 0, st>>>(kind, A2, n, L, k0, n0, Q, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- launch
static int pick_w(int N2) {
  int T = N2 >= 8 ? N2 / 8 : 1;
  int w = 256 / T;
  if (w < 1) w = 1;
  if (w > 8) w = 8;
  return w;
}

template <int N2, int W>
static cudaError_t c1_w(const FarArgs& a, int n_units, int hz, cudaStream_t st) {
  // 8192-point columns (Q = 2^25, the DHT at N = 2^24): 16 points per
  // thread, one CTA per SM, twiddles per use
  constexpr bool BIG = N2 >= 8192;
  constexpr int E = BIG ? 16 : (N2 >= 8 ? 8 : N2);
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  const int smem = (W * (N2 + PAD) + (BIG ? 0 : W * N2)) * 16;   // FFT buffers + four-step twiddles
  constexpr int MB = BIG ? 1 : ((W * (N2 / E)) >= 256 ? 2 : 1);
  auto k = (hz && E >= 8) ? chirp_pass1_kernel<N2, E, W, MB, true, !BIG> : chirp_pass1_kernel<N2, E, W, MB, false, !BIG>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  note_launch(), k<<<dim3(a.L1 / W, n_units), W * (N2 / E), smem, st>>>(a);
  return cudaGetLastError();
}

template <int N2, int W>
static cudaError_t c3_w(const FarArgs& a, int n_ranges, cudaStream_t st) {
  constexpr bool BIG = N2 >= 8192;          // see c1_w
  constexpr int E = BIG ? 16 : (N2 >= 8 ? 8 : N2);
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  const int smem = W * (N2 + PAD) * 16;
  constexpr int MB = BIG ? 1 : ((W * (N2 / E)) >= 256 ? 2 : 1);
  auto k = (g_chirp_variant & 1) ? chirp_pass3_kernel<N2, E, W, 1> : chirp_pass3_kernel<N2, E, W, MB>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  note_launch(), k<<<dim3(a.L1 / W, n_ranges), W * (N2 / E), smem, st>>>(a);
  return cudaGetLastError();
}

template <int N2, int W, int S>
static cudaError_t pp1_w(const double2* in, double2* out, const FarArgs& a, cudaStream_t st) {
  constexpr int E = N2 >= 8 ? 8 : N2;
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  const int smem = W * (N2 + PAD) * 16;
  auto k = plain_pass1_kernel<N2, E, W, S>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  note_launch(), k<<<dim3(a.L1 / W), W * (N2 / E), smem, st>>>(in, out, a);
  return cudaGetLastError();
}

// W must divide L1 (Q1); choose the largest power of two <= min(cap, Q1).
#define FHTB_W_DISPATCH(FN, N2, ...)                                             \
  do {                                                                           \
    int w_ = pick_w(N2);                                                         \
    while (w_ > a.L1) w_ >>= 1;                                                  \
    switch (w_) {                                                                \
      case 8: return FN<N2, 8>(__VA_ARGS__);                                     \
      case 4: return FN<N2, 4>(__VA_ARGS__);                                     \
      case 2: return FN<N2, 2>(__VA_ARGS__);                                     \
      default: return FN<N2, 1>(__VA_ARGS__);                                    \
    }                                                                            \
  } while (0)

#define FHTB_SIZE_SWITCH(LOG, MACRO)                                             \
  switch (LOG) {                                                                 \
    case 1: MACRO(2); case 2: MACRO(4); case 3: MACRO(8); case 4: MACRO(16);     \
    case 5: MACRO(32); case 6: MACRO(64); case 7: MACRO(128); case 8: MACRO(256);\
    case 9: MACRO(512); case 10: MACRO(1024); case 11: MACRO(2048);              \
    case 12: MACRO(4096); case 13: MACRO(8192);                                  \
  }

cudaError_t launch_chirp_pass1(const FarArgs& a, int logN2, int n_units, int hz, cudaStream_t st) {
#define M1(N) FHTB_W_DISPATCH(c1_w, N, a, n_units, hz, st)
  FHTB_SIZE_SWITCH(logN2, M1)
#undef M1
  return cudaErrorInvalidValue;
}

cudaError_t launch_chirp_pass3(const FarArgs& a, int logN2, int n_ranges, cudaStream_t st) {
#define M3(N) FHTB_W_DISPATCH(c3_w, N, a, n_ranges, st)
  FHTB_SIZE_SWITCH(logN2, M3)
#undef M3
  return cudaErrorInvalidValue;
}

template <int N1>
static cudaError_t c2_t(const FarArgs& a, int n_units, cudaStream_t st) {
  constexpr int E = N1 >= 8 ? 8 : N1;
  const int smem = 3 * N1 * 16;
  constexpr int MB = N1 / E <= 32 ? 16 : (N1 / E <= 64 ? 8 : (N1 / E <= 128 ? 4 : 2));
  auto k = chirp_pass2_kernel<N1, E, MB>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  note_launch(), k<<<dim3(a.L2, n_units), N1 / E, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_chirp_pass2(const FarArgs& a, int logN1, int n_units, cudaStream_t st) {
#define M2(N) return c2_t<N>(a, n_units, st);
  FHTB_SIZE_SWITCH(logN1, M2)
#undef M2
  return cudaErrorInvalidValue;
}

template <int N1, int S>
static cudaError_t pp2_t(const double2* in, double2* out, const FarArgs& a, int tr, cudaStream_t st) {
  constexpr int E = N1 >= 8 ? 8 : N1;
  const int smem = N1 * 16;
  auto k = plain_pass2_kernel<N1, E, S>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  note_launch(), k<<<dim3(a.L2), N1 / E, smem, st>>>(in, out, a, tr);
  return cudaGetLastError();
}

// Forward (sign -1) FFT of length Q = L1*L2 of a device vector, out-of-place
// through `tmp`.  Used to build the chirp filter spectra.
cudaError_t launch_plain_fft(const FarArgs& a, int logN1, int logN2, const double2* in, double2* tmp,
                             double2* out, int transposed, cudaStream_t st) {
  cudaError_t e = cudaErrorInvalidValue;
#define PP1(N) { FHTB_W_DISPATCH_P1(N); }
#define FHTB_W_DISPATCH_P1(N)                                                    \
  do {                                                                           \
    int w_ = pick_w(N);                                                          \
    while (w_ > a.L1) w_ >>= 1;                                                  \
    switch (w_) {                                                                \
      case 8: e = pp1_w<N, 8, -1>(in, tmp, a, st); break;                        \
      case 4: e = pp1_w<N, 4, -1>(in, tmp, a, st); break;                        \
      case 2: e = pp1_w<N, 2, -1>(in, tmp, a, st); break;                        \
      default: e = pp1_w<N, 1, -1>(in, tmp, a, st); break;                       \
    }                                                                            \
  } while (0); break;
  switch (logN2) {
    case 1: PP1(2) case 2: PP1(4) case 3: PP1(8) case 4: PP1(16) case 5: PP1(32) case 6: PP1(64)
    case 7: PP1(128) case 8: PP1(256) case 9: PP1(512) case 10: PP1(1024) case 11: PP1(2048)
    case 12: PP1(4096) case 13: PP1(8192)
    default: return cudaErrorInvalidValue;
  }
#undef PP1
#undef FHTB_W_DISPATCH_P1
  if (e != cudaSuccess) return e;
#define PP2(N) e = pp2_t<N, -1>(tmp, out, a, transposed, st); break;
  switch (logN1) {
    case 1: PP2(2) case 2: PP2(4) case 3: PP2(8) case 4: PP2(16) case 5: PP2(32) case 6: PP2(64)
    case 7: PP2(128) case 8: PP2(256) case 9: PP2(512) case 10: PP2(1024) case 11: PP2(2048)
    case 12: PP2(4096) case 13: PP2(8192)
    default: return cudaErrorInvalidValue;
  }
#undef PP2
  return e;
}

cudaError_t launch_chirp_filter(double2* h, long long Q, long long Mn, long long J, long long s, long long L,
                                cudaStream_t st) {
  long long b = (Q + 255) / 256;
  if (b > 148 * 64) b = 148 * 64;
  note_launch(), chirp_filter_kernel<<<(int)b, 256, 0, st>>>(h, Q, Mn, J, s, L);
  return cudaGetLastError();
}

template <int N>
static cudaError_t trig_t(int kind, long long n, long long L, long long k0, long long n0, const double* v,
                          double* out, long long batch, const double2* H, const double2* tw, cudaStream_t st) {
  constexpr int E = N >= 16 ? 16 : N;
  const int smem = N * 16;
  auto k = trig_kernel<N, E>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  note_launch(), k<<<(unsigned)batch, N / E, smem, st>>>(kind, n, L, k0, n0, v, out, H, tw);
  return cudaGetLastError();
}

cudaError_t launch_trig(int kind, int logQ, long long n, long long L, long long k0, long long n0, const double* v,
                        double* out, long long batch, const double2* H, const double2* tw, cudaStream_t st) {
#define TT(N) return trig_t<N>(kind, n, L, k0, n0, v, out, batch, H, tw, st);
  FHTB_SIZE_SWITCH(logQ, TT)
#undef TT
  return cudaErrorInvalidValue;
}

}  // namespace fhtb
