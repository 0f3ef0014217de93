// fhtb_misc.cu -- element-wise Bessel kernels, J0 roots, twiddle tables and
// a batched power-of-two FFT utility.
//
//   bessel_j          bessel.py:232-260  (array path)
//   hankel_asy_eval   bessel.py:72-91
//   taylor_eval       bessel.py:133-146
//   bessel_roots_j0   bessel.py:295-321  (Newton from (n - 1/4) pi)
#include "fhtb_bessel.cuh"
#include "fhtb_core.cuh"
#include "fhtb_launch.h"

namespace fhtb {

static inline int grid_for(long long n, int threads) {
  long long b = (n + threads - 1) / threads;
  if (b > 148LL * 64) b = 148LL * 64;
  return (int)(b < 1 ? 1 : b);
}

__global__ void bessel_j_kernel(int nu, JOrder c, const double* __restrict__ z, long long n,
                                double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = jn(nu, z[i], c);
}

__global__ void bessel_multi_kernel(int omax, const JOrder* __restrict__ tab, const double* __restrict__ z,
                                    long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double v[kMaxOrd];
    jn_all<kMaxOrd>(omax, z[i], tab, v);
#pragma unroll
    for (int o = 0; o < kMaxOrd; ++o)
      if (o <= omax) out[(long long)o * n + i] = v[o];
  }
}

__global__ void hankel_eval_kernel(int nu, int mt, const double* __restrict__ coef,
                                   const double* __restrict__ z, long long n, double* __restrict__ out) {
  // coef: ae[0..mt), ao[0..mt)   (signed a_{2m}, a_{2m+1})
  const double phi = (2 * nu + 1) * (3.141592653589793 / 4.0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double x = z[i];
    const double w = 1.0 / (x * x);
    double pe = coef[mt - 1], po = coef[2 * mt - 1];
    for (int m = mt - 2; m >= 0; --m) {
      pe = pe * w + coef[m];
      po = po * w + coef[mt + m];
    }
    double s, c;
    sincos(x - phi, &s, &c);
    out[i] = FHTB_SQRT_2_OVER_PI / sqrt(x) * (c * pe - s * po / x);
  }
}

__global__ void taylor_eval_kernel(int nu, int nt, double inv_fact, const double* __restrict__ z,
                                   long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double h = 0.5 * z[i];
    double term = inv_fact;
    for (int k = 0; k < nu; ++k) term *= h;
    double acc = term;
    const double hh = h * h;
    for (int t = 1; t < nt; ++t) {
      term = -term * hh / (double)(t * (t + nu));
      acc += term;
    }
    out[i] = acc;
  }
}

// Newton on J0 from (n - 1/4) pi, J0' = -J1.  Per-element stopping at the
// reference's global criterion |step| <= 4 * 2^-52 * z_max (bessel.py:311).
__global__ void roots_j0_kernel(const JOrder* __restrict__ tab, long long count, double* __restrict__ roots,
                                double* __restrict__ pert, unsigned long long* resid_bits) {
  const double zmax = ((double)count - 0.25) * 3.141592653589793;
  const double stop = 4.0 * 2.220446049250313e-16 * zmax;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x) {
    const double g = ((double)(i + 1) - 0.25) * 3.141592653589793;
    double x = g;
    for (int it = 0; it < 20; ++it) {
      const double d = jn(0, x, tab[0]) / jn(1, x, tab[1]);
      x += d;
      if (fabs(d) <= stop) break;
    }
    roots[i] = x;
    pert[i] = x - g;
    const double r = fabs(jn(0, x, tab[0]));
    atomicMax(resid_bits, (unsigned long long)__double_as_longlong(r));
    // residual against the tolerance this root can meet in fp64: the
    // reference's 1e-13 (bessel.py:313), or, once the root's own rounding
    // dominates (|J0(x)| ~ |J1(x)| ulp(x) reaches 1e-13 near x ~ 2e6, i.e.
    // N ~ 2^20 roots), two ulps of x times |J1(x)|
    const double tol = fmax(1e-13, 2.0 * fabs(jn(1, x, tab[1])) * (fabs(x) * 2.220446049250313e-16));
    atomicMax(resid_bits + 1, (unsigned long long)__double_as_longlong(r / tol));
  }
}

// twiddle pool: table for N = 2^l (l = 1..max_log) at offset N - 2, e^{+2 pi i m / N}
__global__ void twiddle_kernel(double2* pool, int max_log) {
  const long long total = (1LL << (max_log + 1)) - 2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    // find l with 2^l - 2 <= i < 2^{l+1} - 2
    int l = 1;
    while ((1LL << (l + 1)) - 2 <= i) ++l;
    const long long N = 1LL << l;
    const long long m = i - (N - 2);
    double s, c;
    sincospi(2.0 * (double)m / (double)N, &s, &c);
    pool[i] = make_double2(c, s);
  }
}

__global__ void qtwiddle_kernel(double2* qlo, double2* qhi, int logQ, int qbits, int sign) {
  const long long Q = 1LL << logQ;
  const long long nlo = 1LL << qbits, nhi = Q >> qbits;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nlo + nhi;
       i += (long long)gridDim.x * blockDim.x) {
    const long long m = i < nlo ? i : (i - nlo) << qbits;
    double s, c;
    sincospi(2.0 * (double)m / (double)Q, &s, &c);
    const double2 v = make_double2(c, sign * s);
    if (i < nlo) qlo[i] = v; else qhi[i - nlo] = v;
  }
}

// Batched power-of-two FFT (N <= 4096), one CTA per transform.  Utility
// used by the tests to pin the FFT core against numpy, and for small
// filter spectra.
template <int N, int S>
__global__ void fft_batch_kernel(const double2* __restrict__ in, double2* __restrict__ out,
                                 const double2* __restrict__ tw_pool) {
  constexpr int E = N >= 16 ? 16 : N;
  constexpr int T = N / E;
  __shared__ double2 sm[N];
  const int t = threadIdx.x;
  const double2* x = in + (long long)blockIdx.x * N;
  double2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = x[t + T * e];
  block_fft<N, E, S>(v, sm, t, tw_pool + (N - 2));
  double2* y = out + (long long)blockIdx.x * N;
#pragma unroll
  for (int s = 0; s < E; ++s) y[fft_out_index<N, E>(t, s)] = v[s];
}

template <int N>
static cudaError_t fftb_t(int sign, const double2* in, double2* out, long long batch,
                          const double2* tw, cudaStream_t st) {
  constexpr int E = N >= 16 ? 16 : N;
  if (sign > 0) note_launch(), fft_batch_kernel<N, 1><<<(unsigned)batch, N / E, 0, st>>>(in, out, tw);
  else note_launch(), fft_batch_kernel<N, -1><<<(unsigned)batch, N / E, 0, st>>>(in, out, tw);
  return cudaGetLastError();
}

cudaError_t launch_fft_batch(int logN, int sign, const double2* in, double2* out, long long batch,
                             const double2* tw, cudaStream_t st) {
  switch (logN) {
    case 1: return fftb_t<2>(sign, in, out, batch, tw, st);
    case 2: return fftb_t<4>(sign, in, out, batch, tw, st);
    case 3: return fftb_t<8>(sign, in, out, batch, tw, st);
    case 4: return fftb_t<16>(sign, in, out, batch, tw, st);
    case 5: return fftb_t<32>(sign, in, out, batch, tw, st);
    case 6: return fftb_t<64>(sign, in, out, batch, tw, st);
    case 7: return fftb_t<128>(sign, in, out, batch, tw, st);
    case 8: return fftb_t<256>(sign, in, out, batch, tw, st);
    case 9: return fftb_t<512>(sign, in, out, batch, tw, st);
    case 10: return fftb_t<1024>(sign, in, out, batch, tw, st);
    case 11: return fftb_t<2048>(sign, in, out, batch, tw, st);
  }
  return cudaErrorInvalidValue;
}

// Planning statistics of one coefficient row (fourier_bessel.py:208-225,
// dht.py:140-157 take them with numpy on the host): out[3v] = sum |c_n|,
// out[3v+1] = max |b_n| over the n >= n_split with c_n != 0, out[3v+2] = 1 if
// any such n exists.  One CTA per row, fixed-order tree (deterministic).
__global__ void __launch_bounds__(256)
coef_stats_kernel(const double* __restrict__ C, long long ldc, long long n, long long n_split,
                  const double* __restrict__ b, long long nb, double* __restrict__ out) {
  const double* c = C + (long long)blockIdx.x * ldc;
  double l1 = 0.0, bm = 0.0, nz = 0.0;
  for (long long i = threadIdx.x; i < n; i += 256) {
    const double x = c[i];
    l1 += fabs(x);
    if (i >= n_split && x != 0.0) {
      nz = 1.0;
      if (b && i < nb) bm = fmax(bm, fabs(b[i]));
    }
  }
  __shared__ double s[3][256];
  s[0][threadIdx.x] = l1;
  s[1][threadIdx.x] = bm;
  s[2][threadIdx.x] = nz;
  __syncthreads();
  for (int h = 128; h; h >>= 1) {
    if (threadIdx.x < h) {
      s[0][threadIdx.x] += s[0][threadIdx.x + h];
      s[1][threadIdx.x] = fmax(s[1][threadIdx.x], s[1][threadIdx.x + h]);
      s[2][threadIdx.x] = fmax(s[2][threadIdx.x], s[2][threadIdx.x + h]);
    }
    __syncthreads();
  }
  if (threadIdx.x < 3) out[3 * (long long)blockIdx.x + threadIdx.x] = s[threadIdx.x][0];
}

cudaError_t launch_coef_stats(const double* C, long long ldc, int n_vec, long long n, long long n_split,
                              const double* b, long long nb, double* out, cudaStream_t st) {
  if (n_vec == 0) return cudaSuccess;
  note_launch(), coef_stats_kernel<<<n_vec, 256, 0, st>>>(C, ldc, n, n_split, b, nb, out);
  return cudaGetLastError();
}

// out[v][i] = alpha * a[v][i] * w[i]  (dht.py:188-190: the diagonal D_v of the self-inverse check)
__global__ void mul_rows_kernel(double* __restrict__ out, long long ldo, const double* __restrict__ a, long long lda,
                                const double* __restrict__ w, double alpha, long long n, int n_vec) {
  const long long tot = n * n_vec;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long v = e / n, i = e % n;
    out[v * ldo + i] = alpha * a[v * lda + i] * (w ? w[i] : 1.0);
  }
}

cudaError_t launch_mul_rows(double* out, long long ldo, const double* a, long long lda, const double* w, double alpha,
                            long long n, int n_vec, cudaStream_t st) {
  if (n * n_vec == 0) return cudaSuccess;
  note_launch(), mul_rows_kernel<<<grid_for(n * n_vec, 256), 256, 0, st>>>(out, ldo, a, lda, w, alpha, n, n_vec);
  return cudaGetLastError();
}

// res[0] = max_i |alpha * a[i] - b[i]|  (bit pattern of a non-negative double, atomicMax)
__global__ void max_abs_diff_kernel(const double* __restrict__ a, double alpha, const double* __restrict__ b,
                                    long long n, unsigned long long* res) {
  double m = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(alpha * a[i] - b[i]));
#pragma unroll
  for (int off = 16; off; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(res, (unsigned long long)__double_as_longlong(m));
}

cudaError_t launch_max_abs_diff(const double* a, double alpha, const double* b, long long n, unsigned long long* res,
                                cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  note_launch(), max_abs_diff_kernel<<<grid_for(n, 256), 256, 0, st>>>(a, alpha, b, n, res);
  return cudaGetLastError();
}

cudaError_t launch_twiddles(double2* pool, int max_log, cudaStream_t st) {
  const long long total = (1LL << (max_log + 1)) - 2;
  note_launch(), twiddle_kernel<<<grid_for(total, 256), 256, 0, st>>>(pool, max_log);
  return cudaGetLastError();
}

cudaError_t launch_qtwiddles(double2* qlo, double2* qhi, int logQ, int qbits, int sign, cudaStream_t st) {
  const long long n = (1LL << qbits) + ((1LL << logQ) >> qbits);
  note_launch(), qtwiddle_kernel<<<grid_for(n, 256), 256, 0, st>>>(qlo, qhi, logQ, qbits, sign);
  return cudaGetLastError();
}

cudaError_t launch_bessel_j(int nu, const JOrder& c, const double* z, long long n, double* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  note_launch(), bessel_j_kernel<<<grid_for(n, 256), 256, 0, st>>>(nu, c, z, n, out);
  return cudaGetLastError();
}

cudaError_t launch_bessel_multi(int omax, const JOrder* tab, const double* z, long long n, double* out,
                                cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  note_launch(), bessel_multi_kernel<<<grid_for(n, 256), 256, 0, st>>>(omax, tab, z, n, out);
  return cudaGetLastError();
}

cudaError_t launch_hankel_eval(int nu, int mt, const double* coef, const double* z, long long n, double* out,
                               cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  note_launch(), hankel_eval_kernel<<<grid_for(n, 256), 256, 0, st>>>(nu, mt, coef, z, n, out);
  return cudaGetLastError();
}

cudaError_t launch_taylor_eval(int nu, int nt, double inv_fact, const double* z, long long n, double* out,
                               cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  note_launch(), taylor_eval_kernel<<<grid_for(n, 256), 256, 0, st>>>(nu, nt, inv_fact, z, n, out);
  return cudaGetLastError();
}

cudaError_t launch_roots_j0(const JOrder* tab, long long count, double* roots, double* pert,
                            unsigned long long* resid_bits, cudaStream_t st) {
  note_launch(), roots_j0_kernel<<<grid_for(count, 256), 256, 0, st>>>(tab, count, roots, pert, resid_bits);
  return cudaGetLastError();
}

}  // namespace fhtb
