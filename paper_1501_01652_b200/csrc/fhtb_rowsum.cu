// fhtb_rowsum.cu -- far field, narrow-row blocks in fully fused form
// (reference behaviour: schlomilch.py:301-329 block application restricted to
// a block with few rows; see fhtb_far.cu for the general two-pass form).
#include "fhtb_core.cuh"
#include "fhtb_launch.h"
#include "fhtb_far.cuh"

namespace fhtb {

// ------------------------------------------- narrow rows, fully fused form
//
// A block whose rows all lie below L2 = 2^lr (lr <= 12) needs, per column n1,
// only the bin k1 = 0 of pass 2 and its partner:
//     Z_p[k]          = S0_p[k]      = sum_n1 t(n1, k)      F_{p,n1}[k]
//     conj Z_p[2L-k]  = conj S1_p[k'] , S1_p[k'] = sum_n1 t(n1, k' - L2) F_{p,n1}[k'],  k' = L2 - k
// with F_{p,n1} the L2-point column FFT of pair p and t(n1, m) = e^{2 pi i n1 m / Q}.
// The row epilogue is linear in Z_p[k] and antilinear in Z_p[2L-k]:
//     U_k = sum_p (L/k)^{2p} [ alpha_p(k) S0_p[k] + beta_p(k) conj S1_p[L2-k] ],
//     alpha_p = c0_p - i (L/k) c1_p,  beta_p = c0_p + i (L/k) c1_p,  c_i = a_i - i b_i,
// so the sum over the pairs is folded PER COLUMN, in the registers of the
// thread that holds FFT output k2, before the sum over the columns:
//     A_n1[k2] = sum_p (L/k)^{2p} alpha_p(k) F_{p,n1}[k2]            (k = k2      in the block rows)
//     B_n1[k2] = sum_p (L/k)^{2p} conj(beta_p(k)) F_{p,n1}[k2]       (k = L2 - k2 in the block rows)
//     U_k = sum_n1 t(n1, k) A_n1[k]  +  conj( sum_n1 t(n1, -k) B_n1[L2-k] ).
// One CTA = W columns of one unit (as pass 1): the coefficients are loaded
// once, the M column FFTs run back to back with Horner's rule over the pairs
// from the last one down, and only the folded values of the block's rows
// leave the CTA: P[unit][A|B][row][n1] (2 * rows * L1 complex per unit
// instead of M * 2L, no pass 2, no row sums over the intermediate).
// far_rowsum_fin_kernel sums P over n1 in a fixed order and finishes the row.
//
// The pairs run downwards (Horner), so the inputs of pair p are formed from
// the pair-0 state by binary powering, x_n omega_n^{-1/2} (omega_n^{-2})^p
// (the bits of p are uniform over the CTA): an underflow of a high pair only
// drops that negligible pair, and the leading pair is exact.
// A k2 that serves both a row k2 and a row L2 - k2 (L2 - r1 < k2 < r1) keeps
// its second accumulator in shared memory (thread-private slot).
template <int EH>
__device__ __forceinline__ void pair_inputs(int p, const double (&u)[EH], const double (&iw)[EH], double us,
                                            double iws, double sig, double2 (&z)[2 * EH], double2& extra) {
  double b[EH], bs = iws * iws;
#pragma unroll
  for (int e = 0; e < EH; ++e) {
    b[e] = iw[e] * iw[e];
    z[e].x = u[e];
  }
  for (int q = p; q; q >>= 1) {
    if (q & 1) {
#pragma unroll
      for (int e = 0; e < EH; ++e) z[e].x *= b[e];
      us *= bs;
    }
#pragma unroll
    for (int e = 0; e < EH; ++e) b[e] *= b[e];
    bs *= bs;
  }
#pragma unroll
  for (int e = 0; e < EH; ++e) {
    z[e].y = (z[e].x * iw[e]) * sig;        // term 2p+1, carried times sig (BlockDesc)
    z[e + EH] = make_double2(0.0, 0.0);
  }
  extra = make_double2(us, (us * iws) * sig);
}

template <int N2, int W, int MINB, int E = 16>
__global__ void __launch_bounds__(W * (N2 / E), MINB)
far_rowsum_kernel(FarArgs a) {
  constexpr int T = N2 / E, EH = E / 2, NTH = W * T;
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  constexpr int NP = N2 + PAD;
  extern __shared__ __align__(16) double2 sm2[];
  double* wA = reinterpret_cast<double*>(sm2 + W * NP);     // [s][tid]: L/k, k = k2
  double* wB = wA + E * NTH;                                // [s][tid]: L/k, k = N2 - k2
  double2* A2 = reinterpret_cast<double2*>(wB + E * NTH);   // [s][tid]: B where A and B share a k2
  const int tid = threadIdx.x, w = tid % W, tt = tid / W;
  const int L1 = a.L1;
  const long long n1 = (long long)blockIdx.x * W + w;
  const int ul = blockIdx.y;
  const UnitDesc U = a.units[a.u0 + ul];
  const ReqDesc& R = a.reqs[U.req];
  const BlockDesc& B = a.blocks[U.block];
  const double bsig = B.sig, bisig = B.isig;
  long long cA, cB;
  unit_cols(a, R, B, cA, cB);
  const int R0 = (int)max(B.r0, 1LL), R1 = (int)min(B.r1, (long long)N2);
  unsigned m0 = 0, m1 = 0;
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int k2 = fft_out_index<N2, E>(tt, s), kb = N2 - k2;
    const bool t0 = k2 >= R0 && k2 < R1, t1 = k2 >= 1 && kb >= R0 && kb < R1;
    m0 |= (unsigned)t0 << s;
    m1 |= (unsigned)t1 << s;
    wA[s * NTH + tid] = t0 ? a.Ld / (double)k2 : 0.0;
    wB[s * NTH + tid] = t1 ? a.Ld / (double)kb : 0.0;
    A2[s * NTH + tid] = make_double2(0.0, 0.0);
  }
  // column state of pair 0: u = x omega^{-1/2}, iw = 1/omega
  double u[EH], iw[EH], us = 0.0, iws = 0.0;
#pragma unroll
  for (int e = 0; e < EH; ++e) load_col(a, R, cA, cB, n1 + (long long)L1 * (tt + T * e), u[e], iw[e]);
  if (tt == 0 && n1 == 0) load_col(a, R, cA, cB, (long long)L1 * (T * EH), us, iws);
  double2 A[E];
#pragma unroll
  for (int s = 0; s < E; ++s) A[s] = make_double2(0.0, 0.0);
  const double2* tw = a.tw + (N2 - 2);
  double2* sm = sm2 + w * NP;
  for (int p = a.p1 - 1; p >= a.p0; --p) {
    double2 z[E];
    double2 extra;
    pair_inputs<EH>(p, u, iw, us, iws, bsig, z, extra);
    // (the barrier after the register-only first radix pass separates the
    // previous pair's last shared-memory reads from this pair's writes)
    block_fft<N2, E, 1, true, true>(z, sm, tt, tw, extra);
    const double c0x = R.ac[2 * p], c0y = -R.bc[2 * p];
    const double c1x = R.ac[2 * p + 1] * bisig, c1y = -R.bc[2 * p + 1] * bisig;
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const bool t0 = (m0 >> s) & 1u, t1 = (m1 >> s) & 1u;
      if (t0 || t1) {
        // alpha = c0 - i wk c1 (row k2), or conj(beta) = conj(c0) - i wk conj(c1) (row N2 - k2)
        const double wk = t0 ? wA[s * NTH + tid] : wB[s * NTH + tid];
        const double gx = t0 ? fma(wk, c1y, c0x) : fma(-wk, c1y, c0x);
        const double gy = t0 ? fma(-wk, c1x, c0y) : fma(-wk, c1x, -c0y);
        const double w2 = wk * wk;
        A[s].x = fma(A[s].x, w2, fma(gx, z[s].x, -gy * z[s].y));
        A[s].y = fma(A[s].y, w2, fma(gx, z[s].y, gy * z[s].x));
      }
      if (t0 && t1) {
        const double wk = wB[s * NTH + tid];
        const double gx = fma(-wk, c1y, c0x), gy = fma(-wk, c1x, -c0y), w2 = wk * wk;
        double2 t = A2[s * NTH + tid];
        t.x = fma(t.x, w2, fma(gx, z[s].x, -gy * z[s].y));
        t.y = fma(t.y, w2, fma(gx, z[s].y, gy * z[s].x));
        A2[s * NTH + tid] = t;
      }
    }
  }
  // four-step twiddles, once per column, and the folded rows out
  const long long qm = (1LL << a.logQ) - 1;
  double2* P0 = a.G + ((long long)(2 * ul) * a.rs) * L1 + n1;
  double2* P1 = a.G + ((long long)(2 * ul + 1) * a.rs) * L1 + n1;
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const bool t0 = (m0 >> s) & 1u, t1 = (m1 >> s) & 1u;
    const int k2 = fft_out_index<N2, E>(tt, s), kb = N2 - k2;
    if (t0) P0[(long long)(k2 - R0) * L1] = cmul(A[s], qtw(a, (n1 * k2) & qm));
    if (t1) {
      const double2 b = t0 ? A2[s * NTH + tid] : A[s];
      P1[(long long)(kb - R0) * L1] = cmul(b, qtw(a, (n1 * (long long)(k2 - N2)) & qm));
    }
  }
}

// High-occupancy form for column FFTs of up to 2048 points.  The folded
// accumulators live in thread-private shared-memory slots instead of 64
// registers (read-modify-write once per pair and needed output: ~26 B of
// shared-memory traffic per point against the 32 + 16 B of pass 1's twiddle
// table and tensor-store staging), omega_n^2 is recomputed per pair, and the
// row factors L/k come from one table per CTA; that leaves the registers of
// pass 1, so three CTAs fit on an SM.  OVS: second-accumulator slots per
// thread for the k2 that serve two rows (0: none can occur, host-checked:
// 2 r1 <= N2 + 1; 2: at most two per thread, 2 r1 - N2 - 1 <= N2 / 16).
template <int N2, int W, int MINB, int OVS>
__global__ void __launch_bounds__(W * (N2 / 16), MINB)
far_rowsum2_kernel(FarArgs a) {
  constexpr int E = 16, T = N2 / E, EH = E / 2, NTH = W * T;
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  constexpr int NP = N2 + PAD;
  extern __shared__ __align__(16) double2 sm2[];
  double2* As = sm2 + W * NP;                               // [s][tid]
  double2* A2s = As + E * NTH;                              // [j < OVS][tid]
  double* wt = reinterpret_cast<double*>(A2s + OVS * NTH);  // [k - R0]: L/k
  const int tid = threadIdx.x, w = tid % W, tt = tid / W;
  const int L1 = a.L1;
  const long long n1 = (long long)blockIdx.x * W + w;
  const int ul = blockIdx.y;
  const UnitDesc U = a.units[a.u0 + ul];
  const ReqDesc& R = a.reqs[U.req];
  const BlockDesc& B = a.blocks[U.block];
  const double bsig = B.sig, bisig = B.isig;
  long long cA, cB;
  unit_cols(a, R, B, cA, cB);
  const int R0 = (int)max(B.r0, 1LL), R1 = (int)min(B.r1, (long long)N2);
  unsigned m0 = 0, m1 = 0;
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int k2 = fft_out_index<N2, E>(tt, s), kb = N2 - k2;
    m0 |= (unsigned)(k2 >= R0 && k2 < R1) << s;
    m1 |= (unsigned)(k2 >= 1 && kb >= R0 && kb < R1) << s;
    As[s * NTH + tid] = make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int j = 0; j < OVS; ++j) A2s[j * NTH + tid] = make_double2(0.0, 0.0);
  for (int j = tid; j < R1 - R0; j += NTH) wt[j] = a.Ld / (double)(R0 + j);
  // column state of pair 0: u = x omega^{-1/2}, iw = 1/omega
  double u[EH], iw[EH], us = 0.0, iws = 0.0;
  const long long nb = n1 + (long long)L1 * tt, nstep = (long long)L1 * T;
#pragma unroll
  for (int e = 0; e < EH; ++e) load_col(a, R, cA, cB, nb + nstep * e, u[e], iw[e]);
  if (tt == 0 && n1 == 0) load_col(a, R, cA, cB, nstep * EH, us, iws);
  const double2* tw = a.tw + (N2 - 2);
  double2* sm = sm2 + w * NP;
  const unsigned mo = m0 & m1;
  __syncthreads();                                          // wt
  for (int p = a.p1 - 1; p >= a.p0; --p) {
    double2 z[E];
    double2 extra;
    pair_inputs<EH>(p, u, iw, us, iws, bsig, z, extra);
    const double c0x = R.ac[2 * p], c0y = -R.bc[2 * p];
    const double c1x = R.ac[2 * p + 1] * bisig, c1y = -R.bc[2 * p + 1] * bisig;
    block_fft<N2, E, 1, true, true>(z, sm, tt, tw, extra);
#pragma unroll
    for (int s = 0; s < E; ++s) {
      const bool t0 = (m0 >> s) & 1u, t1 = (m1 >> s) & 1u;
      const int k2 = fft_out_index<N2, E>(tt, s), kb = N2 - k2;
      if (t0 || t1) {
        const double wk = wt[(t0 ? k2 : kb) - R0];
        const double gx = fma(t0 ? wk : -wk, c1y, c0x);
        const double gy = fma(-wk, c1x, t0 ? c0y : -c0y);
        const double w2 = wk * wk;
        double2 t = As[s * NTH + tid];
        t.x = fma(t.x, w2, fma(gx, z[s].x, -gy * z[s].y));
        t.y = fma(t.y, w2, fma(gx, z[s].y, gy * z[s].x));
        As[s * NTH + tid] = t;
      }
      if (OVS > 0 && t0 && t1) {
        const int j = __popc(mo & ((1u << s) - 1u));
        if (j < OVS) {
          const double wk = wt[kb - R0];
          const double gx = fma(-wk, c1y, c0x), gy = fma(-wk, c1x, -c0y), w2 = wk * wk;
          double2 t = A2s[j * NTH + tid];
          t.x = fma(t.x, w2, fma(gx, z[s].x, -gy * z[s].y));
          t.y = fma(t.y, w2, fma(gx, z[s].y, gy * z[s].x));
          A2s[j * NTH + tid] = t;
        }
      }
    }
  }
  const long long qm = (1LL << a.logQ) - 1;
  double2* P0 = a.G + ((long long)(2 * ul) * a.rs) * L1 + n1;
  double2* P1 = a.G + ((long long)(2 * ul + 1) * a.rs) * L1 + n1;
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const bool t0 = (m0 >> s) & 1u, t1 = (m1 >> s) & 1u;
    const int k2 = fft_out_index<N2, E>(tt, s), kb = N2 - k2;
    if (t0) P0[(long long)(k2 - R0) * L1] = cmul(As[s * NTH + tid], qtw(a, (n1 * k2) & qm));
    if (t1) {
      double2 b = As[s * NTH + tid];
      if (t0) {
        const int j = __popc(mo & ((1u << s) - 1u));
        b = (OVS > 0 && j < OVS) ? A2s[(OVS > 0 ? j : 0) * NTH + tid] : make_double2(0.0, 0.0);
      }
      P1[(long long)(kb - R0) * L1] = cmul(b, qtw(a, (n1 * (long long)(k2 - N2)) & qm));
    }
  }
}

// U_k = sum_n1 P[A][row][n1] + conj(sum_n1 P[B][row][n1]), the row scale
// (1/2) post_k (L/k)^{1/2 + 2 p0} and the gamma rotation; one CTA per
// (row, unit), n1 summed by strided threads and a fixed-order tree.
__global__ void __launch_bounds__(128)
far_rowsum_fin_kernel(FarArgs a) {
  const int ul = blockIdx.y;
  const UnitDesc U = a.units[a.u0 + ul];
  const ReqDesc& R = a.reqs[U.req];
  const BlockDesc& B = a.blocks[U.block];
  const double bsig = B.sig, bisig = B.isig;
  const int R0 = (int)max(B.r0, 1LL), R1 = (int)min(B.r1, (long long)a.L2);
  const int k = R0 + (int)blockIdx.x;
  if (k >= R1) return;
  const int L1 = a.L1, tid = threadIdx.x;
  const double2* P0 = a.G + ((long long)(2 * ul) * a.rs + blockIdx.x) * L1;
  const double2* P1 = a.G + ((long long)(2 * ul + 1) * a.rs + blockIdx.x) * L1;
  double2 s0 = make_double2(0.0, 0.0), s1 = make_double2(0.0, 0.0);
#pragma unroll 4
  for (int n1 = tid; n1 < L1; n1 += 128) {
    s0 = cadd(s0, P0[n1]);
    s1 = cadd(s1, P1[n1]);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    s0.x += __shfl_xor_sync(0xffffffffu, s0.x, off);
    s0.y += __shfl_xor_sync(0xffffffffu, s0.y, off);
    s1.x += __shfl_xor_sync(0xffffffffu, s1.x, off);
    s1.y += __shfl_xor_sync(0xffffffffu, s1.y, off);
  }
  __shared__ double2 red[4][2];
  if ((tid & 31) == 0) {
    red[tid >> 5][0] = s0;
    red[tid >> 5][1] = s1;
  }
  __syncthreads();
  if (tid) return;
  s0 = cadd(cadd(red[0][0], red[1][0]), cadd(red[2][0], red[3][0]));
  s1 = cadd(cadd(red[0][1], red[1][1]), cadd(red[2][1], red[3][1]));
  const double ux = s0.x + s1.x, uy = s0.y - s1.y;
  const double ir = a.Ld / (double)k;
  double post = 1.0;
  if (R.pr) post = ipow_f((double)k / a.Ld, R.pr);
  if (R.post_e && R.pe) post *= ipow_f(R.post_e[k - 1], R.pe);
  double r0 = 0.5 * post * sqrt(ir);
  for (int p = 0; p < a.p0; ++p) r0 = (r0 * ir) * ir;           // (L/k)^{2 p0}
  double v = ux * r0;
  if (a.cs_tab) {
    const double2 th = __ldg(a.cs_tab + (k - 1));
    v = v * th.x + (uy * r0) * th.y;
  }
  a.part[(long long)ul * a.part_stride + (k - 1)] = v;
}

template <int N2, int W, int MINB, int E = 16>
static cudaError_t rowsum_t(const FarArgs& a, int n_units, cudaStream_t st) {
  constexpr int T = N2 / E, NTH = W * T;
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  const int smem = W * (N2 + PAD) * 16 + E * NTH * (8 + 8 + 16);   // FFT buffers + L/k tables + second accumulators
  auto k = far_rowsum_kernel<N2, W, MINB, E>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  if (a.L1 % W) return cudaErrorInvalidValue;
  note_launch(), k<<<dim3(a.L1 / W, n_units), NTH, smem, st>>>(a);
  return cudaGetLastError();
}

template <int N2, int W, int MINB, int OVS>
static cudaError_t rowsum2_t(const FarArgs& a, int n_units, cudaStream_t st) {
  constexpr int T = N2 / 16, NTH = W * T;
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  // FFT buffers + accumulators (+ second slots) + L/k table of the block rows
  const int smem = W * (N2 + PAD) * 16 + (16 + OVS) * NTH * 16 + ((a.rs + 1) & ~1) * 8;
  auto k = far_rowsum2_kernel<N2, W, MINB, OVS>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  if (a.L1 % W) return cudaErrorInvalidValue;
  note_launch(), k<<<dim3(a.L1 / W, n_units), NTH, smem, st>>>(a);
  return cudaGetLastError();
}

template <int OVS>
static cudaError_t rowsum2_d(const FarArgs& a, int logN2, int n_units, cudaStream_t st) {
  switch (logN2) {
    case 7: return rowsum2_t<128, 16, 3, OVS>(a, n_units, st);
    case 8: return rowsum2_t<256, 8, 3, OVS>(a, n_units, st);
    case 9: return rowsum2_t<512, 4, 3, OVS>(a, n_units, st);
    case 10: return rowsum2_t<1024, 2, 3, OVS>(a, n_units, st);
    case 11: return rowsum2_t<2048, 1, 3, OVS>(a, n_units, st);
  }
  return cudaErrorInvalidValue;
}

// Fused narrow-row units: column FFTs of 2^logN2 points, folded rows to P (a.G).
// form 0: accumulators in registers, any overlap of the two row types (1 or 2
// CTAs per SM); 1 / 2: high-occupancy form without / with two overlap slots.
cudaError_t launch_far_rowsum(const FarArgs& a, int logN2, int form, int n_units, cudaStream_t st) {
  if (form == 1) return rowsum2_d<0>(a, logN2, n_units, st);
  if (form == 2) return rowsum2_d<2>(a, logN2, n_units, st);
  switch (logN2) {
    case 7: return rowsum_t<128, 16, 2>(a, n_units, st);
    case 8: return rowsum_t<256, 8, 2>(a, n_units, st);
    case 9: return rowsum_t<512, 4, 2>(a, n_units, st);
    case 10: return rowsum_t<1024, 2, 2>(a, n_units, st);
    case 11:
      // as at 4096 points: 8 points per thread (256 threads, 2 CTAs = 16 warps per SM, no
      // spills) instead of 16 (128 threads at 255 registers, 8 warps)
      if (g_far_variant & 0x20000) return rowsum_t<2048, 1, 2>(a, n_units, st);
      return rowsum_t<2048, 1, 2, 8>(a, n_units, st);
    case 12:
      // 8 points per thread: 512 threads (16 warps) on the one CTA an SM holds,
      // one more shared-memory exchange (variant bit 17 selects 16 points, 8 warps)
      if (g_far_variant & 0x20000) return rowsum_t<4096, 1, 1>(a, n_units, st);
      return rowsum_t<4096, 1, 1, 8>(a, n_units, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_far_rowsum_fin(const FarArgs& a, int n_units, cudaStream_t st) {
  note_launch(), far_rowsum_fin_kernel<<<dim3(a.rs, n_units), 128, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace fhtb
