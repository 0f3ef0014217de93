// fhtb_far.cu -- far field of the Schlomilch application, direct mode.
//
// Reference behaviour (schlomilch.py:301-329, :470-502): for each block and
// each term i < 2M, u_i = col_w[i] * c on the block columns, C u_i (DCT-I,
// N+1) and S u_i (DST-I, N-1) via rfft embeddings (trig.py:59-77), then
// out[rows] += sum_i A_i * C u_i + B_i * S u_i.
//
// B200 formulation.  C u + i S u = sum_n u_n e^{+i pi k n / L}, i.e. a
// length-2L DFT of the zero-padded column vector.  Terms 2p and 2p+1 are
// real, so they share ONE complex FFT z = u_{2p} + i u_{2p+1}; the two
// spectra are separated in the epilogue from Z[k] and conj Z[2L-k].
// The column weights omega_n^{-i-1/2} (and the Fourier-Bessel / DHT
// pre-multipliers) are generated in registers while loading c (no 2M x N
// materialisation, cf. schlomilch.py:251-257), and the row weights
// (L/k)^{i+1/2}, the gamma-shift diagonals cos/sin(theta_k + (2o+1)pi/4)
// (Remark 1), the order combination (schlomilch.py:280-299) and the
// post-multipliers r^u / e^u (fourier_bessel.py:240-242, dht.py:167-174) are
// applied in the epilogue of the last FFT pass, which reduces all 2M terms
// of a (request, block) unit in registers and writes one partial row.
//
//   one-pass  (2L <= 8192): one CTA per unit, whole FFT in shared memory.
//   two-pass  (2L  > 8192): Q = 2L = L1*L2 four-step.
//      pass 1: per column n1, L2-point FFT over n2 (n = n1 + L1 n2), twiddle
//              e^{2 pi i n1 k2 / Q}, store G[unit][p][k2][n1].
//      pass 2: per (column pair {k2, L2-k2}, unit), L1-point FFTs over n1,
//              the fused DCT/DST separation and the row epilogue.
//   reduce:  F[vec][j] += sum of the unit partials of that vector, in unit
//            order (deterministic).
#include <cuda.h>
#include <algorithm>
#include <cstring>

#include "fhtb_core.cuh"
#include "fhtb_launch.h"
#include "fhtb_far.cuh"

namespace fhtb {

// ------------------------------------------------------------------ pass 1
// TMA: the twiddled outputs of the CTA's W columns are staged in shared
// memory as rows [k2][w] (reusing the FFT buffer) and written to G by 2D
// tensor stores (boxes of 2W doubles x BR rows), so the strided W*16-byte row
// segments do not go through the LSU path one warp instruction at a time.
// QT: four-step twiddles staged in shared memory (else computed per use,
// for the large columns whose table would not fit beside the FFT buffer).
template <int N2, int E, int W, int MINB, bool TMA, bool QT = true>
__global__ void __launch_bounds__(W * (N2 / E), MINB)
far_pass1_kernel(FarArgs a, const __grid_constant__ CUtensorMap gmap) {
  constexpr int T = N2 / E;
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  constexpr int NP = N2 + PAD;
  constexpr int BR = N2 < 256 ? N2 : 256;           // tensor-store box rows
  extern __shared__ __align__(128) double2 sm2[];
  const int tid = threadIdx.x, w = tid % W, tt = tid / W;
  const int L1 = a.L1;
  const long long n1 = a.xn1 + (long long)blockIdx.x * W + w;
  const int ul = blockIdx.y;
  const UnitDesc U = a.units[a.u0 + ul];
  const ReqDesc& R = a.reqs[U.req];
  const BlockDesc& B = a.blocks[U.block];
  const double bsig = B.sig, bisig = B.isig;
  long long cA, cB;
  unit_cols(a, R, B, cA, cB);
  // n = n1 + L1 n2 <= L  <=>  n2 < L2/2, or n2 = L2/2 with n1 = 0 (n = L):
  // the upper half of every thread's slots is zero (2L = L1 L2), except one
  // element carried separately.
  constexpr int EH = E / 2;
  double v[EH], iw[EH], vs = 0.0, iws = 0.0;
#pragma unroll
  for (int e = 0; e < EH; ++e) load_col(a, R, cA, cB, n1 + (long long)L1 * (tt + T * e), v[e], iw[e]);
  if (tt == 0 && n1 == 0) load_col(a, R, cA, cB, (long long)L1 * (T * EH), vs, iws);
  double2* sm = sm2 + w * NP;
  const double2* tw = a.tw + (N2 - 2);
  // four-step twiddles e^{2 pi i n1 k2/Q} of this thread's outputs are the
  // same for every pair: build them once into shared memory (thread-private
  // slots, no synchronisation needed)
  // slot-major so that a warp's accesses are unit stride (conflict free)
  double2* qt = sm2 + W * NP + tid;
  constexpr int NTH = W * T;
#pragma unroll
  for (int s = 0; s < E; ++s)
    if (QT) qt[s * NTH] = qtw(a, n1 * fft_out_index<N2, E>(tt, s));
  for (int p = 0; p < a.p0; ++p) {          // advance to the shard's first pair
#pragma unroll
    for (int e = 0; e < EH; ++e) v[e] = (v[e] * iw[e]) * iw[e];
    vs = (vs * iws) * iws;
  }
  for (int p = a.p0; p < a.p1; ++p) {
    double2 z[E];
#pragma unroll
    for (int e = 0; e < EH; ++e) {
      const double im = v[e] * iw[e];
      z[e] = make_double2(v[e], im * bsig);
      v[e] = im * iw[e];
      z[e + EH] = make_double2(0.0, 0.0);
    }
    const double ims = vs * iws;
    const double2 extra = make_double2(vs, ims * bsig);
    vs = ims * iws;
    if (TMA) {
      // the previous pair's tensor store may still read the staging area:
      // waited for after the register-only first radix pass (SYNC0)
      block_fft<N2, E, 1, true, true>(z, sm, tt, tw, extra);
    } else {
      __syncthreads();
      block_fft<N2, E, 1, true>(z, sm, tt, tw, extra);
    }
    if (TMA) {
      __syncthreads();
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int k2 = fft_out_index<N2, E>(tt, s);
        sm2[k2 * W + w] = cmul(z[s], QT ? qt[s * NTH] : qtw(a, n1 * k2));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        const int row0 = (ul * a.M + p) * a.L2;
        const int c0 = 2 * (int)(blockIdx.x * W);
#pragma unroll
        for (int r = 0; r < N2; r += BR) {
          const unsigned sa = (unsigned)__cvta_generic_to_shared(sm2 + r * W);
          asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];"
                       :: "l"(&gmap), "r"(sa), "r"(c0), "r"(row0 + r) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else if (a.xw) {
      // exchange mode: row k2 goes to its owner's chunk, at the owner's row j
      const long long nl = n1 - a.xn1;
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int k2 = fft_out_index<N2, E>(tt, s);
        const int2 oj = __ldg(a.xrow + k2);
        a.G[oj.x * a.xchunk + (((long long)(ul * a.M + p) * a.xrows + oj.y) << a.xlog) + nl] =
            cmul(z[s], QT ? qt[s * NTH] : qtw(a, n1 * k2));
      }
    } else {
      double2* G = a.G + ((long long)(ul * a.M + p) * N2) * L1;
#pragma unroll
      for (int s = 0; s < E; ++s) {
        const int k2 = fft_out_index<N2, E>(tt, s);
        G[(long long)k2 * L1 + n1] = cmul(z[s], QT ? qt[s * NTH] : qtw(a, n1 * k2));
      }
    }
  }
  if (TMA && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// Pass 1, one CTA per (column group, unit, pair p): no per-element state is
// carried across pairs, so registers hold only the FFT data.  The column
// weights come from the grid tables W0[n-1] = omega_n^{-1/2}, IW[n-1] =
// 1/omega_n (L2 resident) and omega_n^{-2p} = IW^{2p} by binary powering.
template <int N2, int E, int W, int MINB>
__global__ void __launch_bounds__(W * (N2 / E), MINB)
far_pass1p_kernel(FarArgs a) {
  constexpr int T = N2 / E;
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  constexpr int NP = N2 + PAD;
  extern __shared__ double2 sm2[];
  const int tid = threadIdx.x, w = tid % W, tt = tid / W;
  const int L1 = a.L1;
  const long long n1 = (long long)blockIdx.x * W + w;
  const int ul = blockIdx.y / a.M, p = blockIdx.y % a.M;
  if (p < a.p0 || p >= a.p1) return;
  const UnitDesc U = a.units[a.u0 + ul];
  const ReqDesc& R = a.reqs[U.req];
  const BlockDesc& B = a.blocks[U.block];
  const double bsig = B.sig, bisig = B.isig;
  long long cA, cB;
  unit_cols(a, R, B, cA, cB);
  double2 z[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const long long n = n1 + (long long)L1 * (tt + T * e);
    z[e] = make_double2(0.0, 0.0);
    if (n >= cA && n < cB) {
      double x = a.C[(long long)R.vec * a.ldc + (n - 1)];
      if (R.preA) x *= ipow_f(R.preA[n - 1], R.pa);
      if (R.preB) x *= ipow_f(R.preB[n - 1], R.pb);
      const double iw = __ldg(a.iw_tab + (n - 1));
      double v = x * __ldg(a.w0_tab + (n - 1));
      // v *= iw^(2p), binary powering
      double b2 = iw * iw;
      for (int q = p; q; q >>= 1) {
        if (q & 1) v *= b2;
        b2 *= b2;
      }
      z[e] = make_double2(v, (v * iw) * bsig);
    }
  }
  double2* sm = sm2 + w * NP;
  block_fft<N2, E, 1>(z, sm, tt, a.tw + (N2 - 2));
  double2* G = a.G + ((long long)(ul * a.M + p) * N2) * L1;
#pragma unroll
  for (int s = 0; s < E; ++s) {
    const int k2 = fft_out_index<N2, E>(tt, s);
    G[(long long)k2 * L1 + n1] = cmul(z[s], qtw(a, n1 * k2));
  }
}

// mbarrier / bulk-copy helpers (column tables of the narrow-column blocks)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// global -> shared bulk copy of `bytes` (multiple of 16, both 16-byte aligned), completion on `bar`
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// --------------------------------------------- pass 2 / one-pass epilogue
//
// MODE 0: two-pass, columns read from G.
// MODE 1: one-pass (L2 == 1, N1 == 2L): one column generated from c.
// MODE 2: block whose columns all lie below L1 (narrow-column side block):
//         pass 1 degenerates to G[n1][k2] = u[n1] e^{2 pi i n1 k2/Q}, so the
//         columns are formed here from the per-unit table u (colgen_prep)
//         and no intermediate exists.
//
// Epilogue algebra.  Term i of row k adds r_i (a_i Y.x + b_i Y.y) to the
// cosine part and r_i (as_i Y.x + bs_i Y.y) to the sine part of the gamma
// rotation, with as_i = -b_i, bs_i = a_i (pack_requests).  Both are one
// complex sum U = sum_i r_i (a_i - i b_i) Y_i: cosine part Re U, sine part
// Im U.  With r_{2p} = r_0 (L/k)^{2p}, r_{2p+1} = r_{2p} L/k, U is folded by
// Horner's rule over the pairs from the last one down (MODE 0 / 2; MODE 1
// generates its columns by a forward recurrence and keeps r explicitly);
// r_0 and the MODE-2 column-shift phase phi_k are applied once at the end.
// MODE 3: MODE 0 in exchange mode (distributed four-step): column pairs from
//         a.xc0, rows assembled from the received chunks of all ranks.
// step-table twiddles for narrow-column blocks: always at E = 16; at E = 8
// only in the high-occupancy shapes (MINB >= 5), which need the registers
#define TQS_ON(MODE, E, MINB) ((MODE) == 2 && ((E) >= 16 || (MINB) >= 5))
#define TQS_SMEM(MODE, E) ((MODE) == 2 && (E) >= 16)
#define IRS_K(E, MODE) false
// narrow-column blocks: the Horner accumulators live in thread-private shared-memory
// slots (read-modify-write once per pair and row) instead of NQ complex registers;
// at the register caps of these shapes (128 at 2048 points, 96 at 512) ncu counted
// as many local (spill) loads and stores as global loads (variant bit 18 turns it off)
// (template parameter ACS of the kernel)
// UBLT: template parameter (library option far_bulk_tables); measured on cfg2: far field
// 63.95 -> 64.85 ms with the bulk-copied tables (the table hits in L1 either way; the
// copy adds a shared-memory read per point to kernels bound by that pipe), so off
#define UBL_ON(MODE, E, MINB, N1, ACS, UBLT) ((UBLT) && (ACS) && (MODE) == 2 && TQS_ON(MODE, E, MINB) && (N1) <= 1024)
// HP (half pairing): every thread finishes the rows of its OWN lower-half FFT outputs
// (k1 < N1/2, i.e. k = k2 + L2 k1 < L) straight from its registers; only the upper-half
// outputs go through shared memory, once, as the partners conj Z[2L-k] = conj Z_b[N1-1-k1] of
// the other column's rows: 8 + 8 bytes of shared-memory traffic per point for the
// Z[k] / Z[2L-k] pairing instead of 16 + 16.  The CTA of column 0 (its own partner, plus row
// L) keeps the general form: HP kernels cover the column pairs k2a >= 1.
template <int N1, int E, int MODE, int MINB, bool ACS = false, bool UBLT = false, bool HP = false>
__global__ void __launch_bounds__((MODE == 1 ? 1 : 2) * (N1 / E), MINB)
far_pass2_kernel(FarArgs a) {
  constexpr bool ONEPASS = (MODE == 1);
  constexpr bool HOR = (MODE != 1);
  constexpr bool XCH = (MODE == 3);
  constexpr int T = N1 / E;
  constexpr int NCOL = ONEPASS ? 1 : 2;
  constexpr int NT = NCOL * T;
  constexpr int NQ = E / 2 > 0 ? E / 2 : 1;     // output slots per thread
  constexpr int HALF = N1 / 2;
  constexpr int NP = N1 + 4;
  constexpr int LOGE = ilog2c(E);
  extern __shared__ double2 sm2[];
  const int tid = threadIdx.x, h = tid / T, tt = tid % T;
  const int L = (int)a.L;
  const int L2 = a.L2;
  const int k2a = (XCH ? a.xc0 + (int)blockIdx.x : (int)blockIdx.x) + (HP ? 1 : 0), k2b = (L2 - k2a) % L2;
  const bool selfp = (k2a == k2b);
  const int myk2 = h == 0 ? k2a : k2b;
  const int ul = blockIdx.y;
  const UnitDesc U = a.units[a.u0 + ul];
  const ReqDesc& R = a.reqs[U.req];
  const BlockDesc& B = a.blocks[U.block];
  const double bsig = B.sig, bisig = B.isig;
  const double2* tw = a.tw + (N1 - 2);
  const int xj = XCH ? __ldg(a.xrow + myk2).y : 0;
  // L2 = Q / N1 is a power of two: k / L2 as a shift (a runtime division
  // costs ~20 integer instructions per output and pair)
  const int lgL2 = a.logQ - ilog2c(N1);

  // E <= 8: the shared-memory offsets of Z[k] and Z[2L-k] are kept per slot
  // (registers allow it); E = 16 recomputes them per pair
  constexpr bool PRE = (E <= 8 && N1 >= 1024) && !HP;
  constexpr int RLH = FftShape<N1, E>::RL / 2 > 0 ? FftShape<N1, E>::RL / 2 : 1;   // HP: lower-half slots per radix group
  int kq[IRS_K(E, MODE) ? 1 : NQ], oz[PRE ? NQ : 1], op[PRE ? NQ : 1];
  // IRS (E = 16, Horner modes): the row factors L/k live in shared memory
  // ([q][tid] after the FFT buffers) instead of NQ registers, which the
  // 16-point state cannot spare without spilling
  constexpr bool IRS = false;   // (measured: 18.05 -> 18.30 ms at 2048 points; with the accumulators in shared memory 64.5 -> 66.6 ms far field, so off)
  double* irs = reinterpret_cast<double*>(sm2 + NCOL * NP + (TQS_ON(MODE, E, MINB) ? NCOL * E : 0));
  int* kqs = reinterpret_cast<int*>(irs + (IRS ? NQ * NT : 0));      // IRS: row indices too
  double ir[IRS ? 1 : NQ], rp[HOR ? 1 : NQ];
  constexpr bool ACSC = ACS, acs = ACS;
  // UBL: the column table u_p of a narrow-column unit (N1 complex per pair, read by
  // both columns of every CTA) arrives by bulk copy into a two-slot shared-memory
  // buffer, pair p+1 while pair p is transformed (mbarrier per slot), instead of
  // LDG.128 through L1 by both halves of the CTA
  constexpr bool UBL = UBL_ON(MODE, E, MINB, N1, ACS, UBLT);
  double2* accs = reinterpret_cast<double2*>(kqs + (IRS ? NQ * NT : 0)) + tid;   // [q * NT]
  double2 acc[ACS ? 1 : NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int o = tid + NT * q;
    const int hh = o / HALF, qq = o % HALF;
    int k = 0;
    if (HP) {
      // row of this thread's q-th lower-half output slot
      const int s = (q / RLH) * (2 * RLH) + (q % RLH);
      if (!(selfp && h == 1)) {
        k = myk2 + L2 * fft_out_index<N1, E>(tt, s);
        if (k < 1 || k > L || k < B.r0 || k >= B.r1) k = 0;
      }
    } else if (hh < NCOL && !(selfp && hh == 1)) {
      const int k2 = hh == 0 ? k2a : k2b;
      const int k1 = (k2 == 0) ? qq + 1 : qq;
      k = k2 + L2 * k1;
      if (k < 1 || k > L || k < B.r0 || k >= B.r1) k = 0;
    }
    if (IRS) kqs[q * NT + tid] = k;
    else kq[IRS ? 0 : q] = k;
    if (ACS) accs[q * NT] = make_double2(0.0, 0.0);
    else acc[ACS ? 0 : q] = make_double2(0.0, 0.0);
    const double irq = k ? a.Ld / (double)k : 0.0;
    if (IRS) irs[q * NT + tid] = irq;
    else ir[IRS ? 0 : q] = irq;
    if (PRE) {
      const int kp = 2 * L - k;
      oz[PRE ? q : 0] = k ? (((k & (L2 - 1)) == k2a) ? 0 : NP) + swz<LOGE>(k >> lgL2) : 0;
      op[PRE ? q : 0] = k ? (((kp & (L2 - 1)) == k2a) ? 0 : NP) + swz<LOGE>(kp >> lgL2) : 0;
    }
    if (!HOR) {
      double post = 1.0;
      if (k && R.pr) post = ipow_f((double)k / a.Ld, R.pr);
      if (k && R.post_e && R.pe) post *= ipow_f(R.post_e[k - 1], R.pe);
      rp[HOR ? 0 : q] = k ? 0.5 * post * sqrt(irq) : 0.0;
    }
  }
  // column sources
  //   MODE 1: v = x omega^{-1/2}, iw = 1/omega kept per element (z = v (1, iw),
  //           v *= iw^2 per pair)
  //   MODE 2: tq = e^{2 pi i m k2/Q} per element; z = u_p[m] tq
  //   MODE 2, E >= 16 (TQS): tq = tb * st[e], tb = e^{2 pi i tt k2/Q} per
  //           thread and st[e] = e^{2 pi i T e k2/Q} per column in shared
  //           memory (broadcast reads): E complex registers fewer, which
  //           lets the column FFT run with E = 16 (one radix pass fewer)
  constexpr bool TQS = TQS_ON(MODE, E, MINB);
  double v[ONEPASS ? E : 1], iw[ONEPASS ? E : 1];
  double2 tq[(MODE == 2 && !TQS) ? E : 1];
  double2 tb = make_double2(1.0, 0.0);
  if (ONEPASS) {
    long long cA, cB;
    unit_cols(a, R, B, cA, cB);
#pragma unroll
    for (int e = 0; e < E; ++e) load_col(a, R, cA, cB, tt + T * e, v[ONEPASS ? e : 0], iw[ONEPASS ? e : 0]);
  }
  double2* ub = reinterpret_cast<double2*>(accs - tid + (ACS ? NQ * NT : 0));        // [2][N1]
  unsigned long long* ubar = reinterpret_cast<unsigned long long*>(ub + 2 * N1);   // [2]
  if (MODE == 2 && TQS) {
    double2* st = sm2 + NCOL * NP + h * E;
    if (tt < E) st[tt] = myk2 ? qtw(a, (long long)T * tt * myk2) : make_double2(1.0, 0.0);
    tb = myk2 ? qtw(a, (long long)tt * myk2) : make_double2(1.0, 0.0);
    if (UBL && tid == 0) {
      mbar_init(ubar, 1);
      mbar_init(ubar + 1, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (UBL && tid == 0 && a.p1 > a.p0)
      bulk_load(ub, a.G + (long long)(ul * a.M + (a.p1 - 1)) * N1, N1 * 16, ubar);
  } else if (MODE == 2) {
#pragma unroll
    for (int e = 0; e < E; ++e)
      tq[(MODE == 2 && !TQS) ? e : 0] = myk2 ? qtw(a, (long long)(tt + T * e) * myk2) : make_double2(1.0, 0.0);
  }
  if (!HOR) {
    for (int p = 0; p < a.p0; ++p) {        // advance to the shard's first pair
#pragma unroll
      for (int e = 0; e < E; ++e) v[ONEPASS ? e : 0] = (v[ONEPASS ? e : 0] * iw[ONEPASS ? e : 0]) * iw[ONEPASS ? e : 0];
#pragma unroll
      for (int q = 0; q < NQ; ++q) rp[HOR ? 0 : q] = (rp[HOR ? 0 : q] * ir[IRS ? 0 : q]) * ir[IRS ? 0 : q];
    }
  }
  for (int pi = 0; pi < a.p1 - a.p0; ++pi) {
    const int p = HOR ? a.p1 - 1 - pi : a.p0 + pi;
    double2 z[E];
    if (ONEPASS) {
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const double im = v[ONEPASS ? e : 0] * iw[ONEPASS ? e : 0];
        z[e] = make_double2(v[ONEPASS ? e : 0], im * bsig);
        v[ONEPASS ? e : 0] = im * iw[ONEPASS ? e : 0];
      }
    } else if (MODE == 2) {
      const double2* u = a.G + (long long)(ul * a.M + p) * N1;
      if (UBL) {
        while (!mbar_try_wait(ubar + (pi & 1), (pi >> 1) & 1)) {}
        u = ub + (pi & 1) * N1;
      }
      if (TQS) {
        const double2* st = sm2 + NCOL * NP + h * E;
#pragma unroll
        for (int e = 0; e < E; ++e) z[e] = cmul(cmul(u[tt + T * e], tb), st[e]);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) z[e] = cmul(u[tt + T * e], tq[(MODE == 2 && !TQS) ? e : 0]);
      }
    } else if (XCH) {
      // row myk2 assembled from the chunks of all source ranks
      const long long row = ((long long)(ul * a.M + p) * a.xrows + xj) << a.xlog;
      const int msk = (1 << a.xlog) - 1;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int n1 = tt + T * e;
        z[e] = a.xin[(n1 >> a.xlog) * a.xchunk + row + (n1 & msk)];
      }
    } else {
      const double2* G = a.G + ((long long)(ul * a.M + p) * L2 + myk2) * N1;
#pragma unroll
      for (int e = 0; e < E; ++e) z[e] = G[tt + T * e];
    }
    // E <= 8: the pair's row coefficients are loaded before the transform
    // (their latency hides behind it); E = 16 has no registers to spare
    // (measured: pass 2 at 2048 points 16.9 -> 18.3 ms with the early loads)
    const int i0 = 2 * p, i1 = 2 * p + 1;
    double ac0, bc0, ac1, bc1;
    if (E <= 8) {
      ac0 = R.ac[i0], bc0 = R.bc[i0];
      ac1 = R.ac[i1] * bisig, bc1 = R.bc[i1] * bisig;
    }
    __syncthreads();
    if (UBL && tid == 0 && pi + 1 < a.p1 - a.p0) {
      // every thread has read slot (pi+1)&1 (pair pi-1) before the barrier above
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bulk_load(ub + ((pi + 1) & 1) * N1, a.G + (long long)(ul * a.M + (p - 1)) * N1, N1 * 16, ubar + ((pi + 1) & 1));
    }
    block_fft<N1, E, 1>(z, sm2 + h * NP, tt, tw);
    __syncthreads();
    if (HP) {
      // upper-half outputs Z[k1 >= N1/2] of this column at index k1 - N1/2
#pragma unroll
      for (int s = 0; s < E; ++s)
        if ((s % (2 * RLH)) >= RLH) sm2[h * NP + fft_out_index<N1, E>(tt, s) - HALF] = z[s];
    } else {
#pragma unroll
      for (int s = 0; s < E; ++s) sm2[h * NP + swz<LOGE>(fft_out_index<N1, E>(tt, s))] = z[s];
    }
    __syncthreads();
    if (E > 8) {
      ac0 = R.ac[i0], bc0 = R.bc[i0];
      ac1 = R.ac[i1] * bisig, bc1 = R.bc[i1] * bisig;
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int k = IRS ? kqs[q * NT + tid] : kq[IRS ? 0 : q];
      if (!k) continue;
      const int kp = 2 * L - k;
      double2 Zk, Zp;
      if (HP) {
        // own register; partner Z_b[N1 - 1 - k1] from the other column (this one if self-paired)
        const int s = (q / RLH) * (2 * RLH) + (q % RLH);
        Zk = z[s];
        Zp = cconj(sm2[(selfp ? h : 1 - h) * NP + (HALF - 1 - fft_out_index<N1, E>(tt, s))]);
      } else {
        Zk = sm2[PRE ? oz[PRE ? q : 0] : (((k & (L2 - 1)) == k2a) ? 0 : NP) + swz<LOGE>(k >> lgL2)];
        Zp = cconj(sm2[PRE ? op[PRE ? q : 0] : (((kp & (L2 - 1)) == k2a) ? 0 : NP) + swz<LOGE>(kp >> lgL2)]);
      }
      // 2 Ya, 2 Yb (the factor 1/2 is folded into r_0)
      double2 Ya = make_double2(Zk.x + Zp.x, Zk.y + Zp.y);
      double2 Yb = make_double2(Zk.y - Zp.y, Zp.x - Zk.x);
      if (k == L) { Ya.y = 0.0; Yb.y = 0.0; }      // S u has no row N (schlomilch.py:314-316)
      // t0 = (a0 - i b0) Ya, t1 = (a1 - i b1) Yb
      const double t0x = fma(ac0, Ya.x, bc0 * Ya.y), t0y = fma(ac0, Ya.y, -bc0 * Ya.x);
      const double t1x = fma(ac1, Yb.x, bc1 * Yb.y), t1y = fma(ac1, Yb.y, -bc1 * Yb.x);
      const double w = IRS ? irs[q * NT + tid] : ir[IRS ? 0 : q];
      if (HOR) {
        const double w2 = w * w;
        if (ACSC && acs) {
          double2 t = accs[q * NT];
          t.x = fma(t.x, w2, fma(w, t1x, t0x));
          t.y = fma(t.y, w2, fma(w, t1y, t0y));
          accs[q * NT] = t;
        } else {
          acc[ACS ? 0 : q].x = fma(acc[ACS ? 0 : q].x, w2, fma(w, t1x, t0x));
          acc[ACS ? 0 : q].y = fma(acc[ACS ? 0 : q].y, w2, fma(w, t1y, t0y));
        }
      } else {
        const double r0 = rp[HOR ? 0 : q], r1 = r0 * w;
        acc[ACS ? 0 : q].x = fma(r0, t0x, fma(r1, t1x, acc[ACS ? 0 : q].x));
        acc[ACS ? 0 : q].y = fma(r0, t0y, fma(r1, t1y, acc[ACS ? 0 : q].y));
        rp[HOR ? 0 : q] = r1 * w;
      }
    }
  }
  long long sh = 0;
  if (MODE == 2) {
    long long cA, cB;
    unit_cols(a, R, B, cA, cB);
    sh = cA;
  }
  double* part = a.part + (long long)ul * a.part_stride;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int k = IRS ? kqs[q * NT + tid] : kq[IRS ? 0 : q];
    if (!k) continue;
    double2 u = ACS ? accs[q * NT] : acc[ACS ? 0 : q];
    if (HOR) {
      double post = 1.0;
      if (R.pr) post = ipow_f((double)k / a.Ld, R.pr);
      if (R.post_e && R.pe) post *= ipow_f(R.post_e[k - 1], R.pe);
      const double irq = IRS ? irs[q * NT + tid] : ir[IRS ? 0 : q];
      double r0 = 0.5 * post * sqrt(irq);
      for (int p = 0; p < a.p0; ++p) r0 = (r0 * irq) * irq;    // (L/k)^{2 p0}
      u = make_double2(u.x * r0, u.y * r0);
    }
    if (MODE == 2 && sh) {
      // phi_k = e^{i pi k sh / L}; exactly (-1)^sh at k = L
      const double2 phi = (k == L) ? make_double2((sh & 1) ? -1.0 : 1.0, 0.0)
                                   : qtw(a, ((long long)k * sh) & (2 * a.L - 1));   // 2L = Q, a power of two
      u = cmul(u, phi);
    }
    double val = u.x;
    if (a.cs_tab) {
      const double2 th = __ldg(a.cs_tab + (k - 1));
      val = u.x * th.x + u.y * th.y;
    }
    part[k - 1] = val;
  }
}

// Column table of a narrow-column (MODE 2) unit, shifted to its first column
// sh: u_p[m] = x_n omega_n^{-1/2} omega_n^{-2p} (1, 1/omega_n), n = m + sh,
// p < M, m < L1 (terms 2p and 2p+1 as the real and imaginary part).
__global__ void colgen_prep_kernel(FarArgs a) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int ul = blockIdx.y;
  if (m >= a.L1) return;
  const UnitDesc U = a.units[a.u0 + ul];
  const ReqDesc& R = a.reqs[U.req];
  const BlockDesc& B = a.blocks[U.block];
  const double bsig = B.sig, bisig = B.isig;
  long long cA, cB;
  unit_cols(a, R, B, cA, cB);
  const long long n = m + cA;
  double v, iw;
  load_col(a, R, cA, cB, n, v, iw);
  double2* u = a.G + (long long)(ul * a.M) * a.L1 + m;
  for (int p = 0; p < a.M; ++p) {
    const double im = v * iw;
    u[(long long)p * a.L1] = make_double2(v, im * bsig);
    v = im * iw;
  }
}

// Pass 2 of a block whose rows all lie below K*L2 (narrow-row side block):
// only the FFT bins k1 < K of each column (and their partners near L1) are
// needed, i.e. 2K weighted sums over n1 per column instead of an L1-point FFT:
//   Z[c + L2 j]       = sum_n1 G[c][n1] e^{+2 pi i n1 j / L1}        (j < K)
//   Z[2L - (c + L2 j)] = sum_n1 G[L2-c][n1] e^{-2 pi i n1 (j+1) / L1}  (c != 0)
//                      = sum_n1 G[0][n1] e^{-2 pi i n1 j / L1}       (c == 0)
// CTA = (column pair {c, L2-c}, unit); warps 0-3 sum column c, warps 4-7
// column L2-c, each over a quarter of n1, for all pairs first (loads of all
// pairs in flight together), then 2K threads combine the quarters in fixed
// order and run the epilogue (same algebra as far_pass2_kernel).
// KB: compile-time bound on the bins of the chunk's units (1, 2 or 4).
// Measured on cfg2: the 3-bin form of the block with rows [539, 2488)
// (15.4 ms per 64 vectors) loses to its full pass 2 (8.4 ms), so the
// default keeps one bin per column (far_rowdot_bins = 1).
constexpr int kMaxPairs = 16;
template <int KB>
__global__ void __launch_bounds__(256)
far_rowdot_kernel(FarArgs a, int c_lo) {
  constexpr int kMaxBins = KB;
  const int L = (int)a.L;
  const int L1 = a.L1, L2 = a.L2;
  const int c = c_lo + blockIdx.x;
  const int ul = blockIdx.y;
  const UnitDesc U = a.units[a.u0 + ul];
  const ReqDesc& R = a.reqs[U.req];
  const BlockDesc& B = a.blocks[U.block];
  const double bsig = B.sig, bisig = B.isig;
  // all KB bins are summed (compile-time trip counts keep the loads of the
  // unrolled n1 loop in flight together); bins past the block rows are not
  // written
  constexpr int K = KB;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int cb = (L2 - c) % L2;
  // outputs k = c + L2 j and k = cb + L2 j (cb != c), j < K, inside the block
  bool any = false;
  for (int j = 0; j < K; ++j) {
    const int kA = c + L2 * j, kB = cb + L2 * j;
    any |= kA >= 1 && kA <= L && kA >= B.r0 && kA < B.r1;
    any |= cb != c && kB >= 1 && kB <= L && kB >= B.r0 && kB < B.r1;
  }
  if (!any) return;
  __shared__ double2 part_s[8][kMaxPairs][2 * kMaxBins];
  const int side_w = wid >> 2, quarter = wid & 3;
  const int col = side_w == 0 ? c : cb;
  const double2* rot = a.tw + (L1 - 2);   // e^{+2 pi i m / L1}
  const int msk = L1 - 1;
  const int qlen = (L1 + 3) / 4;
  const int lo = quarter * qlen, hi = min(L1, lo + qlen);
  for (int p = a.p0; p < a.p1; ++p) {
    const double2* g = a.G + ((long long)(ul * a.M + p) * L2 + col) * L1;
    double2 sp[kMaxBins], sn[kMaxBins];
#pragma unroll
    for (int j = 0; j < kMaxBins; ++j) sp[j] = sn[j] = make_double2(0.0, 0.0);
#pragma unroll 4
    for (int n1 = lo + lane; n1 < hi; n1 += 32) {
      const double2 v = g[n1];
      sp[0] = cadd(sp[0], v);
#pragma unroll
      for (int j = 1; j <= kMaxBins; ++j) {
        const double2 t = __ldg(rot + ((n1 * j) & msk));
        if (j < K) sp[j] = cadd(sp[j], cmul(v, t));
        sn[j - 1] = cadd(sn[j - 1], cmul(v, cconj(t)));
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxBins; ++j) {
#pragma unroll
      for (int off = 16; off; off >>= 1) {
        sp[j].x += __shfl_xor_sync(0xffffffffu, sp[j].x, off);
        sp[j].y += __shfl_xor_sync(0xffffffffu, sp[j].y, off);
        sn[j].x += __shfl_xor_sync(0xffffffffu, sn[j].x, off);
        sn[j].y += __shfl_xor_sync(0xffffffffu, sn[j].y, off);
      }
      if (lane == 0) {
        part_s[wid][p][j] = sp[j];
        part_s[wid][p][kMaxBins + j] = sn[j];
      }
    }
  }
  __syncthreads();
  const int side = threadIdx.x / K, j = threadIdx.x % K;
  if (side >= 2) return;
  if (side == 1 && cb == c) return;
  const int kcol = side == 0 ? c : cb;
  const int k = kcol + L2 * j;
  if (!(k >= 1 && k <= L && k >= B.r0 && k < B.r1)) return;
  // Z[k] from this side's column; conj Z[2L-k] from the partner column
  // (itself when cb == c) at the minus sum j+1, or column 0's own minus sum j
  const int sk = side, spn = side ^ (cb != c ? 1 : 0);
  const int zi = (kcol == 0) ? kMaxBins + j - 1 : kMaxBins + j;
  const double ir = a.Ld / (double)k;
  double2 acc = make_double2(0.0, 0.0);
  for (int p = a.p1 - 1; p >= a.p0; --p) {
    double2 Zk = part_s[4 * sk][p][j], Zp = part_s[4 * spn][p][zi];
#pragma unroll
    for (int w = 1; w < 4; ++w) {
      Zk = cadd(Zk, part_s[4 * sk + w][p][j]);
      Zp = cadd(Zp, part_s[4 * spn + w][p][zi]);
    }
    Zp = cconj(Zp);
    double2 Ya = make_double2(Zk.x + Zp.x, Zk.y + Zp.y);
    double2 Yb = make_double2(Zk.y - Zp.y, Zp.x - Zk.x);
    if (k == L) { Ya.y = 0.0; Yb.y = 0.0; }
    const int i0 = 2 * p, i1 = 2 * p + 1;
    const double ac0 = R.ac[i0], bc0 = R.bc[i0], ac1 = R.ac[i1] * bisig, bc1 = R.bc[i1] * bisig;
    const double t0x = fma(ac0, Ya.x, bc0 * Ya.y), t0y = fma(ac0, Ya.y, -bc0 * Ya.x);
    const double t1x = fma(ac1, Yb.x, bc1 * Yb.y), t1y = fma(ac1, Yb.y, -bc1 * Yb.x);
    const double w2 = ir * ir;
    acc.x = fma(acc.x, w2, fma(ir, t1x, t0x));
    acc.y = fma(acc.y, w2, fma(ir, t1y, t0y));
  }
  double post = 1.0;
  if (R.pr) post = ipow_f((double)k / a.Ld, R.pr);
  if (R.post_e && R.pe) post *= ipow_f(R.post_e[k - 1], R.pe);
  double r0 = 0.5 * post * sqrt(ir);
  for (int p = 0; p < a.p0; ++p) r0 = (r0 * ir) * ir;           // (L/k)^{2 p0}
  double v = acc.x * r0;
  if (a.cs_tab) {
    const double2 th = __ldg(a.cs_tab + (k - 1));
    v = v * th.x + (acc.y * r0) * th.y;
  }
  a.part[(long long)ul * a.part_stride + (k - 1)] = v;
}

// One bin per column (the default narrow-row form): the single-bin kernel
// keeps both loads of four unrolled iterations in flight (the general
// far_rowdot_kernel<1> measured 5.9 vs 3.9 ms on cfg2).
__global__ void __launch_bounds__(256)
far_rowdot1_kernel(FarArgs a, int c_lo) {
  const int L = (int)a.L;
  const int L1 = a.L1, L2 = a.L2;
  const int c = c_lo + blockIdx.x;
  const int ul = blockIdx.y;
  const UnitDesc U = a.units[a.u0 + ul];
  const ReqDesc& R = a.reqs[U.req];
  const BlockDesc& B = a.blocks[U.block];
  const double bsig = B.sig, bisig = B.isig;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int cb = (L2 - c) % L2;
  // outputs: k = c (needs Z[c] = S0(c), conj Z[2L-c] = conj S1(cb)) and
  //          k = cb (needs Z[cb] = S0(cb), conj Z[2L-cb] = conj S1(c))
  const int kA = c, kB = (cb != c) ? cb : 0;
  const bool okA = kA >= 1 && kA <= L && kA >= B.r0 && kA < B.r1;
  const bool okB = kB >= 1 && kB <= L && kB >= B.r0 && kB < B.r1;
  if (!okA && !okB) return;
  __shared__ double2 part_s[8][kMaxPairs][2];
  const int side_w = wid >> 2, quarter = wid & 3;
  const int col = side_w == 0 ? c : cb;
  const double2* rot = a.tw + (L1 - 2);   // e^{+2 pi i n1 / L1}
  const int qlen = (L1 + 3) / 4;
  const int lo = quarter * qlen, hi = min(L1, lo + qlen);
  for (int p = a.p0; p < a.p1; ++p) {
    const double2* g = a.G + ((long long)(ul * a.M + p) * L2 + col) * L1;
    double2 s0 = make_double2(0, 0), s1 = make_double2(0, 0);
#pragma unroll 4
    for (int n1 = lo + lane; n1 < hi; n1 += 32) {
      const double2 v = g[n1];
      s0 = cadd(s0, v);
      s1 = cadd(s1, cmul(v, cconj(__ldg(rot + n1))));
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
      s0.x += __shfl_xor_sync(0xffffffffu, s0.x, off);
      s0.y += __shfl_xor_sync(0xffffffffu, s0.y, off);
      s1.x += __shfl_xor_sync(0xffffffffu, s1.x, off);
      s1.y += __shfl_xor_sync(0xffffffffu, s1.y, off);
    }
    if (lane == 0) {
      part_s[wid][p][0] = s0;
      part_s[wid][p][1] = s1;
    }
  }
  __syncthreads();
  const int side = threadIdx.x;
  if (side >= 2) return;
  const bool ok = side == 0 ? okA : okB;
  if (!ok) return;
  const int k = side == 0 ? kA : kB;
  const double ir = a.Ld / (double)k;
  double2 acc = make_double2(0.0, 0.0);
  for (int p = a.p1 - 1; p >= a.p0; --p) {
    // fixed-order combination of the four quarters; Z[k] from this side's
    // column, conj Z[2L-k] from the partner column
    const int sk = side, sp = side ^ (cb != c ? 1 : 0);
    double2 Zk = part_s[4 * sk][p][0], Zp = part_s[4 * sp][p][1];
#pragma unroll
    for (int w = 1; w < 4; ++w) {
      Zk = cadd(Zk, part_s[4 * sk + w][p][0]);
      Zp = cadd(Zp, part_s[4 * sp + w][p][1]);
    }
    Zp = cconj(Zp);
    double2 Ya = make_double2(Zk.x + Zp.x, Zk.y + Zp.y);
    double2 Yb = make_double2(Zk.y - Zp.y, Zp.x - Zk.x);
    if (k == L) { Ya.y = 0.0; Yb.y = 0.0; }
    const int i0 = 2 * p, i1 = 2 * p + 1;
    const double ac0 = R.ac[i0], bc0 = R.bc[i0], ac1 = R.ac[i1] * bisig, bc1 = R.bc[i1] * bisig;
    const double t0x = fma(ac0, Ya.x, bc0 * Ya.y), t0y = fma(ac0, Ya.y, -bc0 * Ya.x);
    const double t1x = fma(ac1, Yb.x, bc1 * Yb.y), t1y = fma(ac1, Yb.y, -bc1 * Yb.x);
    const double w2 = ir * ir;
    acc.x = fma(acc.x, w2, fma(ir, t1x, t0x));
    acc.y = fma(acc.y, w2, fma(ir, t1y, t0y));
  }
  double post = 1.0;
  if (R.pr) post = ipow_f((double)k / a.Ld, R.pr);
  if (R.post_e && R.pe) post *= ipow_f(R.post_e[k - 1], R.pe);
  double r0 = 0.5 * post * sqrt(ir);
  for (int p = 0; p < a.p0; ++p) r0 = (r0 * ir) * ir;           // (L/k)^{2 p0}
  double v = acc.x * r0;
  if (a.cs_tab) {
    const double2 th = __ldg(a.cs_tab + (k - 1));
    v = v * th.x + (acc.y * r0) * th.y;
  }
  a.part[(long long)ul * a.part_stride + (k - 1)] = v;
}

// ------------------------------------------------- pass 2, paired-lane form
//
// CTA = (column pair {c, L2-c}, unit); lane pairs (2 tt, 2 tt + 1) hold the
// same FFT index k1 of the two columns.  Half 1 transforms
//     h[n1] = conj(G[L2-c][n1]) * e^{2 pi i n1 / L1}     (c != 0; no twiddle for c == 0)
// so that its output V[k1] = conj(Z[2L - (c + L2 k1)]) lands on the same k1
// as U[k1] = Z[c + L2 k1]: the DCT/DST separation of every output row needs
// only one register exchange between the two lanes (no shared-memory round
// trip, no barrier).  Rows c + L2 k1 (k1 < L1/2) are produced by half 0,
// rows (L2-c) + L2 (L1-1-k1) (k1 >= L1/2) by half 1.  The gamma rotation
// (cos th_k, sin th_k) is independent of the term index and is applied once
// at the end (two accumulators).
template <int N1, int E, int MINB>
__global__ void __launch_bounds__(2 * (N1 / E), MINB)
far_pass2x_kernel(FarArgs a) {
  constexpr int T = N1 / E;
  constexpr int NQ = E / 2;
  constexpr int NP = N1 + 4;
  using Sh = FftShape<N1, E>;
  constexpr int RL = Sh::RL;
  extern __shared__ double2 sm2[];
  const int tid = threadIdx.x, h = tid & 1, tt = tid >> 1;
  const int L = (int)a.L;
  const int L2 = a.L2;
  const int c = blockIdx.x;
  const int k2b = (L2 - c) % L2;
  const int ul = blockIdx.y;
  const UnitDesc U = a.units[a.u0 + ul];
  const ReqDesc& R = a.reqs[U.req];
  const BlockDesc& B = a.blocks[U.block];
  const double bsig = B.sig, bisig = B.isig;
  const double2* tw = a.tw + (N1 - 2);

  // computing slots: e' = slot index in "t + T e'" order; half 0 owns
  // e' < E/2 (k1 < L1/2), half 1 owns e' >= E/2.
  int kq[NQ];
  double accC[NQ], accS[NQ], rp[NQ], ir[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int e = h ? q + NQ : q;
    const int k1 = tt + T * e;
    int k = 0;
    if (h == 0) {
      k = c + L2 * k1;
    } else if (c == 0) {
      k = (k1 == N1 / 2) ? L : 0;
    } else if (2 * c != L2) {
      k = k2b + L2 * (N1 - 1 - k1);
    }
    if (k < 1 || k > L || k < B.r0 || k >= B.r1) k = 0;
    kq[q] = k;
    accC[q] = accS[q] = rp[q] = ir[q] = 0.0;
    if (k) {
      const double irk = a.Ld / (double)k;
      double post = 1.0;
      if (R.pr) post = ipow_f((double)k / a.Ld, R.pr);
      if (R.post_e && R.pe) post *= ipow_f(R.post_e[k - 1], R.pe);
      ir[q] = irk;
      rp[q] = post * sqrt(irk);
    }
  }
  const int mycol = h ? k2b : c;
  for (int p = 0; p < a.p0; ++p)
#pragma unroll
    for (int q = 0; q < NQ; ++q) rp[q] = (rp[q] * ir[q]) * ir[q];
  for (int p = a.p0; p < a.p1; ++p) {
    const double2* G = a.G + ((long long)(ul * a.M + p) * L2 + mycol) * N1;
    double2 z[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int n1 = tt + T * e;
      double2 g = G[n1];
      if (h) {
        g = cconj(g);
        if (c != 0) g = cmul(g, __ldg(tw + n1));
      }
      z[e] = g;
    }
    __syncthreads();
    block_fft<N1, E, 1>(z, sm2 + h * NP, tt, tw);
    // slot s holds index tt + T e, e = s/RL + (s%RL)*NB  <=>  s = (e%NB)*RL + e/NB
    constexpr int NB = E / RL;
    double2 own[NQ], oth[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const double2 lo = z[(q % NB) * RL + q / NB];                  // e = q
      const double2 hi = z[((q + NQ) % NB) * RL + (q + NQ) / NB];    // e = q + NQ
      own[q] = h ? hi : lo;
      // partner computes the other half: send it my value at its slot
      const double2 v = h ? lo : hi;
      oth[q].x = __shfl_xor_sync(0xffffffffu, v.x, 1);
      oth[q].y = __shfl_xor_sync(0xffffffffu, v.y, 1);
    }
    const int i0 = 2 * p, i1 = 2 * p + 1;
    const double ac0 = R.ac[i0], as0 = R.as[i0], bc0 = R.bc[i0], bs0 = R.bs[i0];
    const double ac1 = R.ac[i1] * bisig, as1 = R.as[i1] * bisig, bc1 = R.bc[i1] * bisig, bs1 = R.bs[i1] * bisig;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int k = kq[q];
      if (!k) continue;
      // Zk and conj(Z[2L-k]) of output row k
      double2 Zk, Zp;
      if (h == 0) { Zk = own[q]; Zp = oth[q]; }
      else if (c == 0) { Zk = oth[q]; Zp = own[q]; }          // row L
      else { Zk = cconj(own[q]); Zp = cconj(oth[q]); }
      double2 Ya = make_double2(0.5 * (Zk.x + Zp.x), 0.5 * (Zk.y + Zp.y));
      double2 Yb = make_double2(0.5 * (Zk.y - Zp.y), -0.5 * (Zk.x - Zp.x));
      if (k == L) { Ya.y = 0.0; Yb.y = 0.0; }      // S u has no row N (schlomilch.py:314-316)
      const double r0 = rp[q], r1 = r0 * ir[q];
      accC[q] += r0 * (ac0 * Ya.x + bc0 * Ya.y) + r1 * (ac1 * Yb.x + bc1 * Yb.y);
      accS[q] += r0 * (as0 * Ya.x + bs0 * Ya.y) + r1 * (as1 * Yb.x + bs1 * Yb.y);
      rp[q] = r1 * ir[q];
    }
  }
  double* part = a.part + (long long)ul * a.part_stride;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int k = kq[q];
    if (!k) continue;
    double v = accC[q];
    if (a.cs_tab) {
      const double2 th = __ldg(a.cs_tab + (k - 1));
      v = accC[q] * th.x + accS[q] * th.y;
    }
    part[k - 1] = v;
  }
}

// F[vec][j] += each partial of the chunk's units of vec whose block holds row
// j, one at a time in unit order.  Units of one vector are contiguous in the
// chunk.  Adding unit by unit (not the chunk's sum) makes F independent of
// where the chunk boundaries fall, so a vector's result does not depend on
// the rest of the batch (fhtb_apply_host runs vector groups separately).
__global__ void far_reduce_kernel(FarArgs a, int n_units) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= a.n_out) return;
  const long long k = a.first + a.stride * j;
  int u = 0;
  while (u < n_units) {
    const int vec = a.units[a.u0 + u].vec;
    double* f = a.F + (long long)vec * a.ldf + j;
    double s = *f;
    bool any = false;
    while (u < n_units && a.units[a.u0 + u].vec == vec) {
      const BlockDesc& B = a.blocks[a.units[a.u0 + u].block];
      if (k >= B.r0 && k < B.r1) {
        s += a.part[(long long)u * a.part_stride + j];
        any = true;
      }
      ++u;
    }
    if (any) {
      *f = s;
      if (!isfinite(s)) *a.nf = 1;
    }
  }
}

// ---------------------------------------------------------------- launch
// bits 0-3: pass-1 shape at 1024; 4-7: pass-2 shape at 2048; 8-11: paired-lane
// pass 2; 12-15: per-pair pass 1; bit 16: no TMA stores; 20-23: narrow-column
// FFT shape.  Default = best measured on B200.
int g_far_variant = 20 + (3 << 20);
int g_far_bulk = 0;      // narrow-column tables by bulk copy (cp.async.bulk + mbarrier), see UBL_ON
int g_far_hp = 1;        // pass 2: half pairing (HP kernels) for the column pairs k2a >= 1

// 2D tensor map over G viewed as rows of 2*L1 doubles (one row per (unit,
// pair, k2)); cuTensorMapEncodeTiled is fetched through the runtime so the
// library does not link libcuda directly.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

static bool g_tmap(CUtensorMap* m, const FarArgs& a, int n_units, int W, int BR) {
  EncodeTiledFn fn = encode_fn();
  if (!fn || ((unsigned long long)a.G & 127)) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)2 * a.L1, (cuuint64_t)n_units * a.M * a.L2};
  const cuuint64_t strides[1] = {(cuuint64_t)a.L1 * 16};
  const cuuint32_t box[2] = {(cuuint32_t)(2 * W), (cuuint32_t)BR};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)a.G, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int N2, int E, int W, int MINB, bool QT = true>
static cudaError_t p1_t(const FarArgs& a, int n_units, cudaStream_t st) {
  constexpr int T = N2 / E;
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  const int smem = (W * (N2 + PAD) + (QT ? W * N2 : 0)) * 16;   // FFT buffers (staging) + four-step twiddles
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  const bool tma = !a.xw && !(g_far_variant & 0x10000) && g_tmap(&m, a, n_units, W, N2 < 256 ? N2 : 256);
  auto k = tma ? far_pass1_kernel<N2, E, W, MINB, true, QT> : far_pass1_kernel<N2, E, W, MINB, false, QT>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int cols = a.xw ? a.L1 / a.xw : a.L1;      // exchange mode: this rank's column slab
  if (cols % W) return cudaErrorInvalidValue;
  note_launch(), k<<<dim3(cols / W, n_units), W * T, smem, st>>>(a, m);
  return cudaGetLastError();
}

template <int N2>
static cudaError_t p1_d(const FarArgs& a, int n_units, cudaStream_t st) {
  constexpr int E = N2 >= 16 ? 16 : N2;
  // 512-point columns: 128-thread CTAs, 3 per SM (as the tuned 1024 shape);
  // bits 24-27 of the variant select alternatives (tuning sweeps; measured
  // on FB cfg3: default 487, W=8/2 CTAs 470, W=4/2 CTAs 483, W=2/4 CTAs 486)
  if (N2 == 512) {
    switch ((g_far_variant >> 24) & 15) {
      case 1: return p1_t<N2, E, 8, 2>(a, n_units, st);
      case 2: return p1_t<N2, E, 4, 2>(a, n_units, st);
      case 3: return p1_t<N2, E, 2, 4>(a, n_units, st);
      default: return p1_t<N2, E, 4, 3>(a, n_units, st);
    }
  }
  // 2048-point columns: bits 28-30 (default: 2 columns per CTA, 1 CTA/SM;
  // one column at 2 or 3 CTAs/SM measured 8-12% slower on FB cfg3 and cfg2 1e-8)
  if (N2 == 2048) {
    switch ((g_far_variant >> 28) & 7) {
      case 1: return p1_t<N2, E, 1, 2>(a, n_units, st);
      case 2: return p1_t<N2, E, 1, 3>(a, n_units, st);
      default: break;
    }
  }
  // 4096-point columns (narrow-row blocks): twiddles computed per use, 2 CTAs/SM
  if (N2 == 4096) return p1_t<N2, E, 1, 2, false>(a, n_units, st);
  // 8192-point columns (grids 2L = 2^24, 2^25): twiddles per use, one CTA
  // of 512 threads (the staged table would not fit beside the FFT buffer)
  if (N2 == 8192) return p1_t<N2, E, 1, 1, false>(a, n_units, st);
  constexpr int W = N2 >= 4096 ? 1 : 4096 / N2;
  return p1_t<N2, E, W, 1>(a, n_units, st);
}

template <int N1, int E, int MODE, int MINB, bool ACS = false, bool UBLT = false, bool HP = false>
static cudaError_t p2_t(const FarArgs& a, int gx, int gy, cudaStream_t st) {
  constexpr int T = N1 / E;
  constexpr int NCOL = MODE == 1 ? 1 : 2;
  const int smem = (NCOL * (N1 + 4) + (TQS_ON(MODE, E, MINB) ? NCOL * E : 0) + (ACS ? (E / 2) * NCOL * T : 0) +
                    (UBL_ON(MODE, E, MINB, N1, ACS, UBLT) ? 2 * N1 + 1 : 0)) * 16 +
                   (IRS_K(E, MODE) ? (E / 2) * NCOL * T * 12 : 0);   // + IRS row factors, rows
  if constexpr (HP) {
    // column pairs k2a >= 1 by the half-pairing kernel, column 0 by the general one
    if (gx > 1) {
      auto kh = far_pass2_kernel<N1, E, MODE, MINB, ACS, UBLT, true>;
      cudaError_t eh = cudaFuncSetAttribute(kh, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (eh != cudaSuccess) return eh;
      note_launch(), kh<<<dim3(gx - 1, gy), NCOL * T, smem, st>>>(a);
      eh = cudaGetLastError();
      if (eh != cudaSuccess) return eh;
    }
    gx = 1;
  }
  auto k = far_pass2_kernel<N1, E, MODE, MINB, ACS, UBLT>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  note_launch(), k<<<dim3(gx, gy), NCOL * T, smem, st>>>(a);
  return cudaGetLastError();
}

template <int N1, int MODE>
static cudaError_t p2_d(const FarArgs& a, int gx, int gy, cudaStream_t st) {
  if (MODE == 0 && N1 == 2048) {
    switch ((g_far_variant >> 4) & 15) {
      case 2: return p2_t<N1, 8, MODE, 1>(a, gx, gy, st);
      case 3: return p2_t<N1, 16, MODE, 1>(a, gx, gy, st);
      case 4: return p2_t<N1, 8, MODE, 2>(a, gx, gy, st);
      default: break;
    }
  }
  // narrow-column blocks: bits 20-23 of the variant pick E = 16 with the
  // shared step-table twiddles (TQS) for the column FFT
  if constexpr (MODE == 2 && N1 >= 512) {
    switch ((g_far_variant >> 20) & 15) {
      // measured (cfg2, 64 vectors): 2048 columns 11.7 -> 10.4 ms with E = 16;
      // 512 columns 14.6 -> 15.6 ms, so they keep E = 8 under case 1
      case 1: if (N1 >= 1024) return p2_t<N1, 16, MODE, (N1 >= 2048 ? 2 : 3)>(a, gx, gy, st); break;
      case 2: return p2_t<N1, 16, MODE, (N1 >= 2048 ? 2 : N1 >= 1024 ? 3 : 6)>(a, gx, gy, st);
      // case 3 (default): 512 columns at 5 CTAs/SM with step-table twiddles
      // (cfg2 far 70.8 -> 70.6 ms; 6 CTAs/SM 71.4)
      // (bit 18 of the variant: accumulators in registers, the round-1 form)
      case 3: if (g_far_variant & 0x40000) {
                if (N1 == 512) return p2_t<N1, 8, MODE, 5>(a, gx, gy, st);
                if (N1 >= 1024) return p2_t<N1, 16, MODE, (N1 >= 2048 ? 2 : 3)>(a, gx, gy, st);
              } else {
                if (N1 == 512 && g_far_bulk) return p2_t<N1, 8, MODE, 5, true, true>(a, gx, gy, st);
                if (N1 == 512 && g_far_hp) return p2_t<N1, 8, MODE, 5, true, false, true>(a, gx, gy, st);
                if (N1 == 512) return p2_t<N1, 8, MODE, 5, true>(a, gx, gy, st);
                if (N1 == 1024 && g_far_bulk) return p2_t<N1, 16, MODE, 3, true, true>(a, gx, gy, st);
                if (N1 >= 1024 && g_far_hp) return p2_t<N1, 16, MODE, (N1 >= 2048 ? 2 : 3), true, false, true>(a, gx, gy, st);
                if (N1 >= 1024) return p2_t<N1, 16, MODE, (N1 >= 2048 ? 2 : 3), true>(a, gx, gy, st);
              }
              break;
      case 4: if (N1 == 512) return p2_t<N1, 8, MODE, 6>(a, gx, gy, st);
              if (N1 >= 1024) return p2_t<N1, 16, MODE, (N1 >= 2048 ? 2 : 3)>(a, gx, gy, st);
              break;
      default: break;
    }
  }
  // 256-point narrow-column blocks (far_min_cols = 8): 64-thread CTAs, 10 per SM
  if constexpr (MODE == 2 && N1 == 256) {
    // 16 points per thread: two radix-16 passes, one exchange, one-warp CTAs (cfg2 far field
    // with the 91-column block at 256 points: 63.9 ms with 8 points per thread, 63.5 with 16)
    if (g_far_hp) return p2_t<N1, 16, MODE, 16, true, false, true>(a, gx, gy, st);
    return p2_t<N1, 16, MODE, 16, true>(a, gx, gy, st);
  }
  // narrow-column blocks carry a complex state per element: 8 points/thread
  constexpr int E = MODE == 2 ? (N1 >= 8 ? 8 : N1) : (N1 >= 16 ? 16 : N1);
  // two columns of 2048 with E = 16: 256 threads, 2 CTAs/SM measured best
  constexpr int MINB = ((MODE == 0 || MODE == 3) && N1 == 2048) ? 2
                       : ((MODE == 0 || MODE == 3) && N1 == 1024) ? 3
                       : (MODE == 2 && N1 <= 1024) ? (N1 <= 512 ? 4 : 2) : 1;
  // full blocks at 2048 points: accumulators in shared memory as for the narrow-column
  // blocks (128 registers at 2 CTAs/SM spill otherwise; bit 19 of the variant: registers)
  if constexpr ((MODE == 0 || MODE == 3) && N1 == 2048) {
    if (!(g_far_variant & 0x80000) && MODE == 0 && g_far_hp) return p2_t<N1, E, MODE, MINB, true, false, true>(a, gx, gy, st);
    if (!(g_far_variant & 0x80000)) return p2_t<N1, E, MODE, MINB, true>(a, gx, gy, st);
  }
  return p2_t<N1, E, MODE, MINB>(a, gx, gy, st);
}

cudaError_t launch_far_colgen(const FarArgs& a, int logN1, int n_units, cudaStream_t st) {
  note_launch(), colgen_prep_kernel<<<dim3((a.L1 + 255) / 256, n_units), 256, 0, st>>>(a);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return err;
  const int gx = a.L2 / 2 + 1;
  switch (logN1) {
    case 1: return p2_d<2, 2>(a, gx, n_units, st);
    case 2: return p2_d<4, 2>(a, gx, n_units, st);
    case 3: return p2_d<8, 2>(a, gx, n_units, st);
    case 4: return p2_d<16, 2>(a, gx, n_units, st);
    case 5: return p2_d<32, 2>(a, gx, n_units, st);
    case 6: return p2_d<64, 2>(a, gx, n_units, st);
    case 7: return p2_d<128, 2>(a, gx, n_units, st);
    case 8: return p2_d<256, 2>(a, gx, n_units, st);
    case 9: return p2_d<512, 2>(a, gx, n_units, st);
    case 10: return p2_d<1024, 2>(a, gx, n_units, st);
    case 11: return p2_d<2048, 2>(a, gx, n_units, st);
    case 12: return p2_d<4096, 2>(a, gx, n_units, st);
  }
  return cudaErrorInvalidValue;
}

// L2 prefetch of the coefficient rows of a chunk's units, launched just
// before pass 1: the pass-1 prologue loads c strided by L1 columns at CTA
// start, where its DRAM latency is exposed (~16% of pass-1 stall samples).
__global__ void prefetch_rows_kernel(FarArgs a) {
  const UnitDesc U = a.units[a.u0 + blockIdx.y];
  const ReqDesc& R = a.reqs[U.req];
  const double* row = a.C + (long long)R.vec * a.ldc;
  const long long lines = (a.n_data_cols * 8 + 127) / 128;
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < lines; l += (long long)gridDim.x * blockDim.x)
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(row + l * 16));
}

cudaError_t launch_prefetch_rows(const FarArgs& a, int n_units, cudaStream_t st) {
  const long long lines = (a.n_data_cols * 8 + 127) / 128;
  const int bx = (int)std::min<long long>((lines + 255) / 256, 64);
  note_launch(), prefetch_rows_kernel<<<dim3(bx, n_units), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_far_rowdot(const FarArgs& a, int n_units, int kbins, cudaStream_t st) {
  const dim3 grid(a.L2 / 2 + 1, n_units);
  if (kbins <= 1) note_launch(), far_rowdot1_kernel<<<grid, 256, 0, st>>>(a, 0);
  else if (kbins <= 2) note_launch(), far_rowdot_kernel<2><<<grid, 256, 0, st>>>(a, 0);
  else if (kbins <= 3) note_launch(), far_rowdot_kernel<3><<<grid, 256, 0, st>>>(a, 0);
  else note_launch(), far_rowdot_kernel<4><<<grid, 256, 0, st>>>(a, 0);
  return cudaGetLastError();
}

template <int N2, int E, int W, int MINB>
static cudaError_t p1p_t(const FarArgs& a, int n_units, cudaStream_t st) {
  constexpr int T = N2 / E;
  constexpr int PAD = 8 / W > 0 ? 8 / W : 0;
  const int smem = W * (N2 + PAD) * 16;
  auto k = far_pass1p_kernel<N2, E, W, MINB>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  note_launch(), k<<<dim3(a.L1 / W, n_units * a.M), W * T, smem, st>>>(a);
  return cudaGetLastError();
}

template <int N2>
static cudaError_t p1p_d(const FarArgs& a, int n_units, cudaStream_t st) {
  constexpr int E = N2 >= 16 ? 16 : N2;
  switch ((g_far_variant >> 12) & 15) {
    case 2: return p1p_t<N2, E, (N2 >= 2048 ? 1 : 2048 / N2), 1>(a, n_units, st);
    case 3: return p1p_t<N2, E, (N2 >= 1024 ? 1 : 1024 / N2), 2>(a, n_units, st);
    case 4: return p1p_t<N2, E, (N2 >= 4096 ? 1 : 4096 / N2), 1>(a, n_units, st);
    default: return p1p_t<N2, E, (N2 >= 2048 ? 1 : 2048 / N2), 2>(a, n_units, st);
  }
}

cudaError_t launch_far_pass1(const FarArgs& a, int logN2, int n_units, cudaStream_t st) {
  if (((g_far_variant >> 12) & 15) && a.w0_tab && !a.xw) {
    switch (logN2) {
      case 6: return p1p_d<64>(a, n_units, st);
      case 7: return p1p_d<128>(a, n_units, st);
      case 8: return p1p_d<256>(a, n_units, st);
      case 9: return p1p_d<512>(a, n_units, st);
      case 10: return p1p_d<1024>(a, n_units, st);
      case 11: return p1p_d<2048>(a, n_units, st);
      case 12: return p1p_d<4096>(a, n_units, st);
      case 13: return p1p_d<8192>(a, n_units, st);
    }
    return cudaErrorInvalidValue;
  }
  switch (logN2) {
    case 6: return p1_d<64>(a, n_units, st);
    case 7: return p1_d<128>(a, n_units, st);
    case 8: return p1_d<256>(a, n_units, st);
    case 9: return p1_d<512>(a, n_units, st);
    case 10:
      switch (g_far_variant & 15) {
        case 1: return p1_t<1024, 16, 2, 2>(a, n_units, st);
        case 4: return p1_t<1024, 16, 2, 3>(a, n_units, st);
        case 5: return p1_t<1024, 16, 1, 4>(a, n_units, st);
        case 6: return p1_t<1024, 16, 1, 6>(a, n_units, st);
        case 2: return p1_t<1024, 8, 2, 2>(a, n_units, st);
        case 3: return p1_t<1024, 8, 4, 1>(a, n_units, st);
        default: return p1_d<1024>(a, n_units, st);
      }
    case 11: return p1_d<2048>(a, n_units, st);
    case 12: return p1_d<4096>(a, n_units, st);
    case 13: return p1_d<8192>(a, n_units, st);
  }
  return cudaErrorInvalidValue;
}

template <int N1, int E, int MINB>
static cudaError_t p2x_t(const FarArgs& a, int gx, int gy, cudaStream_t st) {
  constexpr int T = N1 / E;
  const int smem = 2 * (N1 + 4) * 16;
  auto k = far_pass2x_kernel<N1, E, MINB>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  note_launch(), k<<<dim3(gx, gy), 2 * T, smem, st>>>(a);
  return cudaGetLastError();
}

template <int N1>
static cudaError_t p2x_d(const FarArgs& a, int gx, int gy, cudaStream_t st) {
  switch ((g_far_variant >> 8) & 15) {
    case 2: return p2x_t<N1, 16, 2>(a, gx, gy, st);
    case 3: return p2x_t<N1, 8, 1>(a, gx, gy, st);
    case 4: return p2x_t<N1, 8, 2>(a, gx, gy, st);
    default: return p2x_t<N1, 16, 1>(a, gx, gy, st);
  }
}

cudaError_t launch_far_pass2x_range(const FarArgs& a, int logN1, int n_pairs, int n_units, cudaStream_t st) {
  switch (logN1) {
    case 7: return p2_d<128, 3>(a, n_pairs, n_units, st);
    case 8: return p2_d<256, 3>(a, n_pairs, n_units, st);
    case 9: return p2_d<512, 3>(a, n_pairs, n_units, st);
    case 10: return p2_d<1024, 3>(a, n_pairs, n_units, st);
    case 11: return p2_d<2048, 3>(a, n_pairs, n_units, st);
    case 12: return p2_d<4096, 3>(a, n_pairs, n_units, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_far_pass2(const FarArgs& a, int logN1, int n_units, cudaStream_t st) {
  const int gx = a.L2 / 2 + 1;
  if ((g_far_variant >> 8) & 15) {
    switch (logN1) {
      case 7: return p2x_d<128>(a, gx, n_units, st);
      case 8: return p2x_d<256>(a, gx, n_units, st);
      case 9: return p2x_d<512>(a, gx, n_units, st);
      case 10: return p2x_d<1024>(a, gx, n_units, st);
      case 11: return p2x_d<2048>(a, gx, n_units, st);
      case 12: return p2x_d<4096>(a, gx, n_units, st);
    }
    return cudaErrorInvalidValue;
  }
  switch (logN1) {
    case 1: return p2_d<2, 0>(a, gx, n_units, st);
    case 2: return p2_d<4, 0>(a, gx, n_units, st);
    case 3: return p2_d<8, 0>(a, gx, n_units, st);
    case 4: return p2_d<16, 0>(a, gx, n_units, st);
    case 5: return p2_d<32, 0>(a, gx, n_units, st);
    case 6: return p2_d<64, 0>(a, gx, n_units, st);
    case 7: return p2_d<128, 0>(a, gx, n_units, st);
    case 8: return p2_d<256, 0>(a, gx, n_units, st);
    case 9: return p2_d<512, 0>(a, gx, n_units, st);
    case 10: return p2_d<1024, 0>(a, gx, n_units, st);
    case 11: return p2_d<2048, 0>(a, gx, n_units, st);
    case 12: return p2_d<4096, 0>(a, gx, n_units, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_far_onepass(const FarArgs& a, int logN1, int n_units, cudaStream_t st) {
  switch (logN1) {
    case 1: return p2_d<2, 1>(a, 1, n_units, st);
    case 2: return p2_d<4, 1>(a, 1, n_units, st);
    case 3: return p2_d<8, 1>(a, 1, n_units, st);
    case 4: return p2_d<16, 1>(a, 1, n_units, st);
    case 5: return p2_d<32, 1>(a, 1, n_units, st);
    case 6: return p2_d<64, 1>(a, 1, n_units, st);
    case 7: return p2_d<128, 1>(a, 1, n_units, st);
    case 8: return p2_d<256, 1>(a, 1, n_units, st);
    case 9: return p2_d<512, 1>(a, 1, n_units, st);
    case 10: return p2_d<1024, 1>(a, 1, n_units, st);
    case 11: return p2_d<2048, 1>(a, 1, n_units, st);
    case 12: return p2_d<4096, 1>(a, 1, n_units, st);
    case 13: return p2_d<8192, 1>(a, 1, n_units, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_far_reduce(const FarArgs& a, int n_units, cudaStream_t st) {
  const long long b = (a.n_out + 255) / 256;
  note_launch(), far_reduce_kernel<<<(unsigned)b, 256, 0, st>>>(a, n_units);
  return cudaGetLastError();
}

__global__ void cs_table_kernel(double2* cs, long long L, double gamma, double pi_over_L) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < L; i += (long long)gridDim.x * blockDim.x) {
    double s, c;
    sincos(-gamma * (double)(i + 1) * pi_over_L, &s, &c);
    cs[i] = make_double2(c, s);
  }
}

__global__ void col_tables_kernel(double* w0, double* iw, long long L, double gamma) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < L; i += (long long)gridDim.x * blockDim.x) {
    const double om = ((double)(i + 1) + gamma) * 3.141592653589793;
    iw[i] = 1.0 / om;
    w0[i] = 1.0 / sqrt(om);
  }
}

cudaError_t launch_col_tables(double* w0, double* iw, long long L, double gamma, cudaStream_t st) {
  long long b = (L + 255) / 256;
  if (b > 148 * 64) b = 148 * 64;
  note_launch(), col_tables_kernel<<<(unsigned)b, 256, 0, st>>>(w0, iw, L, gamma);
  return cudaGetLastError();
}

cudaError_t launch_cs_table(double2* cs, long long L, double gamma, double pi_over_L, cudaStream_t st) {
  long long b = (L + 255) / 256;
  if (b > 148 * 64) b = 148 * 64;
  note_launch(), cs_table_kernel<<<(unsigned)b, 256, 0, st>>>(cs, L, gamma, pi_over_L);
  return cudaGetLastError();
}

}  // namespace fhtb
