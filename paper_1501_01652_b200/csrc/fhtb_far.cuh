// fhtb_far.cuh -- device helpers shared by the far-field translation units
// (fhtb_far.cu, fhtb_rowsum.cu): column state, four-step twiddles.
#pragma once
#include "fhtb_core.cuh"
#include "fhtb_launch.h"

namespace fhtb {

// x^p by binary powering (pre/post multipliers reach p = 10 per element)
__device__ __forceinline__ double ipow_f(double x, int p) {
  double r = 1.0;
  for (; p; p >>= 1) {
    if (p & 1) r *= x;
    x *= x;
  }
  return r;
}

// Four-step twiddle e^{+2 pi i m / Q}.
__device__ __forceinline__ double2 qtw(const FarArgs& a, long long m) {
  const int lo = (int)(m & ((1LL << a.qbits) - 1));
  const long long hi = m >> a.qbits;
  double2 w = __ldg(a.qlo + lo);
  if (hi) w = cmul(w, __ldg(a.qhi + hi));
  return w;
}

// Column state of grid column n for request R on block B:
//   v = x_n * omega_n^{-1/2},  iw = 1/omega_n   (0 outside the block)
__device__ __forceinline__ void load_col(const FarArgs& a, const ReqDesc& R, long long cA, long long cB,
                                         long long n, double& v, double& iw) {
  v = 0.0;
  iw = 0.0;
  if (n >= cA && n < cB) {
    double x = a.C[(long long)R.vec * a.ldc + (n - 1)];
    if (R.preA) x *= ipow_f(R.preA[n - 1], R.pa);
    if (R.preB) x *= ipow_f(R.preB[n - 1], R.pb);
    // (computing beats loading w0_tab/iw_tab here: pass 1 28.1 vs 29.6 ms, cfg2)
    const double om = ((double)n + a.gamma) * 3.141592653589793;
    iw = 1.0 / om;
    v = x * (1.0 / sqrt(om));
  }
}

__device__ __forceinline__ void unit_cols(const FarArgs& a, const ReqDesc& R, const BlockDesc& B,
                                          long long& cA, long long& cB) {
  cA = max(max(B.c0, R.col_lo), 1LL);
  cB = min(B.c1, min(a.n_data_cols + 1, a.L + 1));
}

}  // namespace fhtb
