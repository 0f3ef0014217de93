// fhtb_bessel.cuh -- fp64 J_nu(z) evaluators for integer nu >= 0, z >= 0.
//
// Same three-branch method as the reference point evaluator
// (bessel.py:232-260): 10-term Taylor series below t_{nu,10}(2^-52)
// (bessel.py:133-146), 10-pair Hankel asymptotic expansion above
// s_{nu,10}(2^-52) (bessel.py:72-91), Miller's backward recurrence with the
// J0 + 2 sum J_2k = 1 normalisation in between (bessel.py:197-229).
// Differences (rounding level only): the Miller start order is chosen per
// element instead of from the tile maximum, and the Hankel phase is formed by
// rotating (cos z, sin z) by the exact octant angle (2nu+1)pi/4.
//
// jn_all(): one Miller sweep that yields J_0..J_omax together (used by the
// multi-order near field of the Fourier-Bessel / DHT engines, where the
// reference re-runs Miller once per order, schlomilch.py:512-523).
#pragma once
#include <cuda_runtime.h>

namespace fhtb {

constexpr int kAsyPairs = 10;      // bessel.py:40  _ASY_TERMS
constexpr int kTaylorTerms = 10;   // bessel.py:39  _TAYLOR_TERMS
constexpr int kMaxOrder = 1023;    // orders held by the per-device constant table (engine universes)

// Per-order constants, filled on the host (fhtb_host.cpp).
struct JOrder {
  double tlo;               // taylor_cutoff(nu, 10, 2^-52)
  double shi;               // asy_cutoff(nu, 10, 2^-52)
  double inv_fact;          // 1 / nu!
  double cphi, sphi;        // cos, sin of (2nu+1) pi/4
  double ae[kAsyPairs];     // (-1)^m a_{2m}(nu)
  double ao[kAsyPairs];     // (-1)^m a_{2m+1}(nu)
};

#define FHTB_SQRT_2_OVER_PI 0.79788456080286535588

__device__ __forceinline__ double jn_taylor(int nu, double z, const JOrder& c) {
  const double h = 0.5 * z;
  double term = c.inv_fact;
  for (int i = 0; i < nu; ++i) term *= h;
  double acc = term;
  const double hh = h * h;
#pragma unroll
  for (int t = 1; t < kTaylorTerms; ++t) {
    term = -term * hh / (double)(t * (t + nu));
    acc += term;
  }
  return acc;
}

// Hankel expansion given (cos z, sin z).
__device__ __forceinline__ double jn_hankel_cs(double z, double cz, double sz, const JOrder& c) {
  const double w = 1.0 / (z * z);
  double pe = c.ae[kAsyPairs - 1], po = c.ao[kAsyPairs - 1];
#pragma unroll
  for (int m = kAsyPairs - 2; m >= 0; --m) {
    pe = fma(pe, w, c.ae[m]);
    po = fma(po, w, c.ao[m]);
  }
  const double cm = cz * c.cphi + sz * c.sphi;   // cos(z - phi)
  const double sm = sz * c.cphi - cz * c.sphi;   // sin(z - phi)
  return FHTB_SQRT_2_OVER_PI * rsqrt(z) * (cm * pe - sm * po / z);
}

__device__ __forceinline__ double jn_hankel(double z, const JOrder& c) {
  double s, co;
  sincos(z, &s, &co);
  return jn_hankel_cs(z, co, s, c);
}

__device__ __forceinline__ int miller_start(double b) {
  // b + 10 + 11 b^{1/3} (bessel.py:197-229), the cube root in single precision
  // scaled up by more than its error (1 ulp + the rounding of b), so that the
  // start order is never below the reference's and equals it except when
  // the exact value lies within ~3e-7 relative of an integer
  return (int)ceil(b + 10.0 + 11.0 * ((double)cbrtf((float)b) * (1.0 + 3e-7)));
}

// Miller for a single order nu, mid-range z > 0.
__device__ __forceinline__ double jn_miller(int nu, double z) {
  const double b = fmax((double)nu, z);
  const int k0 = miller_start(b);
  const double rz = __drcp_rn(z);          // = 1.0 / z, correctly rounded
  double up = 0.0, cur = 1e-30, nrm = 0.0, cap = 0.0;
  // orders above nu: two steps per trip, no capture, one overflow check
  int k = k0;
  if ((k - nu - 1) & 1) {
    const double lo = fma((2.0 * k) * rz, cur, -up);
    up = cur;
    cur = lo;
    if (((k - 1) & 1) == 0) nrm += 2.0 * cur;
    --k;
  }
  // the even order of every two-step trip has the same parity slot
  const bool ev1 = ((k - 1) & 1) == 0;
  double tk = 2.0 * k;                      // 2k, exact, counted down in doubles (no I2F per step)
  // eight steps per trip with one overflow check while the growth of eight
  // steps, at most (2 k0 / z)^8 < 1e48, stays inside the 1e58 headroom
  if (tk * rz < 1e6) {
    for (; k > nu + 8; k -= 8) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const double lo = fma(tk * rz, cur, -up);
        const double lo2 = fma((tk - 2.0) * rz, lo, -cur);
        nrm += 2.0 * (ev1 ? lo : lo2);
        up = lo;
        cur = lo2;
        tk -= 4.0;
      }
      if (fabs(cur) > 1e250) {
        cur *= 1e-250; up *= 1e-250; nrm *= 1e-250;
      }
    }
  }
  for (; k > nu + 1; k -= 2) {
    const double lo = fma(tk * rz, cur, -up);
    const double lo2 = fma((tk - 2.0) * rz, lo, -cur);
    nrm += 2.0 * (ev1 ? lo : lo2);
    up = lo;
    cur = lo2;
    tk -= 4.0;
    if (fabs(cur) > 1e250) {
      cur *= 1e-250; up *= 1e-250; nrm *= 1e-250;
    }
  }
  // orders nu .. 0
  for (; k > 0; --k) {
    const double lo = fma((2.0 * k) * rz, cur, -up);
    up = cur;
    cur = lo;
    const int o = k - 1;
    if (o == nu) cap = cur;
    if ((o & 1) == 0) nrm += (o == 0) ? cur : 2.0 * cur;
    if (fabs(cur) > 1e250) {
      cur *= 1e-250; up *= 1e-250; nrm *= 1e-250; cap *= 1e-250;
    }
  }
  return cap / nrm;
}

// J_nu(z), reference dispatch (bessel.py:245-256).
__device__ __forceinline__ double jn(int nu, double z, const JOrder& c) {
  if (z <= c.tlo) return jn_taylor(nu, z, c);
  if (z >= c.shi) return jn_hankel(z, c);
  return jn_miller(nu, z);
}

// J_0..J_{omax}(z) into out[] (omax < OMAX).  Branch per element: Taylor is
// not needed (Miller is accurate for all small z > 0); Hankel per order
// where z clears that order's cutoff, sharing one sincos.
template <int OMAX>
__device__ __forceinline__ void jn_all(int omax, double z, const JOrder* __restrict__ tab,
                                        double (&out)[OMAX]) {
  if (z == 0.0) {
#pragma unroll
    for (int o = 0; o < OMAX; ++o) out[o] = (o == 0) ? 1.0 : 0.0;
    return;
  }
  if (z >= tab[omax].shi) {
    double s, co;
    sincos(z, &s, &co);
#pragma unroll
    for (int o = 0; o < OMAX; ++o) out[o] = (o <= omax) ? jn_hankel_cs(z, co, s, tab[o]) : 0.0;
    return;
  }
  const double b = fmax((double)omax, z);
  // start at least at OMAX so the capture phase below has static indices
  const int k0 = max(miller_start(b), OMAX);
  const double rz = __drcp_rn(z);          // = 1.0 / z, correctly rounded
  double up = 0.0, cur = 1e-30, nrm = 0.0;
  // phase 1: k = k0 .. OMAX+1 produce f_{k-1} for orders >= OMAX (no capture);
  // two steps per trip (one even order), overflow check once per trip (the
  // growth of two steps stays far below the 1e58 headroom)
  int k = k0;
  if ((k - OMAX) & 1) {
    const double lo = fma((2.0 * k) * rz, cur, -up);
    up = cur;
    cur = lo;
    if (((k - 1) & 1) == 0) nrm += 2.0 * cur;
    --k;
  }
  // orders k-1 and k-2: exactly one of them is even, the same slot every trip
  const bool ev1 = ((k - 1) & 1) == 0;
  double tk = 2.0 * k;                      // 2k, exact (no I2F per step)
  // eight steps per overflow check while (2 k0 / z)^8 < 1e48 (jn_miller)
  if (tk * rz < 1e6) {
    for (; k > OMAX + 7; k -= 8) {
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        const double lo = fma(tk * rz, cur, -up);
        const double lo2 = fma((tk - 2.0) * rz, lo, -cur);
        nrm += 2.0 * (ev1 ? lo : lo2);
        up = lo;
        cur = lo2;
        tk -= 4.0;
      }
      if (fabs(cur) > 1e250) {
        cur *= 1e-250; up *= 1e-250; nrm *= 1e-250;
      }
    }
  }
  for (; k > OMAX; k -= 2) {
    const double lo = fma(tk * rz, cur, -up);
    const double lo2 = fma((tk - 2.0) * rz, lo, -cur);
    nrm += 2.0 * (ev1 ? lo : lo2);
    up = lo;
    cur = lo2;
    tk -= 4.0;
    if (fabs(cur) > 1e250) {
      cur *= 1e-250; up *= 1e-250; nrm *= 1e-250;
    }
  }
  // phase 2: k = OMAX .. 1 produce f_{OMAX-1} .. f_0, captured with static indices
#pragma unroll
  for (int o = OMAX - 1; o >= 0; --o) {
    const double lo = fma((2.0 * (o + 1)) * rz, cur, -up);
    up = cur;
    cur = lo;
    out[o] = cur;
    if ((o & 1) == 0) nrm += (o == 0) ? cur : 2.0 * cur;
    if (fabs(cur) > 1e250) {
      cur *= 1e-250; up *= 1e-250; nrm *= 1e-250;
#pragma unroll
      for (int q = o; q < OMAX; ++q) out[q] *= 1e-250;
    }
  }
  const double inv = 1.0 / nrm;
#pragma unroll
  for (int o = 0; o < OMAX; ++o) out[o] = (o <= omax) ? out[o] * inv : 0.0;
}

// J_{omin}..J_{omin+W-1}(z) into out[] (orders above omax are returned as 0):
// jn_all for a window of orders that does not start at 0 (Fourier-Bessel /
// DHT engines of order nu > 0 use the universe |nu -/+ j|, j < K).  One Miller
// sweep: down to the window without capture, W captured steps with static
// indices, then on to order 0 for the normalisation.
template <int W>
__device__ __forceinline__ void jn_window(int omin, int omax, double z, const JOrder* __restrict__ tab,
                                           double (&out)[W]) {
  if (z == 0.0) {
#pragma unroll
    for (int j = 0; j < W; ++j) out[j] = (omin + j == 0) ? 1.0 : 0.0;
    return;
  }
  if (z >= tab[omax].shi) {
    double s, co;
    sincos(z, &s, &co);
#pragma unroll
    for (int j = 0; j < W; ++j) out[j] = (omin + j <= omax) ? jn_hankel_cs(z, co, s, tab[omin + j]) : 0.0;
    return;
  }
  const int top = omin + W;                 // first order above the window
  const double b = fmax((double)omax, z);
  const int k0 = max(miller_start(b), top);
  const double rz = __drcp_rn(z);          // = 1.0 / z, correctly rounded
  double up = 0.0, cur = 1e-30, nrm = 0.0;
  // phase 1: k = k0 .. top+1 produce f_{k-1} for orders >= top (no capture)
  for (int k = k0; k > top; --k) {
    const double lo = fma((2.0 * k) * rz, cur, -up);
    up = cur;
    cur = lo;
    if (((k - 1) & 1) == 0) nrm += 2.0 * cur;
    if (fabs(cur) > 1e250) {
      cur *= 1e-250; up *= 1e-250; nrm *= 1e-250;
    }
  }
  // phase 2: orders top-1 .. omin, captured with static indices
#pragma unroll
  for (int j = W - 1; j >= 0; --j) {
    const int o = omin + j;
    const double lo = fma((2.0 * (o + 1)) * rz, cur, -up);
    up = cur;
    cur = lo;
    out[j] = cur;
    if ((o & 1) == 0) nrm += (o == 0) ? cur : 2.0 * cur;
    if (fabs(cur) > 1e250) {
      cur *= 1e-250; up *= 1e-250; nrm *= 1e-250;
#pragma unroll
      for (int q = j; q < W; ++q) out[q] *= 1e-250;
    }
  }
  // phase 3: orders omin-1 .. 0 (normalisation only)
  for (int o = omin - 1; o >= 0; --o) {
    const double lo = fma((2.0 * (o + 1)) * rz, cur, -up);
    up = cur;
    cur = lo;
    if ((o & 1) == 0) nrm += (o == 0) ? cur : 2.0 * cur;
    if (fabs(cur) > 1e250) {
      cur *= 1e-250; up *= 1e-250; nrm *= 1e-250;
#pragma unroll
      for (int q = 0; q < W; ++q) out[q] *= 1e-250;
    }
  }
  const double inv = 1.0 / nrm;
#pragma unroll
  for (int j = 0; j < W; ++j) out[j] = (omin + j <= omax) ? out[j] * inv : 0.0;
}

}  // namespace fhtb
