// fhtb_types.h -- plain-old-data descriptors shared by host (fhtb_host.cpp)
// and device (fhtb_*.cu) code.  No torch types, no STL.
#pragma once
#include <cstdint>

namespace fhtb {

constexpr int kMaxOrd = 16;     // order-universe size handled by one request
constexpr int kMaxTerms = 32;   // 2M terms per request (M <= 16)

// One (order_weights, coefficients) request of a Schlomilch application
// (schlomilch.py:436-468), with the Fourier-Bessel / DHT diagonal pre- and
// post-multipliers fused (fourier_bessel.py:215-242, dht.py:151-174):
//
//   x_n  = C[vec][n-1] * preA[n-1]^pa * preB[n-1]^pb      (n >= col_lo)
//   out[vec][j] += (k/L)^pr * post_e[j]^pe * sum_n G(k, n) x_n,
//   G(k, n) = sum_o w[o] J_o(k (n+gamma) pi / L),   k = first + stride*j.
struct ReqDesc {
  int vec;
  int pa, pb, pr, pe;
  int pad_;
  long long col_lo;
  const double* preA;
  const double* preB;
  const double* post_e;
  double w[kMaxOrd];        // weight per universe order (near field)
  // far field: per term i < 2M, row combination A_i = rp_i (ac cos th + as sin th),
  // B_i = rp_i (bc cos th + bs sin th), rp_i = (L/k)^(i+1/2)   (schlomilch.py:280-299)
  double ac[kMaxTerms], as[kMaxTerms], bc[kMaxTerms], bs[kMaxTerms];
};

// Asymptotic block, 1-based half-open (schlomilch.py:119-152), plus the
// chirp-z parameters used when the grid is not a power of two.
struct BlockDesc {
  long long r0, r1, c0, c1;
  // chirp mode: rows k = first + stride*j (j < J), columns n = c0 + m (m < Mn)
  long long J, Mn;
  int logQ;                 // convolution length Q = 2^logQ
  int pad_;
  const double2* H;         // FFT_Q of the chirp filter (device)
  // direct mode: four-step split 2L = 2^dlogL1 * 2^(logQ2L - dlogL1) and the
  // pruned form of the block: 0 full two-pass, 1 narrow columns (no pass 1),
  // 2 narrow rows (pass 2 = two sums per column)
  int dmode;
  int dlogL1;
  // dmode 2: FFT bins k1 < kbins of each column are needed (rows k < kbins * L2)
  int kbins;
  // direct mode: terms 2p (real part) and 2p+1 (imaginary part) share one
  // complex FFT; u_{2p+1} = u_{2p} / omega_n is smaller by omega_n, and what the
  // separation Z[k] -/+ conj Z[2L-k] loses is amplified by the row factor L/k
  // (1e-10 relative at N = 2^24, k ~ 10).  The imaginary part is therefore
  // carried times sig = 2^floor(log2 omega_{c0}) (exact) and the odd-term
  // coefficients times isig = 1/sig.
  double sig, isig;
  int pad2_;
};

// Work unit of the far field: one request on one block.
struct UnitDesc {
  int req;
  int block;
  int vec;
  int pad_;
};

// Near-field / direct tile: output rows [j0, j0+nrows) of one segment,
// columns [na, nb) (1-based grid columns).
struct NearTile {
  int seg;
  int nrows;
  long long j0;
  long long na, nb;
  long long part;           // partial-sum slot base (-1: write F directly)
};

}  // namespace fhtb
