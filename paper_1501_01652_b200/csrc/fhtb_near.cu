// fhtb_near.cu -- near-field ("border") and direct-summation kernel.
//
//   out[vec][j] (+)= post_q(k) * sum_n sum_o w_q[o] J_o(rowf(k) * colf(n)) x_q[n]
//
// over a list of tiles (output rows x grid columns).  This single kernel is
// the GPU form of
//   * the Schlomilch border  _eval_segments / SchlomilchEngine._mask_streamed
//     (schlomilch.py:193-220, 504-531),
//   * schlomilch_direct (schlomilch.py:223-229),
//   * the Fourier-Bessel low columns _direct_columns_many
//     (fourier_bessel.py:148-172),
//   * the DHT direct rows _rows_direct (dht.py:82-94).
//
// Bessel values are generated in registers (one Miller sweep yields every
// order of the universe), staged in shared memory, and contracted against
// the weighted coefficient tile with fp64 tensor-core MMA (wmma m8n8k4 ->
// DMMA).  The reduction order over columns is fixed, so results are
// reproducible run to run.
#include <mma.h>

#include "fhtb_bessel.cuh"
#include "fhtb_core.cuh"
#include "fhtb_launch.h"

namespace fhtb {

using namespace nvcuda;

constexpr int kRT = kNearRT;   // output rows per tile
constexpr int kNearThreads = 256;

// JT: request columns per CTA (64, or 128 when a vector group needs more,
// e.g. Fourier-Bessel and DHT batches -- the Bessel tile is then generated
// once for all of them).
// Shared-memory row strides are padded so that the m8n8k4 fp64 fragment
// loads are bank-conflict free: A rows (8 rows x 4 doubles per fragment) by
// 4 doubles, B rows (4 rows x 8 doubles) by 8 doubles.
template <int NORD, int JT> struct NearCfg {
  static constexpr int NK = NORD <= 2 ? 16 : (NORD <= 4 ? 8 : 4);   // grid columns per step
  static constexpr int K = NK * NORD;                                // MMA depth per step
  static constexpr int KA = K + 4;                                   // As row stride
  static constexpr int JB = JT + 8;                                  // Bs / Cs row stride
  static constexpr int A_ELEMS = kRT * KA;
  static constexpr int B_ELEMS = K * JB;
  static constexpr int C_ELEMS = kRT * JB;
  static constexpr int SMEM = 8 * ((A_ELEMS + B_ELEMS) > C_ELEMS ? (A_ELEMS + B_ELEMS) : C_ELEMS);
};

// x^p by binary powering (the DHT pre-multipliers reach p = 10 per element
// and column step; the repeated product was 9% of the DHT near-field samples)
__device__ __forceinline__ double ipow(double x, int p) {
  double r = 1.0;
  for (; p; p >>= 1) {
    if (p & 1) r *= x;
    x *= x;
  }
  return r;
}

template <int NORD, int JT>
__global__ void __launch_bounds__(kNearThreads, (NORD == 1 && JT == 64) ? 3 : 2)
near_kernel(NearArgs a) {
  using Cfg = NearCfg<NORD, JT>;
  constexpr int NK = Cfg::NK, K = Cfg::K, KA = Cfg::KA, JB = Cfg::JB;
  extern __shared__ double smem[];
  double* As = smem;                       // [kRT][K]
  double* Bs = smem + Cfg::A_ELEMS;        // [K][JT]
  double* Cs = smem;                       // [kRT][JT] (epilogue, aliases As/Bs)

  const NearTile tile = a.tiles[blockIdx.x];
  const int g = blockIdx.y;
  const int q0 = a.grp_q0[g], q1 = a.grp_q0[g + 1];
  const int nq = q1 - q0;
  // order-parity classes (universe {0..n-1}): the group's columns are
  // [0, fe*8) requests of even orders only, [fe*8, fo*8) odd orders only,
  // then mixed.  The K dimension is laid out even orders first (PE of them),
  // so each class contracts only its half of K.
  constexpr int PE = (NORD + 1) / 2;
  const bool split = a.grp_cls != nullptr;
  int fe = 0, fo = 0;
  if (split) {
    const int2 cl = a.grp_cls[g];
    fe = cl.x >> 3;
    fo = cl.y >> 3;
  }
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  if (a.n_shards > 1 && (int)(blockIdx.x % a.n_shards) != a.shard) {
    // another shard's tile: contribute zeros to the partial slot (if any)
    if (tile.part >= 0) {
      const int v0 = a.grp_v0[g], nv = a.grp_v0[g + 1] - v0;
      for (int e = tid; e < kRT * nv; e += kNearThreads)
        a.part[tile.part * a.part_stride + (long long)(v0 + e / kRT) * kRT + e % kRT] = 0.0;
    }
    return;
  }

  // 2D warp tiling of the kRT x JT output: WR x WC warps, each FR x FC
  // fragments of 8 x 8, so that a warp loads FR A- and FC B-fragments per
  // k-step for FR*FC DMMAs (8 rows x JT columns per warp loaded every B
  // fragment once per row fragment: 1 + JT/8 loads for JT/8 DMMAs)
  constexpr int WC = JT >= 128 ? 4 : 2;
  constexpr int WR = (kNearThreads / 32) / WC;
  constexpr int FR = (kRT / 8) / WR;
  constexpr int FC = (JT / 8) / WC;
  const int wr = warp / WC, wc = warp % WC;
  wmma::fragment<wmma::accumulator, 8, 8, 4, double> acc[FR][FC];
#pragma unroll
  for (int r = 0; r < FR; ++r)
#pragma unroll
    for (int c = 0; c < FC; ++c) wmma::fill_fragment(acc[r][c], 0.0);
  const int nfrag = (nq + 7) >> 3;

  constexpr int NBE = (NK * JT + kNearThreads - 1) / kNearThreads;   // Bs elements per thread
  for (long long n0 = tile.na; n0 < tile.nb; n0 += NK) {
    // ---- coefficients of this step, loaded into registers first so their
    // latency hides behind the Bessel tile (stored to Bs after it)
    double xv[NBE];
#pragma unroll
    for (int t = 0; t < NBE; ++t) {
      const int e = tid + t * kNearThreads;
      const int q = e / JT, c = e % JT;
      const long long n = n0 + q;
      double x = 0.0;
      if (e < NK * JT && c < nq && n < tile.nb) {
        const ReqDesc* r = a.reqs + q0 + c;
        if (n >= r->col_lo && n <= a.n_data_cols) {
          x = a.C[(long long)r->vec * a.ldc + (n - 1)];
          if (r->preA) x *= ipow(r->preA[n - 1], r->pa);
          if (r->preB) x *= ipow(r->preB[n - 1], r->pb);
        }
      }
      xv[t] = x;
    }
    // ---- Bessel tile: As[i][u*NK + q] = J_{orders[u]}(z_{i,q})
    for (int e = tid; e < kRT * NK; e += kNearThreads) {
      const int i = e / NK, q = e % NK;
      const long long n = n0 + q;
      const long long j = tile.j0 + i;
      double vals[NORD];
#pragma unroll
      for (int u = 0; u < NORD; ++u) vals[u] = 0.0;
      if (i < tile.nrows && n < tile.nb) {
        const long long k = a.first + a.stride * j;
        const double rf = a.rowv ? a.rowv[k - 1] : (double)k;
        const double cf = a.colv ? a.colv[n - 1] : ((double)n + a.gamma) * a.scale;
        const double z = rf * cf;
        if (NORD == 1) {
          vals[0] = jn(a.orders[0], z, a.jtab[a.orders[0]]);
        } else if (a.orders_identity) {
          // universe {0, 1, ..., n-1}: one Miller sweep of NORD orders, static indices
          jn_all<NORD>(a.omax, z, a.jtab, vals);
        } else {
          // any universe inside a window of kMaxOrd orders [omin, omin + kMaxOrd)
          double all[kMaxOrd];
          jn_window<kMaxOrd>(a.omin, a.omax, z, a.jtab, all);
#pragma unroll
          for (int u = 0; u < NORD; ++u)
            if (u < a.n_orders) {
              double v = 0.0;
#pragma unroll
              for (int o = 0; o < kMaxOrd; ++o)
                if (o == a.orders[u] - a.omin) v = all[o];
              vals[u] = v;
            }
        }
      }
#pragma unroll
      for (int u = 0; u < NORD; ++u) {
        const int pu = split ? ((u & 1) ? PE + (u >> 1) : (u >> 1)) : u;
        As[i * KA + pu * NK + q] = vals[u];
      }
    }
    // ---- weighted coefficient tile: Bs[u*NK + q][c] = w_c[u] * x_c[n]
#pragma unroll
    for (int t = 0; t < NBE; ++t) {
      const int e = tid + t * kNearThreads;
      if (e >= NK * JT) break;
      const int q = e / JT, c = e % JT;
      const long long n = n0 + q;
      const ReqDesc* r = (c < nq && n < tile.nb) ? a.reqs + q0 + c : nullptr;
#pragma unroll
      for (int u = 0; u < NORD; ++u) {
        const int pu = split ? ((u & 1) ? PE + (u >> 1) : (u >> 1)) : u;
        Bs[(pu * NK + q) * JB + c] = r ? r->w[u] * xv[t] : 0.0;
      }
    }
    __syncthreads();
    // ---- DMMA: warp (wr, wc) owns row fragments wr*FR.. and column
    // fragments wc*FC..  Column fragment f of class 0 (even orders)
    // contracts only k-steps < KE, class 1 (odd) only >= KE.
    constexpr int KE = (PE * NK) / 4;     // k-steps of the even-order half
#pragma unroll
    for (int kk = 0; kk < K / 4; ++kk) {
      wmma::fragment<wmma::matrix_a, 8, 8, 4, double, wmma::row_major> fa[FR];
#pragma unroll
      for (int r = 0; r < FR; ++r) wmma::load_matrix_sync(fa[r], As + ((wr * FR + r) * 8) * KA + kk * 4, KA);
#pragma unroll
      for (int c = 0; c < FC; ++c) {
        const int f = wc * FC + c;
        const bool on = f < nfrag && (kk < KE ? f < fe || f >= fo : f >= fe);
        if (on) {
          wmma::fragment<wmma::matrix_b, 8, 8, 4, double, wmma::row_major> fb;
          wmma::load_matrix_sync(fb, Bs + (kk * 4) * JB + f * 8, JB);
#pragma unroll
          for (int r = 0; r < FR; ++r) wmma::mma_sync(acc[r][c], fa[r], fb, acc[r][c]);
        }
      }
    }
    __syncthreads();
  }
  // ---- epilogue: reduce request columns into vectors with post factors
#pragma unroll
  for (int r = 0; r < FR; ++r)
#pragma unroll
    for (int c = 0; c < FC; ++c)
      wmma::store_matrix_sync(Cs + ((wr * FR + r) * 8) * JB + (wc * FC + c) * 8, acc[r][c], JB, wmma::mem_row_major);
  __syncthreads();
  const int v0 = a.grp_v0[g], v1 = a.grp_v0[g + 1];
  const int nv = v1 - v0;
  for (int e = tid; e < kRT * nv; e += kNearThreads) {
    const int i = e % kRT, vl = e / kRT;
    if (i >= tile.nrows) continue;
    const int vec = v0 + vl;
    const long long j = tile.j0 + i;
    const long long k = a.first + a.stride * j;
    double s = 0.0;
    for (int idx = a.vstart[vec]; idx < a.vstart[vec + 1]; ++idx) {
      const int c = a.vcol[idx];
      const ReqDesc* r = a.reqs + q0 + c;
      double p = Cs[i * JB + c];
      if (r->pr) p *= ipow((double)k / a.Ld, r->pr);
      if (r->post_e && r->pe) p *= ipow(r->post_e[j], r->pe);
      s += p;
    }
    if (tile.part >= 0) {
      a.part[tile.part * a.part_stride + (long long)vec * kRT + i] = s;
    } else {
      double* dst = a.F + (long long)vec * a.ldf + j;
      s = a.overwrite ? s : *dst + s;
      *dst = s;
      if (!isfinite(s)) *a.nf = 1;
    }
  }
}

// F[v][j] += Fn[v][j]
__global__ void add_rows_kernel(double* F, long long ldf, const double* Fn, long long ldn, int n_vec,
                                long long n, int* nf) {
  const long long tot = (long long)n_vec * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
    const long long v = e / n, j = e % n;
    const double s = F[v * ldf + j] + Fn[v * ldn + j];
    F[v * ldf + j] = s;
    if (!isfinite(s)) *nf = 1;
  }
}

cudaError_t launch_add_rows(double* F, long long ldf, const double* Fn, long long ldn, int n_vec, long long n,
                            int* nf, cudaStream_t st) {
  const long long tot = (long long)n_vec * n;
  long long b = (tot + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  if (b < 1) return cudaSuccess;
  note_launch(), add_rows_kernel<<<(unsigned)b, 256, 0, st>>>(F, ldf, Fn, ldn, n_vec, n, nf);
  return cudaGetLastError();
}

// Sum column-chunk partials of one row tile in chunk order.
__global__ void near_reduce_kernel(const NearRowTile* rt, const double* part, double* F,
                                   long long ldf, int n_vec, int overwrite, int* nf) {
  const NearRowTile t = rt[blockIdx.x];
  for (int e = threadIdx.x; e < kRT * n_vec; e += blockDim.x) {
    const int i = e % kRT, v = e / kRT;
    if (i >= t.nrows) continue;
    double s = 0.0;
    for (int c = 0; c < t.nchunks; ++c)
      s += part[(t.part + c) * (long long)n_vec * kRT + (long long)v * kRT + i];
    double* dst = F + (long long)v * ldf + t.j0 + i;
    s = overwrite ? s : *dst + s;
    *dst = s;
    if (!isfinite(s)) *nf = 1;
  }
}

template <int NORD, int JT>
static cudaError_t launch_near_t(const NearArgs& a, int n_tiles, int n_groups, cudaStream_t st) {
  constexpr int smem = NearCfg<NORD, JT>::SMEM;
  cudaError_t e = cudaFuncSetAttribute(near_kernel<NORD, JT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  note_launch(), near_kernel<NORD, JT><<<dim3(n_tiles, n_groups), kNearThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int JT>
static cudaError_t launch_near_j(const NearArgs& a, int n_tiles, int n_groups, cudaStream_t st) {
  if (a.n_orders <= 1) return launch_near_t<1, JT>(a, n_tiles, n_groups, st);
  if (a.n_orders <= 2) return launch_near_t<2, JT>(a, n_tiles, n_groups, st);
  if (a.n_orders <= 4) return launch_near_t<4, JT>(a, n_tiles, n_groups, st);
  if (a.n_orders <= 6) return launch_near_t<6, JT>(a, n_tiles, n_groups, st);
  if (a.n_orders <= 8) return launch_near_t<8, JT>(a, n_tiles, n_groups, st);
  if (a.n_orders <= 12) return launch_near_t<12, JT>(a, n_tiles, n_groups, st);
  return launch_near_t<16, JT>(a, n_tiles, n_groups, st);
}

cudaError_t launch_near(const NearArgs& a, int n_tiles, int n_groups, int max_cols, cudaStream_t st) {
  if (n_tiles == 0 || n_groups == 0) return cudaSuccess;
  if (max_cols <= 64) return launch_near_j<64>(a, n_tiles, n_groups, st);
  return launch_near_j<128>(a, n_tiles, n_groups, st);
}

cudaError_t launch_near_reduce(const NearRowTile* rt, int n_rt, const double* part, double* F,
                               long long ldf, int n_vec, int overwrite, int* nf, cudaStream_t st) {
  if (n_rt == 0) return cudaSuccess;
  note_launch(), near_reduce_kernel<<<n_rt, 256, 0, st>>>(rt, part, F, ldf, n_vec, overwrite, nf);
  return cudaGetLastError();
}

}  // namespace fhtb
