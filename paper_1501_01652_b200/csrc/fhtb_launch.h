// fhtb_launch.h -- kernel argument blocks and launch entry points
// (implemented in fhtb_*.cu, called from the host runtime fhtb_host.cpp).
#pragma once
#include <cuda_runtime.h>

#include "fhtb_types.h"

namespace fhtb {

// Cumulative count of kernels launched by the library (fhtb_launch_count).
void note_launch();

struct JOrder;

struct NearRowTile {
  long long j0;
  int nrows;
  int nchunks;
  long long part;
};

struct NearArgs {
  const NearTile* tiles;
  long long first, stride;      // output index j -> grid row k = first + stride*j
  const double* rowv;           // null: row factor k; else rowv[k-1]
  const double* colv;           // null: column factor (n+gamma)*scale; else colv[n-1]
  double gamma, scale, Ld;
  int n_orders, omax;
  int orders_identity;          // universe == {0, 1, ..., n_orders-1}
  int omin;                     // smallest universe order (window [omin, omin + kMaxOrd) holds them all)
  int orders[kMaxOrd];
  const JOrder* jtab;           // indexed by order
  const ReqDesc* reqs;
  const int* grp_q0;            // requests of group g: [grp_q0[g], grp_q0[g+1])
  const int* grp_v0;            // vectors of group g
  const int2* grp_cls;          // per group: end columns of the even / odd order classes (or null)
  const int* vstart;            // columns of vector v: vcol[vstart[v] .. vstart[v+1]) (group-local)
  const int* vcol;
  const double* C;
  long long ldc, n_data_cols;
  double* F;
  long long ldf;
  double* part;
  long long part_stride;         // n_vec * 64 doubles per partial slot
  int overwrite;
  int shard, n_shards;          // tiles t with t % n_shards == shard are computed
  int* nf;                      // device flag: a non-finite value was written to F
};

struct FarArgs {
  long long L;                  // grid length
  int L1, L2;                   // FFT split: Q = L1 * L2 (2L in direct mode)
  int M;                        // term pairs (direct) / 2M terms (chirp)
  int logQ;
  double gamma, Ld, pi_over_L;
  long long first, stride;      // output rows
  long long n_out;
  long long n_data_cols;
  const UnitDesc* units;
  const ReqDesc* reqs;
  const BlockDesc* blocks;
  const int2* vranges;          // unit ranges per grid.y
  int u0;                       // first unit of the chunk (G is indexed by unit - u0)
  const double* C;
  long long ldc;
  double* F;
  long long ldf;
  double2* G;                   // intermediate
  double* part;                 // chirp mode: per-unit partial rows
  long long part_stride;
  const double2* tw;            // twiddle pool: table for N at offset N-2
  const double2* qlo;           // four-step twiddles e^{2 pi i m / Q}, m = hi*4096 + lo
  const double2* qhi;
  int qbits;                    // number of lo bits (<= 12)
  const double2* cs_tab;        // (cos, sin)(-gamma k pi / L) for k = 1..L (null if gamma == 0)
  const double* w0_tab;         // omega_n^{-1/2}, n = 1..L (direct mode)
  const double* iw_tab;         // 1/omega_n
  int p0, p1;                   // pair range of this shard (direct: pairs p; chirp: terms 2p0 .. 2p1-1)
  // distributed four-step (exchange mode, xw > 0 ranks): pass 1 covers the
  // column slab n1 in [xn1, xn1 + L1/xw) and writes X[peer][unit][pair][j][n1 - xn1];
  // pass 2 covers the column pairs c in [xc0, xc0 + gridDim.x) and reads the
  // received X[src][unit][pair][j][n1 local]; xrow[k2] = (owner, j).
  int xw, xlog, xrows, xc0;
  long long xn1, xchunk;
  const int2* xrow;
  const double2* xin;
  int* nf;                      // device flag: a non-finite value was written to F
  int rs;                       // fused narrow rows: row stride of P = G[unit][A|B][rs][L1]
};
cudaError_t launch_col_tables(double* w0, double* iw, long long L, double gamma, cudaStream_t st);

extern int g_far_variant;         // tuning knob for the hot far-field sizes
extern int g_far_bulk;            // narrow-column tables by bulk copy into shared memory
extern int g_far_hp;              // pass 2 half pairing
extern int g_chirp_variant;       // tuning knob for the chirp-z passes

cudaError_t launch_near(const NearArgs& a, int n_tiles, int n_groups, int max_cols, cudaStream_t st);
cudaError_t launch_add_rows(double* F, long long ldf, const double* Fn, long long ldn, int n_vec, long long n,
                            int* nf, cudaStream_t st);
constexpr int kNearMaxCols = 128;   // request columns per near-field CTA (largest tile)
cudaError_t launch_near_reduce(const NearRowTile* rt, int n_rt, const double* part, double* F,
                               long long ldf, int n_vec, int overwrite, int* nf, cudaStream_t st);
constexpr int kNearRT = 64;

// direct mode (2L power of two, unit-stride rows)
cudaError_t launch_far_onepass(const FarArgs& a, int logN1, int n_units, cudaStream_t st);
cudaError_t launch_far_pass1(const FarArgs& a, int logN2, int n_units, cudaStream_t st);
cudaError_t launch_far_pass2(const FarArgs& a, int logN1, int n_units, cudaStream_t st);
// exchange mode: pass 2 over n_pairs column pairs starting at a.xc0
cudaError_t launch_far_pass2x_range(const FarArgs& a, int logN1, int n_pairs, int n_units, cudaStream_t st);
cudaError_t launch_far_reduce(const FarArgs& a, int n_units, cudaStream_t st);
cudaError_t launch_far_colgen(const FarArgs& a, int logN1, int n_units, cudaStream_t st);
cudaError_t launch_far_rowdot(const FarArgs& a, int n_units, int kbins, cudaStream_t st);
cudaError_t launch_far_rowsum(const FarArgs& a, int logN2, int form, int n_units, cudaStream_t st);
cudaError_t launch_far_rowsum_fin(const FarArgs& a, int n_units, cudaStream_t st);
cudaError_t launch_prefetch_rows(const FarArgs& a, int n_units, cudaStream_t st);
cudaError_t launch_cs_table(double2* cs, long long L, double gamma, double pi_over_L, cudaStream_t st);

// chirp mode (any grid length, strided output rows)
// hz: every unit's columns fit in the lower half of Q (half-zero first pass)
cudaError_t launch_chirp_pass1(const FarArgs& a, int logN2, int n_units, int hz, cudaStream_t st);
cudaError_t launch_chirp_pass2(const FarArgs& a, int logN1, int n_units, cudaStream_t st);
cudaError_t launch_chirp_pass3(const FarArgs& a, int logN2, int n_units, cudaStream_t st);
cudaError_t launch_chirp_reduce(const FarArgs& a, int n_units, cudaStream_t st);
cudaError_t launch_chirp_filter(double2* h, long long Q, long long Mn, long long J, long long s, long long L,
                                cudaStream_t st);
cudaError_t launch_plain_fft(const FarArgs& a, int logN1, int logN2, const double2* in, double2* tmp,
                             double2* out, int transposed, cudaStream_t st);
cudaError_t launch_trig(int kind, int logQ, long long n, long long L, long long k0, long long n0, const double* v,
                        double* out, long long batch, const double2* H, const double2* tw, cudaStream_t st);
// trig lengths with Q > 8192: elementwise stages around plain_fft
cudaError_t launch_trig_pre(const double* x, long long n, long long L, long long k0, long long Q, double2* A,
                            cudaStream_t st);
cudaError_t launch_trig_mid(const double2* A2, const double2* H, long long Q, double2* A, cudaStream_t st);
cudaError_t launch_trig_post(int kind, const double2* A2, long long n, long long L, long long k0, long long n0,
                             long long Q, double* out, cudaStream_t st);

// utilities
cudaError_t launch_twiddles(double2* tw_pool, int max_log, cudaStream_t st);
cudaError_t launch_qtwiddles(double2* qlo, double2* qhi, int logQ, int qbits, int sign, cudaStream_t st);
cudaError_t launch_bessel_j(int nu, const JOrder& c, const double* z, long long n, double* out, cudaStream_t st);
cudaError_t launch_bessel_multi(int omax, const JOrder* tab, const double* z, long long n, double* out, cudaStream_t st);
cudaError_t launch_hankel_eval(int nu, int m_terms, const double* coef, const double* z, long long n,
                               double* out, cudaStream_t st);
cudaError_t launch_taylor_eval(int nu, int n_terms, double inv_fact, const double* z, long long n,
                               double* out, cudaStream_t st);
cudaError_t launch_coef_stats(const double* C, long long ldc, int n_vec, long long n, long long n_split,
                              const double* b, long long nb, double* out, cudaStream_t st);
cudaError_t launch_mul_rows(double* out, long long ldo, const double* a, long long lda, const double* w, double alpha,
                            long long n, int n_vec, cudaStream_t st);
cudaError_t launch_max_abs_diff(const double* a, double alpha, const double* b, long long n, unsigned long long* res,
                                cudaStream_t st);
cudaError_t launch_roots_j0(const JOrder* tab, long long count, double* roots, double* pert,
                            unsigned long long* resid_bits, cudaStream_t st);
cudaError_t launch_fft_batch(int logN, int sign, const double2* in, double2* out, long long batch,
                             const double2* tw_pool, cudaStream_t st);

}  // namespace fhtb
