/* fhtb200.h -- C ABI of libfhtb200.so, the B200 (sm_100a, fp64) engine behind
 * the fasthankel-compatible Python package paper_1501_01652_b200.
 *
 * The reference (fasthankel, pure Python/NumPy) has no FFI of its own: its
 * "operator API" is the Python function surface (__init__.py:44-85).  Each
 * entry point below replaces the N-length numerical core of one reference
 * function; the cited file:line is the reference code it stands in for.
 * All array arguments are DEVICE pointers (fp64, row-major, batch-leading);
 * `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 * asynchronous on `stream` unless stated otherwise.  Return value: FHTB_OK
 * or an FHTB_E* code; fhtb_last_error() gives a thread-local message.
 */
#ifndef FHTB200_H
#define FHTB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FHTB_OK 0
#define FHTB_EINVAL 1      /* bad argument            -> Python ValueError   */
#define FHTB_ECUDA 2       /* CUDA launch/runtime     -> Python RuntimeError */
#define FHTB_ENONFINITE 3  /* non-finite result       -> Python RuntimeError */
#define FHTB_ECONVERGE 4   /* Newton did not converge -> Python RuntimeError */

#define FHTB_DCT1 0
#define FHTB_DST1 1

/* apply flags */
#define FHTB_FAR 1         /* asymptotic blocks (DCT-I/DST-I far field)     */
#define FHTB_NEAR 2        /* pointwise border segments (near field)        */
#define FHTB_OVERWRITE 4   /* direct: F = result instead of F += result     */

int fhtb_abi_version(void);
const char* fhtb_last_error(void);
/* Non-finite outputs (reference contract: cli.py:128-130, exit code 3 when the
 * output holds a non-finite value).  Every kernel that writes final values to
 * F (far/chirp reductions, near-field reduction and add) sets a per-device
 * flag when it writes inf or NaN.  fhtb_nonfinite_check synchronises `stream`
 * on the current device, clears the flag and returns FHTB_ENONFINITE if it
 * was set since the previous check (FHTB_OK otherwise). */
int fhtb_nonfinite_check(void* stream);
/* Cumulative number of CUDA kernels this library has launched (all devices). */
int64_t fhtb_launch_count(void);
/* Prepare per-device tables (twiddles, Bessel order constants) on the
 * current device.  Idempotent; synchronous. */
int fhtb_init(void);
/* Tunables: "far_chunk_bytes" (two-pass intermediate budget), ...;
 * "kernel_timing" 1/0 turns on CUDA-event timing of every apply launch;
 * "serial" 1/0 issues every launch on the caller's stream in plan order (no
 * chunk pipeline, near field after the far field) so that those per-launch
 * times are exclusive.  Results are bit-identical either way. */
int fhtb_set_option(const char* key, int64_t value);
/* Kernel-family timing (no reference counterpart; bench.py roofline):
 * with "kernel_timing" on, every far/near launch of fhtb_apply* is bracketed
 * by CUDA events on its own stream and tagged with the algorithmic bytes it
 * moves.  fhtb_kernel_times synchronises on the recorded events, writes the
 * per-family sums (ms of event time, bytes, nominal FFT flops at 5 n log2 n
 * per executed n-point transform, launches; arrays of n_fam) and
 * clears the record.  Family i is named by fhtb_kernel_family_name(i). */
int32_t fhtb_kernel_families(void);
const char* fhtb_kernel_family_name(int32_t i);
int fhtb_kernel_times(double* ms, double* bytes, double* flops, int64_t* launches, int32_t n_fam);

/* ---------------------------------------------------------------- L1 --- */
/* Planning statistics of coefficient rows C[v][0..n) on the device, returned
 * to the host (synchronises `stream`): out_host[3v] = sum |c|, [3v+1] = max
 * |b[i]| over i >= n_split with c[i] != 0 (b: nb device values, may be null),
 * [3v+2] = 1 if any such i.  Replaces the numpy scans of
 * fourier_bessel.py:208-225 and dht.py:140-157 (norm1, b_max, nonzero). */
int fhtb_coef_stats(const double* C, int64_t ldc, int32_t n_vec, int64_t n, int64_t n_split, const double* b,
                    int64_t nb, double* out_host, void* stream);
/* out[v][i] = alpha * a[v][i] * w[i] (w may be null), and max_i |alpha a[i] - b[i]| returned to
 * the host: the diagonal scalings and the residual of dht_self_inverse_residual (dht.py:179-194). */
int fhtb_mul_rows(double* out, int64_t ldo, const double* a, int64_t lda, const double* w, double alpha, int64_t n,
                  int32_t n_vec, void* stream);
int fhtb_max_abs_diff(const double* a, double alpha, const double* b, int64_t n, double* out_host, void* stream);
/* F[v][0..n) = 0 for v < n_vec (stream-ordered memset of result rows). */
int fhtb_zero_rows(double* F, int64_t ldf, int32_t n_vec, int64_t n, void* stream);
/* out[i] = J_nu(z[i]); replaces bessel.py:232-260 (bessel_j, array path). */
int fhtb_bessel_j(int nu, const double* z, int64_t n, double* out, void* stream);
/* out[o*n + i] = J_o(z[i]) for o <= nu_max (one Miller sweep). */
int fhtb_bessel_j_multi(int nu_max, const double* z, int64_t n, double* out, void* stream);
/* replaces bessel.py:72-91 (hankel_asy_eval) */
int fhtb_hankel_asy_eval(int nu, int m_terms, const double* z, int64_t n, double* out, void* stream);
/* replaces bessel.py:133-146 (taylor_eval) */
int fhtb_taylor_eval(int nu, int n_terms, const double* z, int64_t n, double* out, void* stream);
/* First `count` roots of J0 and b_n = j_{0,n} - (n-1/4)pi; replaces
 * bessel.py:295-321.  Synchronous: *resid_max (host) = max |J0(root)|;
 * returns FHTB_ECONVERGE when a root's residual exceeds 1e-13
 * (bessel.py:313-317) -- or, for roots beyond ~2e6 where the rounding of
 * the root itself leaves |J0| above 1e-13, 2 ulp(root) |J1(root)|. */
int fhtb_roots_j0(int64_t count, double* roots, double* perturb, double* resid_max, void* stream);
/* Batched complex FFT (interleaved re/im), n = 2^k <= 2048, X_k = sum x_n e^{sign 2 pi i nk/n}.
 * Utility behind the FFT-core tests. */
int fhtb_fft(int64_t n, int sign, const double* in, double* out, int64_t batch, void* stream);
/* DCT-I / DST-I of `batch` rows of length `length`; replaces trig.py:80-92
 * (apply) for real rows.  Workspace from fhtb_trig_workspace. */
size_t fhtb_trig_workspace(int kind, int64_t length, int64_t batch);
int fhtb_trig_apply(int kind, int64_t length, const double* v, int64_t batch, double* out,
                    void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------ L2 engine ----- */
/* A grid = the partitioned Schlomilch matrix of one (L, gamma, eps, order
 * universe) problem: schlomilch.py:139-170 (build_partition) plus the
 * _AsyWork state of schlomilch.py:244-270, kept on the device. */
typedef struct fhtb_grid fhtb_grid;

typedef struct fhtb_grid_desc {
  int64_t L;                 /* grid length N (or 4N+3 for the DHT)          */
  double gamma;              /* frequency shift: omega_n = (n+gamma) pi      */
  int32_t m_terms;           /* M: 2M asymptotic terms per block             */
  int32_t n_blocks;          /* blocks[4*b..]: r0, r1, c0, c1 (1-based, half-open) */
  const int64_t* blocks;     /* host */
  int32_t n_segments;        /* segments[3*s..]: r0, r1, c_end               */
  const int64_t* segments;   /* host */
  int64_t row_first;         /* output j <-> grid row k = row_first + row_stride*j */
  int64_t row_stride;
  int64_t n_out;
  int64_t n_data_cols;       /* columns n > n_data_cols hold zero coefficients */
  int32_t n_orders;          /* order universe (schlomilch.py:422-431)       */
  const int32_t* orders;     /* host */
} fhtb_grid_desc;

/* One (order_weights, coefficients) request (schlomilch.py:436-468) with the
 * fused diagonal pre/post multipliers of fourier_bessel.py:215-242 and
 * dht.py:151-174:  x_n = C[vec][n-1] * pre_a[n-1]^pre_a_pow * pre_b[n-1]^pre_b_pow
 * for n >= col_lo;  F[vec][j] += (k/L)^post_r_pow * post_e[j]^post_e_pow * y_k. */
typedef struct fhtb_request {
  int32_t vec;
  int32_t n_terms;           /* weighted orders */
  const int32_t* orders;     /* host, each in the grid universe */
  const double* weights;     /* host */
  int64_t col_lo;
  const double* pre_a;       /* device or NULL */
  int32_t pre_a_pow;
  const double* pre_b;
  int32_t pre_b_pow;
  int32_t post_r_pow;
  const double* post_e;      /* device or NULL, indexed by output j */
  int32_t post_e_pow;
} fhtb_request;

int fhtb_grid_create(const fhtb_grid_desc* desc, fhtb_grid** out);
void fhtb_grid_destroy(fhtb_grid* g);
/* Algorithmic DRAM bytes of one request's far-field application in the
 * formulation this grid executes (pruned side blocks included), following
 * the SURVEY 8(d) byte model: intermediates written and read, coefficient
 * reads, partial rows and output. */
double fhtb_grid_far_model_bytes(const fhtb_grid* g);
size_t fhtb_apply_workspace(const fhtb_grid* g, int32_t n_req, int32_t n_vec, int32_t flags);
/* F[vec][j] += Schlomilch application of each request (far and/or near
 * field per flags).  F must be initialised by the caller (zeros for a plain
 * evaluation).  Deterministic reduction order. */
int fhtb_apply(const fhtb_grid* g, const fhtb_request* reqs, int32_t n_req, const double* C,
               int64_t ldc, int32_t n_vec, double* F, int64_t ldf, int32_t flags, void* ws,
               size_t ws_bytes, void* stream);
/* One shard of fhtb_apply for splitting a single application over several
 * devices: shard s of n computes the asymptotic term pairs
 * [M s/n, M (s+1)/n) of every far-field unit and the near-field tiles
 * t = s (mod n); the n partial results sum (e.g. ncclAllReduce) to the
 * fhtb_apply result up to rounding.  F is accumulated into as fhtb_apply;
 * same workspace size.  fhtb_apply == fhtb_apply_part(..., 0, 1, ...). */
int fhtb_apply_part(const fhtb_grid* g, const fhtb_request* reqs, int32_t n_req, const double* C,
                    int64_t ldc, int32_t n_vec, double* F, int64_t ldf, int32_t flags, int32_t shard,
                    int32_t n_shards, void* ws, size_t ws_bytes, void* stream);

/* Distributed four-step (exchange mode) -- SURVEY 8(e): one application
 * split over `world` ranks where the full (unpruned) far-field blocks of a
 * power-of-two grid run as a distributed FFT: rank r computes pass 1 for its
 * column slab n1 in [r L1/world, (r+1) L1/world) into `send`, laid out as
 * world equal chunks (one per destination rank: the rows k2 of the column
 * pairs {c, L2-c} that rank owns); the library then calls
 * exchange(user, round, bytes_per_peer), which must perform the all-to-all
 * (recv chunk s <- chunk r of rank s's send, e.g. ncclAllToAll or
 * dist.all_to_all_single) ordered on `stream`; pass 2 of rank r's column pairs
 * reads `recv`.  Pruned side blocks and near-field tiles are split as in
 * fhtb_apply_part; the world partial F sum to the fhtb_apply result up to
 * rounding.  xbytes = size of send (== size of recv), a multiple of
 * fhtb_apply_x_unit_bytes (units per exchange round); workspace from
 * fhtb_apply_x_workspace.  Grids without full two-pass blocks (one-pass,
 * chirp) or with L1 not divisible into 16-column slabs never call
 * exchange (plain fhtb_apply_part split); unit_bytes is then 0. */
typedef int (*fhtb_exchange_fn)(void* user, int32_t round, size_t bytes_per_peer);
size_t fhtb_apply_x_unit_bytes(const fhtb_grid* g, int32_t world);
size_t fhtb_apply_x_workspace(const fhtb_grid* g, int32_t n_req, int32_t n_vec, int32_t flags, int32_t world,
                              size_t xbytes);
int fhtb_apply_x(const fhtb_grid* g, const fhtb_request* reqs, int32_t n_req, const double* C, int64_t ldc,
                 int32_t n_vec, double* F, int64_t ldf, int32_t flags, int32_t rank, int32_t world, void* send,
                 void* recv, size_t xbytes, fhtb_exchange_fn exchange, void* user, void* ws, size_t ws_bytes,
                 void* stream);

/* fhtb_apply(FAR|NEAR) from HOST memory to HOST memory: the end-to-end
 * form of schlomilch.py:389-396 / :436-468 for a caller holding host arrays
 * (the reference's own calling convention, numpy in and out).  C_host
 * (n_vec rows of n_data_cols, leading dimension ldc_host) is copied in
 * n_groups vector groups on a copy stream; the far field of group g starts
 * as soon as its rows have landed, the near field of the whole batch runs on
 * its own stream once all rows are in, and the finished rows of group g are
 * copied out to F_host (n_vec rows of n_out, overwritten) while later groups
 * compute.  Pinned host memory gives the overlap; pageable memory is
 * accepted (copies then serialise).  The result equals fhtb_apply on device
 * copies of C, F = 0, bit for bit (reductions are independent of the
 * grouping).  Device buffers are carved from ws
 * (fhtb_apply_host_workspace).  Asynchronous on `stream`: F_host is valid
 * after the stream synchronises. */
size_t fhtb_apply_host_workspace(const fhtb_grid* g, int32_t n_req, int32_t n_vec, int32_t flags);
int fhtb_apply_host(const fhtb_grid* g, const fhtb_request* reqs, int32_t n_req, const double* C_host,
                    int64_t ldc_host, int32_t n_vec, double* F_host, int64_t ldf_host, int32_t flags,
                    int32_t n_groups, void* ws, size_t ws_bytes, void* stream);

/* Direct sums with rank-1 arguments z = row_val[k] * col_val[n] over a full
 * n_rows x n_cols rectangle: fourier_bessel.py:148-172 (low columns),
 * dht.py:82-94 (direct rows), and the O(N^2) oracles schlomilch.py:223-229,
 * fourier_bessel.py:292-309.  Requests use the same structure (orders must
 * be in the given universe; col_lo, pre/post as above, post_r_pow uses
 * k/r_scale). */
typedef struct fhtb_direct_desc {
  int64_t n_rows;
  const double* row_val;     /* device */
  int64_t n_cols;
  const double* col_val;     /* device */
  int64_t n_data_cols;
  double r_scale;
  int32_t n_orders;
  const int32_t* orders;     /* host */
} fhtb_direct_desc;

size_t fhtb_direct_workspace(const fhtb_direct_desc* d, int32_t n_req, int32_t n_vec);
int fhtb_direct_apply(const fhtb_direct_desc* d, const fhtb_request* reqs, int32_t n_req,
                      const double* C, int64_t ldc, int32_t n_vec, double* F, int64_t ldf,
                      int32_t flags, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FHTB200_H */
