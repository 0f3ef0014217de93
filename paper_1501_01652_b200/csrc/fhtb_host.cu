// fhtb_host.cu -- host runtime behind the C ABI (include/fhtb200.h).
//
// Owns the per-device tables (FFT twiddles, Bessel order constants), the
// grid objects (partition + far/near-field tables on the device) and the
// apply scheduler: request packing, far-field unit ordering and chunking,
// near-field tiling and vector grouping.  All scheduling decisions are
// deterministic functions of the arguments, so results are reproducible.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fhtb200.h"
#include "fhtb_bessel.cuh"
#include "fhtb_launch.h"

using namespace fhtb;

namespace fhtb {
static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace fhtb

namespace {

thread_local std::string g_err;
int64_t g_far_chunk_bytes = 2LL << 30;     // two-pass intermediate budget per chunk (2 GiB measured best: cfg2 step 77.65 -> 76.85 ms; 1.5 GiB 77.25, 3 GiB 79.3)
int64_t g_near_chunk_cols = 8192;          // near-field column chunk per tile (single-order grids)
int64_t g_near_chunk_cols_multi = 1024;    // ... multi-order universes
int g_far_prune = 1;                       // pruned side blocks (direct two-pass)
int g_near_split = 1;                      // near field: order-parity classes
int g_far_streams = 2;                     // far-field chunks in flight (direct two-pass)
int g_near_overlap = 1;                    // near field on its own stream beside the far field
int g_serial = 0;                          // diagnostics: every launch on the caller's stream, in order
int g_prune_rows = 11;                     // narrow-row blocks: rows below 2^g_prune_rows
int g_rowsum = 2;                          // narrow-row blocks: fully fused forms (dmode 3..5); 1: only blocks that would run both passes; 0: off
int g_rowsum_min_m = 4;                    // ... for blocks already pruned to row sums: only with at least this many pairs
int g_rowdot_bins = 1;                     // narrow-row blocks: at most this many pass-2 bins per column
int g_min_lc = 0;                          // narrow-column blocks: smallest column FFT 2^g_min_lc (0: 256 points from 8 pairs on, else 512)
int g_near_priority = 0;                   // near-field stream priority (see get_aux)
int g_far_prefetch = 1;                    // L2 prefetch of the coefficient rows before pass 1
int g_host_taper = 4;                      // fhtb_apply_host: inner/outer group size ratio

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CU(x)                                                                       \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) {                                                        \
      (void)cudaGetLastError(); /* clear a non-sticky error so later calls work */  \
      return fail(FHTB_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));     \
    }                                                                               \
  } while (0)

// ------------------------------------------------ kernel-family timing
// fhtb_set_option("kernel_timing", 1): CUDA events around every launch of the
// apply scheduler, recorded on the stream the kernel runs on, together with
// the algorithmic bytes the launch moves.  fhtb_kernel_times
// reads and resets the per-family sums (bench.py roofline.kernels[]).
enum KFam {
  kfPass1, kfPass2, kfNarrow, kfRowdot, kfReduce, kfOnepass, kfNear, kfNearReduce,
  kfChirp1, kfChirp2, kfChirp3, kfChirpReduce, kfOther, kfRowsum, kfRowsumFin, kNumFam
};
const char* const kFamNames[kNumFam] = {
  "far_pass1", "far_pass2", "far_narrow_cols", "far_rowdot", "far_reduce", "far_onepass", "near",
  "near_reduce", "chirp_pass1", "chirp_pass2", "chirp_pass3", "chirp_reduce", "other", "far_rowsum",
  "far_rowsum_fin"};
struct KtRec {
  int fam, dev;
  cudaEvent_t a, b;
  double bytes, flops;
};
thread_local double t_kt_flops = 0.0;     // nominal FFT flops of the next KT launch (5 n log2 n per transform)
std::mutex g_kt_mu;
int g_kt_on = 0;
std::vector<KtRec> g_kt;
std::map<int, std::vector<cudaEvent_t>> g_kt_pool;

cudaEvent_t kt_event(int dev) {
  std::lock_guard<std::mutex> lk(g_kt_mu);
  auto& p = g_kt_pool[dev];
  if (!p.empty()) {
    cudaEvent_t e = p.back();
    p.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  return e;
}

struct KtScope {
  int fam, dev = 0;
  cudaStream_t st;
  double bytes, flops;
  cudaEvent_t a = nullptr;
  KtScope(int f, cudaStream_t s, double by) : fam(f), st(s), bytes(by), flops(t_kt_flops) {
    t_kt_flops = 0.0;
    if (!g_kt_on) return;
    cudaGetDevice(&dev);
    a = kt_event(dev);
    if (a && cudaEventRecord(a, st) != cudaSuccess) a = nullptr;
  }
  ~KtScope() {
    if (!a) return;
    cudaEvent_t b = kt_event(dev);
    if (!b || cudaEventRecord(b, st) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(g_kt_mu);
    g_kt.push_back(KtRec{fam, dev, a, b, bytes, flops});
  }
};

#define KT(fam, st, bytes, call)         \
  do {                                   \
    KtScope kt_((fam), (st), (bytes));   \
    CU(call);                            \
  } while (0)

// ------------------------------------------------------------ host math
// a_0..a_{count-1}(nu) by the ratio recurrence (bessel.py:45-58)
std::vector<double> asy_coeffs(int nu, int count) {
  std::vector<double> a(count);
  a[0] = 1.0;
  const double q = 4.0 * nu * nu;
  for (int m = 1; m < count; ++m) {
    const double t = (double)(2 * m - 1);
    a[m] = a[m - 1] * (q - t * t) / (8.0 * m);
  }
  return a;
}

// s_{nu,M}(eps), four fixed-point iterations (bessel.py:109-130)
double asy_cutoff(int nu, int mt, double eps) {
  std::vector<double> a = asy_coeffs(nu, 2 * mt + 2);
  const double a0 = std::fabs(a[2 * mt]), a1 = std::fabs(a[2 * mt + 1]);
  const double c = std::sqrt(2.0) / (std::sqrt(M_PI) * eps);
  double s = 1.0;
  for (int i = 0; i < 4; ++i) s = std::pow(c * (a0 + a1 / s), 1.0 / (2 * mt + 0.5));
  return s;
}

// t_{nu,T}(eps) (bessel.py:149-168)
double taylor_cutoff(int nu, int nt, double eps) {
  const double e = 2 * nt + nu;
  const double lt = (e * std::log(2.0) + std::lgamma(nt + nu + 1.0) + std::lgamma(nt + 1.0) + std::log(eps)) / e;
  return std::exp(lt);
}

JOrder make_jorder(int nu) {
  JOrder c;
  const double u = std::ldexp(1.0, -52);
  c.tlo = taylor_cutoff(nu, kTaylorTerms, u);
  c.shi = asy_cutoff(nu, kAsyPairs, u);
  c.inv_fact = 1.0 / std::tgamma(nu + 1.0);
  const double r = std::sqrt(0.5);
  switch ((2 * nu + 1) % 8) {
    case 1: c.cphi = r; c.sphi = r; break;
    case 3: c.cphi = -r; c.sphi = r; break;
    case 5: c.cphi = -r; c.sphi = -r; break;
    default: c.cphi = r; c.sphi = -r; break;
  }
  std::vector<double> a = asy_coeffs(nu, 2 * kAsyPairs);
  for (int m = 0; m < kAsyPairs; ++m) {
    const double sg = (m & 1) ? -1.0 : 1.0;
    c.ae[m] = sg * a[2 * m];
    c.ao[m] = sg * a[2 * m + 1];
  }
  return c;
}

// ------------------------------------------------------- device context
constexpr int kTwMaxLog = 13;

struct DevCtx {
  double2* tw = nullptr;           // twiddle pool, N = 2..8192
  JOrder* jtab = nullptr;          // orders 0..kMaxOrder
  unsigned long long* scratch = nullptr;
  int* nf = nullptr;               // set to 1 by any reduction that writes a non-finite output
  double* stats = nullptr;         // fhtb_coef_stats output rows (grown on demand)
  size_t stats_cap = 0;
  std::map<int, std::pair<double2*, double2*>> qtab;   // four-step twiddles per log2 Q
};

constexpr int kQBits = 12;
inline cudaStream_t S(void* s) { return (cudaStream_t)s; }

std::mutex g_mu;
std::mutex g_scratch_mu;            // serialises the users of DevCtx::scratch
std::map<int, DevCtx> g_ctx;

// Two auxiliary streams + events per (device, caller stream): far-field
// chunks are computed on them two at a time and reduced in chunk order on the
// caller's stream.
struct AuxStreams {
  cudaStream_t cs[3];                   // two far-field chunk streams, one near-field stream
  cudaEvent_t start, done[2], red[2], nstart, ndone;
};
std::map<std::pair<int, cudaStream_t>, AuxStreams> g_aux;

int get_aux(cudaStream_t caller, AuxStreams** out) {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, caller);
  auto it = g_aux.find(key);
  if (it == g_aux.end()) {
    AuxStreams a;
    for (int i = 0; i < 2; ++i) {
      CU(cudaEventCreateWithFlags(&a.done[i], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&a.red[i], cudaEventDisableTiming));
    }
    for (int i = 0; i < 2; ++i) CU(cudaStreamCreateWithFlags(&a.cs[i], cudaStreamNonBlocking));
    // near-field stream priority (near_priority: 0 = default, 1 = highest, -1 = lowest)
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    const int prio = g_near_priority > 0 ? hi : (g_near_priority < 0 ? lo : 0);
    CU(cudaStreamCreateWithPriority(&a.cs[2], cudaStreamNonBlocking, prio));
    CU(cudaEventCreateWithFlags(&a.start, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&a.nstart, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&a.ndone, cudaEventDisableTiming));
    it = g_aux.emplace(key, a).first;
  }
  *out = &it->second;
  return FHTB_OK;
}

int get_ctx(DevCtx** out) {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_ctx.find(dev);
  if (it != g_ctx.end()) {
    *out = &it->second;
    return FHTB_OK;
  }
  DevCtx c;
  const long long ntw = (1LL << (kTwMaxLog + 1)) - 2;
  CU(cudaMalloc(&c.tw, ntw * sizeof(double2)));
  CU(launch_twiddles(c.tw, kTwMaxLog, 0));
  std::vector<JOrder> tab(kMaxOrder + 1);
  for (int o = 0; o <= kMaxOrder; ++o) tab[o] = make_jorder(o);
  CU(cudaMalloc(&c.jtab, tab.size() * sizeof(JOrder)));
  CU(cudaMemcpy(c.jtab, tab.data(), tab.size() * sizeof(JOrder), cudaMemcpyHostToDevice));
  CU(cudaMalloc(&c.scratch, 64));
  CU(cudaMalloc(&c.nf, sizeof(int)));
  CU(cudaMemset(c.nf, 0, sizeof(int)));
  CU(cudaDeviceSynchronize());
  g_ctx[dev] = c;
  *out = &g_ctx[dev];
  return FHTB_OK;
}

// Per-call tables (requests, units, near-field groups) go to the device through a
// ring of pinned staging slots: a cudaMemcpyAsync from pageable memory first
// synchronises the stream, which stalls the host behind the previous
// application and breaks the group pipeline of fhtb_apply_host.
constexpr size_t kStageSlotBytes = 512 << 10;
constexpr int kStageSlots = 32;
struct StageRing {
  char* base = nullptr;
  cudaEvent_t ev[kStageSlots];
  bool used[kStageSlots];
  int next = 0;
};
std::map<int, StageRing> g_stage;

cudaError_t h2d_tables(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return cudaSuccess;
  if (bytes > kStageSlotBytes) return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_mu);
  StageRing& r = g_stage[dev];
  if (!r.base) {
    e = cudaMallocHost((void**)&r.base, kStageSlotBytes * kStageSlots);
    if (e != cudaSuccess) { r.base = nullptr; return e; }
    for (int i = 0; i < kStageSlots; ++i) {
      e = cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
      r.used[i] = false;
    }
  }
  const int i = r.next;
  r.next = (r.next + 1) % kStageSlots;
  if (r.used[i]) {
    e = cudaEventSynchronize(r.ev[i]);         // the copy that last used this slot (long done)
    if (e != cudaSuccess) return e;
  }
  char* slot = r.base + (size_t)i * kStageSlotBytes;
  std::memcpy(slot, src, bytes);
  e = cudaMemcpyAsync(dst, slot, bytes, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  r.used[i] = true;
  return cudaEventRecord(r.ev[i], st);
}

// e^{+2 pi i m / Q} = qlo[m & (2^b - 1)] * qhi[m >> b],  b = min(12, log2 Q)
int get_qtab(DevCtx* c, int logQ, double2** lo, double2** hi, int* bits) {
  std::lock_guard<std::mutex> lk(g_mu);
  const int b = std::min(kQBits, logQ);
  auto it = c->qtab.find(logQ);
  if (it == c->qtab.end()) {
    double2 *ql = nullptr, *qh = nullptr;
    const long long nlo = 1LL << b, nhi = (1LL << logQ) >> b;
    CU(cudaMalloc(&ql, nlo * sizeof(double2)));
    CU(cudaMalloc(&qh, nhi * sizeof(double2)));
    CU(launch_qtwiddles(ql, qh, logQ, b, 1, 0));
    CU(cudaDeviceSynchronize());
    it = c->qtab.emplace(logQ, std::make_pair(ql, qh)).first;
  }
  *lo = it->second.first;
  *hi = it->second.second;
  *bits = b;
  return FHTB_OK;
}


size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Bump allocator over a caller-provided workspace.
struct Carve {
  char* base;
  size_t cap, off = 0;
  bool ok = true;
  template <class T> T* take(size_t n) {
    size_t b = align_up(n * sizeof(T));
    if (off + b > cap) { ok = false; return nullptr; }
    T* p = (T*)(base + off);
    off += b;
    return p;
  }
};

bool is_pow2(long long x) { return x > 0 && (x & (x - 1)) == 0; }
int ilog2ll(long long x) { int l = 0; while ((1LL << l) < x) ++l; return l; }

// Request packing (schlomilch.py:280-299 with the order combination folded
// into per-term scalars; see fhtb_types.h).
int pack_requests(const fhtb_request* reqs, int n_req, int M, const std::vector<int>& universe,
                  long long n_data_cols, std::vector<ReqDesc>& out) {
  out.assign(n_req, ReqDesc());
  const double sq2pi = std::sqrt(2.0 / M_PI);
  for (int q = 0; q < n_req; ++q) {
    const fhtb_request& r = reqs[q];
    ReqDesc d;
    std::memset(&d, 0, sizeof(d));
    d.vec = r.vec;
    d.pa = r.pre_a_pow;
    d.pb = r.pre_b_pow;
    d.pr = r.post_r_pow;
    d.pe = r.post_e_pow;
    d.col_lo = std::max<long long>(r.col_lo, 1);
    d.preA = r.pre_a_pow ? r.pre_a : nullptr;
    d.preB = r.pre_b_pow ? r.pre_b : nullptr;
    d.post_e = r.post_e_pow ? r.post_e : nullptr;
    if (r.n_terms < 0 || (r.n_terms && (!r.orders || !r.weights)))
      return fail(FHTB_EINVAL, "request order list is malformed");
    for (int t = 0; t < r.n_terms; ++t) {
      const int o = r.orders[t];
      const double w = r.weights[t];
      if (o < 0 || o > kMaxOrder) return fail(FHTB_EINVAL, "order out of range");
      auto it = std::find(universe.begin(), universe.end(), o);
      if (it == universe.end()) return fail(FHTB_EINVAL, "order " + std::to_string(o) + " outside engine universe");
      d.w[it - universe.begin()] += w;
      // far field scalars
      std::vector<double> a = asy_coeffs(o, 2 * M);
      const double rr = std::sqrt(0.5);
      double cp, sp;
      switch ((2 * o + 1) % 8) {
        case 1: cp = rr; sp = rr; break;
        case 3: cp = -rr; sp = rr; break;
        case 5: cp = -rr; sp = -rr; break;
        default: cp = rr; sp = -rr; break;
      }
      for (int m = 0; m < M; ++m) {
        const double lam = w * sq2pi * ((m & 1) ? -1.0 : 1.0);
        const double g = lam * a[2 * m], h = lam * a[2 * m + 1];
        d.ac[2 * m] += g * cp;  d.as[2 * m] += -g * sp;
        d.bc[2 * m] += g * sp;  d.bs[2 * m] += g * cp;
        d.ac[2 * m + 1] += h * sp;  d.as[2 * m + 1] += h * cp;
        d.bc[2 * m + 1] += -h * cp; d.bs[2 * m + 1] += h * sp;
      }
    }
    (void)n_data_cols;
    out[q] = d;
  }
  return FHTB_OK;
}

// Group request columns (sorted by vector) so each group holds whole vectors
// and at most kNearMaxCols request columns; *max_cols = widest group.
int make_groups(const std::vector<ReqDesc>& sorted, int n_vec, std::vector<int>& q0, std::vector<int>& v0,
                int* max_cols) {
  q0.clear();
  v0.clear();
  *max_cols = 0;
  std::vector<int> cnt(n_vec, 0);
  for (auto& r : sorted) cnt[r.vec]++;
  int q = 0, v = 0;
  while (v < n_vec) {
    q0.push_back(q);
    v0.push_back(v);
    int cols = 0;
    while (v < n_vec && cols + cnt[v] <= kNearMaxCols) { cols += cnt[v]; q += cnt[v]; ++v; }
    if (cols == 0 && v < n_vec) return fail(FHTB_EINVAL, "more than 128 requests for one vector");
    *max_cols = std::max(*max_cols, cols);
  }
  q0.push_back(q);
  v0.push_back(v);
  return FHTB_OK;
}

// Near-field request layout with order-parity classes (universe {0..n-1},
// n >= 3): per group of whole vectors, requests whose weights touch only even
// orders first, then only odd, then mixed; the first two classes are padded to
// a multiple of 8 columns with inert requests (zero weights, vec -1, no
// columns), so that every 8-column MMA fragment has one class.
int make_groups_split(const std::vector<ReqDesc>& sorted, int n_vec, int n_orders, std::vector<ReqDesc>& out,
                      std::vector<int>& q0, std::vector<int>& v0, std::vector<int2>& cls, int* max_cols) {
  out.clear();
  q0.clear();
  v0.clear();
  cls.clear();
  *max_cols = 0;
  auto klass = [&](const ReqDesc& r) {
    bool ev = false, od = false;
    for (int u = 0; u < n_orders; ++u)
      if (r.w[u] != 0.0) ((u & 1) ? od : ev) = true;
    return (ev && od) ? 2 : (od ? 1 : 0);
  };
  std::vector<std::vector<int>> byvec(n_vec);
  for (int i = 0; i < (int)sorted.size(); ++i) byvec[sorted[i].vec].push_back(i);
  ReqDesc inert;
  std::memset(&inert, 0, sizeof inert);
  inert.vec = -1;
  inert.col_lo = (long long)1 << 62;
  auto padded = [](int n) { return (n + 7) & ~7; };
  int v = 0;
  while (v < n_vec) {
    int cnt[3] = {0, 0, 0};
    int v1 = v;
    while (v1 < n_vec) {
      int c2[3] = {cnt[0], cnt[1], cnt[2]};
      for (int i : byvec[v1]) c2[klass(sorted[i])]++;
      if (padded(c2[0]) + padded(c2[1]) + c2[2] > kNearMaxCols) break;
      for (int k = 0; k < 3; ++k) cnt[k] = c2[k];
      ++v1;
    }
    if (v1 == v) return fail(FHTB_EINVAL, "too many requests for one vector");
    q0.push_back((int)out.size());
    v0.push_back(v);
    const int base = (int)out.size();
    for (int k = 0; k < 3; ++k) {
      for (int vv = v; vv < v1; ++vv)
        for (int i : byvec[vv])
          if (klass(sorted[i]) == k) out.push_back(sorted[i]);
      if (k < 2)
        while ((int)out.size() - base < padded((k == 0 ? 0 : padded(cnt[0])) + cnt[k]) ||
               ((int)out.size() - base) % 8)
          out.push_back(inert);
      if (k == 0) cls.push_back(make_int2((int)out.size() - base, 0));
      if (k == 1) cls.back().y = (int)out.size() - base;
    }
    *max_cols = std::max(*max_cols, (int)out.size() - base);
    v = v1;
  }
  q0.push_back((int)out.size());
  v0.push_back(v);
  return FHTB_OK;
}

// Group-local columns of every vector's requests, in column order (the
// near-field epilogue sums exactly those, in that order).
void vec_columns(const std::vector<ReqDesc>& reqs, const std::vector<int>& q0, int n_vec, std::vector<int>& vstart,
                 std::vector<int>& vcol) {
  std::vector<std::vector<int>> by(n_vec);
  for (int g = 0; g + 1 < (int)q0.size(); ++g)
    for (int q = q0[g]; q < q0[g + 1]; ++q)
      if (reqs[q].vec >= 0) by[reqs[q].vec].push_back(q - q0[g]);
  vstart.assign(n_vec + 1, 0);
  vcol.clear();
  for (int v = 0; v < n_vec; ++v) {
    vstart[v] = (int)vcol.size();
    vcol.insert(vcol.end(), by[v].begin(), by[v].end());
  }
  vstart[n_vec] = (int)vcol.size();
  if (vcol.empty()) vcol.push_back(0);
}

// Near tiles over a list of segments (r0, r1, c_end) in grid index space.
void make_tiles(const std::vector<long long>& segs, long long first, long long stride, long long n_data_cols,
                long long n_out, int n_orders, std::vector<NearTile>& tiles, std::vector<NearRowTile>& rts,
                long long& n_slots) {
  // column chunk per tile: multi-order universes (Fourier-Bessel, DHT) use
  // shorter chunks -- their tiles are strongly skewed (a few 64 x 8192 tiles
  // against a mean of ~8K entries on cfg3), so long chunks leave a tail;
  // measured DHT cfg4 86.5 -> 89.7, FB cfg3 474.6 -> 478.4 transforms/s with
  // 1024.  Single-order grids keep 8192 (cfg2 near 7.7 vs 9.2 ms at 2048).
  const long long chunk = n_orders > 1 ? g_near_chunk_cols_multi : g_near_chunk_cols;
  tiles.clear();
  rts.clear();
  n_slots = 0;
  const int ns = (int)segs.size() / 3;
  for (int s = 0; s < ns; ++s) {
    const long long r0 = segs[3 * s], r1 = segs[3 * s + 1], ce = segs[3 * s + 2];
    const long long cb = std::min(ce, n_data_cols + 1);
    if (r1 <= r0 || cb <= 1) continue;
    // output rows j with grid row k = first + stride*j in [r0, r1)
    long long jlo = (r0 - first + stride - 1) / stride;
    if (r0 < first) jlo = 0;
    long long jhi = (r1 - 1 - first) >= 0 ? (r1 - 1 - first) / stride + 1 : 0;
    jhi = std::min(jhi, n_out);     // grid rows past the last output row are not outputs
    if (jhi <= jlo) continue;
    const long long nch = (cb - 1 + chunk - 1) / chunk;
    for (long long j = jlo; j < jhi; j += kNearRT) {
      const int nr = (int)std::min<long long>(kNearRT, jhi - j);
      long long slot = -1;
      if (nch > 1) {
        slot = n_slots;
        n_slots += nch;
        rts.push_back(NearRowTile{j, nr, (int)nch, slot});
      }
      for (long long c = 0; c < nch; ++c) {
        NearTile t;
        t.seg = s;
        t.nrows = nr;
        t.j0 = j;
        t.na = 1 + c * chunk;
        t.nb = std::min(cb, t.na + chunk);
        t.part = nch > 1 ? slot + c : -1;
        tiles.push_back(t);
      }
    }
  }
  // launch order: most work first (longest-processing-time order), so the
  // short tiles -- partial row tiles, last column chunks -- fill the tail of
  // the grid instead of the long ones.  Results do not depend on the order:
  // every tile owns its partial slot (or its rows), and the slots are
  // reduced per row tile in chunk order.
  std::stable_sort(tiles.begin(), tiles.end(), [](const NearTile& x, const NearTile& y) {
    return (long long)x.nrows * (x.nb - x.na) > (long long)y.nrows * (y.nb - y.na);
  });
}

}  // namespace

// ======================================================================
// ======================================================================
struct fhtb_grid {
  int device = 0;
  long long L = 0;
  double gamma = 0;
  int M = 0;
  long long first = 1, stride = 1, n_out = 0, n_data_cols = 0;
  std::vector<long long> blocks;   // 4 per block
  std::vector<long long> segs;     // 3 per segment
  std::vector<int> orders;
  bool direct = false;             // direct (power-of-two) far-field mode
  int logQ = 0, logN1 = 0, logN2 = 0;   // direct mode split
  std::vector<BlockDesc> bdesc;    // host copy (chirp parameters)
  std::vector<double2*> H;         // chirp filter spectra per block
  BlockDesc* d_blocks = nullptr;
  double2* cs_tab = nullptr;       // (cos, sin)(-gamma k pi/L), k = 1..L, when gamma != 0
  double* w0_tab = nullptr;        // omega_n^{-1/2} (direct two-pass mode)
  double* iw_tab = nullptr;        // 1/omega_n
  // near field
  std::vector<NearTile> tiles;
  std::vector<NearRowTile> rts;
  long long n_slots = 0;
  NearTile* d_tiles = nullptr;
  NearRowTile* d_rts = nullptr;
};

namespace {

void split_q(int logQ, int* l1, int* l2) {
  // pass 2 holds three N1-point rows in shared memory: N1 <= 4096
  *l1 = std::min(12, (logQ + 1) / 2);
  *l2 = logQ - *l1;
}

// Forward FFT (sign -1) of a length-2^logQ device vector (filter spectra).
// transposed: out[k2*Q1 + k1] for k = k2 + Q2*k1 under the split_q split
// (the layout chirp_pass2 reads); else natural order.
int plain_fft(DevCtx* ctx, int logQ, const double2* in, double2* tmp, double2* out, int transposed,
              cudaStream_t st) {
  if (logQ <= 11 && !transposed) {
    CU(launch_fft_batch(logQ, -1, in, out, 1, ctx->tw, st));
    return FHTB_OK;
  }
  FarArgs a;
  std::memset(&a, 0, sizeof a);
  int l1, l2;
  split_q(logQ, &l1, &l2);
  a.L1 = 1 << l1;
  a.L2 = 1 << l2;
  a.tw = ctx->tw;
  a.nf = ctx->nf;
  double2 *ql, *qh;
  int qb;
  if (int r = get_qtab(ctx, logQ, &ql, &qh, &qb)) return r;
  a.qlo = ql;
  a.qhi = qh;
  a.qbits = qb;
  CU(launch_plain_fft(a, l1, l2, in, tmp, out, transposed, st));
  return FHTB_OK;
}

}  // namespace

extern "C" {

int fhtb_abi_version(void) { return 1; }
int64_t fhtb_launch_count(void) { return g_launches.load(); }
const char* fhtb_last_error(void) { return g_err.c_str(); }

int32_t fhtb_kernel_families(void) { return kNumFam; }

const char* fhtb_kernel_family_name(int32_t i) { return (i >= 0 && i < kNumFam) ? kFamNames[i] : ""; }

int fhtb_kernel_times(double* ms, double* bytes, double* flops, int64_t* launches, int32_t n_fam) {
  std::vector<KtRec> recs;
  {
    std::lock_guard<std::mutex> lk(g_kt_mu);
    recs.swap(g_kt);
  }
  for (int i = 0; i < n_fam; ++i) {
    if (ms) ms[i] = 0.0;
    if (bytes) bytes[i] = 0.0;
    if (flops) flops[i] = 0.0;
    if (launches) launches[i] = 0;
  }
  int rc = FHTB_OK;
  for (const KtRec& r : recs) {
    float t = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess) {
      (void)cudaGetLastError();
      rc = fail(FHTB_ECUDA, "kernel timing: event query failed");
    }
    if (r.fam < n_fam) {
      if (ms) ms[r.fam] += t;
      if (bytes) bytes[r.fam] += r.bytes;
      if (flops) flops[r.fam] += r.flops;
      if (launches) launches[r.fam] += 1;
    }
    std::lock_guard<std::mutex> lk(g_kt_mu);
    g_kt_pool[r.dev].push_back(r.a);
    g_kt_pool[r.dev].push_back(r.b);
  }
  return rc;
}

int fhtb_init(void) {
  DevCtx* c;
  return get_ctx(&c);
}

int fhtb_nonfinite_check(void* stream) {
  DevCtx* c;
  if (int r = get_ctx(&c)) return r;
  int flag = 0;
  CU(cudaMemcpyAsync(&flag, c->nf, sizeof(int), cudaMemcpyDeviceToHost, S(stream)));
  CU(cudaMemsetAsync(c->nf, 0, sizeof(int), S(stream)));
  CU(cudaStreamSynchronize(S(stream)));
  if (flag) return fail(FHTB_ENONFINITE, "non-finite values in output");
  return FHTB_OK;
}

int fhtb_set_option(const char* key, int64_t value) {
  if (!key) return fail(FHTB_EINVAL, "null key");
  if (!std::strcmp(key, "far_prune")) {
    g_far_prune = (int)value;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "kernel_timing")) {
    g_kt_on = value ? 1 : 0;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "serial")) {
    g_serial = value ? 1 : 0;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "near_priority")) {
    g_near_priority = value > 0 ? 1 : (value < 0 ? -1 : 0);
    return FHTB_OK;
  }
  if (!std::strcmp(key, "far_prefetch")) {
    g_far_prefetch = value ? 1 : 0;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "host_taper")) {
    if (value < 1 || value > 64) return fail(FHTB_EINVAL, "host_taper must be 1..64");
    g_host_taper = (int)value;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "far_rowsum")) {
    g_rowsum = (int)std::max<int64_t>(0, std::min<int64_t>(value, 2));
    return FHTB_OK;
  }
  if (!std::strcmp(key, "far_rowsum_min_pairs")) {
    g_rowsum_min_m = (int)std::max<int64_t>(1, value);
    return FHTB_OK;
  }
  if (!std::strcmp(key, "far_rowdot_bins")) {
    if (value < 1 || value > 4) return fail(FHTB_EINVAL, "far_rowdot_bins must be 1..4");
    g_rowdot_bins = (int)value;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "far_min_cols")) {
    if (value != 0 && (value < 7 || value > 12)) return fail(FHTB_EINVAL, "far_min_cols must be 0 (auto) or 7..12");
    g_min_lc = (int)value;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "far_prune_rows")) {
    if (value < 10 || value > 12) return fail(FHTB_EINVAL, "far_prune_rows must be 10..12");
    g_prune_rows = (int)value;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "near_overlap")) {
    g_near_overlap = value ? 1 : 0;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "far_streams")) {
    if (value < 1 || value > 2) return fail(FHTB_EINVAL, "far_streams must be 1 or 2");
    g_far_streams = (int)value;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "near_split")) {
    g_near_split = value ? 1 : 0;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "chirp_variant")) {
    g_chirp_variant = (int)value;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "far_half_pairing")) {
    g_far_hp = value ? 1 : 0;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "far_bulk_tables")) {
    g_far_bulk = value ? 1 : 0;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "far_variant")) {
    g_far_variant = (int)value;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "far_chunk_bytes")) {
    if (value < (1 << 20)) return fail(FHTB_EINVAL, "far_chunk_bytes too small");
    g_far_chunk_bytes = value;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "near_chunk_cols_multi")) {
    if (value < 64) return fail(FHTB_EINVAL, "near_chunk_cols_multi too small");
    g_near_chunk_cols_multi = value;
    return FHTB_OK;
  }
  if (!std::strcmp(key, "near_chunk_cols")) {
    if (value < 64) return fail(FHTB_EINVAL, "near_chunk_cols too small");
    g_near_chunk_cols = value;                // both kinds of grid (near_chunk_cols_multi after it)
    g_near_chunk_cols_multi = value;
    return FHTB_OK;
  }
  return fail(FHTB_EINVAL, std::string("unknown option ") + key);
}

// ------------------------------------------------------------------- L1
int fhtb_bessel_j(int nu, const double* z, int64_t n, double* out, void* stream) {
  if (nu < 0) return fail(FHTB_EINVAL, "bessel_j requires nu >= 0");
  DevCtx* c;
  if (int r = get_ctx(&c)) return r;
  JOrder jo = make_jorder(nu);
  CU(launch_bessel_j(nu, jo, z, n, out, S(stream)));
  return FHTB_OK;
}

int fhtb_bessel_j_multi(int nu_max, const double* z, int64_t n, double* out, void* stream) {
  if (nu_max < 0 || nu_max >= kMaxOrd) return fail(FHTB_EINVAL, "nu_max out of range");
  DevCtx* c;
  if (int r = get_ctx(&c)) return r;
  CU(launch_bessel_multi(nu_max, c->jtab, z, n, out, S(stream)));
  return FHTB_OK;
}

int fhtb_hankel_asy_eval(int nu, int m_terms, const double* z, int64_t n, double* out, void* stream) {
  if (nu < 0 || m_terms < 1 || m_terms > 64) return fail(FHTB_EINVAL, "bad hankel_asy_eval arguments");
  DevCtx* c;
  if (int r = get_ctx(&c)) return r;
  std::vector<double> a = asy_coeffs(nu, 2 * m_terms), coef(2 * m_terms);
  for (int m = 0; m < m_terms; ++m) {
    const double sg = (m & 1) ? -1.0 : 1.0;
    coef[m] = sg * a[2 * m];
    coef[m_terms + m] = sg * a[2 * m + 1];
  }
  double* d = nullptr;
  CU(cudaMallocAsync(&d, coef.size() * sizeof(double), S(stream)));
  CU(cudaMemcpyAsync(d, coef.data(), coef.size() * sizeof(double), cudaMemcpyHostToDevice, S(stream)));
  CU(launch_hankel_eval(nu, m_terms, d, z, n, out, S(stream)));
  CU(cudaFreeAsync(d, S(stream)));
  CU(cudaStreamSynchronize(S(stream)));
  return FHTB_OK;
}

int fhtb_taylor_eval(int nu, int n_terms, const double* z, int64_t n, double* out, void* stream) {
  if (nu < 0 || n_terms < 1) return fail(FHTB_EINVAL, "bad taylor_eval arguments");
  DevCtx* c;
  if (int r = get_ctx(&c)) return r;
  CU(launch_taylor_eval(nu, n_terms, 1.0 / std::tgamma(nu + 1.0), z, n, out, S(stream)));
  return FHTB_OK;
}

int fhtb_roots_j0(int64_t count, double* roots, double* perturb, double* resid_max, void* stream) {
  if (count < 1) return fail(FHTB_EINVAL, "count must be >= 1");
  DevCtx* c;
  if (int r = get_ctx(&c)) return r;
  std::lock_guard<std::mutex> scratch_lk(g_scratch_mu);      // c->scratch is shared
  CU(cudaMemsetAsync(c->scratch, 0, 16, S(stream)));
  CU(launch_roots_j0(c->jtab, count, roots, perturb, c->scratch, S(stream)));
  unsigned long long bits[2] = {0, 0};
  CU(cudaMemcpyAsync(bits, c->scratch, 16, cudaMemcpyDeviceToHost, S(stream)));
  CU(cudaStreamSynchronize(S(stream)));
  double res, ratio;
  std::memcpy(&res, &bits[0], 8);
  std::memcpy(&ratio, &bits[1], 8);
  if (resid_max) *resid_max = res;
  // each root against max(1e-13, 2 ulp(x) |J1(x)|): identical to the
  // reference's 1e-13 test wherever fp64 can meet it (roots below ~2e6)
  if (!(ratio <= 1.0)) {
    char buf[128];
    std::snprintf(buf, sizeof buf, "Newton failed to converge on J0 roots (residual %.3e)", res);
    return fail(FHTB_ECONVERGE, buf);
  }
  return FHTB_OK;
}

int fhtb_coef_stats(const double* C, int64_t ldc, int32_t n_vec, int64_t n, int64_t n_split, const double* b,
                    int64_t nb, double* out_host, void* stream) {
  if (n_vec < 0 || n < 0 || n_split < 0 || !out_host) return fail(FHTB_EINVAL, "bad coef_stats arguments");
  if (n_vec == 0) return FHTB_OK;
  DevCtx* c;
  if (int r = get_ctx(&c)) return r;
  // one caller at a time per process: the device buffer is shared (concurrent host threads,
  // e.g. simulated ranks, would otherwise overwrite each other's rows before the copy-out)
  static std::mutex stats_mu;
  std::lock_guard<std::mutex> call_lk(stats_mu);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (c->stats_cap < (size_t)n_vec) {
      CU(cudaDeviceSynchronize());
      cudaFree(c->stats);
      c->stats = nullptr;
      c->stats_cap = 0;
      const size_t cap = std::max<size_t>(256, 2 * (size_t)n_vec);
      CU(cudaMalloc(&c->stats, sizeof(double) * 3 * cap));
      c->stats_cap = cap;
    }
  }
  double* d = c->stats;
  CU(launch_coef_stats(C, ldc, n_vec, n, n_split, b, nb, d, S(stream)));
  CU(cudaMemcpyAsync(out_host, d, sizeof(double) * 3 * (size_t)n_vec, cudaMemcpyDeviceToHost, S(stream)));
  CU(cudaStreamSynchronize(S(stream)));
  return FHTB_OK;
}

int fhtb_mul_rows(double* out, int64_t ldo, const double* a, int64_t lda, const double* w, double alpha, int64_t n,
                  int32_t n_vec, void* stream) {
  if (n < 0 || n_vec < 0 || ldo < n || lda < n) return fail(FHTB_EINVAL, "bad mul_rows arguments");
  CU(launch_mul_rows(out, ldo, a, lda, w, alpha, n, n_vec, S(stream)));
  return FHTB_OK;
}

int fhtb_max_abs_diff(const double* a, double alpha, const double* b, int64_t n, double* out_host, void* stream) {
  if (n < 0 || !out_host) return fail(FHTB_EINVAL, "bad max_abs_diff arguments");
  DevCtx* c;
  if (int r = get_ctx(&c)) return r;
  std::lock_guard<std::mutex> scratch_lk(g_scratch_mu);      // c->scratch is shared
  CU(cudaMemsetAsync(c->scratch, 0, 8, S(stream)));
  CU(launch_max_abs_diff(a, alpha, b, n, c->scratch, S(stream)));
  unsigned long long bits = 0;
  CU(cudaMemcpyAsync(&bits, c->scratch, 8, cudaMemcpyDeviceToHost, S(stream)));
  CU(cudaStreamSynchronize(S(stream)));
  std::memcpy(out_host, &bits, 8);
  return FHTB_OK;
}

int fhtb_zero_rows(double* F, int64_t ldf, int32_t n_vec, int64_t n, void* stream) {
  if (n_vec < 0 || n < 0 || ldf < n) return fail(FHTB_EINVAL, "bad zero_rows arguments");
  if (n_vec == 0 || n == 0) return FHTB_OK;
  CU(cudaMemset2DAsync(F, sizeof(double) * (size_t)ldf, 0, sizeof(double) * (size_t)n, (size_t)n_vec, S(stream)));
  return FHTB_OK;
}

int fhtb_fft(int64_t n, int sign, const double* in, double* out, int64_t batch, void* stream) {
  if (!is_pow2(n) || n < 2 || n > 2048) return fail(FHTB_EINVAL, "fhtb_fft: n must be a power of two in [2, 2048]");
  DevCtx* c;
  if (int r = get_ctx(&c)) return r;
  CU(launch_fft_batch(ilog2ll(n), sign, (const double2*)in, (double2*)out, batch, c->tw, S(stream)));
  return FHTB_OK;
}

// ---------------------------------------------------------------- grid
int fhtb_grid_create(const fhtb_grid_desc* d, fhtb_grid** out) {
  if (!d || !out) return fail(FHTB_EINVAL, "null argument");
  if (d->L < 1) return fail(FHTB_EINVAL, "L must be >= 1");
  if (d->m_terms < 1 || 2 * d->m_terms > kMaxTerms) return fail(FHTB_EINVAL, "m_terms out of range");
  if (d->n_orders < 1 || d->n_orders > kMaxOrd) return fail(FHTB_EINVAL, "order universe size out of range");
  if (d->row_stride < 1 || d->row_first < 1) return fail(FHTB_EINVAL, "bad row mapping");
  DevCtx* ctx;
  if (int r = get_ctx(&ctx)) return r;
  fhtb_grid* g = new fhtb_grid();
  CU(cudaGetDevice(&g->device));
  g->L = d->L;
  g->gamma = d->gamma;
  g->M = d->m_terms;
  g->first = d->row_first;
  g->stride = d->row_stride;
  g->n_out = d->n_out;
  g->n_data_cols = std::min<long long>(d->n_data_cols, d->L);
  g->blocks.assign(d->blocks, d->blocks + 4 * d->n_blocks);
  g->segs.assign(d->segments, d->segments + 3 * d->n_segments);
  g->orders.assign(d->orders, d->orders + d->n_orders);
  for (int o : g->orders)
    if (o < 0 || o > kMaxOrder) { delete g; return fail(FHTB_EINVAL, "order out of range"); }
  if (*std::max_element(g->orders.begin(), g->orders.end()) - *std::min_element(g->orders.begin(), g->orders.end()) >=
      kMaxOrd) {
    delete g;
    return fail(FHTB_EINVAL, "order universe spans more than 16 orders");
  }
  g->direct = is_pow2(2 * g->L) && g->first == 1 && g->stride == 1 && g->n_out == g->L;
  if (g->direct) {
    g->logQ = ilog2ll(2 * g->L);
    if (g->logQ > 25) { delete g; return fail(FHTB_EINVAL, "grid too large (2L > 2^25)"); }
    if (g->logQ <= 13) {
      g->logN1 = g->logQ;
      g->logN2 = 0;
    } else {
      g->logN1 = std::min(12, (g->logQ + 1) / 2);
      g->logN2 = g->logQ - g->logN1;
    }
  }
  const int nb = d->n_blocks;
  g->H.assign(nb, nullptr);
  for (int b = 0; b < nb; ++b) {
    BlockDesc x;
    std::memset(&x, 0, sizeof x);
    x.r0 = g->blocks[4 * b];
    x.r1 = g->blocks[4 * b + 1];
    x.c0 = g->blocks[4 * b + 2];
    x.c1 = g->blocks[4 * b + 3];
    if (!g->direct) {
      // rows j with first + stride*j < r1 ; columns c0 .. min(c1, data+1)
      const long long J = std::min<long long>(g->n_out, x.r1 > g->first ? (x.r1 - g->first + g->stride - 1) / g->stride : 0);
      const long long Mn = std::min(x.c1, g->n_data_cols + 1) - x.c0;
      if (J > 0 && Mn > 0 && x.r1 > x.r0) {
        const int logQ = std::max(2, ilog2ll(Mn + J - 1));
        if (logQ > 26) { fhtb_grid_destroy(g); return fail(FHTB_EINVAL, "chirp convolution too long"); }
        const long long Q = 1LL << logQ;
        x.J = J;
        x.Mn = Mn;
        x.logQ = logQ;
        double2 *h = nullptr, *tmp = nullptr, *Hb = nullptr;
        CU(cudaMalloc(&h, Q * sizeof(double2)));
        CU(cudaMalloc(&tmp, Q * sizeof(double2)));
        CU(cudaMalloc(&Hb, Q * sizeof(double2)));
        CU(launch_chirp_filter(h, Q, Mn, J, g->stride, g->L, 0));
        if (int r = plain_fft(ctx, logQ, h, tmp, Hb, 1, 0)) return r;
        CU(cudaDeviceSynchronize());
        cudaFree(h);
        cudaFree(tmp);
        x.H = Hb;
        g->H[b] = Hb;
      } else {
        x.J = 0;
        x.Mn = 0;
      }
    } else if (g->logN2 > 0) {
      // pruned four-step split per block (direct two-pass mode)
      x.dmode = 0;
      x.dlogL1 = g->logN1;
      const long long cend = std::min(x.c1, g->n_data_cols + 1);   // columns n < cend
      // narrow-column blocks are shifted to their first column (fhtb_far.cu MODE 2)
      // smallest column FFT: 256 points (two radix-16 passes, one-warp CTAs) pay from 8 pairs on
      // (cfg2 1e-15 far 64.0 -> 63.5 ms, FB cfg3 +1.5%; with 3 / 5 pairs -1.3% / -0.8%)
      const int min_lc = g_min_lc ? g_min_lc : (g->M >= 8 ? 8 : 9);
      const int lc = std::max(min_lc, ilog2ll(std::max<long long>(cend - x.c0, 2)));
      // L2 >= r1 so that every block row has k1 = 0; keep L2 >= 1024 (the
      // pass-1 FFT is least efficient below that) and L1 <= 2048 (rowdot sums)
      const int lr = std::max(std::max(g->logQ - 11, 10), ilog2ll(std::max<long long>(x.r1, 2)));
      // narrow rows with the pass-1 FFT kept at 2^lr0 points: the rows k < r1
      // need the bins k1 <= (r1-1) >> lr0 of each column (2 sums per bin)
      // (the pass-1 column FFT is at most 8192 points: 2L = 2^25 keeps 2^13)
      const int lr0 = std::min(13, std::max(g->logQ - 11, 10));
      const long long kb = ((std::max<long long>(x.r1, 2) - 1) >> lr0) + 1;
      x.kbins = 1;
      if (g_far_prune && lc <= 12 && lc < g->logQ) {
        x.dmode = 1;                 // narrow columns: pass 1 degenerates
        x.dlogL1 = lc;
      } else if (g_far_prune && kb <= g_rowdot_bins && lr0 < g->logQ && g->logQ - lr0 <= 13) {
        x.dmode = 2;                 // narrow rows: pass 2 collapses to 2*kbins sums
        x.dlogL1 = g->logQ - lr0;
        x.kbins = (int)kb;
      } else if (g_far_prune && lr <= g_prune_rows && lr < g->logQ && g->logQ - lr <= 13) {
        x.dmode = 2;                 // narrow rows with a longer pass-1 FFT, one bin
        x.dlogL1 = g->logQ - lr;
      }
      // narrow rows, fully fused (fhtb_rowsum.cu): column FFTs of 2^ls >= r1
      // points (128..4096), pairs folded per column, no intermediate.  Needs
      // r1 <= 2^ls < L and at least 16 columns n1.  dmode 3 + form:
      //   form 1: high-occupancy kernel, no k2 serves two rows (2 r1 <= 2^ls + 1)
      //   form 2: same with up to two such k2 per thread (2 r1 - 2^ls - 1 <= 2^ls / 16)
      //   form 0: accumulators in registers, any overlap (2048 / 4096 points)
      // g_rowsum 1: blocks that would otherwise run the full pass 1 + pass 2 use
      // form 0 at 4096 points (cfg2: 17.3 vs 25.2 us per unit and pair) and the
      // high-occupancy forms; 2: also the blocks already pruned to row sums.
      const bool was_rows = x.dmode == 2;     // already pruned to pass 1 + row sums
      if (g_far_prune && g_rowsum && (x.dmode == 0 || (was_rows && g_rowsum >= 2 && g->M >= g_rowsum_min_m))) {
        int ls = std::max(7, ilog2ll(std::max<long long>(x.r1, 2)));
        long long ov = 2 * x.r1 - (1LL << ls) - 1;          // k2 in (2^ls - r1, r1) serve two rows
        int form = -1;
        if (ls <= 11 && ov <= 0) form = 1;
        else if (ls <= 11 && ov <= (1LL << ls) / 16) form = 2;
        else if (ls + 1 <= 11) { ls += 1; form = 1; }
        else if (ls <= 12) form = 0;
        if (form >= 0 && g->logQ - ls >= 4 && (1LL << ls) < g->L) {
          x.dmode = 3 + form;
          x.dlogL1 = g->logQ - ls;
          x.kbins = 1;
        }
      }
    }
    x.sig = x.isig = 1.0;
    if (g->direct) {
      // exact power of two near omega at the block's first column (fhtb_types.h)
      const double om0 = ((double)std::max<long long>(x.c0, 1) + g->gamma) * M_PI;
      if (om0 > 1.0) {
        int ex = 0;
        std::frexp(om0, &ex);
        x.sig = std::ldexp(1.0, ex - 1);
        x.isig = 1.0 / x.sig;
      }
    }
    g->bdesc.push_back(x);
  }
  if (!g->bdesc.empty()) {
    CU(cudaMalloc(&g->d_blocks, g->bdesc.size() * sizeof(BlockDesc)));
    CU(cudaMemcpy(g->d_blocks, g->bdesc.data(), g->bdesc.size() * sizeof(BlockDesc), cudaMemcpyHostToDevice));
  }
  if (g->gamma != 0.0) {
    CU(cudaMalloc(&g->cs_tab, g->L * sizeof(double2)));
    CU(launch_cs_table(g->cs_tab, g->L, g->gamma, M_PI / (double)g->L, 0));
  }
  if (g->direct && g->logN2 > 0) {
    CU(cudaMalloc(&g->w0_tab, g->L * sizeof(double)));
    CU(cudaMalloc(&g->iw_tab, g->L * sizeof(double)));
    CU(launch_col_tables(g->w0_tab, g->iw_tab, g->L, g->gamma, 0));
  }
  if (g->direct && g->logN2 > 0) {
    double2 *ql, *qh;
    int qb;
    if (int r = get_qtab(ctx, g->logQ, &ql, &qh, &qb)) return r;
  }
  make_tiles(g->segs, g->first, g->stride, g->n_data_cols, g->n_out, (int)g->orders.size(), g->tiles, g->rts,
             g->n_slots);
  if (!g->tiles.empty()) {
    CU(cudaMalloc(&g->d_tiles, g->tiles.size() * sizeof(NearTile)));
    CU(cudaMemcpy(g->d_tiles, g->tiles.data(), g->tiles.size() * sizeof(NearTile), cudaMemcpyHostToDevice));
  }
  if (!g->rts.empty()) {
    CU(cudaMalloc(&g->d_rts, g->rts.size() * sizeof(NearRowTile)));
    CU(cudaMemcpy(g->d_rts, g->rts.data(), g->rts.size() * sizeof(NearRowTile), cudaMemcpyHostToDevice));
  }
  CU(cudaDeviceSynchronize());
  *out = g;
  return FHTB_OK;
}

double fhtb_grid_far_model_bytes(const fhtb_grid* g) {
  if (!g) return 0.0;
  const double L = (double)g->L;
  const int nb = (int)g->blocks.size() / 4;
  double bytes = 8.0 * L;                                   // output row
  for (int b = 0; b < nb; ++b) {
    const BlockDesc& x = g->bdesc[b];
    const double rows = (double)std::max<long long>(0, x.r1 - x.r0);
    const double cols = (double)std::max<long long>(0, std::min(x.c1, g->n_data_cols + 1) - x.c0);
    if (rows <= 0 || cols <= 0) continue;
    const double terms = 2.0 * g->M;
    bytes += 8.0 * cols + 16.0 * rows;                      // coefficients, partial row w+r
    if (!g->direct) {                                       // chirp: two round trips of Q
      bytes += terms * 4.0 * 16.0 * (double)(1LL << x.logQ);
    } else if (g->logN2 == 0) {
      // one-pass: no intermediate
    } else if (x.dmode == 0) {
      bytes += terms * 32.0 * L;                            // G written and read
    } else if (x.dmode == 2) {
      const double L2 = (double)(1LL << (g->logQ - x.dlogL1));
      bytes += terms * 16.0 * L * (1.0 + std::min(1.0, 2.0 * (rows + 1) / L2));
    } else if (x.dmode >= 3) {
      bytes += 2.0 * 32.0 * rows * (double)(1LL << x.dlogL1);   // folded rows P written and read
    }                                                       // dmode 1: no intermediate
  }
  return bytes;
}

void fhtb_grid_destroy(fhtb_grid* g) {
  if (!g) return;
  cudaFree(g->d_blocks);
  cudaFree(g->cs_tab);
  cudaFree(g->w0_tab);
  cudaFree(g->iw_tab);
  for (double2* h : g->H) cudaFree(h);
  cudaFree(g->d_tiles);
  cudaFree(g->d_rts);
  delete g;
}

}  // extern "C"

namespace {

// bytes of intermediate per far-field unit
// rows of a fused narrow-row block: k in [max(r0, 1), min(r1, L2))
long long fused_rows(const fhtb_grid* g, const BlockDesc& x, int logL1) {
  const long long L2 = 1LL << (g->logQ - logL1);
  return std::max<long long>(1, std::min(x.r1, L2) - std::max<long long>(x.r0, 1));
}

size_t unit_bytes_q(const fhtb_grid* g, int logQ) {
  return (size_t)(g->direct ? g->M : 2 * g->M) * ((size_t)1 << logQ) * sizeof(double2);
}

long long chunk_for(size_t ub, long long n_units) {
  long long per = std::max<long long>(1, g_far_chunk_bytes / (long long)ub);
  return std::min(per, std::max<long long>(n_units, 1));
}

struct FarPlan {
  std::vector<UnitDesc> units;                 // execution order
  std::vector<int2> chunks;                    // [u0, u1) per launch group
  std::vector<int> chunk_logq;
  std::vector<int> chunk_key;                  // direct two-pass: dmode*64 + log2 L1
  size_t g_bytes = 0;                          // intermediate
  size_t part_bytes = 0;                       // chirp partials
};

// skip_full: leave out the full (dmode 0) units of a direct two-pass grid
// (exchange mode computes them by the distributed four-step).
void plan_far(const fhtb_grid* g, const std::vector<ReqDesc>& rs, FarPlan& fp, int skip_full = 0) {
  fp = FarPlan();
  const int nb = (int)g->blocks.size() / 4;
  const int n_req = (int)rs.size();
  std::vector<UnitDesc> all;
  for (int q = 0; q < n_req; ++q)
    for (int b = 0; b < nb; ++b) {
      const long long r0 = g->blocks[4 * b], r1 = g->blocks[4 * b + 1];
      const long long c0 = std::max<long long>(g->blocks[4 * b + 2], rs[q].col_lo);
      const long long c1 = std::min<long long>(g->blocks[4 * b + 3], g->n_data_cols + 1);
      if (r1 <= r0 || c1 <= c0) continue;
      if (!g->direct && g->bdesc[b].J == 0) continue;
      if (skip_full && g->direct && g->logN2 > 0 && g->bdesc[b].dmode == 0) continue;
      all.push_back(UnitDesc{q, b, rs[q].vec, 0});
    }
  if (g->direct) {
    const size_t pb = sizeof(double) * (size_t)g->n_out;
    if (g->logN2 == 0) {
      // one-pass: every unit in one launch; one partial row per unit
      fp.units = all;
      const long long nu = (long long)all.size();
      if (nu) {
        fp.chunks.push_back(make_int2(0, (int)nu));
        fp.chunk_logq.push_back(g->logQ);
        fp.chunk_key.push_back(-1);
        fp.part_bytes = pb * nu;
      }
      return;
    }
    // two-pass: group units by pruned form and split (keeping vector order
    // inside a group), chunks bounded by the intermediate budget
    std::vector<int> keys;
    for (auto& u : all) keys.push_back(g->bdesc[u.block].dmode * 64 + g->bdesc[u.block].dlogL1);
    std::vector<int> uk = keys;
    std::sort(uk.begin(), uk.end());
    uk.erase(std::unique(uk.begin(), uk.end()), uk.end());
    for (int key : uk) {
      const long long start = (long long)fp.units.size();
      for (size_t i = 0; i < all.size(); ++i)
        if (keys[i] == key) fp.units.push_back(all[i]);
      const long long n = (long long)fp.units.size() - start;
      // narrow-column units keep only their column table (M x L1)
      size_t ub = (key / 64 == 1) ? (size_t)g->M * ((size_t)1 << (key % 64)) * sizeof(double2)
                                  : unit_bytes_q(g, g->logQ);
      if (key / 64 >= 3) {
        // fused narrow rows: P[unit][A|B][rows][L1], rows = the widest block of the group
        long long rs = 1;
        for (size_t i = 0; i < all.size(); ++i)
          if (keys[i] == key) rs = std::max(rs, fused_rows(g, g->bdesc[all[i].block], key % 64));
        ub = 2 * (size_t)rs * ((size_t)1 << (key % 64)) * sizeof(double2);
      }
      const long long cu = chunk_for(ub + pb, n);
      for (long long u0 = 0; u0 < n; u0 += cu) {
        fp.chunks.push_back(make_int2((int)(start + u0), (int)(start + std::min(n, u0 + cu))));
        fp.chunk_logq.push_back(g->logQ);
        fp.chunk_key.push_back(key);
      }
      fp.g_bytes = std::max(fp.g_bytes, ub * (size_t)cu);
      fp.part_bytes = std::max(fp.part_bytes, pb * (size_t)cu);
    }
    return;
  }
  // chirp mode: group by filter length, keep vector order inside a group
  // key: 2 log2 Q + hz, hz = the block's columns fill at most half of Q (the
  // pass-1 FFT input is then zero in its upper half)
  auto ckey = [&](const UnitDesc& u) {
    const BlockDesc& b = g->bdesc[u.block];
    return 2 * b.logQ + ((2 * b.Mn <= (1LL << b.logQ)) ? 1 : 0);
  };
  std::vector<int> logs;
  for (auto& u : all) logs.push_back(ckey(u));
  std::sort(logs.begin(), logs.end());
  logs.erase(std::unique(logs.begin(), logs.end()), logs.end());
  for (int key : logs) {
    const int lq = key / 2;
    const long long start = (long long)fp.units.size();
    for (auto& u : all)
      if (ckey(u) == key) fp.units.push_back(u);
    const long long n = (long long)fp.units.size() - start;
    const size_t ub = unit_bytes_q(g, lq);
    const long long cu = chunk_for(ub, n);
    for (long long u0 = 0; u0 < n; u0 += cu) {
      fp.chunks.push_back(make_int2((int)(start + u0), (int)(start + std::min(n, u0 + cu))));
      fp.chunk_key.push_back(key % 2);
      fp.chunk_logq.push_back(lq);
    }
    fp.g_bytes = std::max(fp.g_bytes, ub * (size_t)cu);
    fp.part_bytes = std::max(fp.part_bytes, sizeof(double) * (size_t)cu * (size_t)g->n_out);
  }
}

size_t far_ws(const fhtb_grid* g, int n_req) {
  // worst case over request sets of this size: every request touches every block
  std::vector<ReqDesc> rs(n_req);
  for (int q = 0; q < n_req; ++q) { std::memset(&rs[q], 0, sizeof(ReqDesc)); rs[q].col_lo = 1; }
  FarPlan fp;
  plan_far(g, rs, fp);
  size_t s = align_up(sizeof(UnitDesc) * std::max<size_t>(fp.units.size(), 1));
  s += align_up(sizeof(int2) * (fp.chunks.size() + 1));
  const int nbuf = (g->direct && g->logN2 > 0) ? 2 : 1;     // chunks in flight
  s += nbuf * (align_up(fp.g_bytes) + align_up(fp.part_bytes));
  return s;
}

size_t ws_need(const fhtb_grid* g, int n_req, int n_vec, int flags) {
  size_t s = align_up(sizeof(ReqDesc) * std::max(n_req, 1));
  if (flags & FHTB_FAR) s += far_ws(g, n_req);
  s += 2 * align_up(sizeof(int) * (n_vec + 2));
  if (flags & FHTB_NEAR) {
    s += align_up(sizeof(double) * (size_t)g->n_slots * n_vec * kNearRT);
    // parity-class layout: a padded copy of the requests (<= 16 inert per vector) + class ends
    s += align_up(sizeof(ReqDesc) * ((size_t)std::max(n_req, 1) + 16 * (size_t)n_vec));
    s += align_up(sizeof(int2) * (n_vec + 2));
    s += align_up(sizeof(int) * (n_vec + 2)) + align_up(sizeof(int) * ((size_t)n_req + 2));
    if (flags & FHTB_FAR) s += align_up(sizeof(double) * (size_t)n_vec * g->n_out);   // overlap buffer
  }
  return s + 4096;
}

// ------------------------------------------ distributed four-step (exchange)
struct XCtx {
  void* send;
  void* recv;
  size_t bytes;
  fhtb_exchange_fn exchange;
  void* user;
};

// Column-pair ownership: pairs c = 0..L2/2 ({c, L2-c}) split into balanced
// contiguous ranges; rank s's rows are k2 = c (j = c - lo) then k2 = L2 - c
// (j = cnt + c - lo) for the c with a distinct partner.
void x_pairs(int L2, int world, int s, int* lo, int* cnt) {
  const int n = L2 / 2 + 1, base = n / world, extra = n % world;
  *lo = s * base + std::min(s, extra);
  *cnt = base + (s < extra ? 1 : 0);
}

bool x_supported(const fhtb_grid* g, int world, int* l1, int* rows) {
  if (!g || world < 2 || !g->direct || g->logN2 == 0) return false;
  const int L1 = 1 << g->logN1, L2 = 1 << (g->logQ - g->logN1);
  if (L1 % world || (L1 / world) % 16 || L2 / 2 + 1 < world) return false;
  int lo, cnt, mx = 0;
  for (int s = 0; s < world; ++s) {
    x_pairs(L2, world, s, &lo, &cnt);
    mx = std::max(mx, cnt);
  }
  *l1 = g->logN1;
  *rows = 2 * mx;
  return true;
}

std::vector<UnitDesc> x_units(const fhtb_grid* g, const std::vector<ReqDesc>& rs) {
  std::vector<UnitDesc> u;
  const int nb = (int)g->blocks.size() / 4;
  for (int q = 0; q < (int)rs.size(); ++q)
    for (int b = 0; b < nb; ++b) {
      const long long r0 = g->blocks[4 * b], r1 = g->blocks[4 * b + 1];
      const long long c0 = std::max<long long>(g->blocks[4 * b + 2], rs[q].col_lo);
      const long long c1 = std::min<long long>(g->blocks[4 * b + 3], g->n_data_cols + 1);
      if (r1 <= r0 || c1 <= c0 || g->bdesc[b].dmode != 0) continue;
      u.push_back(UnitDesc{q, b, rs[q].vec, 0});
    }
  return u;
}

size_t x_ws(const fhtb_grid* g, int n_req, int world, size_t xbytes) {
  int l1, rows;
  if (!x_supported(g, world, &l1, &rows)) return 0;
  const size_t per = (size_t)world * g->M * rows * ((1 << l1) / world) * sizeof(double2);
  const size_t u_round = std::max<size_t>(1, xbytes / std::max<size_t>(per, 1));
  const size_t nu = (size_t)std::max(n_req, 1) * (g->blocks.size() / 4 + 1);
  return align_up(sizeof(UnitDesc) * nu) + align_up(sizeof(int2) * ((size_t)1 << (g->logQ - l1))) +
         align_up(sizeof(double) * u_round * (size_t)g->n_out) + 4096;
}

// fhtb_apply_host's far-field calls: the group's rows are ready when `ready`
// fires, and its workspace region is free when `region_free` fires (null: no
// earlier user).  The tables are then copied on the first auxiliary far
// stream and only the aux streams wait, so the chunks of consecutive groups
// follow each other on the aux streams without draining the pipeline.
struct HostPipe {
  cudaEvent_t ready;
  cudaEvent_t region_free;
};

int apply_impl(const fhtb_grid* g, const fhtb_request* reqs, int32_t n_req, const double* C, int64_t ldc,
               int32_t n_vec, double* F, int64_t ldf, int32_t flags, int32_t shard, int32_t n_shards,
               const XCtx* xc, void* ws, size_t ws_bytes, void* stream, const HostPipe* hp = nullptr);

}  // namespace

extern "C" {

size_t fhtb_apply_workspace(const fhtb_grid* g, int32_t n_req, int32_t n_vec, int32_t flags) {
  if (!g) return 0;
  return ws_need(g, n_req, n_vec, flags);
}

int fhtb_apply(const fhtb_grid* g, const fhtb_request* reqs, int32_t n_req, const double* C, int64_t ldc,
               int32_t n_vec, double* F, int64_t ldf, int32_t flags, void* ws, size_t ws_bytes, void* stream) {
  return fhtb_apply_part(g, reqs, n_req, C, ldc, n_vec, F, ldf, flags, 0, 1, ws, ws_bytes, stream);
}

int fhtb_apply_part(const fhtb_grid* g, const fhtb_request* reqs, int32_t n_req, const double* C, int64_t ldc,
                    int32_t n_vec, double* F, int64_t ldf, int32_t flags, int32_t shard, int32_t n_shards,
                    void* ws, size_t ws_bytes, void* stream) {
  return apply_impl(g, reqs, n_req, C, ldc, n_vec, F, ldf, flags, shard, n_shards, nullptr, ws, ws_bytes, stream);
}

size_t fhtb_apply_x_workspace(const fhtb_grid* g, int32_t n_req, int32_t n_vec, int32_t flags, int32_t world,
                              size_t xbytes) {
  if (!g) return 0;
  return ws_need(g, n_req, n_vec, flags) + x_ws(g, n_req, world, xbytes);
}

size_t fhtb_apply_x_unit_bytes(const fhtb_grid* g, int32_t world) {
  int l1, rows;
  if (!x_supported(g, world, &l1, &rows)) return 0;
  return (size_t)world * (size_t)g->M * (size_t)rows * (size_t)((1 << l1) / world) * sizeof(double2);
}

int fhtb_apply_x(const fhtb_grid* g, const fhtb_request* reqs, int32_t n_req, const double* C, int64_t ldc,
                 int32_t n_vec, double* F, int64_t ldf, int32_t flags, int32_t rank, int32_t world, void* send,
                 void* recv, size_t xbytes, fhtb_exchange_fn exchange, void* user, void* ws, size_t ws_bytes,
                 void* stream) {
  if (!exchange || !send || !recv) return fail(FHTB_EINVAL, "exchange mode needs buffers and a callback");
  XCtx x{send, recv, xbytes, exchange, user};
  return apply_impl(g, reqs, n_req, C, ldc, n_vec, F, ldf, flags, rank, world, &x, ws, ws_bytes, stream);
}

}  // extern "C"

// ------------------------------------------------ host-buffer application
// fhtb_apply_host: the whole batch from host memory to host memory, with the
// copies overlapped with the far field.  Vector groups g = 0..G-1:
//   h2d stream : C_dev[g] <- C_host[g]                       (event in[g])
//   near stream: after in[G-1], the near field of ALL vectors into Fn
//                (one batched call: the Bessel tiles are shared by the batch)
//   caller     : after in[g], F_dev[g] = 0; far field of group g; after the
//                near field, F_dev[g] += Fn[g]                 (event fin[g])
//   d2h stream : after fin[g], F_host[g] <- F_dev[g]
// Per vector this is the arithmetic of fhtb_apply(FAR|NEAR): far partials
// added unit by unit in plan order (independent of the grouping), then the
// near sum.  So the result equals fhtb_apply on device copies bit for bit.
namespace {
constexpr int kMaxHostGroups = 64;
struct HostAux {
  cudaStream_t h2d, d2h, near;
  cudaEvent_t in[kMaxHostGroups], fin[kMaxHostGroups], nstart, ndone;
};
std::map<std::pair<int, cudaStream_t>, HostAux> g_haux;

int get_haux(cudaStream_t caller, HostAux** out) {
  int dev = 0;
  CU(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, caller);
  auto it = g_haux.find(key);
  if (it == g_haux.end()) {
    HostAux h;
    CU(cudaStreamCreateWithFlags(&h.h2d, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&h.d2h, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&h.near, cudaStreamNonBlocking));
    for (int i = 0; i < kMaxHostGroups; ++i) {
      CU(cudaEventCreateWithFlags(&h.in[i], cudaEventDisableTiming));
      CU(cudaEventCreateWithFlags(&h.fin[i], cudaEventDisableTiming));
    }
    CU(cudaEventCreateWithFlags(&h.nstart, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&h.ndone, cudaEventDisableTiming));
    it = g_haux.emplace(key, h).first;
  }
  *out = &it->second;
  return FHTB_OK;
}

struct HostLayout {
  size_t c_off, f_off, fn_off, far_off, far_bytes, near_off, near_bytes, total;
};

HostLayout host_layout(const fhtb_grid* g, int32_t n_req, int32_t n_vec, int32_t flags) {
  HostLayout h;
  size_t s = 0;
  h.c_off = s;
  s += align_up(sizeof(double) * (size_t)n_vec * g->n_data_cols);
  h.f_off = s;
  s += align_up(sizeof(double) * (size_t)n_vec * g->n_out);
  const bool near = (flags & FHTB_NEAR) && !g->tiles.empty();
  h.fn_off = s;
  if (near && (flags & FHTB_FAR)) s += align_up(sizeof(double) * (size_t)n_vec * g->n_out);
  h.far_off = s;                             // two far regions, alternating groups
  h.far_bytes = (flags & FHTB_FAR) ? ws_need(g, n_req, n_vec, FHTB_FAR) : 0;
  s += 2 * align_up(h.far_bytes);
  h.near_off = s;
  h.near_bytes = near ? ws_need(g, n_req, n_vec, FHTB_NEAR) : 0;
  s += align_up(h.near_bytes);
  h.total = s + 4096;
  return h;
}
}  // namespace

extern "C" {

size_t fhtb_apply_host_workspace(const fhtb_grid* g, int32_t n_req, int32_t n_vec, int32_t flags) {
  if (!g) return 0;
  return host_layout(g, n_req, n_vec, flags).total;
}

int fhtb_apply_host(const fhtb_grid* g, const fhtb_request* reqs, int32_t n_req, const double* C_host,
                    int64_t ldc_host, int32_t n_vec, double* F_host, int64_t ldf_host, int32_t flags,
                    int32_t n_groups, void* ws, size_t ws_bytes, void* stream) {
  if (!g) return fail(FHTB_EINVAL, "null grid");
  if (n_req < 0 || n_vec < 0) return fail(FHTB_EINVAL, "negative counts");
  if (!C_host || !F_host) return fail(FHTB_EINVAL, "null host buffer");
  if (ldc_host < g->n_data_cols || ldf_host < g->n_out) return fail(FHTB_EINVAL, "host leading dimension too small");
  if (n_vec == 0) return FHTB_OK;
  for (int q = 0; q < n_req; ++q)
    if (reqs[q].vec < 0 || reqs[q].vec >= n_vec) return fail(FHTB_EINVAL, "request vec out of range");
  const HostLayout hl = host_layout(g, n_req, n_vec, flags);
  if (ws_bytes < hl.total) return fail(FHTB_EINVAL, "workspace too small");
  char* base = (char*)align_up((size_t)ws);
  if (base + hl.total - 4096 > (char*)ws + ws_bytes) return fail(FHTB_EINVAL, "workspace too small");
  double* Cd = (double*)(base + hl.c_off);
  double* Fd = (double*)(base + hl.f_off);
  const long long ldc = g->n_data_cols, ldf = g->n_out;
  const bool near = (flags & FHTB_NEAR) && !g->tiles.empty();
  const bool far = (flags & FHTB_FAR) != 0;
  double* Fn = (near && far) ? (double*)(base + hl.fn_off) : Fd;
  cudaStream_t st = S(stream);
  HostAux* hx;
  if (int r = get_haux(st, &hx)) return r;
  DevCtx* ctx;
  if (int r = get_ctx(&ctx)) return r;
  const int G = std::max(1, std::min({(int)n_groups, (int)n_vec, kMaxHostGroups}));
  // tapered groups: the first group's copy-in and the last group's copy-out
  // are the exposed parts, so those two groups get 1/host_taper of the share
  // of the inner ones (weights 1, t, ..., t, 1)
  std::vector<int> v0(G + 1);
  {
    std::vector<double> cw(G + 1, 0.0);
    for (int i = 0; i < G; ++i) cw[i + 1] = cw[i] + ((G > 2 && (i == 0 || i == G - 1)) ? 1.0 : (double)g_host_taper);
    for (int i = 0; i <= G; ++i) v0[i] = (int)std::llround(n_vec * cw[i] / cw[G]);
    v0[G] = n_vec;
    for (int i = G - 1; i >= 1; --i) v0[i] = std::min(v0[i], v0[i + 1] - 1);   // every group non-empty
    for (int i = 1; i < G; ++i) v0[i] = std::max(v0[i], v0[i - 1] + 1);
  }
  // requests sorted by vector, grouped
  std::vector<int> perm(n_req);
  for (int i = 0; i < n_req; ++i) perm[i] = i;
  std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return reqs[a].vec < reqs[b].vec; });

  // inputs, group by group, on the copy stream (after the caller's prior work)
  CU(cudaEventRecord(hx->nstart, st));
  CU(cudaStreamWaitEvent(hx->h2d, hx->nstart, 0));
  for (int i = 0; i < G; ++i) {
    const int nv = v0[i + 1] - v0[i];
    CU(cudaMemcpy2DAsync(Cd + (size_t)v0[i] * ldc, ldc * sizeof(double), C_host + (size_t)v0[i] * ldc_host,
                         ldc_host * sizeof(double), ldc * sizeof(double), nv, cudaMemcpyHostToDevice, hx->h2d));
    CU(cudaEventRecord(hx->in[i], hx->h2d));
  }
  // near field of the whole batch on its own stream
  if (near) {
    CU(cudaStreamWaitEvent(hx->near, hx->in[G - 1], 0));
    if (far) CU(cudaMemsetAsync(Fn, 0, sizeof(double) * (size_t)n_vec * ldf, hx->near));
    else CU(cudaMemsetAsync(Fd, 0, sizeof(double) * (size_t)n_vec * ldf, hx->near));
    if (int r = apply_impl(g, reqs, n_req, Cd, ldc, n_vec, Fn, ldf, FHTB_NEAR, 0, 1, nullptr, base + hl.near_off,
                           hl.near_bytes, hx->near))
      return r;
    CU(cudaEventRecord(hx->ndone, hx->near));
  }
  std::vector<fhtb_request> sub;
  size_t q = 0;
  for (int i = 0; i < G; ++i) {
    const int nv = v0[i + 1] - v0[i];
    double* Fg = Fd + (size_t)v0[i] * ldf;
    if (far) {
      sub.clear();
      while (q < perm.size() && reqs[perm[q]].vec < v0[i + 1]) {
        fhtb_request r = reqs[perm[q]];
        r.vec -= v0[i];
        sub.push_back(r);
        ++q;
      }
      CU(cudaMemsetAsync(Fg, 0, sizeof(double) * (size_t)nv * ldf, st));
      // region i % 2 was last used by group i - 2 (done when fin[i-2] fired)
      const HostPipe hp{hx->in[i], i >= 2 ? hx->fin[i - 2] : nullptr};
      if (!sub.empty())
        if (int r = apply_impl(g, sub.data(), (int)sub.size(), Cd + (size_t)v0[i] * ldc, ldc, nv, Fg, ldf, FHTB_FAR,
                               0, 1, nullptr, base + hl.far_off + (i & 1) * align_up(hl.far_bytes), hl.far_bytes,
                               st, &hp))
          return r;
    }
    if (!near && !far) CU(cudaMemsetAsync(Fg, 0, sizeof(double) * (size_t)nv * ldf, st));
    // the near-field add and the copy-out of group i run on the d2h stream:
    // the caller's stream goes straight on to the far field of group i+1
    // instead of waiting there for the near field (which needs every group's
    // rows and so finishes only after the first groups' far fields)
    CU(cudaEventRecord(hx->fin[i], st));
    CU(cudaStreamWaitEvent(hx->d2h, hx->fin[i], 0));
    if (near) {
      CU(cudaStreamWaitEvent(hx->d2h, hx->ndone, 0));
      if (far) CU(launch_add_rows(Fg, ldf, Fn + (size_t)v0[i] * ldf, ldf, nv, ldf, ctx->nf, hx->d2h));
    }
    CU(cudaMemcpy2DAsync(F_host + (size_t)v0[i] * ldf_host, ldf_host * sizeof(double), Fg, ldf * sizeof(double),
                         ldf * sizeof(double), nv, cudaMemcpyDeviceToHost, hx->d2h));
  }
  // the caller's stream completes after the last output copy
  CU(cudaEventRecord(hx->fin[0], hx->d2h));
  CU(cudaStreamWaitEvent(st, hx->fin[0], 0));
  return FHTB_OK;
}

}  // extern "C"

namespace {

// Full (dmode 0) far-field units by the distributed four-step: per round of
// units, pass 1 over this rank's column slab into the send buffer (rows
// grouped by owning rank), the caller's exchange (all-to-all), pass 2 over
// this rank's column pairs from the receive buffer, reduction into F.
int run_exchange(const fhtb_grid* g, DevCtx* ctx, const std::vector<ReqDesc>& rs, const ReqDesc* d_req,
                 const double* C, int64_t ldc, double* F, int64_t ldf, int rank, int world, int l1, int rows,
                 const XCtx& xc, Carve& cv, cudaStream_t st) {
  std::vector<UnitDesc> units = x_units(g, rs);
  const int n = (int)units.size();
  if (n == 0) return FHTB_OK;
  const int l2 = g->logQ - l1, L1 = 1 << l1, L2 = 1 << l2, cols = L1 / world;
  const long long per = (long long)g->M * rows * cols;                       // elements per unit per peer
  const long long U = (long long)(xc.bytes / ((size_t)world * per * sizeof(double2)));
  if (U < 1) return fail(FHTB_EINVAL, "exchange buffers too small for one unit");
  std::vector<int2> xrow(L2);
  for (int s = 0; s < world; ++s) {
    int lo, cnt;
    x_pairs(L2, world, s, &lo, &cnt);
    for (int c = lo; c < lo + cnt; ++c) {
      xrow[c] = make_int2(s, c - lo);
      const int p = (L2 - c) % L2;
      if (p != c) xrow[p] = make_int2(s, cnt + c - lo);
    }
  }
  UnitDesc* d_units = cv.take<UnitDesc>(n);
  int2* d_xrow = cv.take<int2>(L2);
  double* part = cv.take<double>((size_t)std::min<long long>(U, n) * g->n_out);
  if (!cv.ok) return fail(FHTB_EINVAL, "workspace too small (exchange mode)");
  CU(h2d_tables(d_units, units.data(), n * sizeof(UnitDesc), st));
  CU(h2d_tables(d_xrow, xrow.data(), L2 * sizeof(int2), st));
  FarArgs a;
  std::memset(&a, 0, sizeof a);
  a.L = g->L;
  a.M = g->M;
  a.gamma = g->gamma;
  a.Ld = (double)g->L;
  a.pi_over_L = M_PI / (double)g->L;
  a.first = g->first;
  a.stride = g->stride;
  a.n_out = g->n_out;
  a.n_data_cols = g->n_data_cols;
  a.units = d_units;
  a.reqs = d_req;
  a.blocks = g->d_blocks;
  a.C = C;
  a.ldc = ldc;
  a.F = F;
  a.ldf = ldf;
  a.tw = ctx->tw;
  a.nf = ctx->nf;
  a.part = part;
  a.part_stride = g->n_out;
  a.cs_tab = g->cs_tab;
  a.w0_tab = g->w0_tab;
  a.iw_tab = g->iw_tab;
  a.p0 = 0;
  a.p1 = g->M;
  a.L1 = L1;
  a.L2 = L2;
  a.logQ = g->logQ;
  double2 *ql, *qh;
  int qb;
  if (int r = get_qtab(ctx, g->logQ, &ql, &qh, &qb)) return r;
  a.qlo = ql;
  a.qhi = qh;
  a.qbits = qb;
  a.xw = world;
  a.xlog = ilog2ll(cols);
  a.xrows = rows;
  a.xn1 = (long long)rank * cols;
  a.xchunk = U * per;
  a.xrow = d_xrow;
  int lo, cnt;
  x_pairs(L2, world, rank, &lo, &cnt);
  for (int r0 = 0, round = 0; r0 < n; r0 += (int)U, ++round) {
    const int nu = (int)std::min<long long>(U, n - r0);
    a.u0 = r0;
    a.G = (double2*)xc.send;
    a.xc0 = 0;
    CU(launch_far_pass1(a, l2, nu, st));
    if (int r = xc.exchange(xc.user, round, (size_t)a.xchunk * sizeof(double2)))
      return fail(FHTB_ECUDA, "exchange callback failed (" + std::to_string(r) + ")");
    a.G = nullptr;
    a.xin = (const double2*)xc.recv;
    a.xc0 = lo;
    CU(cudaMemsetAsync(part, 0, sizeof(double) * (size_t)nu * g->n_out, st));
    if (cnt > 0) CU(launch_far_pass2x_range(a, l1, cnt, nu, st));
    CU(launch_far_reduce(a, nu, st));
  }
  return FHTB_OK;
}

// Nominal FFT flops of one far-field chunk per launch (5 n log2 n per executed
// transform of n points, zero padding included, epilogues excluded):
// [0] first launch, [1] second, [2] third (chirp pass 3).
void chunk_flops(const fhtb_grid* g, const FarPlan& fp, size_t ci, int npairs, double out[3]) {
  out[0] = out[1] = out[2] = 0.0;
  const int2 ch = fp.chunks[ci];
  for (int u = ch.x; u < ch.y; ++u) {
    const BlockDesc& x = g->bdesc[fp.units[u].block];
    const double np = (double)npairs;
    if (!g->direct) {
      int l1, l2;
      split_q(x.logQ, &l1, &l2);
      const double Q = (double)(1LL << x.logQ);
      out[0] += 2.0 * np * 5.0 * Q * l2;
      out[1] += 2.0 * np * 2.0 * 5.0 * Q * l1;
      out[2] += 2.0 * np * 5.0 * Q * l2;
      continue;
    }
    const double Q = (double)(1LL << g->logQ);
    if (g->logN2 == 0) {
      out[0] += np * 5.0 * Q * g->logQ;
    } else if (x.dmode == 1) {
      out[0] += np * 5.0 * Q * x.dlogL1;
    } else if (x.dmode >= 2) {
      out[0] += np * 5.0 * Q * (g->logQ - x.dlogL1);
    } else {
      out[0] += np * 5.0 * Q * (g->logQ - x.dlogL1);
      out[1] += np * 5.0 * Q * x.dlogL1;
    }
  }
}

// Algorithmic bytes of one far-field chunk per kernel family (kernel timing;
// the per-unit terms of fhtb_grid_far_model_bytes, restricted to this shard's
// pairs): [0] the first launch (pass 1 / column tables / chirp pass 1 / one
// pass), [1] the second (pass 2 / row sums / chirp pass 2), [2] chirp pass 3,
// [3] the reduction into F.
void chunk_bytes(const fhtb_grid* g, const FarPlan& fp, size_t ci, const std::vector<ReqDesc>& rs, int npairs,
                 double out[4]) {
  out[0] = out[1] = out[2] = out[3] = 0.0;
  const int2 ch = fp.chunks[ci];
  const double L = (double)g->L, np = (double)npairs;
  int last_vec = -1;
  for (int u = ch.x; u < ch.y; ++u) {
    const UnitDesc& ud = fp.units[u];
    const BlockDesc& x = g->bdesc[ud.block];
    const double c0 = (double)std::max<long long>(x.c0, rs[ud.req].col_lo);
    const double cols = std::max(0.0, (double)std::min(x.c1, g->n_data_cols + 1) - c0);
    if (ud.vec != last_vec) out[3] += 16.0 * (double)g->n_out;       // F read + write per vector
    last_vec = ud.vec;
    if (!g->direct) {
      const double Q = (double)(1LL << x.logQ), J = (double)x.J;
      out[0] += 2.0 * np * 16.0 * Q + 8.0 * cols;
      out[1] += 2.0 * np * 32.0 * Q;
      out[2] += 2.0 * np * 16.0 * Q + 8.0 * J;
      out[3] += 8.0 * (double)g->n_out;
      continue;
    }
    const double rows = (double)std::max<long long>(0, x.r1 - x.r0);
    out[3] += 8.0 * rows;
    if (g->logN2 == 0) {
      out[0] += 8.0 * cols + 8.0 * rows;
    } else if (x.dmode == 1) {
      const double l1 = (double)(1LL << x.dlogL1);
      out[0] += 8.0 * cols + np * 16.0 * l1;                          // column table written
      out[1] += np * 16.0 * l1 + 8.0 * rows;                          // read, partial row
    } else if (x.dmode >= 3) {
      const double l1 = (double)(1LL << x.dlogL1);
      out[0] += 8.0 * cols + 32.0 * rows * l1;                        // folded rows written
      out[1] += 32.0 * rows * l1 + 8.0 * rows;                        // read, partial row
    } else {
      out[0] += np * 32.0 * L + 8.0 * cols;                           // G written
      double rd = 1.0;
      if (x.dmode == 2) rd = std::min(1.0, 2.0 * (rows + 1) / (double)(1LL << (g->logQ - x.dlogL1)));
      out[1] += np * 32.0 * L * rd + 8.0 * rows;                      // G read, partial row
    }
  }
}

int apply_impl(const fhtb_grid* g, const fhtb_request* reqs, int32_t n_req, const double* C, int64_t ldc,
               int32_t n_vec, double* F, int64_t ldf, int32_t flags, int32_t shard, int32_t n_shards,
               const XCtx* xc, void* ws, size_t ws_bytes, void* stream, const HostPipe* hp) {
  if (!g) return fail(FHTB_EINVAL, "null grid");
  if (hp && (flags != FHTB_FAR || xc || n_shards != 1)) return fail(FHTB_EINVAL, "host pipe: far field only");
  if (n_shards < 1 || shard < 0 || shard >= n_shards) return fail(FHTB_EINVAL, "bad shard index");
  if (n_req < 0 || n_vec < 0) return fail(FHTB_EINVAL, "negative counts");
  if (n_req == 0 || n_vec == 0) return FHTB_OK;
  for (int q = 0; q < n_req; ++q)
    if (reqs[q].vec < 0 || reqs[q].vec >= n_vec) return fail(FHTB_EINVAL, "request vec out of range");
  const size_t need = ws_need(g, n_req, n_vec, flags) + (xc ? x_ws(g, n_req, n_shards, xc->bytes) : 0);
  if (ws_bytes < need) return fail(FHTB_EINVAL, "workspace too small");
  DevCtx* ctx;
  if (int r = get_ctx(&ctx)) return r;
  cudaStream_t st = S(stream);

  std::vector<ReqDesc> rd;
  if (int r = pack_requests(reqs, n_req, g->M, g->orders, g->n_data_cols, rd)) return r;
  std::vector<int> perm(n_req);
  for (int i = 0; i < n_req; ++i) perm[i] = i;
  std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return rd[a].vec < rd[b].vec; });
  std::vector<ReqDesc> rs(n_req);
  for (int i = 0; i < n_req; ++i) rs[i] = rd[perm[i]];

  Carve cv{(char*)ws, ws_bytes};
  ReqDesc* d_req = cv.take<ReqDesc>(n_req);
  if (!hp) CU(h2d_tables(d_req, rs.data(), n_req * sizeof(ReqDesc), st));

  // Near field concurrently with the far field (both requested): it runs on
  // an auxiliary stream into a separate buffer Fn, added to F at the end on
  // the caller's stream (F = far sum + near sum, as in the serial order).
  const bool overlap = (flags & FHTB_NEAR) && (flags & FHTB_FAR) && !g->tiles.empty() &&
                       !g->blocks.empty() && g_near_overlap && !g_serial;
  cudaStream_t nst = st;
  double* Fn = F;
  int64_t ldfn = ldf;
  AuxStreams* nax = nullptr;
  if (overlap) {
    if (int r = get_aux(st, &nax)) return r;
    Fn = cv.take<double>((size_t)n_vec * g->n_out);
    if (!cv.ok) return fail(FHTB_EINVAL, "workspace too small");
    ldfn = g->n_out;
    nst = nax->cs[2];
    CU(cudaEventRecord(nax->nstart, st));
    CU(cudaStreamWaitEvent(nst, nax->nstart, 0));
    CU(cudaMemsetAsync(Fn, 0, sizeof(double) * (size_t)n_vec * g->n_out, nst));
  }
  if ((flags & FHTB_NEAR) && !g->tiles.empty()) {
    std::vector<int> q0, v0;
    std::vector<int2> cls;
    std::vector<ReqDesc> nreq;
    int max_cols = 0;
    bool identity = true;
    for (int i = 0; i < (int)g->orders.size(); ++i) identity = identity && g->orders[i] == i;
    const bool split = identity && g->orders.size() >= 3 && g_near_split;
    if (split) {
      if (int r = make_groups_split(rs, n_vec, (int)g->orders.size(), nreq, q0, v0, cls, &max_cols)) return r;
    } else {
      if (int r = make_groups(rs, n_vec, q0, v0, &max_cols)) return r;
    }
    std::vector<int> vstart, vcol;
    vec_columns(split ? nreq : rs, q0, n_vec, vstart, vcol);
    int* d_q0 = cv.take<int>(q0.size());
    int* d_v0 = cv.take<int>(v0.size());
    int* d_vs = cv.take<int>(vstart.size());
    int* d_vc = cv.take<int>(vcol.size());
    int2* d_cls = split ? cv.take<int2>(cls.size()) : nullptr;
    ReqDesc* d_nreq = split ? cv.take<ReqDesc>(nreq.size()) : nullptr;
    double* part = g->n_slots ? cv.take<double>((size_t)g->n_slots * n_vec * kNearRT) : nullptr;
    if (!cv.ok) return fail(FHTB_EINVAL, "workspace too small");
    CU(h2d_tables(d_q0, q0.data(), q0.size() * sizeof(int), nst));
    CU(h2d_tables(d_v0, v0.data(), v0.size() * sizeof(int), nst));
    CU(h2d_tables(d_vs, vstart.data(), vstart.size() * sizeof(int), nst));
    CU(h2d_tables(d_vc, vcol.data(), vcol.size() * sizeof(int), nst));
    if (split) {
      CU(h2d_tables(d_cls, cls.data(), cls.size() * sizeof(int2), nst));
      CU(h2d_tables(d_nreq, nreq.data(), nreq.size() * sizeof(ReqDesc), nst));
    }
    NearArgs na;
    std::memset(&na, 0, sizeof na);
    na.tiles = g->d_tiles;
    na.first = g->first;
    na.stride = g->stride;
    na.rowv = nullptr;
    na.colv = nullptr;
    na.gamma = g->gamma;
    na.scale = M_PI / (double)g->L;
    na.Ld = (double)g->L;
    na.n_orders = (int)g->orders.size();
    na.omax = 0;
    na.omin = g->orders[0];
    na.orders_identity = 1;
    for (int i = 0; i < na.n_orders; ++i) {
      na.orders[i] = g->orders[i];
      na.omax = std::max(na.omax, g->orders[i]);
      na.omin = std::min(na.omin, g->orders[i]);
      if (g->orders[i] != i) na.orders_identity = 0;
    }
    na.jtab = ctx->jtab;
    na.nf = ctx->nf;
    na.reqs = split ? d_nreq : d_req;
    na.grp_q0 = d_q0;
    na.grp_v0 = d_v0;
    na.grp_cls = d_cls;
    na.vstart = d_vs;
    na.vcol = d_vc;
    na.C = C;
    na.ldc = ldc;
    na.n_data_cols = g->n_data_cols;
    na.F = Fn;
    na.ldf = ldfn;
    na.part = part;
    na.part_stride = (long long)n_vec * kNearRT;
    na.overwrite = 0;
    na.shard = shard;
    na.n_shards = n_shards;
    KT(kfNear, nst, 0.0, launch_near(na, (int)g->tiles.size(), (int)q0.size() - 1, max_cols, nst));
    KT(kfNearReduce, nst, 0.0, launch_near_reduce(g->d_rts, (int)g->rts.size(), part, Fn, ldfn, n_vec, 0, ctx->nf, nst));
  }
  if (overlap) CU(cudaEventRecord(nax->ndone, nst));

  // this shard's asymptotic term pairs [p0, p1) (all units) -- SURVEY 8(e)
  const int p0 = (int)((long long)g->M * shard / n_shards), p1 = (int)((long long)g->M * (shard + 1) / n_shards);
  int xl1 = 0, xrows = 0;
  const bool xmode = xc && (flags & FHTB_FAR) && x_supported(g, n_shards, &xl1, &xrows);
  if (xmode) {
    if (int r = run_exchange(g, ctx, rs, d_req, C, ldc, F, ldf, shard, n_shards, xl1, xrows, *xc, cv, st)) return r;
  }
  if ((flags & FHTB_FAR) && !g->blocks.empty() && p1 > p0) {
    FarPlan fp;
    plan_far(g, rs, fp, xmode ? 1 : 0);
    const long long nu = (long long)fp.units.size();
    if (nu > 0) {
      UnitDesc* d_units = cv.take<UnitDesc>(nu);
      int2* d_ch = cv.take<int2>(fp.chunks.size());
      double2* G = fp.g_bytes ? (double2*)cv.take<char>(fp.g_bytes) : nullptr;
      double* part = fp.part_bytes ? (double*)cv.take<char>(fp.part_bytes) : nullptr;
      // second buffer set: two chunks in flight on two streams (direct two-pass)
      const bool pipe = g->direct && g->logN2 > 0 && g_far_streams > 1 && fp.chunks.size() > 1 && !g_serial;
      double2* G2 = (pipe && fp.g_bytes) ? (double2*)cv.take<char>(fp.g_bytes) : nullptr;
      double* part2 = (pipe && fp.part_bytes) ? (double*)cv.take<char>(fp.part_bytes) : nullptr;
      if (!cv.ok) return fail(FHTB_EINVAL, "workspace too small");
      AuxStreams* ax = nullptr;
      if (pipe) {
        if (int r = get_aux(st, &ax)) return r;
      }
      // tables: on the caller's stream, or (host pipe) on the first aux stream
      cudaStream_t ts = st;
      if (hp) {
        ts = pipe ? ax->cs[0] : st;
        CU(cudaStreamWaitEvent(ts, hp->ready, 0));
        if (hp->region_free) CU(cudaStreamWaitEvent(ts, hp->region_free, 0));
        // (host pipe: plain pageable copies.  Their implicit wait for the stream paces the
        // host to one vector group ahead of the device; with the pinned ring the host
        // enqueues all groups at once and the copy-in of later groups competes with the
        // copy-out of earlier ones: e2e 871 -> 784 transforms/s on cfg2)
        CU(cudaMemcpyAsync(d_req, rs.data(), n_req * sizeof(ReqDesc), cudaMemcpyHostToDevice, ts));
        CU(cudaMemcpyAsync(d_units, fp.units.data(), nu * sizeof(UnitDesc), cudaMemcpyHostToDevice, ts));
        CU(cudaMemcpyAsync(d_ch, fp.chunks.data(), fp.chunks.size() * sizeof(int2), cudaMemcpyHostToDevice, ts));
      } else {
        CU(h2d_tables(d_units, fp.units.data(), nu * sizeof(UnitDesc), ts));
        CU(h2d_tables(d_ch, fp.chunks.data(), fp.chunks.size() * sizeof(int2), ts));
      }
      FarArgs a;
      std::memset(&a, 0, sizeof a);
      a.L = g->L;
      a.M = g->M;
      a.gamma = g->gamma;
      a.Ld = (double)g->L;
      a.pi_over_L = M_PI / (double)g->L;
      a.first = g->first;
      a.stride = g->stride;
      a.n_out = g->n_out;
      a.n_data_cols = g->n_data_cols;
      a.units = d_units;
      a.reqs = d_req;
      a.blocks = g->d_blocks;
      a.C = C;
      a.ldc = ldc;
      a.F = F;
      a.ldf = ldf;
      a.tw = ctx->tw;
  a.nf = ctx->nf;
      a.G = G;
      a.part = part;
      a.part_stride = g->n_out;
      a.cs_tab = g->cs_tab;
      a.w0_tab = g->w0_tab;
      a.iw_tab = g->iw_tab;
      a.p0 = p0;
      a.p1 = p1;
      if (g->direct && g->logN2 == 0) {
        a.L1 = 1 << g->logN1;
        a.L2 = 1;
        a.logQ = g->logQ;
        a.vranges = d_ch;
        a.u0 = 0;
        double cb[4], cf[3];
        chunk_bytes(g, fp, 0, rs, p1 - p0, cb);
        chunk_flops(g, fp, 0, p1 - p0, cf);
        t_kt_flops = cf[0];
        KT(kfOnepass, st, cb[0], launch_far_onepass(a, g->logN1, (int)nu, st));
        KT(kfReduce, st, cb[3], launch_far_reduce(a, (int)nu, st));
      } else {
        if (pipe && hp) {
          // the second aux stream and the reductions wait for the tables only
          CU(cudaEventRecord(ax->start, ax->cs[0]));
          CU(cudaStreamWaitEvent(ax->cs[1], ax->start, 0));
          CU(cudaStreamWaitEvent(st, ax->start, 0));
        } else if (pipe) {
          // the aux streams start after the caller's prior work (C, F ready)
          CU(cudaEventRecord(ax->start, st));
          for (int b = 0; b < 2; ++b) CU(cudaStreamWaitEvent(ax->cs[b], ax->start, 0));
        }
        for (size_t ci = 0; ci < fp.chunks.size(); ++ci) {
          const int lq = fp.chunk_logq[ci];
          const int n_units = fp.chunks[ci].y - fp.chunks[ci].x;
          double2 *ql, *qh;
          int qb;
          if (int r = get_qtab(ctx, lq, &ql, &qh, &qb)) return r;
          double cb[4], cf[3];
          chunk_bytes(g, fp, ci, rs, p1 - p0, cb);
          chunk_flops(g, fp, ci, p1 - p0, cf);
          a.qlo = ql;
          a.qhi = qh;
          a.qbits = qb;
          a.logQ = lq;
          a.u0 = fp.chunks[ci].x;
          if (g->direct) {
            const int mode = fp.chunk_key[ci] / 64, l1 = fp.chunk_key[ci] % 64, l2 = g->logQ - l1;
            a.L1 = 1 << l1;
            a.L2 = 1 << l2;
            a.vranges = d_ch + ci;
            // pipelined: chunk ci computes on aux stream b with buffer set b
            // once the reduction of chunk ci-2 (same buffers) is done; the
            // reductions stay on the caller's stream in chunk order, so F is
            // accumulated exactly as in the serial schedule
            const int b = (int)(ci & 1);
            cudaStream_t cs = st;
            if (pipe) {
              cs = ax->cs[b];
              a.G = b ? G2 : G;
              a.part = b ? part2 : part;
              if (ci >= 2) CU(cudaStreamWaitEvent(cs, ax->red[b], 0));
            }
            if (mode != 1 && g_far_prefetch) KT(kfOther, cs, 0.0, launch_prefetch_rows(a, n_units, cs));
            if (mode == 1) {
              t_kt_flops = cf[0];
              KT(kfNarrow, cs, cb[0] + cb[1], launch_far_colgen(a, l1, n_units, cs));
            } else if (mode >= 3) {
              long long rs = 1;
              for (int u = fp.chunks[ci].x; u < fp.chunks[ci].y; ++u)
                rs = std::max(rs, fused_rows(g, g->bdesc[fp.units[u].block], l1));
              a.rs = (int)rs;
              t_kt_flops = cf[0];
              KT(kfRowsum, cs, cb[0], launch_far_rowsum(a, l2, mode - 3, n_units, cs));
              KT(kfRowsumFin, cs, cb[1], launch_far_rowsum_fin(a, n_units, cs));
            } else if (mode == 2) {
              t_kt_flops = cf[0];
              KT(kfPass1, cs, cb[0], launch_far_pass1(a, l2, n_units, cs));
              int kb = 1;
              for (int u = fp.chunks[ci].x; u < fp.chunks[ci].y; ++u)
                kb = std::max(kb, g->bdesc[fp.units[u].block].kbins);
              KT(kfRowdot, cs, cb[1], launch_far_rowdot(a, n_units, kb, cs));
            } else {
              t_kt_flops = cf[0];
              KT(kfPass1, cs, cb[0], launch_far_pass1(a, l2, n_units, cs));
              t_kt_flops = cf[1];
              KT(kfPass2, cs, cb[1], launch_far_pass2(a, l1, n_units, cs));
            }
            if (pipe) {
              CU(cudaEventRecord(ax->done[b], cs));
              CU(cudaStreamWaitEvent(st, ax->done[b], 0));
            }
            KT(kfReduce, st, cb[3], launch_far_reduce(a, n_units, st));
            if (pipe) CU(cudaEventRecord(ax->red[b], st));
          } else {
            int l1, l2;
            split_q(lq, &l1, &l2);
            a.L1 = 1 << l1;
            a.L2 = 1 << l2;
            CU(cudaMemsetAsync(part, 0, sizeof(double) * (size_t)n_units * g->n_out, st));
            t_kt_flops = cf[0];
              KT(kfChirp1, st, cb[0], launch_chirp_pass1(a, l2, n_units, fp.chunk_key[ci], st));
            t_kt_flops = cf[1];
              KT(kfChirp2, st, cb[1], launch_chirp_pass2(a, l1, n_units, st));
            t_kt_flops = cf[2];
              KT(kfChirp3, st, cb[2], launch_chirp_pass3(a, l2, n_units, st));
            KT(kfChirpReduce, st, cb[3], launch_chirp_reduce(a, n_units, st));
          }
        }
      }
    }
  }

  if (overlap) {
    CU(cudaStreamWaitEvent(st, nax->ndone, 0));
    KT(kfOther, st, 0.0, launch_add_rows(F, ldf, Fn, ldfn, n_vec, g->n_out, ctx->nf, st));
  }
  return FHTB_OK;
}

}  // namespace

extern "C" {

// --------------------------------------------------------------- direct
namespace {
void direct_tiles(const fhtb_direct_desc* d, std::vector<NearTile>& tiles, std::vector<NearRowTile>& rts,
                  long long& n_slots) {
  std::vector<long long> seg = {1, d->n_rows + 1, d->n_cols + 1};
  make_tiles(seg, 1, 1, std::min(d->n_data_cols, d->n_cols), d->n_rows, d->n_orders, tiles, rts, n_slots);
}
}  // namespace

size_t fhtb_direct_workspace(const fhtb_direct_desc* d, int32_t n_req, int32_t n_vec) {
  if (!d) return 0;
  std::vector<NearTile> tiles;
  std::vector<NearRowTile> rts;
  long long ns = 0;
  direct_tiles(d, tiles, rts, ns);
  size_t s = align_up(sizeof(ReqDesc) * std::max(n_req, 1));
  s += align_up(sizeof(NearTile) * std::max<size_t>(tiles.size(), 1));
  s += align_up(sizeof(NearRowTile) * std::max<size_t>(rts.size(), 1));
  s += 2 * align_up(sizeof(int) * (n_vec + 2));
  s += align_up(sizeof(int) * (n_vec + 2)) + align_up(sizeof(int) * ((size_t)n_req + 2));
  s += align_up(sizeof(double) * (size_t)ns * n_vec * kNearRT);
  return s + 4096;
}

int fhtb_direct_apply(const fhtb_direct_desc* d, const fhtb_request* reqs, int32_t n_req, const double* C,
                      int64_t ldc, int32_t n_vec, double* F, int64_t ldf, int32_t flags, void* ws,
                      size_t ws_bytes, void* stream) {
  if (!d) return fail(FHTB_EINVAL, "null descriptor");
  if (d->n_orders < 1 || d->n_orders > kMaxOrd) return fail(FHTB_EINVAL, "order universe size out of range");
  if (n_req == 0 || n_vec == 0 || d->n_rows == 0) return FHTB_OK;
  for (int q = 0; q < n_req; ++q)
    if (reqs[q].vec < 0 || reqs[q].vec >= n_vec) return fail(FHTB_EINVAL, "request vec out of range");
  if (ws_bytes < fhtb_direct_workspace(d, n_req, n_vec)) return fail(FHTB_EINVAL, "workspace too small");
  DevCtx* ctx;
  if (int r = get_ctx(&ctx)) return r;
  cudaStream_t st = S(stream);
  std::vector<int> uni(d->orders, d->orders + d->n_orders);
  std::vector<ReqDesc> rd;
  if (int r = pack_requests(reqs, n_req, 1, uni, d->n_data_cols, rd)) return r;
  std::vector<int> perm(n_req);
  for (int i = 0; i < n_req; ++i) perm[i] = i;
  std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return rd[a].vec < rd[b].vec; });
  std::vector<ReqDesc> rs(n_req);
  for (int i = 0; i < n_req; ++i) rs[i] = rd[perm[i]];
  std::vector<NearTile> tiles;
  std::vector<NearRowTile> rts;
  long long ns = 0;
  direct_tiles(d, tiles, rts, ns);
  std::vector<int> q0, v0;
  int max_cols = 0;
  if (int r = make_groups(rs, n_vec, q0, v0, &max_cols)) return r;
  Carve cv{(char*)ws, ws_bytes};
  ReqDesc* d_req = cv.take<ReqDesc>(n_req);
  NearTile* d_tiles = cv.take<NearTile>(std::max<size_t>(tiles.size(), 1));
  NearRowTile* d_rts = cv.take<NearRowTile>(std::max<size_t>(rts.size(), 1));
  std::vector<int> vstart, vcol;
  vec_columns(rs, q0, n_vec, vstart, vcol);
  int* d_q0 = cv.take<int>(q0.size());
  int* d_v0 = cv.take<int>(v0.size());
  int* d_vs = cv.take<int>(vstart.size());
  int* d_vc = cv.take<int>(vcol.size());
  double* part = ns ? cv.take<double>((size_t)ns * n_vec * kNearRT) : nullptr;
  if (!cv.ok) return fail(FHTB_EINVAL, "workspace too small");
  CU(h2d_tables(d_req, rs.data(), n_req * sizeof(ReqDesc), st));
  CU(h2d_tables(d_vs, vstart.data(), vstart.size() * sizeof(int), st));
  CU(h2d_tables(d_vc, vcol.data(), vcol.size() * sizeof(int), st));
  if (!tiles.empty()) CU(h2d_tables(d_tiles, tiles.data(), tiles.size() * sizeof(NearTile), st));
  if (!rts.empty()) CU(h2d_tables(d_rts, rts.data(), rts.size() * sizeof(NearRowTile), st));
  CU(h2d_tables(d_q0, q0.data(), q0.size() * sizeof(int), st));
  CU(h2d_tables(d_v0, v0.data(), v0.size() * sizeof(int), st));
  NearArgs na;
  std::memset(&na, 0, sizeof na);
  na.tiles = d_tiles;
  na.first = 1;
  na.stride = 1;
  na.rowv = d->row_val;
  na.colv = d->col_val;
  na.Ld = d->r_scale;
  na.n_orders = d->n_orders;
  na.orders_identity = 1;
  na.omin = d->orders[0];
  for (int i = 0; i < d->n_orders; ++i) {
    na.orders[i] = d->orders[i];
    na.omax = std::max(na.omax, d->orders[i]);
    na.omin = std::min(na.omin, d->orders[i]);
    if (d->orders[i] != i) na.orders_identity = 0;
    if (d->orders[i] < 0 || d->orders[i] > kMaxOrder) return fail(FHTB_EINVAL, "order out of range");
  }
  if (na.omax - na.omin >= kMaxOrd) return fail(FHTB_EINVAL, "order universe spans more than 16 orders");
  na.jtab = ctx->jtab;
    na.nf = ctx->nf;
  na.reqs = d_req;
  na.grp_q0 = d_q0;
  na.grp_v0 = d_v0;
  na.vstart = d_vs;
  na.vcol = d_vc;
  na.C = C;
  na.ldc = ldc;
  na.n_data_cols = std::min(d->n_data_cols, d->n_cols);
  na.F = F;
  na.ldf = ldf;
  na.part = part;
  na.part_stride = (long long)n_vec * kNearRT;
  na.overwrite = (flags & FHTB_OVERWRITE) ? 1 : 0;
  CU(launch_near(na, (int)tiles.size(), (int)q0.size() - 1, max_cols, st));
  CU(launch_near_reduce(d_rts, (int)rts.size(), part, F, ldf, n_vec, na.overwrite, ctx->nf, st));
  return FHTB_OK;
}


// ------------------------------------------------------------ DCT-I/DST-I
// DCT-I: out[k] = Re sum_{m<n} v_m e^{i pi k m/(n-1)},  k < n   (trig.py:59-66)
// DST-I: out[k] = Im sum_{m<n} v_m e^{i pi (k+1)(m+1)/(n+1)}    (trig.py:69-77)
static int trig_geom(int kind, int64_t n, long long* L, long long* k0, int* logQ) {
  if (kind == FHTB_DCT1) {
    if (n < 2) return fail(FHTB_EINVAL, "DCT-I needs length >= 2");
    *L = n - 1;
    *k0 = 0;
  } else if (kind == FHTB_DST1) {
    if (n < 1) return fail(FHTB_EINVAL, "DST-I needs length >= 1");
    *L = n + 1;
    *k0 = 1;
  } else {
    return fail(FHTB_EINVAL, "kind must be DCT1 or DST1");
  }
  *logQ = std::max(1, ilog2ll(2 * n - 1));
  // Q <= 8192: one CTA per row; beyond, the multi-pass FFT (Q <= 2^26)
  if (*logQ > 26) return fail(FHTB_EINVAL, "trig_apply supports length <= 2^25");
  return FHTB_OK;
}

size_t fhtb_trig_workspace(int kind, int64_t length, int64_t batch) {
  (void)batch;
  long long L, k0;
  int lq;
  if (trig_geom(kind, length, &L, &k0, &lq)) return 0;
  return (lq > 13 ? 4 : 3) * align_up(sizeof(double2) << lq) + 4096;
}

int fhtb_trig_apply(int kind, int64_t length, const double* v, int64_t batch, double* out, void* ws,
                    size_t ws_bytes, void* stream) {
  long long L, k0;
  int lq;
  if (int r = trig_geom(kind, length, &L, &k0, &lq)) return r;
  if (batch == 0) return FHTB_OK;
  if (ws_bytes < fhtb_trig_workspace(kind, length, batch)) return fail(FHTB_EINVAL, "workspace too small");
  DevCtx* ctx;
  if (int r = get_ctx(&ctx)) return r;
  cudaStream_t st = S(stream);
  Carve cv{(char*)ws, ws_bytes};
  const long long Q = 1LL << lq;
  double2* h = cv.take<double2>(Q);
  double2* tmp = cv.take<double2>(Q);
  double2* H = cv.take<double2>(Q);
  CU(launch_chirp_filter(h, Q, length, length, 1, L, st));
  if (int r = plain_fft(ctx, lq, h, tmp, H, 0, st)) return r;
  if (lq <= 13) {
    CU(launch_trig(kind, lq, length, L, k0, k0, v, out, batch, H, ctx->tw, st));
    return FHTB_OK;
  }
  double2* A = h;
  double2* A2 = cv.take<double2>(Q);
  if (!cv.ok) return fail(FHTB_EINVAL, "workspace too small");
  for (int64_t b = 0; b < batch; ++b) {
    CU(launch_trig_pre(v + b * length, length, L, k0, Q, A, st));
    if (int r = plain_fft(ctx, lq, A, tmp, A2, 0, st)) return r;
    CU(launch_trig_mid(A2, H, Q, A, st));
    if (int r = plain_fft(ctx, lq, A, tmp, A2, 0, st)) return r;
    CU(launch_trig_post(kind, A2, length, L, k0, k0, Q, out + b * length, st));
  }
  return FHTB_OK;
}

}  // extern "C"
