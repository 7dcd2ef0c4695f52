// rq_capi.cu -- C ABI (include/rqmc_b200.h): host tables, device contexts,
// batching of replications and numpy pairwise-sum plans.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rqmc_b200.h"
#include "rq_device.cuh"
#include "rq_internal.h"

namespace {

#include "joe_kuo_421.inc"

thread_local std::string g_err;

// host<->device byte counters and optional per-kernel timing (bench.py)
struct Stats {
  uint64_t h2d = 0, d2h = 0;
  bool timing = false;
  double paths_ms = 0, reduce_ms = 0, setup_ms = 0;
  int64_t paths_launches = 0;
} g_stats;
std::mutex g_stats_mu;
// counters may be bumped from several host threads (one per device)
template <class T>
void stat_add(T &field, T v) {
  std::lock_guard<std::mutex> lk(g_stats_mu);
  field += v;
}

struct KTimer {  // CUDA events on the launching stream when timing is on
  cudaEvent_t a = nullptr, b = nullptr;
  double *acc;
  cudaStream_t s;
  KTimer(double *acc_, cudaStream_t s_) : acc(acc_), s(s_) {
    if (g_stats.timing) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
    }
  }
  ~KTimer() {
    if (a) {
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      stat_add(*acc, (double)ms);
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  }
};

// size knobs, overridable for tests that exercise the batch / group loops
int64_t env_int(const char *name, int64_t dflt) {
  const char *v = std::getenv(name);
  if (!v || !*v) return dflt;
  const long long x = std::atoll(v);
  return x > 0 ? (int64_t)x : dflt;
}

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define RQ_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(RQ_ERR_CUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_),    \
                  __FILE__, __LINE__);                                             \
  } while (0)

// ------------------------------------------------------------------ Halton constants
struct HostTables {
  std::vector<rq::HaltonDim> dims;
  std::vector<double> wts, cscale;
  int total_bases(int dim) const { return dim ? dims[dim - 1].sig_off + dims[dim - 1].base : 0; }
  int total_caps(int dim) const { return dim ? dims[dim - 1].dig_off + dims[dim - 1].cap : 0; }
  int total_sums(int dim) const { return dim ? dims[dim - 1].sum_off + dims[dim - 1].cap + 1 : 0; }
};

// numba `float ** int` (int_power): r = 1; while e: if e & 1: r *= a; e >>= 1; a *= a
double numba_ipow(double a, int64_t e) {
  double r = 1.0;
  while (e != 0) {
    if (e & 1) r = rq::dmul(r, a);
    e >>= 1;
    a = rq::dmul(a, a);
  }
  return r;
}

const HostTables &host_tables() {
  static HostTables T;
  static std::once_flag once;
  std::call_once(once, [] {
    std::vector<int> primes;
    for (int c = 2; (int)primes.size() < rq::MAX_DIM; c++) {
      bool ok = true;
      for (int p : primes) {
        if (p * p > c) break;
        if (c % p == 0) {
          ok = false;
          break;
        }
      }
      if (ok) primes.push_back(c);
    }
    int sig = 0, dig = 0, sum = 0;
    for (int d = 0; d < rq::MAX_DIM; d++) {
      rq::HaltonDim h{};
      int p = primes[d];
      h.base = p;
      int K = 1;
      unsigned __int128 v = p;
      while (v < ((unsigned __int128)1 << 32)) {  // halton.py:59-66
        v *= p;
        K++;
      }
      h.K = K;
      h.cap = K + 8;
      int ell = 0;
      while ((1 << ell) < p) ell++;
      h.ell = ell;
      unsigned __int128 num = ((unsigned __int128)1) << (32 + ell);
      uint64_t m = (uint64_t)((num + p - 1) / p);  // ceil(2^(32+ell)/p) in [2^32, 2^33]
      h.mlo = (uint32_t)m;
      // 64-bit numerators x < 2^46: q = floor(x * M / 2^(46+ell)) with
      // M = ceil(2^(46+ell)/p); stored pre-shifted so q = umulhi64(x, m64)
      unsigned __int128 M = ((((unsigned __int128)1) << (46 + ell)) + p - 1) / p;
      h.m64 = (uint64_t)(M << (18 - ell));
      h.m16 = (uint32_t)(((((uint64_t)1) << 32) + p - 1) / p);  // ceil(2^32/p)
      h.tdig = 0;
      for (int v = 128 / p; v > 0; v /= p) h.tdig++;  // 128 = the device tile (TILE)
      h.sig_off = sig;
      h.dig_off = dig;
      h.sum_off = sum;
      h.inv_p = 1.0 / (double)p;
      h.scale0 = std::pow(h.inv_p, (double)K);  // Python float ** int -> C pow
      T.dims.push_back(h);
      for (int j = 0; j < h.cap + 1; j++) T.wts.push_back(numba_ipow(h.inv_p, j + 1));
      double s = 1.0;
      for (int j = 0; j < h.cap + 1; j++) {
        s = rq::dmul(s, h.inv_p);
        T.cscale.push_back(s);
      }
      sig += p;
      dig += h.cap;
      sum += h.cap + 1;
    }
  });
  return T;
}

// Columns of the XORWOW xorshift transition A (prng.py:97-108) on the
// 160-bit state (x, y, z, w, v), and of A^(2^k) by repeated squaring:
// cols[k][c] = A^(2^k) e_c, padded to XW_COLW words.
std::vector<uint32_t> xorwow_jump_columns() {
  const int W = rq::XW_COLW;
  std::vector<uint32_t> cols((size_t)rq::XW_JUMPS * 160 * W, 0u);
  auto apply = [&](const uint32_t *M, const uint32_t *v, uint32_t *o) {
    uint32_t r[5] = {0, 0, 0, 0, 0};
    for (int c = 0; c < 160; c++)
      if ((v[c / 32] >> (c % 32)) & 1u)
        for (int i = 0; i < 5; i++) r[i] ^= M[c * W + i];
    for (int i = 0; i < 5; i++) o[i] = r[i];
  };
  for (int c = 0; c < 160; c++) {
    uint32_t e[5] = {0, 0, 0, 0, 0};
    e[c / 32] = 1u << (c % 32);
    const uint32_t x = e[0], t = x ^ (x >> 2), v = e[4];
    uint32_t *o = &cols[c * W];
    o[0] = e[1];
    o[1] = e[2];
    o[2] = e[3];
    o[3] = e[4];
    o[4] = (v ^ (v << 4)) ^ (t ^ (t << 1));
  }
  for (int k = 1; k < rq::XW_JUMPS; k++) {
    const uint32_t *M = &cols[(size_t)(k - 1) * 160 * W];
    uint32_t *N = &cols[(size_t)k * 160 * W];
    for (int c = 0; c < 160; c++) apply(M, M + c * W, N + c * W);
  }
  return cols;
}

// ---- Kakutani bracket tables (halton.py:178-193): the correctly rounded
// doubles of the exact rationals 1/p^k and (p + 1 - p^k)/p^k, k = 1..64, as
// the reference computes them with fractions.Fraction; thr = inv + 1e-11
// in double arithmetic (halton.py:231).
using Big = std::vector<uint32_t>;  // little-endian 32-bit limbs
void big_mul_small(Big &a, uint32_t m) {
  uint64_t c = 0;
  for (auto &w : a) {
    uint64_t t = (uint64_t)w * m + c;
    w = (uint32_t)t;
    c = t >> 32;
  }
  if (c) a.push_back((uint32_t)c);
}
int big_bits(const Big &a) {
  for (int i = (int)a.size() - 1; i >= 0; i--)
    if (a[i]) return i * 32 + 32 - __builtin_clz(a[i]);
  return 0;
}
int big_cmp(const Big &a, const Big &b) {
  size_t n = std::max(a.size(), b.size());
  for (int i = (int)n - 1; i >= 0; i--) {
    uint32_t x = i < (int)a.size() ? a[i] : 0u, y = i < (int)b.size() ? b[i] : 0u;
    if (x != y) return x < y ? -1 : 1;
  }
  return 0;
}
void big_sub(Big &a, const Big &b) {  // a -= b, a >= b
  int64_t br = 0;
  for (size_t i = 0; i < a.size(); i++) {
    int64_t t = (int64_t)a[i] - (i < b.size() ? b[i] : 0u) - br;
    br = t < 0;
    a[i] = (uint32_t)(t + (br ? ((int64_t)1 << 32) : 0));
  }
}
Big big_shl(const Big &a, int bits) {
  Big r((size_t)(bits / 32), 0u);
  uint32_t c = 0;
  const int sh = bits % 32;
  for (uint32_t w : a) {
    r.push_back(sh ? (w << sh) | c : w);
    c = sh ? w >> (32 - sh) : 0u;
  }
  if (c) r.push_back(c);
  return r;
}
// n / d rounded to nearest (ties to even), 0 < n < d
double big_ratio(const Big &n, const Big &d) {
  const int ln = big_bits(n), ld = big_bits(d);
  const int s = 54 + ld - ln;  // n 2^s / d in [2^53, 2^55), s >= 54
  Big r = big_shl(n, s - 55 > 0 ? s - 55 : 0);
  const int iters = s < 55 ? s : 55;
  uint64_t q = 0;
  for (int i = 0; i < iters; i++) {
    r = big_shl(r, 1);
    q <<= 1;
    if (big_cmp(r, d) >= 0) {
      big_sub(r, d);
      q |= 1;
    }
  }
  bool sticky = big_bits(r) != 0;
  int e = -s;
  if (q >> 54) {
    sticky |= q & 1;
    q >>= 1;
    e++;
  }
  uint64_t m = q >> 1;
  if ((q & 1) && (sticky || (m & 1))) m++;
  return std::ldexp((double)m, e + 1);
}
void kakutani_tables(int p, double *thr, double *b) {
  Big pk{1u};
  for (int k = 1; k <= rq::KK_TAB; k++) {
    big_mul_small(pk, (uint32_t)p);
    const double inv = big_ratio(Big{1u}, pk);
    thr[k - 1] = inv + 1e-11;  // halton.py:205 _BRACKET_TOL
    if (k == 1) {
      b[0] = inv;  // (p + 1 - p) / p
    } else {
      Big num = pk;  // p^k - p - 1
      big_sub(num, Big{(uint32_t)p + 1u});
      b[k - 1] = -big_ratio(num, pk);
    }
  }
}
// Kakutani bracket tables, [dim][2][KK_TAB], computed on first use of a
// dim range (big-integer powers: ~1.3 ms per dim, 8.5 s for all 6542)
std::mutex g_kk_mu;
std::vector<double> g_kk_T;
int g_kk_n = 0;
void kakutani_grow(int n) {  // caller holds g_kk_mu
  if (n <= g_kk_n) return;
  n = std::min(rq::MAX_DIM, (n + 511) / 512 * 512);
  const HostTables &H = host_tables();
  g_kk_T.resize((size_t)n * 2 * rq::KK_TAB);
  for (int d = g_kk_n; d < n; d++)
    kakutani_tables(H.dims[d].base, &g_kk_T[(size_t)d * 2 * rq::KK_TAB],
                    &g_kk_T[(size_t)d * 2 * rq::KK_TAB + rq::KK_TAB]);
  g_kk_n = n;
}
// device copies of dims [0, n) on the current device
int ensure_kakutani_tables(int n) {
  static std::vector<std::pair<int, int>> done;  // (device, dims uploaded)
  int dev = 0;
  RQ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_kk_mu);
  for (auto &e : done)
    if (e.first == dev && e.second >= n) return RQ_OK;
  kakutani_grow(n);
  const int m = g_kk_n;
  std::vector<double> thr((size_t)m * rq::KK_TAB), b(thr.size());
  for (int d = 0; d < m; d++)
    for (int k = 0; k < rq::KK_TAB; k++) {
      thr[(size_t)d * rq::KK_TAB + k] = g_kk_T[(size_t)d * 2 * rq::KK_TAB + k];
      b[(size_t)d * rq::KK_TAB + k] = g_kk_T[(size_t)d * 2 * rq::KK_TAB + rq::KK_TAB + k];
    }
  RQ_CUDA(rq::upload_kakutani_tables(thr.data(), b.data(), m));
  bool found = false;
  for (auto &e : done)
    if (e.first == dev) e.second = m, found = true;
  if (!found) done.emplace_back(dev, m);
  return RQ_OK;
}

int ensure_device_tables() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  RQ_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return RQ_OK;
  // keep freed cudaMallocAsync memory in the pool across synchronisations
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  const HostTables &T = host_tables();
  RQ_CUDA(rq::upload_halton_dims(T.dims.data(), (int)T.dims.size(), T.wts.data(),
                                 T.cscale.data(), (int)T.wts.size()));
  static const std::vector<uint32_t> xw = xorwow_jump_columns();
  RQ_CUDA(rq::upload_xorwow_jumps(xw.data(), xw.size()));
  done.push_back(dev);
  return RQ_OK;
}

// Joe-Kuo expansion: m-recursion (sobol.py:61-71), v_k = m_k << (32 - k).
int sobol_v(int dim, uint32_t *v) {
  if (dim < 1 || dim > kJoeKuoDims) return fail(RQ_ERR_VALUE, "sobol dim %d outside 1..%d", dim, kJoeKuoDims);
  for (int k = 1; k <= 32; k++) v[k - 1] = 1u << (32 - k);  // dimension 1: m_k = 1
  size_t pos = 0;
  for (int d = 2; d <= dim; d++) {
    int s = (int)kJoeKuoPacked[pos], a = (int)kJoeKuoPacked[pos + 1];
    std::vector<uint64_t> m(kJoeKuoPacked + pos + 2, kJoeKuoPacked + pos + 2 + s);
    pos += 2 + s;
    for (int k = s; k < 32; k++) {
      uint64_t acc = (m[k - s] << s) ^ m[k - s];
      for (int i = 1; i < s; i++)
        if ((a >> (s - 1 - i)) & 1) acc ^= m[k - i] << i;
      m.push_back(acc);
    }
    for (int k = 1; k <= 32; k++) v[(d - 1) * 32 + k - 1] = (uint32_t)(m[k - 1] << (32 - k));
  }
  return RQ_OK;
}

// ------------------------------------------------------------------ pairwise plan
struct HostPlan {
  int64_t n;
  std::vector<int64_t> leaf_start;
  std::vector<int32_t> leaf_len;
  std::vector<int32_t> level_off, node_id, node_l, node_r;
  int32_t root, nnodes;
};

// numpy pairwise_sum recursion: n <= 128 leaf, else split at
// n2 = n/2 - (n/2 % 8).  Leaves get ids 0..L-1 in order; internal nodes
// ids >= L grouped by height so each level only depends on lower ones.
void build_plan(int64_t n, HostPlan &P) {
  P.n = n;
  struct Frame {
    int64_t start, len;
    int state;
  };
  // iterative post-order walk; provisional ids: leaf k -> k, internal k -> -(k+1)
  std::vector<Frame> st;
  std::vector<int32_t> out_stack;
  std::vector<std::pair<int32_t, int32_t>> children;
  std::vector<int32_t> int_height;
  auto height = [&](int32_t id) { return id >= 0 ? 0 : int_height[-id - 1]; };
  st.push_back({0, n, 0});
  while (!st.empty()) {
    Frame &f = st.back();
    if (f.len <= 128) {
      P.leaf_start.push_back(f.start);
      P.leaf_len.push_back((int32_t)f.len);
      out_stack.push_back((int32_t)P.leaf_start.size() - 1);
      st.pop_back();
      continue;
    }
    int64_t n2 = f.len / 2;
    n2 -= n2 % 8;
    if (f.state == 0) {
      f.state = 1;
      st.push_back({f.start, n2, 0});
    } else if (f.state == 1) {
      f.state = 2;
      Frame c{f.start + n2, f.len - n2, 0};
      st.push_back(c);
    } else {
      int32_t r = out_stack.back();
      out_stack.pop_back();
      int32_t l = out_stack.back();
      out_stack.pop_back();
      children.push_back({l, r});
      int_height.push_back(std::max(height(l), height(r)) + 1);
      out_stack.push_back(-(int32_t)children.size());
      st.pop_back();
    }
  }
  int32_t L = (int32_t)P.leaf_len.size();
  int32_t I = (int32_t)children.size();
  auto fin = [&](int32_t id) { return id >= 0 ? id : L + (-id - 1); };
  int32_t H = 0;
  for (int32_t h : int_height) H = std::max(H, h);
  P.level_off.assign(H + 1, 0);
  std::vector<std::vector<int32_t>> by_h(H + 1);
  for (int32_t k = 0; k < I; k++) by_h[int_height[k]].push_back(k);
  for (int32_t h = 1; h <= H; h++) {
    P.level_off[h - 1] = (int32_t)P.node_id.size();
    for (int32_t k : by_h[h]) {
      P.node_id.push_back(L + k);
      P.node_l.push_back(fin(children[k].first));
      P.node_r.push_back(fin(children[k].second));
    }
  }
  if (H >= 1) P.level_off[H] = (int32_t)P.node_id.size();
  P.level_off.resize(H + 1);
  P.root = fin(out_stack.back());
  P.nnodes = L + I;
}

// Stream-ordered device allocation released when it goes out of scope, so
// the early error returns of the entry points leak nothing.
struct DevMem {
  void *p = nullptr;
  cudaStream_t s = nullptr;
  DevMem() = default;
  explicit DevMem(cudaStream_t s_) : s(s_) {}
  DevMem(const DevMem &) = delete;
  DevMem &operator=(const DevMem &) = delete;
  cudaError_t alloc(size_t bytes) { return cudaMallocAsync(&p, bytes, s); }
  template <class T>
  T *as() const { return (T *)p; }
  ~DevMem() {
    if (p) cudaFreeAsync(p, s);
  }
};

struct DevPlan {
  rq::SumPlan p{};
  DevMem buf;
};

int upload_plan(const HostPlan &hp, DevPlan &dp, cudaStream_t s) {
  size_t nl = hp.leaf_start.size(), ni = hp.node_id.size(), nlev = hp.level_off.size();
  size_t bytes = nl * 8 + nl * 4 + nlev * 4 + 3 * ni * 4 + 64;
  dp.buf.s = s;
  RQ_CUDA(dp.buf.alloc(bytes));
  char *b = dp.buf.as<char>();
  std::vector<char> host(bytes);
  size_t off = 0;
  auto put = [&](const void *src, size_t n) {
    std::memcpy(host.data() + off, src, n);
    char *dst = b + off;
    off += (n + 7) & ~(size_t)7;
    return dst;
  };
  dp.p.n = hp.n;
  dp.p.nleaves = (int32_t)nl;
  dp.p.nnodes = hp.nnodes;
  dp.p.nlevels = (int32_t)nlev - 1 > 0 ? (int32_t)nlev - 1 : 0;
  dp.p.root = hp.root;
  dp.p.leaf_start = (const int64_t *)put(hp.leaf_start.data(), nl * 8);
  dp.p.leaf_len = (const int32_t *)put(hp.leaf_len.data(), nl * 4);
  dp.p.level_off = (const int32_t *)put(hp.level_off.data(), nlev * 4);
  dp.p.node_id = (const int32_t *)put(hp.node_id.data(), ni * 4);
  dp.p.node_l = (const int32_t *)put(hp.node_l.data(), ni * 4);
  dp.p.node_r = (const int32_t *)put(hp.node_r.data(), ni * 4);
  RQ_CUDA(cudaMemcpyAsync(dp.buf.p, host.data(), off, cudaMemcpyHostToDevice, s));
  stat_add(g_stats.h2d, (uint64_t)off);
  // the host staging buffer must outlive the copy
  RQ_CUDA(cudaStreamSynchronize(s));
  return RQ_OK;
}

}  // namespace

// ------------------------------------------------------------------ sampler
struct rq_sampler {
  rq::RepTables t{};
  void *mem = nullptr;
  bool owns = true;
};

extern "C" {

const char *rq_last_error(void) { return g_err.c_str(); }
int rq_abi_version(void) { return RQ_ABI_VERSION; }

int rq_sobol_directions(int dim, uint32_t *v_host) { return sobol_v(dim, v_host); }

int rq_halton_divide(int d, uint64_t x, uint64_t *q64, uint32_t *q32) {
  if (d < 0 || d >= rq::MAX_DIM) return fail(RQ_ERR_VALUE, "dim index %d outside 0..%d", d, rq::MAX_DIM - 1);
  const rq::HaltonDim &h = host_tables().dims[d];
  if (q64) *q64 = rq::umulhi64(x, h.m64);
  if (q32) {
    uint32_t t = (uint32_t)x;
    *q32 = (uint32_t)((((uint64_t)rq::umulhi32(t, h.mlo)) + t) >> h.ell);
    if (t < 65536u && rq::umulhi32(t, h.m16) != *q32) *q32 = 0xFFFFFFFFu;  // 16-bit magic check
  }
  return RQ_OK;
}

int rq_kakutani_tables(int dim, double *thr_host, double *b_host) {
  if (dim < 1 || dim > rq::MAX_DIM) return fail(RQ_ERR_VALUE, "dim %d outside 1..%d", dim, rq::MAX_DIM);
  std::lock_guard<std::mutex> lk(g_kk_mu);
  kakutani_grow(dim);
  const std::vector<double> &T = g_kk_T;
  for (int d = 0; d < dim; d++)
    for (int k = 0; k < rq::KK_TAB; k++) {
      if (thr_host) thr_host[(size_t)d * rq::KK_TAB + k] = T[(size_t)d * 2 * rq::KK_TAB + k];
      if (b_host) b_host[(size_t)d * rq::KK_TAB + k] = T[(size_t)d * 2 * rq::KK_TAB + rq::KK_TAB + k];
    }
  return RQ_OK;
}

int rq_halton_constants(int dim, int32_t *base, int32_t *K, double *scale0) {
  if (dim < 1 || dim > rq::MAX_DIM) return fail(RQ_ERR_VALUE, "dim %d outside 1..%d", dim, rq::MAX_DIM);
  const HostTables &T = host_tables();
  for (int d = 0; d < dim; d++) {
    if (base) base[d] = T.dims[d].base;
    if (K) K[d] = T.dims[d].K;
    if (scale0) scale0[d] = T.dims[d].scale0;
  }
  return RQ_OK;
}

int rq_sampler_create(rq_sampler **out, int generator, int dim, uint64_t seed,
                      int64_t rep_first, int32_t rep_count, void *stream) {
  if (!out) return fail(RQ_ERR_VALUE, "out is NULL");
  *out = nullptr;
  if (generator < 0 || generator > rq::GEN_LAST)
    return fail(RQ_ERR_VALUE, "unknown generator id %d", generator);
  if (dim < 1) return fail(RQ_ERR_VALUE, "dimension must be >= 1");
  if (rep_count < 1) return fail(RQ_ERR_VALUE, "rep_count must be >= 1");
  bool rasrap = generator == rq::GEN_RASRAP_RECURSIVE || generator == rq::GEN_RASRAP_COUNTER;
  bool sob = generator == rq::GEN_SOBOL_GRAY || generator == rq::GEN_SOBOL_COUNTER;
  if (rasrap && dim > rq::MAX_DIM)
    return fail(RQ_ERR_VALUE, "rasrap dimension %d exceeds %d", dim, rq::MAX_DIM);
  if (sob && dim > kJoeKuoDims)
    return fail(RQ_ERR_VALUE, "source provides %d dimensions, %d requested", kJoeKuoDims, dim);
  int rc = ensure_device_tables();
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  rq_sampler *S = new rq_sampler();
  rq::RepTables &t = S->t;
  t.gen = generator;
  t.dim = dim;
  t.seed = seed;
  t.rep_first = rep_first;
  t.rep_count = rep_count;
  const HostTables &T = host_tables();
  if (rasrap) {
    t.sig_stride = T.total_bases(dim);
    t.dig_stride = (T.total_caps(dim) + 3) & ~3;
    t.sum_stride = T.total_sums(dim);
    t.sig_stride = (t.sig_stride + 3) & ~3;
    t.sig_chunk_max = 0;
    for (int d0 = 0; d0 < dim; d0 += rq::CHUNK_DIMS) {
      int d1 = std::min(dim, d0 + rq::CHUNK_DIMS) - 1;
      t.sig_chunk_max = std::max(t.sig_chunk_max,
                                 T.dims[d1].sig_off + T.dims[d1].base - T.dims[d0].sig_off);
    }
    size_t b_sig = sizeof(uint16_t) * t.sig_stride * rep_count;
    size_t b_sum = sizeof(double) * t.sum_stride * rep_count;
    size_t b_dig = sizeof(uint16_t) * t.dig_stride * rep_count;
    size_t b_start = sizeof(uint64_t) * dim * rep_count;
    cudaError_t e = cudaMallocAsync(&S->mem, b_start + b_sig + b_sum + b_dig, s);
    if (e != cudaSuccess) {
      delete S;
      return fail(RQ_ERR_CUDA, "allocating rasrap tables (%zu B): %s", b_sig + b_sum + b_dig,
                  cudaGetErrorString(e));
    }
    uint64_t *start = (uint64_t *)S->mem;
    double *sums = (double *)(start + (size_t)dim * rep_count);
    uint16_t *sig = (uint16_t *)(sums + t.sum_stride * rep_count);
    uint16_t *dig = sig + t.sig_stride * rep_count;
    t.sigma = sig;
    t.sums = sums;
    t.digits = dig;
    t.start = start;
    {
      KTimer kt(&g_stats.setup_ms, s);
      std::vector<int> bases(dim);
      for (int d = 0; d < dim; d++) bases[d] = T.dims[d].base;
      e = rq::launch_rasrap_setup(t, sig, dig, sums, start, s, bases.data());
    }
    if (e != cudaSuccess) {
      cudaFreeAsync(S->mem, s);
      delete S;
      return fail(RQ_ERR_CUDA, "rasrap setup: %s", cudaGetErrorString(e));
    }
  } else if (sob) {
    std::vector<uint32_t> v((size_t)dim * 32);
    if ((rc = sobol_v(dim, v.data()))) {
      delete S;
      return rc;
    }
    size_t b_v = sizeof(uint32_t) * dim * 32;
    size_t b_gen = b_v * rep_count, b_sh = sizeof(uint32_t) * dim * rep_count;
    cudaError_t e = cudaMallocAsync(&S->mem, b_v + b_gen + b_sh, s);
    if (e != cudaSuccess) {
      delete S;
      return fail(RQ_ERR_CUDA, "allocating sobol tables: %s", cudaGetErrorString(e));
    }
    uint32_t *vd = (uint32_t *)S->mem;
    uint32_t *gen = vd + (size_t)dim * 32;
    uint32_t *sh = gen + (size_t)dim * 32 * rep_count;
    e = cudaMemcpyAsync(vd, v.data(), b_v, cudaMemcpyHostToDevice, s);
    stat_add(g_stats.h2d, (uint64_t)b_v);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // v is a host temporary
    if (e == cudaSuccess) {
      KTimer kt(&g_stats.setup_ms, s);
      e = rq::launch_sobol_setup(t, vd, gen, sh, s);
    }
    if (e != cudaSuccess) {
      cudaFreeAsync(S->mem, s);
      delete S;
      return fail(RQ_ERR_CUDA, "sobol setup: %s", cudaGetErrorString(e));
    }
    t.sobol_v = gen;
    t.sobol_shift = sh;
  } else if (generator == rq::GEN_KAKUTANI) {
    if (dim > rq::MAX_DIM) {
      delete S;
      return fail(RQ_ERR_VALUE, "kakutani dimension %d exceeds %d", dim, rq::MAX_DIM);
    }
    if ((rc = ensure_kakutani_tables(dim))) {
      delete S;
      return rc;
    }
    cudaError_t e = cudaMallocAsync(&S->mem, sizeof(double) * dim * rep_count, s);
    if (e == cudaSuccess) {
      KTimer kt(&g_stats.setup_ms, s);
      e = rq::launch_kakutani_setup(t, (double *)S->mem, s);
    }
    if (e != cudaSuccess) {
      if (S->mem) cudaFreeAsync(S->mem, s);
      delete S;
      return fail(RQ_ERR_CUDA, "kakutani setup: %s", cudaGetErrorString(e));
    }
    t.kk_x0 = (const double *)S->mem;
  } else if (generator == rq::GEN_XORWOW) {
    cudaError_t e = cudaMallocAsync(&S->mem, sizeof(uint32_t) * 6 * rep_count, s);
    if (e == cudaSuccess) {
      KTimer kt(&g_stats.setup_ms, s);
      e = rq::launch_xorwow_setup(t, (uint32_t *)S->mem, s);
    }
    if (e != cudaSuccess) {
      if (S->mem) cudaFreeAsync(S->mem, s);
      delete S;
      return fail(RQ_ERR_CUDA, "xorwow setup: %s", cudaGetErrorString(e));
    }
    t.xw_state = (const uint32_t *)S->mem;
  }
  *out = S;
  return RQ_OK;
}

// Sequential streams: segment layout, MT19937 snapshots and the per-CTA
// word scratch for paths [p0, p0 + nmax) of batches of <= B replications.
// The snapshot walk is sequential per replication (latency bound), so it is
// launched for a whole group of batches at once (<= 1 GiB of snapshots).
struct SeqRun {
  rq::SeqArgs q{};
  int ctas = 0;
  int64_t grp0 = 0, grpn = 0, grp_cap = 0;
  uint32_t *snap = nullptr;
  size_t per_rep = 0;  // snapshot bytes per replication
  void *mem = nullptr;
  cudaStream_t stream = nullptr;  // the work stream: freed in stream order
  ~SeqRun() {
    if (mem) cudaFreeAsync(mem, stream);
  }
};
static int seq_begin(const rq::RepTables &t, const rq::ModelParams &mp, int B, int64_t p0,
                     int64_t nmax, SeqRun &R, cudaStream_t s) {
  int64_t L;
  int segs;
  rq::seq_layout(t, mp, B, nmax, &L, &segs, &R.ctas);
  R.q.p0 = p0;
  R.q.nmax = nmax;
  R.q.seg_len = L;
  R.q.segs_per_rep = segs;
  if (t.gen == rq::GEN_XORWOW) return RQ_OK;
  const bool mt = t.gen == rq::GEN_TWISTER;
  const size_t per_rep = mt ? sizeof(uint32_t) * rq::MT_N * (size_t)segs
                            : sizeof(double) * t.dim * (size_t)segs *
                                  (rq::kak_runs(t.dim) ? 128 : 1);
  // the walk is latency bound (its time hardly depends on the group size):
  // few, large groups (<= 1 GiB of snapshots)
  int64_t G = std::max<int64_t>(B, env_int("RQ_SNAP_GROUP_BYTES", (int64_t)1024 << 20) /
                                      (int64_t)per_rep / B * B);
  G = std::min<int64_t>(G, t.rep_count);
  R.grp_cap = G;
  // per CTA: [dim][TILE] words (Kakutani: doubles, then the orbit state xs[dim])
  size_t b_scr = mt ? sizeof(uint32_t) * (size_t)R.ctas * t.dim * rq::TILE_PATHS
                    : sizeof(double) * (size_t)R.ctas * t.dim * (rq::TILE_PATHS + 1);
  RQ_CUDA(cudaMallocAsync(&R.mem, per_rep * G + b_scr, s));
  R.stream = s;
  R.snap = (uint32_t *)R.mem;
  R.per_rep = per_rep;
  R.q.scratch = (uint32_t *)((char *)R.mem + per_rep * G);
  R.grpn = 0;
  return RQ_OK;
}
// position the run on local replications [r0, r0 + rn): snapshots + grid
static int seq_batch(const rq::RepTables &t, int r0, int rn, SeqRun &R, int *blocks,
                     int *launched, cudaStream_t s) {
  *blocks = (int)std::min<int64_t>((int64_t)rn * R.q.segs_per_rep, R.ctas);
  if (t.gen == rq::GEN_XORWOW) return RQ_OK;
  const bool mt = t.gen == rq::GEN_TWISTER;
  if (r0 < R.grp0 || r0 + rn > R.grp0 + R.grpn) {
    R.grp0 = r0;
    R.grpn = std::min<int64_t>(R.grp_cap, t.rep_count - r0);
    KTimer kt(&g_stats.setup_ms, s);
    if (mt) RQ_CUDA(rq::launch_mt_snap(t, r0, (int)R.grpn, R.q, R.snap, s));
    else RQ_CUDA(rq::launch_kak_snap(t, r0, (int)R.grpn, R.q, (double *)R.snap, s));
    if (launched) *launched += 1;
  }
  const char *at = (const char *)R.snap + R.per_rep * (size_t)(r0 - R.grp0);
  if (mt) R.q.mt_snap = (const uint32_t *)at;
  else R.q.kk_snap = (const double *)at;
  return RQ_OK;
}

void rq_sampler_destroy(rq_sampler *s) {
  if (!s) return;
  if (s->mem) cudaFree(s->mem);
  delete s;
}

static int check_rep(rq_sampler *s, int32_t rl) {
  if (!s) return fail(RQ_ERR_VALUE, "sampler is NULL");
  if (rl < 0 || rl >= s->t.rep_count)
    return fail(RQ_ERR_VALUE, "replication %d outside the sampler's %d", rl, s->t.rep_count);
  return RQ_OK;
}

int64_t rq_index_limit(int generator) {
  switch (generator) {
    case rq::GEN_PHILOX:
    case rq::GEN_SFC64: return (int64_t)1 << 62;
    case rq::GEN_RASRAP_RECURSIVE:
    case rq::GEN_RASRAP_COUNTER: return (int64_t)1 << 39;
  }
  return (int64_t)1 << 32;
}

int rq_sampler_points(rq_sampler *s, int32_t rep_local, int64_t first, int64_t count,
                      double *out_dev, void *stream) {
  int rc = check_rep(s, rep_local);
  if (rc) return rc;
  if (first < 0 || count < 0) return fail(RQ_ERR_VALUE, "index must be non-negative");
  const int64_t lim = rq_index_limit(s->t.gen);
  if (first > lim || count > lim - first)
    return fail(RQ_ERR_RANGE, "point index %lld exceeds the generator's index range %lld",
                (long long)(first + count), (long long)lim);
  if (count == 0) return RQ_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (rq::gen_sequential(s->t.gen)) {  // _WordSampler.fill: words from the cursor on
    rq::ModelParams mp{};
    mp.kind = rq::MODEL_POINTS;
    mp.dim = s->t.dim;
    SeqRun R;
    int blocks = 0;
    if ((rc = seq_begin(s->t, mp, 1, first, count, R, st))) return rc;
    if ((rc = seq_batch(s->t, rep_local, 1, R, &blocks, nullptr, st))) return rc;
    RQ_CUDA(rq::launch_paths_seq(s->t, mp, rep_local, 1, count, R.q, blocks, out_dev, nullptr, st));
    return RQ_OK;
  }
  RQ_CUDA(rq::launch_points(s->t, rep_local, first, nullptr, count, out_dev, st));
  return RQ_OK;
}

int rq_sampler_points_at(rq_sampler *s, int32_t rep_local, const int64_t *idx_dev,
                         int64_t count, double *out_dev, void *stream) {
  int rc = check_rep(s, rep_local);
  if (rc) return rc;
  if (count <= 0) return count < 0 ? fail(RQ_ERR_VALUE, "count < 0") : RQ_OK;
  if (rq::gen_sequential(s->t.gen))  // harness._WordSampler has no at() (harness.py:37-50)
    return fail(RQ_ERR_VALUE, "sequential word streams have no counter-based at()");
  RQ_CUDA(rq::launch_points(s->t, rep_local, 0, idx_dev, count, out_dev, (cudaStream_t)stream));
  return RQ_OK;
}

int rq_sampler_rasrap_tables(rq_sampler *s, int32_t rep_local, uint16_t *digits_host,
                             uint16_t *sigma_host, double *sums_host) {
  int rc = check_rep(s, rep_local);
  if (rc) return rc;
  const rq::RepTables &t = s->t;
  if (t.gen != rq::GEN_RASRAP_RECURSIVE && t.gen != rq::GEN_RASRAP_COUNTER)
    return fail(RQ_ERR_VALUE, "not a rasrap sampler");
  RQ_CUDA(cudaDeviceSynchronize());
  if (digits_host)
    RQ_CUDA(cudaMemcpy(digits_host, t.digits + rep_local * t.dig_stride,
                       sizeof(uint16_t) * t.dig_stride, cudaMemcpyDeviceToHost));
  if (sigma_host)
    RQ_CUDA(cudaMemcpy(sigma_host, t.sigma + rep_local * t.sig_stride,
                       sizeof(uint16_t) * t.sig_stride, cudaMemcpyDeviceToHost));
  if (sums_host)
    RQ_CUDA(cudaMemcpy(sums_host, t.sums + rep_local * t.sum_stride,
                       sizeof(double) * t.sum_stride, cudaMemcpyDeviceToHost));
  return RQ_OK;
}

static int model_to_params(const rq_model *m, int dim, rq::ModelParams &mp, DevMem &tab,
                           cudaStream_t s) {
  if (!m) return fail(RQ_ERR_VALUE, "model is NULL");
  if (m->kind < 0 || m->kind == rq::MODEL_POINTS || m->kind > rq::MODEL_XHASH)
    return fail(RQ_ERR_VALUE, "unknown model kind %d", m->kind);
  if (m->dim != dim) return fail(RQ_ERR_VALUE, "model dim %d != sampler dim %d", m->dim, dim);
  if (m->kind == rq::MODEL_LIBOR && (m->dim < 1 || m->dim > rq::LIBOR_MAX))
    return fail(RQ_ERR_VALUE, "LIBOR steps %d outside 1..%d", m->dim, rq::LIBOR_MAX);
  mp.kind = m->kind;
  mp.dim = m->dim;
  mp.delta = m->delta;
  mp.sigma = m->sigma;
  mp.strike = m->strike;
  mp.front_factor = m->front_factor;
  mp.i0 = m->i0;
  mp.k0 = m->k0;
  mp.k1 = m->k1;
  mp.k2 = m->k2;
  mp.k3 = m->k3;
  mp.k4 = m->k4;
  mp.sigma_xi = m->sigma_xi;
  mp.payment = m->payment;
  // k0 * exp(sigma_xi z) = sum_k (k0 sigma_xi^k / k!) z^k for |sigma_xi z| <= 0.1
  double c = m->k0;
  for (int k = 0; k < rq::MBS_EXP_TERMS; k++) {
    mp.ecoef[k] = c;
    c = c * m->sigma_xi / (double)(k + 1);
  }
  mp.exp_zlim = m->sigma_xi > 0.0 ? 0.1 / m->sigma_xi : INFINITY;
  mp.table = nullptr;
  if (m->kind == rq::MODEL_LIBOR || m->kind == rq::MODEL_MBS) {
    if (!m->table) return fail(RQ_ERR_VALUE, "model table is NULL");
    tab.s = s;
    RQ_CUDA(tab.alloc(sizeof(double) * m->dim));
    RQ_CUDA(cudaMemcpyAsync(tab.p, m->table, sizeof(double) * m->dim, cudaMemcpyHostToDevice, s));
    stat_add(g_stats.h2d, (uint64_t)(sizeof(double) * m->dim));
    mp.table = tab.as<double>();
  }
  return RQ_OK;
}

static int check_grid(const int64_t *grid, int32_t ngrid) {
  if (!grid || ngrid < 1) return fail(RQ_ERR_VALUE, "n_grid must be a nonempty list of positive sizes");
  for (int g = 0; g < ngrid; g++) {
    if (grid[g] < 1) return fail(RQ_ERR_VALUE, "n_grid must be a nonempty list of positive sizes");
    if (g && grid[g] <= grid[g - 1]) return fail(RQ_ERR_VALUE, "n_grid must be strictly increasing");
  }
  if (grid[ngrid - 1] > ((int64_t)1 << 40)) return fail(RQ_ERR_RANGE, "N exceeds 2^40 paths");
  return RQ_OK;
}

// numpy's pairwise summation of n values (numpy/_core/src/umath/
// loops_utils.h.src: n > 128 splits at n2 = n/2 - (n/2 mod 8)), cut into its
// subtrees of <= seg values: the leaves of the cut in order ...
using rq::TILE_PATHS;  // segment payoff spans are tile-aligned

static void seg_nodes(int64_t a, int64_t n, int64_t seg, std::vector<std::pair<int64_t, int64_t>> &out) {
  if (n <= seg) {
    out.emplace_back(a, n);
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  seg_nodes(a, n2, seg, out);
  seg_nodes(a + n2, n - n2, seg, out);
}
// ... and the sum of their subtree sums in the same tree order.
static double seg_combine(int64_t n, int64_t seg, const double *sums, size_t &k) {
  if (n <= seg) return sums[k++];
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  const double l = seg_combine(n2, seg, sums, k);
  return l + seg_combine(n - n2, seg, sums, k);
}

int rq_estimate(rq_sampler *s, const rq_model *model, const int64_t *grid_host, int32_t ngrid,
                double *theta_dev, int32_t *kernel_launches, void *stream) {
  if (!s) return fail(RQ_ERR_VALUE, "sampler is NULL");
  int rc = check_grid(grid_host, ngrid);
  if (rc) return rc;
  if (grid_host[ngrid - 1] > rq_index_limit(s->t.gen))
    return fail(RQ_ERR_RANGE, "N = %lld exceeds the generator's index range %lld",
                (long long)grid_host[ngrid - 1], (long long)rq_index_limit(s->t.gen));
  cudaStream_t st = (cudaStream_t)stream;
  rq::ModelParams mp{};
  DevMem tab;
  if ((rc = model_to_params(model, s->t.dim, mp, tab, st))) return rc;
  // Grid marks up to SEG paths share one payoff buffer per replication batch
  // (prefixes of one pass); longer marks (counter-based generators) are
  // evaluated in segments, each a subtree of numpy's pairwise tree, so no
  // buffer exceeds SEG payoffs per replication.
  const int64_t SEG = std::max<int64_t>(TILE_PATHS, env_int("RQ_SEG_PATHS", (int64_t)1 << 31));
  const bool seq = rq::gen_sequential(s->t.gen);
  int ns = 0;  // grid marks of the shared pass: grid[0 .. ns)
  while (ns < ngrid && (seq || grid_host[ns] <= SEG)) ns++;
  int launched = 0;
  if (ns > 0) {
    const int64_t nmax = grid_host[ns - 1];
    // replication batch: payoff buffer <= 1 GiB (2^27 paths), >= 1 replication
    int64_t B = std::max<int64_t>(1, env_int("RQ_BATCH_PATHS", (int64_t)128 << 20) / nmax);
    B = std::min<int64_t>(B, s->t.rep_count);
    B = std::min<int64_t>(B, 65535);  // the reduction's grid.y
    std::vector<HostPlan> hplans(ns);
    std::vector<DevPlan> dplans(ns);
    int32_t maxnodes = 1;
    for (int g = 0; g < ns; g++) {
      build_plan(grid_host[g], hplans[g]);
      maxnodes = std::max(maxnodes, hplans[g].nnodes);
      if ((rc = upload_plan(hplans[g], dplans[g], st))) return rc;
    }
    DevMem pay_m(st), scratch_m(st), tickets_m(st);
    RQ_CUDA(pay_m.alloc(sizeof(double) * B * nmax));
    RQ_CUDA(scratch_m.alloc(sizeof(double) * B * maxnodes));
    RQ_CUDA(tickets_m.alloc(sizeof(unsigned) * B));
    double *pay = pay_m.as<double>(), *scratch = scratch_m.as<double>();
    unsigned *tickets = tickets_m.as<unsigned>();
    RQ_CUDA(cudaMemsetAsync(tickets, 0, sizeof(unsigned) * B, st));
    SeqRun R;
    if (seq && (rc = seq_begin(s->t, mp, (int)B, 0, nmax, R, st))) return rc;
    for (int64_t r0 = 0; r0 < s->t.rep_count; r0 += B) {
      int rn = (int)std::min<int64_t>(B, s->t.rep_count - r0);
      cudaError_t e;
      if (seq) {
        int blocks = 0;
        if ((rc = seq_batch(s->t, (int)r0, rn, R, &blocks, &launched, st))) return rc;
        KTimer kt(&g_stats.paths_ms, st);
        e = rq::launch_paths_seq(s->t, mp, (int)r0, rn, nmax, R.q, blocks, pay, &launched, st);
        stat_add(g_stats.paths_launches, (int64_t)1);
      } else {
        KTimer kt(&g_stats.paths_ms, st);
        e = rq::launch_paths(s->t, mp, (int)r0, rn, 0, nmax, pay, &launched, st);
        stat_add(g_stats.paths_launches, (int64_t)1);
      }
      if (e != cudaSuccess) return fail(RQ_ERR_CUDA, "path kernel: %s", cudaGetErrorString(e));
      for (int g = 0; g < ns; g++) {
        KTimer kt(&g_stats.reduce_ms, st);
        e = rq::launch_reduce(dplans[g].p, pay, nmax, rn, theta_dev + r0 * ngrid + g, ngrid,
                              scratch, tickets, st);
        if (e != cudaSuccess) return fail(RQ_ERR_CUDA, "reduce kernel: %s", cudaGetErrorString(e));
        launched++;
      }
    }
  }
  if (ns < ngrid) {  // segmented marks, one replication at a time
    std::vector<std::vector<std::pair<int64_t, int64_t>>> nodes(ngrid);
    std::map<int64_t, DevPlan> plans;  // pairwise plan per subtree length (a few distinct)
    int32_t maxnodes = 1;
    int64_t maxspan = 0;
    size_t maxk = 0;
    for (int g = ns; g < ngrid; g++) {
      seg_nodes(0, grid_host[g], SEG, nodes[g]);
      maxk = std::max(maxk, nodes[g].size());
      for (auto &nd : nodes[g]) {
        const int64_t a0 = nd.first / TILE_PATHS * TILE_PATHS;
        maxspan = std::max(maxspan, (nd.first + nd.second + TILE_PATHS - 1) / TILE_PATHS * TILE_PATHS - a0);
        if (!plans.count(nd.second)) {
          HostPlan hp;
          build_plan(nd.second, hp);
          maxnodes = std::max(maxnodes, hp.nnodes);
          if ((rc = upload_plan(hp, plans[nd.second], st))) return rc;
          plans[nd.second].p.n = 1;  // the subtree's sum, not a mean
        }
      }
    }
    DevMem pay_m(st), scratch_m(st), tickets_m(st), sums_m(st);
    RQ_CUDA(pay_m.alloc(sizeof(double) * maxspan));
    RQ_CUDA(scratch_m.alloc(sizeof(double) * maxnodes));
    RQ_CUDA(tickets_m.alloc(sizeof(unsigned)));
    RQ_CUDA(sums_m.alloc(sizeof(double) * maxk));
    RQ_CUDA(cudaMemsetAsync(tickets_m.p, 0, sizeof(unsigned), st));
    double *pay = pay_m.as<double>(), *sums_dev = sums_m.as<double>();
    std::vector<double> sums(maxk), theta_host(ngrid - ns);
    for (int64_t r = 0; r < s->t.rep_count; r++) {
      for (int g = ns; g < ngrid; g++) {
        for (size_t k = 0; k < nodes[g].size(); k++) {
          const int64_t a = nodes[g][k].first, len = nodes[g][k].second;
          const int64_t a0 = a / TILE_PATHS * TILE_PATHS;  // tile-aligned payoff span
          const int64_t a1 = (a + len + TILE_PATHS - 1) / TILE_PATHS * TILE_PATHS;
          cudaError_t e;
          {
            KTimer kt(&g_stats.paths_ms, st);
            e = rq::launch_paths(s->t, mp, (int)r, 1, a0, a1 - a0, pay, &launched, st);
            stat_add(g_stats.paths_launches, (int64_t)1);
          }
          if (e != cudaSuccess) return fail(RQ_ERR_CUDA, "path kernel: %s", cudaGetErrorString(e));
          {
            KTimer kt(&g_stats.reduce_ms, st);
            e = rq::launch_reduce(plans[len].p, pay + (a - a0), a1 - a0, 1, sums_dev + k, 1,
                                  scratch_m.as<double>(), tickets_m.as<unsigned>(), st);
          }
          if (e != cudaSuccess) return fail(RQ_ERR_CUDA, "reduce kernel: %s", cudaGetErrorString(e));
          launched++;
        }
        RQ_CUDA(cudaMemcpyAsync(sums.data(), sums_dev, sizeof(double) * nodes[g].size(),
                                cudaMemcpyDeviceToHost, st));
        RQ_CUDA(cudaStreamSynchronize(st));
        size_t k = 0;
        theta_host[g - ns] = seg_combine(grid_host[g], SEG, sums.data(), k) / (double)grid_host[g];
      }
      RQ_CUDA(cudaMemcpyAsync(theta_dev + r * ngrid + ns, theta_host.data(),
                              sizeof(double) * (ngrid - ns), cudaMemcpyHostToDevice, st));
      RQ_CUDA(cudaStreamSynchronize(st));  // theta_host is reused
    }
  }
  if (kernel_launches) *kernel_launches += launched;
  return RQ_OK;
}

// Device table bytes of one replication's randomisation (rq_sampler_create).
static size_t sampler_bytes_per_rep(int generator, int dim) {
  if (dim < 1) return 64;
  const HostTables &T = host_tables();
  switch (generator) {
    case rq::GEN_RASRAP_RECURSIVE:
    case rq::GEN_RASRAP_COUNTER:
      if (dim > rq::MAX_DIM) return 64;
      return 2 * (size_t)T.total_bases(dim) + 8 * (size_t)T.total_sums(dim) +
             2 * (size_t)T.total_caps(dim) + 8 * (size_t)dim + 64;
    case rq::GEN_SOBOL_GRAY:
    case rq::GEN_SOBOL_COUNTER: return 4 * 33 * (size_t)dim + 64;
    case rq::GEN_KAKUTANI: return 8 * (size_t)dim + 64;
  }
  return 64;
}

int rq_run_replications(int generator, const rq_model *model, uint64_t seed, int64_t rep_first,
                        int64_t rep_count, const int64_t *grid_host, int32_t ngrid,
                        double *theta_host, int32_t *kernel_launches) {
  if (!theta_host) return fail(RQ_ERR_VALUE, "theta_host is NULL");
  if (rep_count < 1) return fail(RQ_ERR_VALUE, "need at least one replication");
  int rc = check_grid(grid_host, ngrid);
  if (rc) return rc;
  if (generator >= 0 && generator <= rq::GEN_LAST && grid_host[ngrid - 1] > rq_index_limit(generator))
    return fail(RQ_ERR_RANGE, "N = %lld exceeds the generator's index range %lld",
                (long long)grid_host[ngrid - 1], (long long)rq_index_limit(generator));
  // one non-blocking stream per device (a process may drive several GPUs)
  static std::mutex smu;
  static cudaStream_t streams[64] = {};
  int dev = 0;
  RQ_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(RQ_ERR_VALUE, "device ordinal %d out of range", dev);
  cudaStream_t st;
  {
    std::lock_guard<std::mutex> lk(smu);
    if (!streams[dev]) RQ_CUDA(cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking));
    st = streams[dev];
  }
  DevMem theta_m(st);
  RQ_CUDA(theta_m.alloc(sizeof(double) * rep_count * ngrid));
  double *theta_dev = theta_m.as<double>();
  // replication groups bound the randomisation tables to ~256 MiB
  const int dim = model ? model->dim : 0;
  const int64_t G = std::max<int64_t>(
      1, std::min<int64_t>(4096, ((int64_t)256 << 20) / (int64_t)sampler_bytes_per_rep(generator, dim)));
  for (int64_t r0 = 0; r0 < rep_count; r0 += G) {
    int32_t rn = (int32_t)std::min<int64_t>(G, rep_count - r0);
    rq_sampler *S = nullptr;
    if ((rc = rq_sampler_create(&S, generator, dim, seed, rep_first + r0, rn, st))) return rc;
    if (kernel_launches && generator != rq::GEN_PHILOX && generator != rq::GEN_SFC64 &&
        generator != rq::GEN_TWISTER)  // (kakutani / xorwow: their start kernels)
      *kernel_launches += 1;  // the randomisation setup kernel
    rc = rq_estimate(S, model, grid_host, ngrid, theta_dev + r0 * ngrid, kernel_launches, st);
    const cudaError_t e = cudaStreamSynchronize(st);
    rq_sampler_destroy(S);
    if (rc) return rc;
    if (e != cudaSuccess) return fail(RQ_ERR_CUDA, "%s", cudaGetErrorString(e));
  }
  RQ_CUDA(cudaMemcpyAsync(theta_host, theta_dev, sizeof(double) * rep_count * ngrid,
                          cudaMemcpyDeviceToHost, st));
  stat_add(g_stats.d2h, (uint64_t)(sizeof(double) * rep_count * ngrid));
  RQ_CUDA(cudaStreamSynchronize(st));
  for (int64_t k = 0; k < rep_count * ngrid; k++)
    if (!std::isfinite(theta_host[k]))
      return fail(RQ_ERR_NONFINITE, "replication %lld produced a non-finite estimate",
                  (long long)(rep_first + k / ngrid));
  return RQ_OK;
}

int rq_model_payoffs(const rq_model *model, const double *u_dev, int64_t npaths,
                     double *out_dev, void *stream) {
  if (!model) return fail(RQ_ERR_VALUE, "model is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  rq::ModelParams mp{};
  DevMem tab;
  int rc = model_to_params(model, model->dim, mp, tab, st);
  if (rc) return rc;
  if (mp.kind != rq::MODEL_LIBOR && mp.kind != rq::MODEL_MBS)
    return fail(RQ_ERR_VALUE, "payoff kernel only for libor/mbs");
  RQ_CUDA(rq::launch_model_payoffs(mp, u_dev, npaths, out_dev, st));
  return RQ_OK;
}

int rq_inv_normal(const double *u_dev, int64_t n, double *out_dev, void *stream) {
  RQ_CUDA(rq::launch_inv_normal(u_dev, n, out_dev, (cudaStream_t)stream));
  return RQ_OK;
}

int rq_stream_normals(rq_sampler *s, int32_t rep_local, int64_t npoints, double *sum_dev,
                      double *store_dev, void *stream) {
  int rc = check_rep(s, rep_local);
  if (rc) return rc;
  if (npoints < 1 || npoints > ((int64_t)1 << 32)) return fail(RQ_ERR_VALUE, "npoints outside 1..2^32");
  if (rq::gen_sequential(s->t.gen))
    return fail(RQ_ERR_VALUE, "the normals stream is for counter/QMC generators (config 4)");
  cudaStream_t st = (cudaStream_t)stream;
  int blocks = rq::stream_grid_blocks(s->t);
  DevMem bs_m(st);
  RQ_CUDA(bs_m.alloc(sizeof(double) * blocks));
  double *bs = bs_m.as<double>();
  RQ_CUDA(rq::launch_stream_normals(s->t, rep_local, npoints, bs, blocks, store_dev, st));
  return rq_pairwise_sum(bs, blocks, sum_dev, stream);
}

void rq_stats_reset(int timing) {
  std::lock_guard<std::mutex> lk(g_stats_mu);
  g_stats = Stats();
  g_stats.timing = timing != 0;
}

void rq_stats_get(uint64_t *h2d, uint64_t *d2h, double *setup_ms, double *paths_ms,
                  double *reduce_ms, int64_t *paths_launches) {
  std::lock_guard<std::mutex> lk(g_stats_mu);
  if (h2d) *h2d = g_stats.h2d;
  if (d2h) *d2h = g_stats.d2h;
  if (setup_ms) *setup_ms = g_stats.setup_ms;
  if (paths_ms) *paths_ms = g_stats.paths_ms;
  if (reduce_ms) *reduce_ms = g_stats.reduce_ms;
  if (paths_launches) *paths_launches = g_stats.paths_launches;
}

int rq_fp64_peak(double *slots_per_s, double *ms_out) {
  int dev = 0, sms = 0;
  RQ_CUDA(cudaGetDevice(&dev));
  RQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  double *sink = nullptr;
  RQ_CUDA(cudaMalloc(&sink, 256 * sizeof(double)));
  cudaEvent_t a, b;
  RQ_CUDA(cudaEventCreate(&a));
  RQ_CUDA(cudaEventCreate(&b));
  const int blocks = sms * 8, iters = 4096;
  RQ_CUDA(rq::launch_dfma_peak(blocks, 64, sink, 0));  // warm-up / clocks up
  RQ_CUDA(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; r++) {
    RQ_CUDA(cudaEventRecord(a, 0));
    RQ_CUDA(rq::launch_dfma_peak(blocks, iters, sink, 0));
    RQ_CUDA(cudaEventRecord(b, 0));
    RQ_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    RQ_CUDA(cudaEventElapsedTime(&ms, a, b));
    best = std::min(best, ms);
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  double slots = (double)blocks * 256 * iters * rq::PEAK_SLOTS_PER_ITER;
  if (slots_per_s) *slots_per_s = slots / (best * 1e-3);
  if (ms_out) *ms_out = best;
  return RQ_OK;
}

int rq_pairwise_sum_host(const double *a_host, int64_t n, double *out_host) {
  if (n < 1 || !a_host || !out_host) return fail(RQ_ERR_VALUE, "n must be >= 1");
  HostPlan hp;
  build_plan(n, hp);
  std::vector<double> val(hp.nnodes);
  for (size_t k = 0; k < hp.leaf_len.size(); k++) {
    const double *a = a_host + hp.leaf_start[k];
    int m = hp.leaf_len[k];
    double res = 0.0;
    if (m < 8) {
      for (int i = 0; i < m; i++) res += a[i];
    } else {
      double r[8];
      int i;
      for (int j = 0; j < 8; j++) r[j] = a[j];
      for (i = 8; i < m - (m % 8); i += 8)
        for (int j = 0; j < 8; j++) r[j] += a[i + j];
      res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      for (; i < m; i++) res += a[i];
    }
    val[k] = res;
  }
  for (size_t lv = 0; lv + 1 < hp.level_off.size(); lv++)
    for (int32_t e = hp.level_off[lv]; e < hp.level_off[lv + 1]; e++)
      val[hp.node_id[e]] = val[hp.node_l[e]] + val[hp.node_r[e]];
  *out_host = val[hp.root];
  return RQ_OK;
}

int rq_pairwise_sum(const double *a_dev, int64_t n, double *out_dev, void *stream) {
  if (n < 1) return fail(RQ_ERR_VALUE, "n must be >= 1");
  cudaStream_t st = (cudaStream_t)stream;
  HostPlan hp;
  build_plan(n, hp);
  DevPlan dp;
  int rc = upload_plan(hp, dp, st);
  if (rc) return rc;
  DevMem scratch_m(st), tickets_m(st);
  RQ_CUDA(scratch_m.alloc(sizeof(double) * hp.nnodes));
  RQ_CUDA(tickets_m.alloc(sizeof(unsigned)));
  double *scratch = scratch_m.as<double>();
  unsigned *tickets = tickets_m.as<unsigned>();
  RQ_CUDA(cudaMemsetAsync(tickets, 0, sizeof(unsigned), st));
  // theta = sum / n: multiply back by n is not exact, so reduce with n = 1 divisor
  dp.p.n = 1;
  RQ_CUDA(rq::launch_reduce(dp.p, a_dev, n, 1, out_dev, 1, scratch, tickets, st));
  return RQ_OK;
}

}  // extern "C"
