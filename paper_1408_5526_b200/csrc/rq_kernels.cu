// rq_kernels.cu -- sm_100a kernels of the RQMC estimator.
//
// Fused path kernel (k_paths): one CTA owns a tile of TILE consecutive paths
// of one replication and walks its tiles (persistent, grid-stride) in units
// of (tile, chunk of CHUNK dimensions).  Per unit:
//
//   generator   uniforms of the unit into a shared-memory tile zt[dd][t]
//               (Rasrap / Sobol': warp w builds the rows dd = w (mod WARPS)
//               for all TILE points; PRNGs: every thread its own column)
//   normals     warp-cooperative inverse normal of the thread's own column:
//               central branch inline, the ~9% tail inputs compacted into a
//               per-warp queue and evaluated 32 at a time
//   model       thread-per-path state in registers (forward rates / MBS
//               cash-flow state) advanced through the chunk's steps
//
// Two CTA barriers per unit separate the phases; the 4-6 CTAs resident on an
// SM are not in lock-step, so one CTA's generator phase overlaps another's
// FP64-dense model phase.  (A double-buffered variant that generated unit
// u+1 inside unit u's iteration measured slower and was dropped.)  The
// generator's level buffers and the inverse normal's tail queue are never
// live at the same time and share shared memory (PhaseShared).
// The payoff (8 B/path) is the only HBM write; k_reduce then applies
// numpy's pairwise-summation tree to each replication's payoff prefix
// (bit-identical to the reference np.sum).
#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cmath>
#include <vector>
#include <type_traits>

#include "rq_device.cuh"
#include "rq_internal.h"

#ifndef RQ_SOBOL_STREAM_REG
#define RQ_SOBOL_STREAM_REG 1  // config-4 Sobol' stream in register form (k_stream_reg)
#endif
#ifndef RQ_SOBOL_PERSIST
#define RQ_SOBOL_PERSIST 1  // persistent Sobol' tile state for single-chunk models
#endif
#ifndef RQ_REDUCE_WARP
#define RQ_REDUCE_WARP 1  // numpy pairwise leaves: eight lanes per leaf (coalesced)
#endif
#ifndef RQ_MBS_MG
#define RQ_MBS_MG 5  // MBS months evaluated together (ILP across months; 5: +0.5% C3 vs 4)
#endif
#ifndef RQ_LIBOR_SMEM_RATES
#define RQ_LIBOR_SMEM_RATES 40  // LIBOR S=80: forward rates kept in shared memory (0: all in registers)
#endif
#ifndef RQ_LIBOR_STATIC_MAX
#define RQ_LIBOR_STATIC_MAX 20  // LIBOR steps up to which the rate triangle is fully unrolled
#endif
#ifndef RQ_RASRAP_MINB
#define RQ_RASRAP_MINB 5  // CTAs per SM for the persistent Rasrap tile with LIBOR S <= 20
#endif
#ifndef RQ_BASE2
#define RQ_BASE2 1  // base 2 in closed form (bit reversal) instead of the digit tree
#endif
#ifndef RQ_TAIL_CAND
#define RQ_TAIL_CAND 1  // inverse-normal tail test on the high word (exact re-test in the queue)
#endif
#ifndef RQ_G2_FAST
#define RQ_G2_FAST 1  // global-sigma Rasrap tiles: level-pass-free path for J == 1 / small J == 2
#endif
#ifndef RQ_CT_CACHE
#define RQ_CT_CACHE 1  // counter-form tile: high-term tables reused while the prefix H0 is unchanged
#endif
#ifndef RQ_CT_PAIRS
#define RQ_CT_PAIRS 1  // counter-form tile: two dims' sum chains per thread at a time
                       // (+2.4% C2, +3.4% C3, +8.2% C4 rasrap-counter; four: -4% C2)
#endif
#ifndef RQ_SW_TABLES
#define RQ_SW_TABLES 1  // persistent Rasrap tile: sigma*w_0 / sigma*w_1 tables, two-level fast path
#endif
#ifndef RQ_WS
#define RQ_WS 1  // warp-specialised path kernel (producer / consumer warpgroups)
#endif
#ifndef RQ_MINB_SMALL
#define RQ_MINB_SMALL 4  // CTAs per SM targeted for LIBOR S <= 20 (register budget)
#endif

namespace rq {

constexpr int TILE = TILE_PATHS;   // paths per CTA tile = threads per CTA
constexpr int CHUNK = CHUNK_DIMS;  // dimensions per unit (multiple of 4 for Philox)
constexpr int WARPS = TILE / 32;
constexpr double TWO_M32 = 2.3283064365386963e-10;  // 2^-32
constexpr double TWO_M33 = 1.1641532182693481e-10;  // 2^-33
constexpr double TWO_M53 = 1.1102230246251565e-16;  // 2^-53

__constant__ HaltonDim c_hdim[CONST_DIMS];
__device__ HaltonDim g_hdim[MAX_DIM];  // every dim (those >= CONST_DIMS are read from here)
// Dim d's constants: warp-uniform constant-bank reads below CONST_DIMS, L1-
// cached global reads above.  The tile generators take WIDE (samplers of more
// than CONST_DIMS dims, dispatched on the host) as a template parameter, so
// the kernels of every benchmark configuration read c_hdim with no test;
// hdim() serves the once-per-point paths (setup, at()).
template <bool WIDE>
__device__ __forceinline__ HaltonDim hdim_t(int d) {
  if constexpr (WIDE) return g_hdim[d];
  else return c_hdim[d];
}
__device__ __forceinline__ HaltonDim hdim(int d) {
  return d < CONST_DIMS ? c_hdim[d] : g_hdim[d];
}
constexpr int CWTS = 1280;  // binpow weights of the first dims, in the constant bank
static_assert(CHUNK_DIMS <= 40, "persistent Rasrap tiles assume their weights fit c_wts");
static_assert(CHUNK_DIMS <= 20, "persistent Rasrap tiles stage sigma of <= 20 dims (639 entries)");
__constant__ double c_wts[CWTS];
constexpr int WTS_CAP = 81920;  // sum over MAX_DIM dims of cap + 1 (78,909)
__device__ double g_wts[WTS_CAP];     // binpow(inv_p, j+1): numba `x ** int` (halton.py:409)
__device__ double g_cscale[WTS_CAP];  // counter-form scale chain (halton.py:436)

cudaError_t upload_halton_dims(const HaltonDim *dims, int n, const double *wts,
                               const double *cscale, int nw) {
  if (n > MAX_DIM || nw > WTS_CAP) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemcpyToSymbol(c_hdim, dims, sizeof(HaltonDim) * (n < CONST_DIMS ? n : CONST_DIMS));
  if (e != cudaSuccess) return e;
  e = cudaMemcpyToSymbol(g_hdim, dims, sizeof(HaltonDim) * n);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyToSymbol(g_wts, wts, sizeof(double) * nw);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyToSymbol(c_wts, wts, sizeof(double) * (nw < CWTS ? nw : CWTS));
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(g_cscale, cscale, sizeof(double) * nw);
}

// floor(t / base) for t < 2^32 (round-up magic, 33-bit multiplier)
__device__ __forceinline__ uint32_t div_base(uint32_t t, const HaltonDim &h) {
  uint64_t x = (uint64_t)__umulhi(t, h.mlo) + t;
  return (uint32_t)(x >> h.ell);
}
// floor(x / base) for x < 2^46 (64-bit round-up magic, see rq_capi.cu)
__device__ __forceinline__ uint64_t div_base64(uint64_t x, const HaltonDim &h) {
  return __umul64hi(x, h.m64);
}
__device__ __forceinline__ double u16d(uint16_t v) { return (double)v; }
// Thread index within its TILE-thread group (the model side of a path
// kernel: threadIdx.x in k_paths, the consumer half in k_paths_ws).
__device__ __forceinline__ int ctid() { return (int)(threadIdx.x & (TILE - 1)); }
// 32-bit shared-state-space address of a shared object, and a load from it
__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}

// ======================================================================
// Setup kernels (per replication randomisation, on device)
// ======================================================================

// One thread per (replication, dimension): rasrap_config + RasrapStream
// init (halton.py:345-360, 256-278, 139-155; seeding.py:59-65).
// invert_radical (start digits, n0) and the init partial sums of one
// (replication, dim) from its permutation sg (halton.py:139-155, 273-278)
template <class SG>
__device__ void rasrap_start_and_sums(const RepTables &t, int rl, int d, const HaltonDim &h,
                                      uint64_t k53, SG sgv, uint16_t *digits, double *sums,
                                      uint64_t *start) {
  // invert_radical: scaled = floor(k53 * p^K / 2^53), digits reversed
  uint64_t pk = 1;
  for (int i = 0; i < h.K; i++) pk *= (uint64_t)h.base;
  uint64_t lo = k53 * pk, hi = umulhi64(k53, pk);
  uint64_t scaled = (hi << 11) | (lo >> 53);
  uint16_t *dg = digits + (int64_t)rl * t.dig_stride + h.dig_off;
  for (int j = h.K; j < h.cap; j++) dg[j] = 0;
  uint64_t n0 = 0;
  for (int s = 0; s < h.K; s++) {
    uint32_t dgt = (uint32_t)(scaled % (uint64_t)h.base);
    dg[h.K - 1 - s] = (uint16_t)dgt;
    n0 = n0 * (uint64_t)h.base + dgt;
    scaled /= (uint64_t)h.base;
  }
  start[(int64_t)rl * t.dim + d] = n0;
  // init partial sums: scale = pow(1/p, K) then *= p (halton.py:273-278)
  double *sm = sums + (int64_t)rl * t.sum_stride + h.sum_off;
  for (int j = h.K; j <= h.cap; j++) sm[j] = 0.0;
  double scale = h.scale0;
  for (int j = h.K - 1; j >= 0; j--) {
    sm[j] = dadd(sm[j + 1], dmul((double)sgv(dg[j]), scale));
    scale = dmul(scale, (double)h.base);
  }
}

// One thread per (replication, dim) of dims [d_lo, d_hi) (small bases: short
// shuffles).  derive_rng(key, d).random() then .permutation(p).
__global__ void k_rasrap_setup(RepTables t, int d_lo, int d_hi, uint16_t *sigma,
                               uint16_t *digits, double *sums, uint64_t *start) {
  const int nd = d_hi - d_lo;
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)t.rep_count * nd) return;
  int rl = (int)(gid / nd), d = d_lo + (int)(gid % nd);
  const HaltonDim h = hdim(d);
  uint64_t m = (uint64_t)(t.rep_first + rl);
  uint64_t key = derive_key3(t.seed, 4, m);  // harness.py:113, family "rasrap"
  Pcg64 g;
  pcg_seed(g, derive_key2(key, (uint64_t)d));  // derive_rng(seed, i)
  uint64_t k53 = pcg_next64(g) >> 11;          // rng.random() = k53 * 2^-53
  uint16_t *sg = sigma + (int64_t)rl * t.sig_stride + h.sig_off;
  for (int a = 0; a < h.base; a++) sg[a] = (uint16_t)a;
  for (int i = h.base - 1; i >= 1; i--) {  // rng.permutation(p)
    int j = (int)pcg_interval32(g, (uint32_t)i);
    uint16_t tmp = sg[j];
    sg[j] = sg[i];
    sg[i] = tmp;
  }
  rasrap_start_and_sums(t, rl, d, h, k53, [&](uint32_t a) { return sg[a]; }, digits, sums, start);
}

// One warp per (replication, dim) of dims [d_lo, d_hi) (large bases): the
// shuffle is one sequential chain of p draws and swaps, so it runs on lane 0
// against a shared-memory copy (30-cycle instead of L2-latency swaps); the
// lanes initialise and write the permutation out coalesced.
__global__ void k_rasrap_setup_warp(RepTables t, int d_lo, int d_hi, int smax, uint16_t *sigma,
                                    uint16_t *digits, double *sums, uint64_t *start) {
  extern __shared__ uint16_t perm_sm[];
  const int nd = d_hi - d_lo, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t unit = (int64_t)blockIdx.x * (blockDim.x >> 5) + w;
  if (unit >= (int64_t)t.rep_count * nd) return;
  const int rl = (int)(unit / nd), d = d_lo + (int)(unit % nd);
  const HaltonDim h = hdim(d);
  uint16_t *ps = perm_sm + (size_t)w * smax;
  for (int a = lane; a < h.base; a += 32) ps[a] = (uint16_t)a;
  __syncwarp();
  uint64_t k53 = 0;
  if (lane == 0) {
    uint64_t key = derive_key3(t.seed, 4, (uint64_t)(t.rep_first + rl));
    Pcg64 g;
    pcg_seed(g, derive_key2(key, (uint64_t)d));
    k53 = pcg_next64(g) >> 11;
    for (int i = h.base - 1; i >= 1; i--) {
      int j = (int)pcg_interval32(g, (uint32_t)i);
      uint16_t tmp = ps[j];
      ps[j] = ps[i];
      ps[i] = tmp;
    }
  }
  __syncwarp();
  uint16_t *sg = sigma + (int64_t)rl * t.sig_stride + h.sig_off;
  for (int a = lane; a < h.base; a += 32) sg[a] = ps[a];
  if (lane == 0)
    rasrap_start_and_sums(t, rl, d, h, k53, [&](uint32_t a) { return ps[a]; }, digits, sums,
                          start);
}

// One thread per (replication, dimension): random_scramble + pre-scrambled
// direction words (sobol.py:259-275, 236-248).
__global__ void k_sobol_setup(RepTables t, const uint32_t *v, uint32_t *gen_v,
                              uint32_t *shift) {
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)t.rep_count * t.dim) return;
  int rl = (int)(gid / t.dim), d = (int)(gid % t.dim);
  uint64_t m = (uint64_t)(t.rep_first + rl);
  uint64_t key = derive_key3(t.seed, 5, m);
  Pcg64 g;
  pcg_seed(g, derive_key3(key, m, (uint64_t)d));  // derive_rng(seed, replication, d)
  uint32_t cols[SOBOL_BITS];
  for (int c = 0; c < SOBOL_BITS; c++) {
    uint32_t bits = pcg_next32(g);
    uint32_t diag = 1u << (31 - c);
    cols[c] = diag | (bits & (diag - 1u));
  }
  shift[(int64_t)rl * t.dim + d] = pcg_next32(g);
  for (int k = 0; k < SOBOL_BITS; k++) {
    uint32_t y = v[d * SOBOL_BITS + k], z = 0;
    for (int c = 0; c < SOBOL_BITS; c++)
      if (y & (1u << (31 - c))) z ^= cols[c];
    gen_v[((int64_t)rl * t.dim + d) * SOBOL_BITS + k] = z;
  }
}

// ======================================================================
// Generators.  unit(rl, base, path, d0, Dc, zt) writes the uniforms of
// points base..base+TILE-1 (this thread's: path) for dims [d0, d0+Dc) into
// zt[dd*TILE + t].  It is warp-synchronous (no CTA barrier inside), so the
// caller can overlap it with other warps' model work.  "Tiled" generators
// require path == base + threadIdx.x; "direct" ones take any index
// (sampler.at).
// ======================================================================
constexpr int LEVBUF = 66;  // nodes per level buffer (>= TILE/2 + 2)

// Shared memory of the phases that never overlap inside a unit: the
// generator's per-warp ping-pong level buffers and the inverse normal's
// per-warp tail queues.
union PhaseShared {
  double lev[WARPS][2][LEVBUF];
  uint16_t tq[WARPS][CHUNK * 32];
};

constexpr int SIGD_MAX = 640;  // sigma entries staged as doubles (single-chunk dims)
static_assert(CHUNK == 20 && SIGD_MAX >= 639, "the first CHUNK primes sum to 639");

struct RasrapTileShared {
  uint16_t bd[CHUNK][MAX_CAP];     // base-p digits of the tile base B = n0 + base
  int16_t nn[CHUNK][MAX_CAP + 1];  // nodes per level: distinct prefixes floor(n / p^j)
  int32_t J[CHUNK];                // top level (one node shared by the whole tile)
  int32_t hB[CHUNK];               // highest digit where B differs from n0 (-1: B == n0)
  double sJ[CHUNK];                // stream partial sum S_J of the top node
  int32_t st_rl[CHUNK];            // replication the state belongs to (-1: none)
  int32_t stg_rl[WARPS];           // replication whose sigma a warp staged (warp-private)
  uint64_t st_base[CHUNK];         // tile base the state belongs to
  int32_t soff[CHUNK];             // offset of sigma_d in sigd
};
// + the persistent partial sums of the chunk's dims
struct RasrapTilePersistShared : RasrapTileShared {
  double P[CHUNK][MAX_CAP + 1];  // S_j(B), j = 0..cap
};
// + their sigma tables staged as doubles (single-chunk models: the first
// CHUNK dims)
struct RasrapTilePersistSigShared : RasrapTilePersistShared {
  double sigd[SIGD_MAX];
#if RQ_SW_TABLES
  // sigma(a) * w_0 and sigma(a) * w_1 per dim (the products the tree forms
  // at levels 0 and 1, same rounding): a two-level tile (J <= 2) needs no
  // level pass -- every leaf adds its parent's and its own term directly
  double sw0[SIGD_MAX], sw1[SIGD_MAX];
#endif
};
struct RasrapDirectShared {
  uint16_t scr[MAX_CAP][TILE];  // per-thread digits (direct path)
};
struct NoShared {
  int unused;
};

// single-chunk models whose chunk width is a compile-time constant
template <class M>
struct FixedDims {
  template <class T>
  static constexpr int get(decltype(T::FIXED_DIMS) *) { return T::FIXED_DIMS; }
  template <class T>
  static constexpr int get(...) { return 0; }
  static constexpr int value = get<M>(nullptr);
};

// models with a dynamic shared-memory region (after the tile / generator's)
template <class M>
struct ModelDyn {
  template <class T>
  static constexpr bool has(decltype(&T::dyn_bytes)) { return true; }
  template <class T>
  static constexpr bool has(...) { return false; }
  static constexpr bool value = has<M>(nullptr);
  static __host__ __device__ size_t bytes(int dim) {
    if constexpr (value) return M::dyn_bytes(dim);
    else return 0;
  }
  static __device__ __forceinline__ void give(M &m, double *p) {
    if constexpr (value) m.set_dyn(p);
  }
};

// kernels hand the phase-shared buffers to generators that use them
template <class G>
struct HasPhase {
  template <class T>
  static constexpr bool get(decltype(&T::ph)) { return true; }
  template <class T>
  static constexpr bool get(...) { return false; }
  static constexpr bool value = get<G>(nullptr);
};
template <class G>
__device__ __forceinline__ void give_phase(G &g, PhaseShared &p) {
  if constexpr (HasPhase<G>::value) g.ph = &p;
}

// Recursive-form point at an arbitrary index (Alg. 2, halton.py:392-416)
// without replaying the stream: for n = n0 + i let h be the highest digit
// where n and n0 differ (= highest carry the odometer reached).  The stream
// then holds sums[j] = init_sums[j] above h and the chain
// S_j = S_{j+1} + sigma(a_j) * binpow(1/p, j+1) below, so the point is that
// chain started from init_sums[h+1] -- bit-identical to the reference.
// Indices are 64-bit: n = n0 + i stays inside the digit window (p^(K+8) >=
// 2^40) for i < RQ_RASRAP_INDEX_MAX (2^39, checked by the C ABI).
__device__ double rasrap_rec_direct(const RepTables &t, int rl, int d, uint64_t i,
                                    uint16_t *scr) {
  const HaltonDim h = hdim(d);
  const uint16_t *d0 = t.digits + (int64_t)rl * t.dig_stride + h.dig_off;
  const uint16_t *sg = t.sigma + (int64_t)rl * t.sig_stride + h.sig_off;
  const double *sums = t.sums + (int64_t)rl * t.sum_stride + h.sum_off;
  uint64_t r = i;
  uint32_t carry = 0;
  int hi = -1, j = 0;
  while (r != 0u || carry != 0u) {
    const uint64_t q = r >> 32 ? div_base64(r, h) : (uint64_t)div_base((uint32_t)r, h);
    uint32_t a0 = d0[j];
    uint32_t a = a0 + (uint32_t)(r - q * (uint64_t)h.base) + carry;
    carry = a >= (uint32_t)h.base;
    a = carry ? a - (uint32_t)h.base : a;
    scr[j * TILE] = (uint16_t)a;
    hi = (a != a0) ? j : hi;
    r = q;
    j++;
  }
  const double *w = g_wts + h.sum_off;
  double S = sums[hi + 1];
  for (int k = hi; k >= 0; k--) S = dadd(S, dmul(u16d(sg[scr[k * TILE]]), w[k]));
  return S;
}

struct GenRasrapRecDirect {
  using Shared = RasrapDirectShared;
  const RepTables *t;
  Shared *sh;
  __device__ void setup(const RepTables &t_, Shared &s, int = 0) {
    t = &t_;
    sh = &s;
  }
  __device__ void unit(int rl, uint64_t, uint64_t path, int d0, int Dc, double *zt) {
    uint16_t *scr = &sh->scr[0][0] + threadIdx.x;
    for (int dd = 0; dd < Dc; dd++)
      zt[dd * TILE + threadIdx.x] = rasrap_rec_direct(*t, rl, d0 + dd, path, scr);
  }
};

// Tiled recursive form, evaluated level by level over the digit tree of the
// tile's TILE consecutive indices n = B + k, B = n0 + base.
//
// With S_j(n) the stream's partial sum at position j for index n, the
// reference recursion (halton.py:402-414, init sums halton.py:273-278) is
//     S_j(n) = init_sums[j]                               if floor(n/p^j) == floor(n0/p^j)
//            = S_{j+1}(n) + sigma(n_j) * binpow(1/p, j+1)  otherwise
// and S_j only depends on the prefix u = floor(n/p^j).  The tile's indices
// have N_j distinct prefixes at level j (N_0 = TILE, N_{j+1} = floor((b_j +
// N_j - 1)/p) + 1 with b_j the digits of B), so the warp owning a dim
// evaluates the N_j nodes of each level from their parents, top (N_J = 1,
// whose S_J is the chain from init_sums[hB+1]) to level 0 = the points.
// That is ~TILE * p/(p-1) node updates per tile and dim instead of
// TILE * log_p(n) for independent per-point chains, with the same
// operations in the same order as the reference (bit-identical).
template <bool PERSIST, bool SIGSM = PERSIST, bool WIDE = false>
struct GenRasrapRecTile {
  static_assert(!(SIGSM && WIDE), "shared-memory sigma tiles have <= CHUNK dims");
  using Shared = typename std::conditional<
      PERSIST,
      typename std::conditional<SIGSM, RasrapTilePersistSigShared, RasrapTilePersistShared>::type,
      RasrapTileShared>::type;
  const RepTables *t;
  Shared *sh;
  PhaseShared *ph;  // level buffers (aliased with the tail queues, see PhaseShared)
  // PERSIST (dispatch: single-chunk models, <= CHUNK dims): consecutive tiles
  // of one CTA share a persistent stream state and the dims' sigma tables are
  // staged in shared memory as doubles (the first CHUNK primes sum to 639 <=
  // SIGD_MAX).  Compile-time, so the persistent kernel carries no stateless
  // or global-sigma code (instruction-cache footprint).  PERSIST without
  // SIGSM: the chunk-major stream (k_stream_chunks), a CTA owning one chunk
  // of any dims over consecutive tiles, sigma read from global memory.
  static constexpr bool persist = PERSIST;
  static constexpr bool sig_smem = SIGSM;
  __device__ __forceinline__ static HaltonDim hd(int d) { return hdim_t<WIDE>(d); }
  __device__ void setup(const RepTables &t_, Shared &s, int = 0) {
    t = &t_;
    sh = &s;
    for (int k = threadIdx.x; k < CHUNK; k += TILE) s.st_rl[k] = -1;
    for (int k = threadIdx.x; k < WARPS; k += TILE) s.stg_rl[k] = -1;
  }
  // Full state at B = n0 + base: digits, hB, P[j] = S_j(B) (chain from
  // init_sums[hB+1]); used for a CTA's first tile of a replication.
  __device__ void state_full(int rl, uint64_t base, int d, int dd) {
    Shared &R = *sh;
    const HaltonDim h = hd(d);
    const uint32_t p = (uint32_t)h.base;
    const uint16_t *n0d = t->digits + (int64_t)rl * t->dig_stride + h.dig_off;
    const double *ini = t->sums + (int64_t)rl * t->sum_stride + h.sum_off;
    const uint16_t *sg = t->sigma + (int64_t)rl * t->sig_stride + h.sig_off;
    const double *w = g_wts + h.sum_off;
    const uint64_t n0 = t->start[(int64_t)rl * t->dim + d];
    uint64_t qb = n0 + base, qn = n0;
    int j = 0, hB = -1;
#pragma unroll 1
    while (qb != qn) {  // positions where B's prefix still differs from n0's
      uint64_t nb = div_base64(qb, h), nq = div_base64(qn, h);
      uint32_t db = (uint32_t)(qb - nb * p), dn = (uint32_t)(qn - nq * p);
      R.bd[dd][j] = (uint16_t)db;
      hB = db != dn ? j : hB;
      qb = nb;
      qn = nq;
      j++;
    }
#pragma unroll 1
    for (; j < h.cap; j++) R.bd[dd][j] = n0d[j];
#pragma unroll 1
    for (int k = h.cap; k > hB; k--) R.P[dd][k] = ini[k];
    double S = ini[hB + 1];
#pragma unroll 1
    for (int k = hB; k >= 0; k--) {
      S = dadd(S, dmul(u16d(sg[R.bd[dd][k]]), w[k]));
      R.P[dd][k] = S;
    }
    R.hB[dd] = hB;
  }
  // Odometer step B -> B + TILE (the adding machine on the digit vector):
  // add TILE's base-p digits with carry, then re-chain the partial sums
  // below the highest changed digit.
  // Odometer step B -> B + TILE on the digits; returns the highest changed
  // digit (>= h.tdig: the top digit of TILE changes or carries out).
  __device__ int digits_advance(int d, int dd) {
    Shared &R = *sh;
    const HaltonDim h = hd(d);
    const uint32_t p = (uint32_t)h.base;
    uint32_t r = TILE, carry = 0;
    int j = 0, jmax = -1;
#pragma unroll 1
    while (r != 0u || carry != 0u) {
      const uint32_t q = __umulhi(r, h.m16);
      const uint32_t b = R.bd[dd][j];
      uint32_t a = b + (r - q * p) + carry;
      carry = a >= p;
      a = carry ? a - p : a;
      R.bd[dd][j] = (uint16_t)a;
      jmax = a != b ? j : jmax;
      r = q;
      j++;
    }
    int hB = R.hB[dd];
    R.hB[dd] = jmax > hB ? jmax : hB;  // a carry above hB makes that digit exceed n0's
    return jmax;
  }
  // Re-chain the partial sums P[k] = S_k(B) for k = jmax .. kmin.  Only
  // P[J] (this tile's top node) and P[k > tdig] (where every later re-chain
  // starts, since its jmax >= tdig) are ever read again, so the chain stops
  // at kmin = min(J, tdig + 1) instead of 0; P[k < kmin] go stale unused.
  __device__ void rechain(int rl, int d, int dd, int jmax, int kmin) {
    Shared &R = *sh;
    const HaltonDim h = hd(d);
    const double *ini = t->sums + (int64_t)rl * t->sum_stride + h.sum_off;
    const double *w = g_wts + h.sum_off;
    const int hB = R.hB[dd];
    double S = R.P[dd][jmax + 1];
    const double *sgd = sigd_of(dd);
    const uint16_t *sg = t->sigma + (int64_t)rl * t->sig_stride + h.sig_off;
#pragma unroll 1
    for (int k = jmax; k >= kmin; k--) {
      const double sv = sig_smem ? sgd[R.bd[dd][k]] : u16d(sg[R.bd[dd][k]]);
      S = k > hB ? ini[k] : dadd(S, dmul(sv, w[k]));
      R.P[dd][k] = S;
    }
  }
  __device__ __forceinline__ double pers_P(int dd, int j) const {
    if constexpr (PERSIST) return sh->P[dd][j];
    return 0.0;
  }
  __device__ __forceinline__ const double *sigd_of(int dd) const {
    if constexpr (SIGSM) return sh->sigd + sh->soff[dd];
    return nullptr;
  }
  // per-dim tile state (one lane per dim): digits of B, hB, level sizes, S_J
  __device__ void prepare_dim(int rl, uint64_t base, int d, int dd) {
    RasrapTileShared &R = *sh;
    const HaltonDim h = hd(d);
    if (!persist) {  // stateless: digits up to the top level, S_J by one chain
      prepare_stateless(rl, base, d, dd);
      return;
    }
    if constexpr (PERSIST) {
      const bool adv = R.st_rl[dd] == rl && R.st_base[dd] + TILE == base;
      const int jmax = adv ? digits_advance(d, dd) : -1;
      if (!adv) state_full(rl, base, d, dd);
      R.st_rl[dd] = rl;
      R.st_base[dd] = base;
      int N = TILE, J = 0, jr = 1;
      R.nn[dd][0] = (int16_t)N;
#pragma unroll 1
      while (N > 1) {
        N = (int)__umulhi((uint32_t)R.bd[dd][J] + (uint32_t)N - 1u, h.m16) + 1;
        J++;
        R.nn[dd][J] = (int16_t)N;
        jr = N > 32 ? J + 1 : jr;
      }
      if (adv) rechain(rl, d, dd, jmax, J < h.tdig + 1 ? J : h.tdig + 1);
      R.J[dd] = J | jr << 8;
      R.sJ[dd] = sh->P[dd][J];
    }
  }
  __device__ void prepare_stateless(int rl, uint64_t base, int d, int dd) {
    RasrapTileShared &R = *sh;
    const HaltonDim h = hd(d);
    const uint32_t p = (uint32_t)h.base;
    const uint16_t *n0d = t->digits + (int64_t)rl * t->dig_stride + h.dig_off;
    const double *ini = t->sums + (int64_t)rl * t->sum_stride + h.sum_off;
    const uint16_t *sg = t->sigma + (int64_t)rl * t->sig_stride + h.sig_off;
    const double *w = g_wts + h.sum_off;
    const uint64_t n0 = t->start[(int64_t)rl * t->dim + d];
    uint64_t qb = n0 + base, qn = n0;
    int j = 0, hB = -1;
#pragma unroll 1
    while (qb != qn) {  // positions where B's prefix still differs from n0's
      uint64_t nb = div_base64(qb, h), nq = div_base64(qn, h);
      uint32_t db = (uint32_t)(qb - nb * p), dn = (uint32_t)(qn - nq * p);
      R.bd[dd][j] = (uint16_t)db;
      hB = db != dn ? j : hB;
      qb = nb;
      qn = nq;
      j++;
    }
    int N = TILE, J = 0, jr = 1;
    R.nn[dd][0] = (int16_t)N;
#pragma unroll 1
    while (N > 1) {
      uint32_t bj = J < j ? R.bd[dd][J] : n0d[J];
      if (J >= j) R.bd[dd][J] = (uint16_t)bj;
      N = (int)__umulhi(bj + (uint32_t)N - 1u, h.m16) + 1;
      J++;
      R.nn[dd][J] = (int16_t)N;
      jr = N > 32 ? J + 1 : jr;
    }
    double S = ini[hB + 1 > J ? hB + 1 : J];
#pragma unroll 1
    for (int k = hB; k >= J; k--) S = dadd(S, dmul(u16d(sg[R.bd[dd][k]]), w[k]));
    R.J[dd] = J | jr << 8;
    R.hB[dd] = hB;
    R.sJ[dd] = S;
  }
  // Dim of slot k of warp w (-1: none): round-robin.  (Grouping the first
  // chunk's dims over the warps by tree cost measured -0.6..+0.1%.)
  __device__ __forceinline__ static int dim_slot(int warp, int k, int, int Dc) {
    const int dd = warp + k * WARPS;
    return dd < Dc ? dd : -1;
  }
  __device__ void stage_sigma(int rl, int d0, int Dc) {
    // warp w stages the sigma tables of its dims (dim_slot)
    Shared &R = *sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint16_t *gsig = t->sigma + (int64_t)rl * t->sig_stride;
    const int off0 = hd(d0).sig_off;
#pragma unroll 1
    for (int k = 0, dd; (dd = dim_slot(warp, k, d0, Dc)) >= 0; k++) {
      const HaltonDim h = hd(d0 + dd);
      const int o = h.sig_off - off0;
      if constexpr (SIGSM) {
#if RQ_SW_TABLES
        const double w0 = c_wts[h.sum_off], w1 = c_wts[h.sum_off + 1];
#endif
        for (int a = lane; a < h.base; a += 32) {
          const double sv = (double)gsig[h.sig_off + a];
          R.sigd[o + a] = sv;
#if RQ_SW_TABLES
          R.sw0[o + a] = dmul(sv, w0);
          R.sw1[o + a] = dmul(sv, w1);
#endif
        }
      }
      if (lane == 0) R.soff[dd] = o;
    }
    __syncwarp();
  }
  // Base 2 (dimension 0) in closed form.  Every partial sum of the
  // reference recursion is an exact dyadic rational there (weights
  // binpow(0.5, j+1) = 2^-(j+1), init sums from Python 0.5**active times
  // powers of 2, < 1 with <= 40 bits), so the point n = n0 + i is exactly
  // init_sums[h+1] + sum_{j<=h} sigma(n_j) 2^-(j+1) whatever the order of
  // the additions, h = the highest bit where n and n0 differ
  // (halton.py:402-414).  sigma is the identity or the flip on {0, 1}, so
  // the sum is the bit reversal of the low h+1 bits of n ^ flip: a handful
  // of integer ops per point instead of a 7-level tree.
  __device__ __forceinline__ void base2_points(int rl, uint64_t base, double *zd) {
    const int lane = threadIdx.x & 31;
    const HaltonDim &h = c_hdim[0];
    const uint64_t n0 = t->start[(int64_t)rl * t->dim];
    const double *ini = t->sums + (int64_t)rl * t->sum_stride + h.sum_off;
    const uint64_t flip = t->sigma[(int64_t)rl * t->sig_stride + h.sig_off] ? ~0ull : 0ull;
#pragma unroll
    for (int m = 0; m < TILE / 32; m++) {
      const int k = lane + 32 * m;
      const uint64_t n = n0 + base + (uint64_t)k, x = n ^ n0;
      double v;
      if (x == 0) {
        v = __ldg(ini);
      } else {
        const int hb = 63 - __clzll((long long)x);  // highest changed digit
        const uint64_t rev = __brevll((n ^ flip) << (63 - hb));  // bits 0..hb reversed
        // rev = sum_j sigma(n_j) 2^(hb-j) < 2^(hb+1): exact, scaled by 2^-(hb+1)
        const double f = __ull2double_rn(rev) * __hiloint2double((1022 - hb) << 20, 0);
        v = dadd(__ldg(ini + hb + 1), f);
      }
      zd[k] = v;
    }
  }
  __device__ void unit(int rl, uint64_t base, uint64_t, int d0, int Dc, double *zt) {
    RasrapTileShared &R = *sh;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (sig_smem && R.stg_rl[warp] != rl) {  // warp-private flag: no cross-warp read
      stage_sigma(rl, d0, Dc);
      __syncwarp();  // every lane has read the flag before lane 0 rewrites it
      if (lane == 0) R.stg_rl[warp] = rl;
    }
    {  // lane k prepares the dim of slot k (base 2: no tree state)
      const int dd = dim_slot(warp, lane, d0, Dc);
      if (dd >= 0 && (!RQ_BASE2 || d0 + dd != 0)) prepare_dim(rl, base, d0 + dd, dd);
      if (RQ_BASE2 && persist && dd == 0 && d0 == 0) {
        R.st_rl[0] = rl;
        R.st_base[0] = base;
      }
    }
    __syncwarp();
    const uint16_t *gsig = t->sigma + (int64_t)rl * t->sig_stride;
    const double *gsum = t->sums + (int64_t)rl * t->sum_stride;
#pragma unroll 1
    for (int k = 0, dd; (dd = dim_slot(warp, k, d0, Dc)) >= 0; k++) {
      if (RQ_BASE2 && d0 + dd == 0) {
        base2_points(rl, base, zt + dd * TILE);
        continue;
      }
      const HaltonDim h = hd(d0 + dd);
      const uint32_t p = (uint32_t)h.base, m16 = h.m16;
      const uint16_t *sg = gsig + h.sig_off;
      // sigma of the dim staged as doubles: one 32-bit shared address, so the
      // loads below are plain LDS (no generic-to-shared conversion per node)
      const uint32_t sgs = sig_smem ? smem_addr(sigd_of(dd)) : 0u;
      auto sig = [&](uint32_t a) { return sig_smem ? lds_f64(sgs + 8u * a) : u16d(sg[a]); };
      const double *ini = gsum + h.sum_off;
      // weights in the constant bank (always so for a persistent single-chunk
      // model: its <= CHUNK dims use < CWTS weights)
      const bool cw = SIGSM || h.sum_off + h.cap < CWTS;
      const double *w = g_wts + h.sum_off;
      const int J = R.J[dd] & 255, jr = R.J[dd] >> 8, hB = R.hB[dd];
      // the init sum of a level above hB (node 0 is then n0's prefix): for a
      // persistent state P[j] = S_j(B) = init_sums[j] there (shared memory)
      auto init_at = [&](int j) { return persist ? pers_P(dd, j) : ini[j]; };
#if RQ_SW_TABLES
      if constexpr (SIGSM) {
        if (J <= 2) {  // two-level tile: leaf = (S_J [+ sigma(b1 + par) w_1]) + sigma(a) w_0
          const uint32_t sws = smem_addr(sh->sw0 + sh->soff[dd]);
          const uint32_t sws1 = smem_addr(sh->sw1 + sh->soff[dd]) + 8u * (uint32_t)R.bd[dd][1];
          const uint32_t b0 = R.bd[dd][0];
          const double top = R.sJ[dd];
          const double p1 = J == 2 && 1 > hB ? init_at(1) : 0.0;  // level-1 node 0 = n0's prefix
#pragma unroll
          for (int m = 0; m < TILE / 32; m++) {
            const int k = lane + 32 * m;
            const uint32_t x = b0 + (uint32_t)k;
            const uint32_t par = __umulhi(x, m16);
            const uint32_t a = x - par * p;
            double vp = top;  // J == 1: every leaf's parent is the top node
            if (J == 2) vp = par == 0 && 1 > hB ? p1 : dadd(top, lds_f64(sws1 + 8u * par));
            double o = dadd(vp, lds_f64(sws + 8u * a));
            if (0 > hB && k == 0) o = ini[0];
            zt[dd * TILE + k] = o;
          }
          continue;
        }
      }
#endif
#if RQ_G2_FAST
      if constexpr (!SIGSM) {
        // sigma in global memory (large bases): a tile whose top node is at
        // level 1, or at level 2 above <= 2 level-1 nodes, needs no level
        // pass and no shuffles -- the (<= 2) parents are formed per lane
        if (J == 1 || (J == 2 && R.nn[dd][1] <= 2)) {
          const uint32_t b0 = R.bd[dd][0];
          const double w0 = cw ? c_wts[h.sum_off] : w[0];
          const double top = R.sJ[dd];
          double v0 = top, v1 = top;
          if (J == 2) {
            const uint32_t b1 = R.bd[dd][1];
            const double w1 = cw ? c_wts[h.sum_off + 1] : w[1];
            v0 = 1 > hB ? init_at(1) : dadd(top, dmul(u16d(sg[b1]), w1));
            v1 = dadd(top, dmul(u16d(sg[b1 + 1 < p ? b1 + 1 : b1]), w1));
          }
#pragma unroll
          for (int m = 0; m < TILE / 32; m++) {
            const int k = lane + 32 * m;
            const uint32_t x = b0 + (uint32_t)k;
            const uint32_t par = __umulhi(x, m16);
            const uint32_t a = x - par * p;
            double o = dadd(par ? v1 : v0, dmul(u16d(sg[a]), w0));
            if (0 > hB && k == 0) o = ini[0];
            zt[dd * TILE + k] = o;
          }
          continue;
        }
      }
#endif
      double *prev = ph->lev[warp][0], *next = ph->lev[warp][1];
      // Levels of <= 32 nodes live in registers, lane k holding node k, and
      // a child reads its parent with a shuffle (every level above 1 for
      // p >= 5, and level 1 itself); wider levels go through shared memory.
      double v = R.sJ[dd];
      int j = J - 1;
#pragma unroll 1
      for (; j >= jr; j--) {  // register levels: nn[j] <= 32 for j >= jr
        const uint32_t x = (uint32_t)R.bd[dd][j] + (uint32_t)lane;
        const uint32_t par = __umulhi(x, m16);
        const uint32_t a = x - par * p;
        const double sv = sig(a);
        const double wj = cw ? c_wts[h.sum_off + j] : w[j];
        const double vp = __shfl_sync(0xffffffffu, v, (int)par);
        v = dadd(vp, dmul(sv, wj));
        if (j > hB && lane == 0) v = init_at(j);
      }
      if (j == 0) {  // level 0 from the register level 1
        const uint32_t b0 = R.bd[dd][0];
        const double w0 = cw ? c_wts[h.sum_off] : w[0];
        const bool at_n0 = 0 > hB;
#pragma unroll
        for (int m = 0; m < TILE / 32; m++) {
          const int k = lane + 32 * m;
          const uint32_t x = b0 + (uint32_t)k;
          const uint32_t par = __umulhi(x, m16);
          const uint32_t a = x - par * p;
          const double sv = sig(a);
          const double vp = __shfl_sync(0xffffffffu, v, (int)par);
          double o = dadd(vp, dmul(sv, w0));
          if (at_n0 && k == 0) o = ini[0];
          zt[dd * TILE + k] = o;
        }
        continue;
      }
      prev[lane] = v;  // level j + 1 (<= 32 nodes)
      __syncwarp();
      // one node: S_j(prefix) = S_{j+1}(parent) + sigma(digit) * w_j, or the
      // init sum when the prefix is n0's (node 0 of a level above hB)
      auto node = [&](uint32_t bj, int k, double wj, bool at_n0, int j, double *dst) {
        const uint32_t x = bj + (uint32_t)k;  // < 2^16
        const uint32_t par = __umulhi(x, m16);
        const uint32_t a = x - par * p;
        const double sv = sig(a);
        double v = dadd(prev[par], dmul(sv, wj));
        if (at_n0 && k == 0) v = j > 0 ? init_at(j) : ini[0];
        dst[k] = v;
      };
#pragma unroll 1
      for (; j >= 1; j--) {  // wide upper levels: <= TILE/2 + 2 nodes
        const int Nj = R.nn[dd][j];
        const uint32_t bj = R.bd[dd][j];
        const double wj = cw ? c_wts[h.sum_off + j] : w[j];
        const bool at_n0 = j > hB;
#pragma unroll 1
        for (int k = lane; k < Nj; k += 32) node(bj, k, wj, at_n0, j, next);
        __syncwarp();
        double *tmp = prev;
        prev = next;
        next = tmp;
      }
      {  // level 0: the TILE points
        const uint32_t b0 = R.bd[dd][0];
        const double w0 = cw ? c_wts[h.sum_off] : w[0];
        const bool at_n0 = 0 > hB;
#pragma unroll
        for (int m = 0; m < TILE / 32; m++) node(b0, lane + 32 * m, w0, at_n0, 0, zt + dd * TILE);
      }
    }
  }
};

// Rasrap counter form (Alg. 3, halton.py:419-440): sum sigma(a_j)*scale_j
// from the least significant digit up, scale_j = (1/p)^(j+1) by repeated
// multiplication, over max(K, #digits) positions.  The running sum starts
// at the low digits, so no prefix can be shared across a tile: direct.
struct GenRasrapCounter {
  static constexpr int MAXB = 3;  // register-heavy digit loop next to LIBOR(20)
  const RepTables *t;
  using Shared = NoShared;
  __device__ void setup(const RepTables &t_, Shared &, int = 0) { t = &t_; }
  __device__ void unit(int rl, uint64_t, uint64_t path, int d0, int Dc, double *zt) {
    const uint16_t *dig = t->digits + (int64_t)rl * t->dig_stride;
    const uint16_t *sig = t->sigma + (int64_t)rl * t->sig_stride;
#pragma unroll 1
    for (int dd = 0; dd < Dc; dd++) {
      const HaltonDim h = hdim(d0 + dd);
      const uint16_t *n0d = dig + h.dig_off;
      const uint16_t *sg = sig + h.sig_off;
      const double *cs = g_cscale + h.sum_off;
      uint64_t r = path;  // 64-bit index (halton.py:506-512 takes int64)
      uint32_t carry = 0;
      double x = 0.0;
#pragma unroll 1
      for (int j = 0; j < h.K || r != 0u || carry != 0u; j++) {
        const uint64_t q = r >> 32 ? div_base64(r, h) : (uint64_t)div_base((uint32_t)r, h);
        uint32_t a = n0d[j] + (uint32_t)(r - q * (uint64_t)h.base) + carry;
        carry = a >= (uint32_t)h.base;
        a = carry ? a - (uint32_t)h.base : a;
        x = dadd(x, dmul(u16d(sg[a]), cs[j]));
        r = q;
      }
      zt[dd * TILE + threadIdx.x] = x;
    }
  }
};

// Counter form on a tile of TILE consecutive indices n = B + t.  With L the
// number of base-p digits that cover the tile (p^L > TILE), n = H * p^L + r
// where r = (B mod p^L) + t and H = B div p^L + (r >= p^L): only two
// values of H occur in a tile.  The reference's sum runs from the lowest
// digit up, x = (((s(a0) w0 + s(a1) w1) + ...) (halton.py:431-440), so a
// point's low L digits are summed per thread and the high terms
// T_j = s(a_j) w_j of its H (the same products, rounded the same way) are
// formed once per tile and dim and then added in order: bit-identical, with
// L instead of max(K, #digits) digit extractions per point.
constexpr int CT_MAXT = 40;  // high terms per variant (digits of n >> L, n < 2^46)
template <bool WIDE = false>
struct GenRasrapCounterTile {
  static constexpr int MAXB = 4;
  struct Shared {
    double T[CHUNK][2][CT_MAXT];
    int32_t nT[CHUNK][2];
    uint32_t lowB[CHUNK];
    // (replication, dim, H0) the slot's T tables were formed for: a CTA's
    // consecutive tiles share H0 for p^L / TILE tiles, so the high terms are
    // formed once per prefix, not per tile (single-chunk models)
    int32_t c_rl[CHUNK], c_d[CHUNK];
    uint64_t c_h[CHUNK];
  };
  const RepTables *t;
  Shared *sh;
  __device__ void setup(const RepTables &t_, Shared &s, int = 0) {
    t = &t_;
    sh = &s;
    for (int k = threadIdx.x; k < CHUNK; k += TILE) s.c_rl[k] = -1;
  }
  __device__ void prepare(int rl, uint64_t base, int d, int dd) {  // one lane per dim
    const HaltonDim h = hdim_t<WIDE>(d);
    const uint64_t p = (uint64_t)h.base;
    const int L = h.tdig + 1;
    uint64_t pL = 1;
    for (int j = 0; j < L; j++) pL *= p;
    const uint64_t B = t->start[(int64_t)rl * t->dim + d] + base;
    const uint64_t H0 = B / pL;
    sh->lowB[dd] = (uint32_t)(B - H0 * pL);
#if RQ_CT_CACHE
    if (sh->c_rl[dd] == rl && sh->c_d[dd] == d && sh->c_h[dd] == H0) return;
    sh->c_rl[dd] = rl;
    sh->c_d[dd] = d;
    sh->c_h[dd] = H0;
#endif
    const uint16_t *sg = t->sigma + (int64_t)rl * t->sig_stride + h.sig_off;
    const double *cs = g_cscale + h.sum_off;
#pragma unroll 1
    for (int v = 0; v < 2; v++) {
      uint64_t H = H0 + (uint64_t)v;
      int j = L, m = 0;
#pragma unroll 1
      for (; j < h.K || H != 0u; j++, m++) {
        const uint64_t q = div_base64(H, h);
        sh->T[dd][v][m] = dmul(u16d(sg[(uint32_t)(H - q * p)]), cs[j]);
        H = q;
      }
      sh->nT[dd][v] = m;
    }
  }
  __device__ void unit(int rl, uint64_t base, uint64_t, int d0, int Dc, double *zt) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();  // the previous unit's readers of T are done
    {
      const int dd = warp + lane * WARPS;  // 5 dims per warp on lanes 0..4
      if (dd < Dc) prepare(rl, base, d0 + dd, dd);
    }
    __syncthreads();
#if RQ_CT_PAIRS
    // two dims' sum chains interleaved (each chain keeps its own order:
    // bit-identical), so a thread has two independent DADD chains in flight
#pragma unroll 1
    for (int dd = 0; dd + 1 < Dc; dd += 2) {
      int v0, v1;
      double x0 = low_sum(rl, d0 + dd, dd, &v0);
      double x1 = low_sum(rl, d0 + dd + 1, dd + 1, &v1);
      const double *T0 = sh->T[dd][v0], *T1 = sh->T[dd + 1][v1];
      const int n0 = sh->nT[dd][v0], n1 = sh->nT[dd + 1][v1];
      const int nmin = n0 < n1 ? n0 : n1;
      int m = 0;
#pragma unroll 2
      for (; m < nmin; m++) {
        x0 = dadd(x0, T0[m]);
        x1 = dadd(x1, T1[m]);
      }
      for (int k = m; k < n0; k++) x0 = dadd(x0, T0[k]);
      for (int k = m; k < n1; k++) x1 = dadd(x1, T1[k]);
      zt[dd * TILE + threadIdx.x] = x0;
      zt[(dd + 1) * TILE + threadIdx.x] = x1;
    }
    if (Dc & 1) {
      const int dd = Dc - 1;
      int v;
      double x = low_sum(rl, d0 + dd, dd, &v);
      const double *T = sh->T[dd][v];
      const int n = sh->nT[dd][v];
      for (int m = 0; m < n; m++) x = dadd(x, T[m]);
      zt[dd * TILE + threadIdx.x] = x;
    }
#else
#pragma unroll 1
    for (int dd = 0; dd < Dc; dd++) {
      int v;
      double x = low_sum(rl, d0 + dd, dd, &v);
      const double *T = sh->T[dd][v];
      const int n = sh->nT[dd][v];
#pragma unroll 4
      for (int m = 0; m < n; m++) x = dadd(x, T[m]);
      zt[dd * TILE + threadIdx.x] = x;
    }
#endif
  }
  // the point's low L digits, summed from the lowest (sets its variant v)
  __device__ __forceinline__ double low_sum(int rl, int d, int dd, int *v) const {
    const HaltonDim h = hdim_t<WIDE>(d);
    const uint32_t p = (uint32_t)h.base;
    const int L = h.tdig + 1;
    uint32_t pL = 1;
    for (int j = 0; j < L; j++) pL *= p;
    const uint16_t *sg = t->sigma + (int64_t)rl * t->sig_stride + h.sig_off;
    const double *cs = g_cscale + h.sum_off;
    uint32_t r = sh->lowB[dd] + (uint32_t)threadIdx.x;
    *v = r >= pL;
    r = *v ? r - pL : r;
    double x = 0.0;
#pragma unroll 1
    for (int j = 0; j < L; j++) {
      const uint32_t q = __umulhi(r, h.m16);
      x = dadd(x, dmul(u16d(sg[r - q * p]), cs[j]));
      r = q;
    }
    return x;
  }
};

// u = w 2^-32 + 2^-33 (harness.py:66-67), exactly: the double 1 + u has the
// mantissa (w << 20) | 2^19, so it is assembled from w with two integer ops
// and 1 is subtracted exactly (no int->double conversion on the XU pipe).
__device__ __forceinline__ double philox_u(uint32_t w) {
  return __hiloint2double((int)(0x3FF00000u | (w >> 12)), (int)((w << 20) | 0x80000u)) - 1.0;
}

// Philox-4x32-10, counter (b, path_lo, path_hi, 0), u = w 2^-32 + 2^-33
// (prng.py:180-231, harness.py:53-67).
struct GenPhilox {
  const RepTables *t;
  using Shared = NoShared;
  __device__ void setup(const RepTables &t_, Shared &, int = 0) { t = &t_; }
  __device__ void unit(int rl, uint64_t, uint64_t path, int d0, int Dc, double *zt) {
    const uint64_t key = derive_key3(t->seed, 3, (uint64_t)(t->rep_first + rl));
    const uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    double *zcol = zt + threadIdx.x;
    for (int dd = 0; dd < Dc; dd += 4) {  // d0 % 4 == 0
      U4 w = philox4x32_10((uint32_t)((d0 + dd) >> 2), (uint32_t)path, (uint32_t)(path >> 32),
                           0u, k0, k1);
      zcol[dd * TILE] = philox_u(w.x);
      if (dd + 1 < Dc) zcol[(dd + 1) * TILE] = philox_u(w.y);
      if (dd + 2 < Dc) zcol[(dd + 2) * TILE] = philox_u(w.z);
      if (dd + 3 < Dc) zcol[(dd + 3) * TILE] = philox_u(w.w);
    }
  }
  // register form for the normals stream: coordinates d0..d0+3 of `path`
  __device__ __forceinline__ void quad(int rl, uint64_t path, int d0, double u[4]) {
    const uint64_t key = derive_key3(t->seed, 3, (uint64_t)(t->rep_first + rl));
    U4 w = philox4x32_10((uint32_t)(d0 >> 2), (uint32_t)path, (uint32_t)(path >> 32), 0u,
                         (uint32_t)key, (uint32_t)(key >> 32));
    u[0] = philox_u(w.x);
    u[1] = philox_u(w.y);
    u[2] = philox_u(w.z);
    u[3] = philox_u(w.w);
  }
};

// Scrambled Sobol' (sobol.py:313-372): the point at counter index j is the
// XOR of the pre-scrambled direction words over the set bits of j, XOR the
// shift; the Gray-code sampler's point i is the counter point at i^(i>>1).
template <bool GRAY>
__device__ __forceinline__ uint32_t sobol_word(const uint32_t *vd, uint32_t shift, uint64_t i) {
  uint32_t x = shift;
  uint32_t bits = (uint32_t)(GRAY ? (i ^ (i >> 1)) : i);
  for (; bits; bits &= bits - 1u) x ^= vd[__ffs(bits) - 1];
  return x;
}

template <bool GRAY>
struct GenSobolDirect {
  const RepTables *t;
  using Shared = NoShared;
  __device__ void setup(const RepTables &t_, Shared &, int = 0) { t = &t_; }
  __device__ void unit(int rl, uint64_t, uint64_t path, int d0, int Dc, double *zt) {
    const uint32_t *v = t->sobol_v + (int64_t)rl * t->dim * SOBOL_BITS;
    const uint32_t *sh = t->sobol_shift + (int64_t)rl * t->dim;
    for (int dd = 0; dd < Dc; dd++)
      zt[dd * TILE + threadIdx.x] =
          (double)sobol_word<GRAY>(v + (d0 + dd) * SOBOL_BITS, sh[d0 + dd], path) * TWO_M32;
  }
};

// u = w 2^-32 exactly: 1 + u is assembled from the bits of w and 1 is
// subtracted (no int->double conversion on the XU pipe).
__device__ __forceinline__ double sobol_u(uint32_t w) {
  return __hiloint2double((int)(0x3FF00000u | (w >> 12)), (int)(w << 20)) - 1.0;
}

// Tiled Sobol': in a 128-aligned tile the index bits >= 7 are common, so
// the warp owning a dim folds them and the shift into one word.  Lane l
// takes the points t = l + 32m (m < 4, conflict-free tile rows).  For t < 32
// the counter index t + 32m differs from t in bits 5-6 only, and the Gray
// index g(t + 32m) = g(t) ^ (32m ^ 16m) (48, 96, 80: bits 4-6), so each lane
// forms its word for t from seven direction words and the other three
// points by one XOR with a warp-uniform word.  Unaligned tiles
// (sampler.fill from an odd start) use the per-point loop.
template <bool GRAY>
struct GenSobolTile {
  const RepTables *t;
  using Shared = NoShared;
  __device__ void setup(const RepTables &t_, Shared &, int = 0) { t = &t_; }
  __device__ void unit(int rl, uint64_t base, uint64_t, int d0, int Dc, double *zt) {
    const uint32_t *v = t->sobol_v + (int64_t)rl * t->dim * SOBOL_BITS;
    const uint32_t *shp = t->sobol_shift + (int64_t)rl * t->dim;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool aligned = (base & 127u) == 0u;
    const uint64_t bidx = GRAY ? (base ^ (base >> 1)) : base;
    const uint32_t gl = GRAY ? (uint32_t)(lane ^ (lane >> 1)) : (uint32_t)lane;
    for (int dd = warp; dd < Dc; dd += WARPS) {
      const uint32_t *vd = v + (d0 + dd) * SOBOL_BITS;
      if (aligned) {
        // For an aligned base B the (Gray) index of B + t is bidx ^ g(t)
        // (the bits of B and t, and of B>>1 and t>>1, are disjoint), so the
        // lane's low 7 bits are c = (bidx & 127) ^ g(lane)
        uint32_t x = sobol_word<false>(vd, shp[d0 + dd], (bidx >> 7) << 7);
        const uint32_t c = ((uint32_t)bidx & 127u) ^ gl;
#pragma unroll
        for (int k = 0; k < 7; k++) x ^= (c >> k) & 1u ? __ldg(vd + k) : 0u;
        const uint32_t v4 = __ldg(vd + 4), v5 = __ldg(vd + 5), v6 = __ldg(vd + 6);
        const uint32_t w1 = GRAY ? v4 ^ v5 : v5, w2 = GRAY ? v5 ^ v6 : v6;
        const uint32_t w3 = GRAY ? v4 ^ v6 : v5 ^ v6;
        double *row = zt + dd * TILE + lane;
        row[0] = sobol_u(x);
        row[32] = sobol_u(x ^ w1);
        row[64] = sobol_u(x ^ w2);
        row[96] = sobol_u(x ^ w3);
      } else {
        for (int tt = lane; tt < TILE; tt += 32)
          zt[dd * TILE + tt] = sobol_u(sobol_word<GRAY>(vd, shp[d0 + dd], base + (uint64_t)tt));
      }
    }
  }
};

// Persistent Sobol' tile (single-chunk models: a CTA prices contiguous
// tiles, dispatch as for the persistent Rasrap tile).  The warp owning a
// dim keeps, in shared memory, the tile's high word H_d (shift and index
// bits >= 7) and per-replication tables of the low seven bits: T0_d[16] and
// T1_d[8] (XORs of direction words 0-3 and 4-6) and the three warp-uniform
// point offsets of GenSobolTile.  From tile T-1 to T the high (Gray) index
// changes by g(T) ^ g(T-1) = 1 << ctz(T) (counter order: the bits of
// T ^ (T-1)), so H_d takes one XOR per tile instead of a loop over the set
// bits of the index; each lane's word is H_d ^ T0_d[c & 15] ^ T1_d[c >> 4].
// Same words as sobol_word (checked by the points / theta tests).
struct SobolPersistShared {
  uint32_t H[CHUNK];
  uint32_t T0[CHUNK][16];
  uint32_t T1[CHUNK][8];
  uint32_t W[CHUNK][4];  // 0, w1, w2, w3
  int32_t st_rl[WARPS];
  uint32_t st_T[WARPS];
};
template <bool GRAY>
struct GenSobolTileP {
  const RepTables *t;
  SobolPersistShared *sh;
  using Shared = SobolPersistShared;
  __device__ void setup(const RepTables &t_, Shared &s, int = 0) {
    t = &t_;
    sh = &s;
    for (int k = threadIdx.x; k < WARPS; k += TILE) s.st_rl[k] = -1;
  }
  __device__ void unit(int rl, uint64_t base, uint64_t, int d0, int Dc, double *zt) {
    Shared &R = *sh;
    const uint32_t *v = t->sobol_v + (int64_t)rl * t->dim * SOBOL_BITS;
    const uint32_t *shp = t->sobol_shift + (int64_t)rl * t->dim;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t T = (uint32_t)(base >> 7);  // base is tile-aligned; indices < 2^32
    const uint32_t gT = GRAY ? T ^ (T >> 1) : T;
    if (R.st_rl[warp] != rl) {  // new replication: tables and H of the warp's dims
#pragma unroll 1
      for (int dd = warp; dd < Dc; dd += WARPS) {
        const uint32_t *vd = v + (d0 + dd) * SOBOL_BITS;
        uint32_t x = 0;
        if (lane < 16) {
#pragma unroll
          for (int k = 0; k < 4; k++) x ^= (lane >> k) & 1 ? __ldg(vd + k) : 0u;
          R.T0[dd][lane] = x;
        } else if (lane < 24) {
#pragma unroll
          for (int k = 0; k < 3; k++) x ^= ((lane - 16) >> k) & 1 ? __ldg(vd + 4 + k) : 0u;
          R.T1[dd][lane - 16] = x;
        } else if (lane < 28) {
          const uint32_t v4 = __ldg(vd + 4), v5 = __ldg(vd + 5), v6 = __ldg(vd + 6);
          const int m = lane - 24;
          x = m == 0 ? 0u
              : m == 1 ? (GRAY ? v4 ^ v5 : v5)
              : m == 2 ? (GRAY ? v5 ^ v6 : v6)
                       : (GRAY ? v4 ^ v6 : v5 ^ v6);
          R.W[dd][m] = x;
        } else if (lane == 28) {
          R.H[dd] = sobol_word<false>(vd, __ldg(shp + d0 + dd), (uint64_t)gT << 7);
        }
      }
    } else if (T == R.st_T[warp] + 1u) {  // next tile: XOR in the changed high bits
      const uint32_t chg = GRAY ? (T & (0u - T)) : (T ^ (T - 1u));
#pragma unroll 1
      for (int dd = warp + lane * WARPS; dd < Dc; dd += 32 * WARPS) {
        const uint32_t *vd = v + (d0 + dd) * SOBOL_BITS + 7;
        uint32_t x = R.H[dd];
        for (uint32_t b = chg; b; b &= b - 1u) x ^= __ldg(vd + __ffs(b) - 1);
        R.H[dd] = x;
      }
    } else {  // a jump (first tile of the CTA in this replication)
#pragma unroll 1
      for (int dd = warp + lane * WARPS; dd < Dc; dd += 32 * WARPS)
        R.H[dd] = sobol_word<false>(v + (d0 + dd) * SOBOL_BITS, __ldg(shp + d0 + dd),
                                    (uint64_t)gT << 7);
    }
    __syncwarp();  // every lane has read st_rl / st_T before lane 0 rewrites them
    if (lane == 0) {
      R.st_rl[warp] = rl;
      R.st_T[warp] = T;
    }
    __syncwarp();
    const uint32_t c = (GRAY ? (T & 1u) << 6 : 0u) ^ (GRAY ? (uint32_t)(lane ^ (lane >> 1)) : (uint32_t)lane);
    const uint32_t c0 = c & 15u, c1 = c >> 4;
#pragma unroll 1
    for (int dd = warp; dd < Dc; dd += WARPS) {
      const uint32_t x = R.H[dd] ^ R.T0[dd][c0] ^ R.T1[dd][c1];
      double *row = zt + dd * TILE + lane;
      row[0] = sobol_u(x);
      row[32] = sobol_u(x ^ R.W[dd][1]);
      row[64] = sobol_u(x ^ R.W[dd][2]);
      row[96] = sobol_u(x ^ R.W[dd][3]);
    }
  }
};

// Register form of the Sobol' stream (config 4, k_stream_reg): thread t of
// a 128-aligned tile B takes point B + t in every dim.  With the tile
// algebra of GenSobolTile its word is H_d ^ L_d(c): H_d folds the shift and
// the index bits >= 7 (formed once per tile and dim into shared memory by the
// CTA), c = (bidx & 127) ^ g(t) is the thread's low 7 index bits for every
// dim, and L_d(c) = T0_d[c & 15] ^ T1_d[c >> 4] are XORs of the direction
// words of those bits, tabled once per CTA (24 words per dim).  Same words
// as sobol_word, so the same uniforms; three shared loads per coordinate.
template <bool GRAY>
struct GenSobolStream {
  static constexpr bool TILE_HOOK = true;
  const RepTables *t;
  const uint32_t *v, *shp;
  uint32_t *T0, *T1, *H;
  int dim, dpad;
  uint32_t c0, c1;
  using Shared = NoShared;
  static __host__ __device__ size_t dyn_bytes(int dim) {
    return (size_t)((dim + 3) & ~3) * (16 + 8 + 1) * sizeof(uint32_t);
  }
  __device__ void setup(const RepTables &t_, Shared &, int dim_) {
    t = &t_;
    dim = dim_;
    dpad = (dim + 3) & ~3;
    extern __shared__ __align__(16) uint32_t sob_sm[];
    T0 = sob_sm;
    T1 = T0 + dpad * 16;
    H = T1 + dpad * 8;
  }
  // per-CTA tables of replication rl (caller syncs before the first tile)
  __device__ void rep(int rl) {
    v = t->sobol_v + (int64_t)rl * dim * SOBOL_BITS;
    shp = t->sobol_shift + (int64_t)rl * dim;
    for (int e = threadIdx.x; e < dpad * 16; e += TILE) {
      const int d = e >> 4;
      const uint32_t c = (uint32_t)e & 15u;
      uint32_t x = 0;
      if (d < dim)
        for (int k = 0; k < 4; k++) x ^= (c >> k) & 1u ? __ldg(v + d * SOBOL_BITS + k) : 0u;
      T0[e] = x;
    }
    for (int e = threadIdx.x; e < dpad * 8; e += TILE) {
      const int d = e >> 3;
      const uint32_t c = (uint32_t)e & 7u;
      uint32_t x = 0;
      if (d < dim)
        for (int k = 0; k < 3; k++) x ^= (c >> k) & 1u ? __ldg(v + d * SOBOL_BITS + 4 + k) : 0u;
      T1[e] = x;
    }
  }
  // tile base tb (multiple of TILE): H for every dim, this thread's c
  __device__ void tile(uint64_t tb) {
    __syncthreads();  // the previous tile's H reads are done
    const uint64_t bidx = GRAY ? (tb ^ (tb >> 1)) : tb;
    for (int d = threadIdx.x; d < dpad; d += TILE)
      H[d] = d < dim ? sobol_word<false>(v + d * SOBOL_BITS, __ldg(shp + d), (bidx >> 7) << 7) : 0u;
    const uint32_t l = threadIdx.x;
    const uint32_t c = ((uint32_t)bidx & 127u) ^ (GRAY ? l ^ (l >> 1) : l);
    c0 = c & 15u;
    c1 = c >> 4;
    __syncthreads();
  }
  __device__ __forceinline__ void quad(int, uint64_t, int d0, double u[4]) {
    const uint4 h = *reinterpret_cast<const uint4 *>(H + d0);
    const uint32_t hh[4] = {h.x, h.y, h.z, h.w};
#pragma unroll
    for (int k = 0; k < 4; k++)
      u[k] = sobol_u(hh[k] ^ T0[(d0 + k) * 16 + c0] ^ T1[(d0 + k) * 8 + c1]);
  }
};

// SFC64 per-path stream (no reference counterpart; numpy SFC64 core):
// state from derive_words(derive_key(seed, 7, m, path), 6), 12 warm-up
// draws, u = (w >> 11) 2^-53 as numpy Generator.random().  Dims are drawn
// in order, so the state carries over between a path's chunks.
struct GenSfc64 {
  const RepTables *t;
  Sfc64 s;
  using Shared = NoShared;
  __device__ void setup(const RepTables &t_, Shared &, int = 0) { t = &t_; }
  __device__ void unit(int rl, uint64_t, uint64_t path, int d0, int Dc, double *zt) {
    if (d0 == 0) {
      uint64_t km = derive_key3(t->seed, 7, (uint64_t)(t->rep_first + rl));
      sfc_seed(s, splitmix64(km ^ path));
    }
    for (int dd = 0; dd < Dc; dd++)
      zt[dd * TILE + threadIdx.x] = (double)(sfc_next(s) >> 11) * TWO_M53;
  }
  __device__ __forceinline__ void quad(int rl, uint64_t path, int d0, double u[4]) {
    if (d0 == 0) {
      uint64_t km = derive_key3(t->seed, 7, (uint64_t)(t->rep_first + rl));
      sfc_seed(s, splitmix64(km ^ path));
    }
#pragma unroll
    for (int k = 0; k < 4; k++) u[k] = (double)(sfc_next(s) >> 11) * TWO_M53;
  }
};

// ======================================================================
// Sequential word streams (prng.py:40-149).  The reference consumes one
// stream per replication row-major: coordinate d of path i is word
// i * dim + d, u = w 2^-32 + 2^-33 (harness.py:46-50).  Both generators
// work on segments of a replication (SeqArgs): begin_segment() positions
// the stream, unit() yields the uniforms of the thread's current path.
// ======================================================================
constexpr uint32_t XW_WEYL = 362437u;
__device__ uint32_t g_xw_jump[XW_JUMPS * 160 * XW_COLW];  // columns of A^(2^k)

cudaError_t upload_xorwow_jumps(const uint32_t *cols, size_t words) {
  if (words != (size_t)XW_JUMPS * 160 * XW_COLW) return cudaErrorInvalidValue;
  return cudaMemcpyToSymbol(g_xw_jump, cols, sizeof(uint32_t) * words);
}

// Xorwow(key) (prng.py:128-134): derive_words(key, 6), key + 1, ... while
// the xorshift words are all zero.  One thread per replication.
__global__ void k_xorwow_setup(RepTables t, uint32_t *state) {
  const int rl = blockIdx.x * blockDim.x + threadIdx.x;
  if (rl >= t.rep_count) return;
  uint64_t key = derive_key3(t.seed, 2, (uint64_t)(t.rep_first + rl));  // family "xorwow"
  uint32_t w[6];
  for (;;) {
    const uint64_t z1 = splitmix64(key), z2 = splitmix64(z1), z3 = splitmix64(z2);
    w[0] = (uint32_t)z1;
    w[1] = (uint32_t)(z1 >> 32);
    w[2] = (uint32_t)z2;
    w[3] = (uint32_t)(z2 >> 32);
    w[4] = (uint32_t)z3;
    w[5] = (uint32_t)(z3 >> 32);
    if (w[0] | w[1] | w[2] | w[3] | w[4]) break;
    key += 1;
  }
  for (int k = 0; k < 6; k++) state[rl * 6 + k] = w[k];
}

// XORWOW, one stream per replication: thread t of a segment owns the run of
// paths [t * ntile, (t + 1) * ntile) and generates its words in order; the
// state is jumped to the run's first word W by the GF(2) matrices A^(2^k)
// of the xorshift part for the set bits of W (the Weyl counter d advances
// by 362437 W).
struct GenXorwow {
  __device__ void set_dyn(double *) {}
  static __host__ __device__ size_t dyn_bytes(int) { return 0; }
  static constexpr bool RUNS = true;
  using Shared = NoShared;
  const RepTables *t;
  uint32_t x, y, z, w, v, d;
  __device__ void setup(const RepTables &t_, Shared &, uint32_t *) { t = &t_; }
  __device__ void begin_segment(int rl, int, int, int64_t, int64_t my_first_path, int dim) {
    const uint32_t *s0 = t->xw_state + rl * 6;
    uint32_t s[5] = {s0[0], s0[1], s0[2], s0[3], s0[4]};
    const uint64_t W = (uint64_t)my_first_path * (uint64_t)dim;
    d = s0[5] + XW_WEYL * (uint32_t)W;
#pragma unroll 1
    for (int k = 0; k < XW_JUMPS; k++) {
      if (!((W >> k) & 1u)) continue;
      const uint4 *col = reinterpret_cast<const uint4 *>(g_xw_jump + (size_t)k * 160 * XW_COLW);
      uint32_t o0 = 0, o1 = 0, o2 = 0, o3 = 0, o4 = 0;
#pragma unroll
      for (int wd = 0; wd < 5; wd++) {
        const uint32_t bits = s[wd];
#pragma unroll 4
        for (int b = 0; b < 32; b++) {
          const uint4 c = __ldg(col + 2 * (wd * 32 + b));
          const uint32_t c4 = __ldg(reinterpret_cast<const uint32_t *>(col + 2 * (wd * 32 + b) + 1));
          const uint32_t m = 0u - ((bits >> b) & 1u);
          o0 ^= c.x & m;
          o1 ^= c.y & m;
          o2 ^= c.z & m;
          o3 ^= c.w & m;
          o4 ^= c4 & m;
        }
      }
      s[0] = o0;
      s[1] = o1;
      s[2] = o2;
      s[3] = o3;
      s[4] = o4;
    }
    x = s[0];
    y = s[1];
    z = s[2];
    w = s[3];
    v = s[4];
  }
  __device__ __forceinline__ uint32_t next() {  // _xorwow_fill (prng.py:97-110)
    const uint32_t tt = x ^ (x >> 2);
    x = y;
    y = z;
    z = w;
    w = v;
    v = (v ^ (v << 4)) ^ (tt ^ (tt << 1));
    d += XW_WEYL;
    return d + v;
  }
  __device__ void unit(int, int, int, int Dc, double *zt) {
    for (int dd = 0; dd < Dc; dd++) zt[dd * TILE + threadIdx.x] = philox_u(next());
  }
  // words of the path the model does not read (f = x_1 reads one of dim)
  __device__ void skip(int n) {
    for (int k = 0; k < n; k++) next();
  }
};

// MT19937 twist of a whole state block (prng.py:44-51) from `o` into `n`.
// In the reference's in-place loop word j reads o[j], o[j+1] and the word
// at j+397 (mod 624), which is already new for j >= 227.  Following the
// chain j -> j+227 -> j+454 every new word is a function of old words and
// of its own chain's previous link (j = 623 also needs n[0], recomputed by
// that thread from old words), so thread k < 227 produces n[k], n[k+227]
// and n[k+454] with no exchange and the twist costs one CTA barrier.
__device__ __forceinline__ uint32_t mt_mix(uint32_t a, uint32_t b, uint32_t c) {
  const uint32_t yy = (a & 0x80000000u) | (b & 0x7FFFFFFFu);
  return c ^ (yy >> 1) ^ ((yy & 1u) ? 0x9908B0DFu : 0u);
}
__device__ void mt_twist(const uint32_t *o, uint32_t *n) {
  for (int k = threadIdx.x; k < 227; k += blockDim.x) {
    const uint32_t a = mt_mix(o[k], o[k + 1], o[k + 397]);
    const uint32_t b = mt_mix(o[k + 227], o[k + 228], a);
    n[k] = a;
    n[k + 227] = b;
    if (k < MT_N - 454) {
      const uint32_t nxt = k == MT_N - 455 ? mt_mix(o[0], o[1], o[397]) : o[k + 455];
      n[k + 454] = mt_mix(o[k + 454], nxt, b);
    }
  }
  __syncthreads();
}
__device__ __forceinline__ uint32_t mt_temper(uint32_t yv) {
  yv ^= yv >> 11;
  yv ^= (yv << 7) & 0x9D2C5680u;
  yv ^= (yv << 15) & 0xEFC60000u;
  return yv ^ (yv >> 18);
}

// Snapshots for the segments of replications rep_local0.. (one CTA each):
// MT19937(key & 0xFFFFFFFF) (prng.py:66-72), twisted in order; the state
// after the twist that yields word W_s = (p0 + s seg_len) dim is stored for
// every segment s (word W_s is then at position W_s mod 624).
__global__ void __launch_bounds__(256) k_mt_snap(RepTables t, int rep_local0, int dim,
                                                 SeqArgs q, uint32_t *snap) {
  __shared__ uint32_t st[2][MT_N];
  const int rl = rep_local0 + blockIdx.x;
  if (threadIdx.x == 0) {
    uint32_t prev = (uint32_t)derive_key3(t.seed, 1, (uint64_t)(t.rep_first + rl));
    st[0][0] = prev;
    for (int i = 1; i < MT_N; i++) {
      prev = 1812433253u * (prev ^ (prev >> 30)) + (uint32_t)i;
      st[0][i] = prev;
    }
  }
  __syncthreads();
  int cur = 0;
  int64_t twists = 0;  // twists applied so far
  for (int sg = 0; sg < q.segs_per_rep; sg++) {
    const int64_t W = (q.p0 + (int64_t)sg * q.seg_len) * dim;
    const int64_t need = W / MT_N + 1;
    for (; twists < need; twists++) {
      mt_twist(st[cur], st[cur ^ 1]);
      cur ^= 1;
    }
    uint32_t *dst = snap + ((int64_t)blockIdx.x * q.segs_per_rep + sg) * MT_N;
    for (int j = threadIdx.x; j < MT_N; j += blockDim.x) dst[j] = st[cur][j];
  }
}

// MT19937, one stream per replication, CTA-cooperative: the CTA owns a
// segment, loads its snapshot and, for every tile of TILE consecutive
// paths, twists and tempers the tile's words (path-major) into a per-CTA
// scratch laid out [dim][TILE], from which every thread reads its path.
struct GenTwister {
  __device__ void set_dyn(double *) {}
  static __host__ __device__ size_t dyn_bytes(int) { return 0; }
  static constexpr bool RUNS = false;
  struct Shared {
    uint32_t st[2][MT_N];
  };
  const RepTables *t;
  Shared *sh;
  uint32_t *scr;  // this CTA's [dim][TILE]
  const SeqArgs *q;
  int cur, pos;   // current state buffer, next word's position in it
  uint32_t dim_m; // ceil(2^32 / dim): k / dim for k < 2^32 / dim
  int dim;
  __device__ void setup(const RepTables &t_, Shared &s, uint32_t *scratch) {
    t = &t_;
    sh = &s;
    scr = scratch;
  }
  __device__ void set_seq(const SeqArgs &q_, int dim_) {
    q = &q_;
    dim = dim_;
    dim_m = (uint32_t)((((uint64_t)1 << 32) + dim_ - 1) / dim_);
  }
  __device__ void begin_segment(int, int rb, int sg, int64_t seg_first_path, int64_t, int) {
    const uint32_t *src = q->mt_snap + ((int64_t)rb * q->segs_per_rep + sg) * MT_N;
    __syncthreads();  // previous segment's readers are done with the state
    for (int j = threadIdx.x; j < MT_N; j += blockDim.x) sh->st[0][j] = src[j];
    cur = 0;
    pos = (int)((seg_first_path * dim) % MT_N);
    __syncthreads();
  }
  // words of tile paths [0, npaths) -> scratch (all threads; CTA barriers)
  __device__ void fill_tile(int npaths) {
    const uint32_t total = (uint32_t)npaths * (uint32_t)dim;
    for (uint32_t k = 0; k < total;) {
      if (pos == MT_N) {
        mt_twist(sh->st[cur], sh->st[cur ^ 1]);
        cur ^= 1;
        pos = 0;
      }
      const uint32_t n = min((uint32_t)(MT_N - pos), total - k);
      const uint32_t *blk = sh->st[cur] + pos;
      for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t kk = k + i;
        const uint32_t pth = __umulhi(kk, dim_m), dd = kk - pth * (uint32_t)dim;
        scr[dd * TILE + pth] = mt_temper(blk[i]);
      }
      pos += (int)n;
      k += n;
    }
    __syncthreads();
  }
  __device__ void skip(int) {}
  __device__ void unit(int, int npaths, int d0, int Dc, double *zt) {
    if (d0 == 0) fill_tile(npaths);
    for (int dd = 0; dd < Dc; dd++)
      zt[dd * TILE + threadIdx.x] = philox_u(__ldcg(scr + (d0 + dd) * TILE + threadIdx.x));
  }
};

// ======================================================================
// Kakutani orbits (halton.py:163-239, 521-542): per dimension the random
// start x0 = derive_rng(key, d).random() and x <- x + b_k with k the
// bracket of 1 - x.  The reference guesses k from a logarithm and then
// corrects it until inv_pow[k-1] + tol < 1 - x <= inv_pow[k-2] + tol holds
// (halton.py:226-235); that k is unique (the smallest k with
// 1 - x > thr[k-1], thr = inv_pow + tol in double), so the device scans the
// thresholds directly.  Orbits are sequential: segments start from
// snapshots taken by k_kak_walk.
// ======================================================================
__device__ double g_kk_thr[MAX_DIM * KK_TAB];
__device__ double g_kk_b[MAX_DIM * KK_TAB];

// cached brackets of the bases of the runs layout, [dim][thr 0..7, b 0..7]:
// warp-uniform reads from the constant bank
__constant__ double c_kk8[KK_RUNS_MAXDIM * 16];

__device__ double g_kk_xthr[MAX_DIM * 8];  // see kak_step_flat

static double kak_xthr(double thr) {  // smallest double x with fl(1 - x) <= thr
  double x = 1.0 - thr;
  while (!(1.0 - x <= thr)) x = std::nextafter(x, 2.0);
  while (x > 0.0 && 1.0 - std::nextafter(x, -1.0) <= thr) x = std::nextafter(x, -1.0);
  return x;
}

cudaError_t upload_kakutani_tables(const double *thr, const double *b, int dims) {
  {
    std::vector<double> xt((size_t)dims * 8);
    for (int d = 0; d < dims; d++)
      for (int j = 0; j < 8; j++) xt[(size_t)d * 8 + j] = kak_xthr(thr[d * KK_TAB + j]);
    cudaError_t e0 = cudaMemcpyToSymbol(g_kk_xthr, xt.data(), sizeof(double) * xt.size());
    if (e0 != cudaSuccess) return e0;
  }
  cudaError_t e = cudaMemcpyToSymbol(g_kk_thr, thr, sizeof(double) * dims * KK_TAB);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyToSymbol(g_kk_b, b, sizeof(double) * dims * KK_TAB);
  if (e != cudaSuccess) return e;
  double c8[KK_RUNS_MAXDIM * 16];
  const int nd = dims < KK_RUNS_MAXDIM ? dims : KK_RUNS_MAXDIM;
  for (int d = 0; d < nd; d++)
    for (int j = 0; j < 8; j++) {
      c8[d * 16 + j] = thr[d * KK_TAB + j];
      c8[d * 16 + 8 + j] = b[d * KK_TAB + j];
    }
  return cudaMemcpyToSymbol(c_kk8, c8, sizeof(double) * 16 * nd);
}

// One orbit step, the first two brackets (probability 1 - 1/p^2) in
// registers, off the L1 latency chain of the sequential orbit.
constexpr int KK_NB = 8;  // brackets held in registers / the constant bank
// One orbit step from cached brackets tc/bc (k < KK_NB) and the global
// tables beyond.  The reference's wrap test (x >= 1 after the step,
// halton.py:236-237) cannot fire in the cached brackets: k = 1 means
// 1 - x > 1/p + tol, so x + b_1 < 1, and b_k < 0 for k >= 2.  The first two
// candidates are formed before the bracket is known (off the latency chain);
// deeper brackets (probability 1/p^2) are found by an unrolled scan.
template <class TC, class BC>
__device__ __forceinline__ double kak_step(double x, TC tc, BC bc, const double *thr,
                                           const double *b) {
  const double om = 1.0 - x;
  const double v0 = x + bc(0), v1 = x + bc(1);
  if (om > tc(0)) return v0;
  if (om > tc(1)) return v1;
  double v = 0.0;
  bool found = false;
#pragma unroll
  for (int j = 2; j < KK_NB; j++) {
    if (!found && om > tc(j)) {
      v = x + bc(j);
      found = true;
    }
  }
  if (!found) {
    int k = KK_NB;
    while (k < KK_TAB - 1 && om <= thr[k]) k++;
    v = x + b[k];
    v = v >= 1.0 ? v - 1.0 : v;
  }
  return v;
}

// Branch-free form for the latency-bound snapshot walks (a warp holds
// orbits of different bases, so the branchy form diverges every step).  As
// fl(1 - x) does not increase with x, the bracket test 1 - x <= thr_j is
// exactly x >= xthr_j (g_kk_xthr, the smallest such double); the tests hold
// exactly for j < k, the increment b_k is picked by a depth-3 select tree
// and added once: the dependent chain per step is a compare, three selects
// and one DADD.
__device__ __forceinline__ double kak_step_flat(double x, const double *xc, const double *bc,
                                                const double *thr, const double *b) {
  bool c[KK_NB];
#pragma unroll
  for (int j = 0; j < KK_NB; j++) c[j] = x >= xc[j];
  if (c[KK_NB - 1]) {  // deeper than the cache: rare
    const double om = 1.0 - x;
    int k = KK_NB;
    while (k < KK_TAB - 1 && om <= thr[k]) k++;
    const double vv = x + b[k];
    return vv >= 1.0 ? vv - 1.0 : vv;
  }
  const double s01 = c[0] ? bc[1] : bc[0], s23 = c[2] ? bc[3] : bc[2];
  const double s45 = c[4] ? bc[5] : bc[4], s67 = c[6] ? bc[7] : bc[6];
  const double s03 = c[1] ? s23 : s01, s47 = c[5] ? s67 : s45;
  return x + (c[3] ? s47 : s03);
}

struct KakDim {  // one base's brackets in registers
  const double *thr, *b;
  double tc[KK_NB], bc[KK_NB];
  __device__ void load(int d) {
    thr = g_kk_thr + d * KK_TAB;
    b = g_kk_b + d * KK_TAB;
#pragma unroll
    for (int j = 0; j < KK_NB; j++) {
      tc[j] = thr[j];
      bc[j] = b[j];
    }
  }
  __device__ __forceinline__ double step(double x) const {
    return kak_step(
        x, [&](int j) { return tc[j]; }, [&](int j) { return bc[j]; }, thr, b);
  }
};

// x0 of every (replication, dim): KakutaniState(p, rng.random()) with
// rng = derive_rng(derive_key(seed, 6, m), d) (halton.py:530-534).
__global__ void k_kakutani_setup(RepTables t, double *x0) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)t.rep_count * t.dim) return;
  const int rl = (int)(gid / t.dim), d = (int)(gid % t.dim);
  const uint64_t key = derive_key3(t.seed, 6, (uint64_t)(t.rep_first + rl));
  Pcg64 g;
  pcg_seed(g, derive_key2(key, (uint64_t)d));
  x0[gid] = pcg_random(g);
}


// Snapshot walk: orbit points at the segment starts P_s = p0 + s seg_len
// (tile layout) or at every run start P = p0 + s seg_len + t ntile_s, t <
// TILE (runs layout); point n is x after n steps.  Each orbit is one
// dependent chain of up to N steps (latency bound), so a thread walks
// KAK_KW orbits interleaved.
constexpr int KAK_KW = 1;  // orbits per thread (4 measured slower: fewer warps, same chain)
template <bool RUNS_LAYOUT>
__global__ void k_kak_walk(RepTables t, int rep_local0, int rep_n, SeqArgs q, double *snap) {
  const int64_t norb = (int64_t)rep_n * t.dim;
  const int64_t o0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * KAK_KW;
  if (o0 >= norb) return;
  double xc[KAK_KW][KK_NB], bc[KAK_KW][KK_NB], x[KAK_KW];
  const double *thr[KAK_KW], *bb[KAK_KW];
  int64_t base[KAK_KW];  // snapshot offset of the orbit
  bool ok[KAK_KW];
#pragma unroll
  for (int w = 0; w < KAK_KW; w++) {
    ok[w] = o0 + w < norb;
    const int64_t o = ok[w] ? o0 + w : o0;
    const int rb = (int)(o / t.dim), d = (int)(o % t.dim);
    thr[w] = g_kk_thr + d * KK_TAB;
    bb[w] = g_kk_b + d * KK_TAB;
#pragma unroll
    for (int j = 0; j < KK_NB; j++) {
      xc[w][j] = g_kk_xthr[d * 8 + j];
      bc[w][j] = bb[w][j];
    }
    x[w] = t.kk_x0[(int64_t)(rep_local0 + rb) * t.dim + d];
    base[w] = (int64_t)rb * q.segs_per_rep * (RUNS_LAYOUT ? TILE : 1) * t.dim + d;
  }
  int64_t pos = 0;
  const int nrun = RUNS_LAYOUT ? TILE : 1;
  for (int sg = 0; sg < q.segs_per_rep; sg++) {
    const int64_t s0 = (int64_t)sg * q.seg_len;
    const int64_t slen = q.seg_len < q.nmax - s0 ? q.seg_len : q.nmax - s0;
    const int64_t ntile = (slen + TILE - 1) / TILE;
    for (int tt = 0; tt < nrun; tt++) {
      int64_t P = q.p0 + s0 + (int64_t)tt * ntile;
      if (P > q.p0 + s0 + slen) P = q.p0 + s0 + slen;  // empty run: never read
#pragma unroll 2
      for (; pos < P; pos++) {
#pragma unroll
        for (int w = 0; w < KAK_KW; w++) x[w] = kak_step_flat(x[w], xc[w], bc[w], thr[w], bb[w]);
      }
      const int64_t slot = ((int64_t)sg * nrun + tt) * t.dim;
#pragma unroll
      for (int w = 0; w < KAK_KW; w++)
        if (ok[w]) snap[base[w] + slot] = x[w];
    }
  }
}

// Per-thread runs (dim <= KK_RUNS_MAXDIM): thread t owns paths
// [t ntile, (t+1) ntile) of a segment and steps each dimension's orbit once
// per path, the orbit values of its dims in the dynamic shared memory
// xs[dim][TILE] next to the tile; the dims' first brackets come from the
// constant bank (warp-uniform).  No barrier and no idle thread in the walk.
struct GenKakutaniRuns {
  static constexpr bool RUNS = true;
  using Shared = NoShared;
  const RepTables *t;
  const SeqArgs *q;
  double *xs;
  int dim;
  __device__ void setup(const RepTables &t_, Shared &, uint32_t *) { t = &t_; }
  __device__ void set_seq(const SeqArgs &q_, int dim_) {
    q = &q_;
    dim = dim_;
  }
  __device__ void set_dyn(double *p) { xs = p; }
  static __host__ __device__ size_t dyn_bytes(int dim_) { return sizeof(double) * dim_ * TILE; }
  __device__ __forceinline__ double step(int d, double x) const {
    const double *c = c_kk8 + d * 16;
    return kak_step(
        x, [&](int j) { return c[j]; }, [&](int j) { return c[8 + j]; },
        g_kk_thr + d * KK_TAB, g_kk_b + d * KK_TAB);
  }
  __device__ void begin_segment(int, int rb, int sg, int64_t, int64_t, int) {
    const double *src = q->kk_snap + (((int64_t)rb * q->segs_per_rep + sg) * TILE + threadIdx.x) * dim;
    for (int d = 0; d < dim; d++) xs[d * TILE + threadIdx.x] = src[d];
  }
  __device__ void unit(int, int, int d0, int Dc, double *zt) {
    for (int dd = 0; dd < Dc; dd++) {
      double *xp = xs + (d0 + dd) * TILE + threadIdx.x;
      const double x = *xp;
      zt[dd * TILE + threadIdx.x] = x;
      *xp = step(d0 + dd, x);
    }
  }
  __device__ void skip(int n) {  // the dims a path-free model does not read
    for (int d = dim - n; d < dim; d++) {
      double *xp = xs + d * TILE + threadIdx.x;
      *xp = step(d, *xp);
    }
  }
};

// Tile layout (TILE consecutive paths): at chunk 0 of a tile, thread t
// advances the orbits of dims t, t + TILE, ... over the tile's paths into
// the per-CTA scratch [dim][TILE] (doubles); chunks read their columns.  The
// orbit state of every dim between tiles, xs[dim], follows the CTA's columns
// in the scratch (any dim up to MAX_DIM; read and written by its own thread).
struct GenKakutani {
  __device__ void set_dyn(double *) {}
  static __host__ __device__ size_t dyn_bytes(int) { return 0; }
  static constexpr bool RUNS = false;
  using Shared = NoShared;
  const RepTables *t;
  double *xs;
  double *scr;
  const SeqArgs *q;
  int dim;
  __device__ void setup(const RepTables &t_, Shared &, uint32_t *) { t = &t_; }
  __device__ void set_seq(const SeqArgs &q_, int dim_) {
    q = &q_;
    dim = dim_;
    // this CTA's slice of the scratch: [dim][TILE] columns, then xs[dim]
    scr = reinterpret_cast<double *>(q_.scratch) + (size_t)blockIdx.x * dim_ * (TILE + 1);
    xs = scr + (size_t)dim_ * TILE;
  }
  __device__ void begin_segment(int, int rb, int sg, int64_t, int64_t, int) {
    const double *src = q->kk_snap + ((int64_t)rb * q->segs_per_rep + sg) * dim;
    __syncthreads();  // the previous segment's last tile is done with the columns
    for (int d = threadIdx.x; d < dim; d += TILE) xs[d] = src[d];
  }
  __device__ void skip(int) {}
  __device__ void fill_tile(int npaths) {
#pragma unroll 1
    for (int d = threadIdx.x; d < dim; d += TILE) {
      KakDim kd;
      kd.load(d);
      double xv = xs[d];
#pragma unroll 4
      for (int j = 0; j < npaths; j++) {
        scr[d * TILE + j] = xv;
        xv = kd.step(xv);
      }
      xs[d] = xv;
    }
    __syncthreads();
  }
  __device__ void unit(int, int npaths, int d0, int Dc, double *zt) {
    if (d0 == 0) fill_tile(npaths);
    for (int dd = 0; dd < Dc; dd++)
      zt[dd * TILE + threadIdx.x] = __ldcg(scr + (d0 + dd) * TILE + threadIdx.x);
  }
};

// ======================================================================
// Warp-cooperative inverse normal over the thread's own column of a chunk.
// Comparisons run on the integer pipe (IEEE order of non-negative doubles
// == order of their bit patterns); four inputs are in flight per pass for
// ILP; the ~9% tail inputs are queued and evaluated 32 at a time.
// ======================================================================
// SUM: the normals are only summed (config-4 stream without a store): each
// goes into *acc where it is formed instead of back into the tile.
// FIXED > 0: Dc == FIXED known at compile time
template <int FIXED = 0, bool UNROLL = false, bool SUM = false>
__device__ __forceinline__ void chunk_to_normals(double *zt, int Dc_, uint16_t *q,
                                                 double *acc = nullptr) {
  const int Dc = FIXED > 0 ? FIXED : Dc_;
  constexpr bool FULL = FIXED > 0 && FIXED % 4 == 0;  // no partial pass: no guards
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int qn = 0;
  auto pass = [&](int d4) {
    double p[4], x[4];
    bool tail[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int dd = d4 + k;
      p[k] = FULL || dd < Dc ? zt[dd * TILE + threadIdx.x] : 0.5;
      tail[k] = (FULL || dd < Dc) && (RQ_TAIL_CAND ? invn_tail_cand(p[k]) : invn_tail_p(p[k]));
    }
#pragma unroll
    for (int k = 0; k < 4; k++) x[k] = invn_central_q(p[k] - 0.5);
#pragma unroll
    for (int k = 0; k < 4; k++) {
      const int dd = d4 + k;
      const int slot = dd * TILE + threadIdx.x;
      unsigned b = __ballot_sync(0xffffffffu, tail[k]);
      if (tail[k]) q[qn + __popc(b & lt)] = (uint16_t)slot;
      else if (FULL || dd < Dc) {
        if constexpr (SUM) *acc += x[k];
        else zt[slot] = x[k];
      }
      qn += __popc(b);
    }
  };
  // A fixed-width chunk (single-chunk LIBOR) keeps one pass body: its path
  // kernel is already long (the unrolled rate triangle), and instruction
  // fetch, not the loop branch, is what costs there (measured: Philox /
  // XORWOW C2 +5%); the persistent Rasrap kernel measured 0.7% better
  // unrolled (UNROLL).
  if constexpr (FIXED > 0 && !UNROLL) {
#pragma unroll 1
    for (int d4 = 0; d4 < Dc; d4 += 4) pass(d4);
  } else {
#pragma unroll
    for (int d4 = 0; d4 < Dc; d4 += 4) pass(d4);
  }
  __syncwarp();
  for (int k = lane; k < qn; k += 32) {
    const int slot = q[k];
    const double x = invn_queued(zt[slot]);  // tail candidates: exact test, then tail
    if constexpr (SUM) *acc += x;
    else zt[slot] = x;
  }
  __syncwarp();
}

// ======================================================================
// Models: thread-per-path state in registers
// ======================================================================

// Scale k of the LIBOR rate state z = k delta L: k = sigma^2 delta, the
// drift's weight, so the drift sum lands directly in the rate multiplier.
// Below 2^-900 (sigma = 0 included) the drift is below one ulp of the
// multiplier 1 + shock whatever k is, and k = 2^-900 keeps z normal and
// 1/k finite.
__device__ __forceinline__ double libor_state_scale(const ModelParams &mp) {
  const double s2d = mp.sigma * mp.sigma * mp.delta;
  return s2d >= 0x1p-900 ? s2d : 0x1p-900;
}

// LIBOR market-model caplet, one-factor Euler (models.py:271-293).  The S
// forward rates live in registers, held as z_n = k delta L_n with k =
// sigma^2 delta: the reference's rate-step (dl = delta L_n; drift +=
// sigma^2 dl / (1 + dl); L_n *= 1 + drift delta + shock) becomes
// f += z_n / (1 + z_n / k); z_n *= f, with f = 1 + shock at the step's start:
// 5 FP64 + MUFU per rate-step instead of 7 (see libor_state_scale).
// For S <= CHUNK the whole step/rate
// triangle is unrolled; above that the step loop is dynamic and the rate
// loop unrolled with uniform guards.  1/(1 + delta L) in the drift uses a
// MUFU seed plus one Newton step (the drift's weight in the path is ~1e-4,
// so the ~2^-44 relative error is far below the 1e-12 parity bar).  The
// deflator prod (1 + delta L_i(T_i)) is formed as a product and inverted
// once (each L_i is frozen after step i, so its final value is its fixing,
// models.py:289-290).
template <int S, int NSR = RQ_LIBOR_SMEM_RATES>
struct ModelLibor {
  static constexpr bool NORMALS = true;
  static constexpr bool SMALL_LIBOR = S <= 20;
  static constexpr int FIXED_DIMS = S <= CHUNK ? S : 0;  // one chunk of exactly S dims
  static constexpr int MINB =
      S <= 20 ? RQ_MINB_SMALL : (S <= 40 ? 3 : (RQ_LIBOR_SMEM_RATES ? 3 : 2));  // CTAs/SM
  struct Shared {
    double l0[S];
  };
  static __host__ __device__ int gen_dims(int dim) { return dim; }
  // S = 80: the first NS rates live in dynamic shared memory Ls[NS][TILE]
  // (they die first: step i only touches rates n >= i), the rest in
  // registers, so a thread needs ~100 fewer registers and three CTAs fit an
  // SM instead of two.
  static constexpr int NS = S >= 80 ? NSR : 0;
  static __host__ __device__ size_t dyn_bytes(int) { return sizeof(double) * NS * TILE; }
  const Shared *sh;
  double *Ls;
  double L[S - NS];
  __device__ void set_dyn(double *p) { Ls = p; }
  __device__ __forceinline__ double &Lr(int n) {
    if (n < NS) return Ls[n * TILE + ctid()];
    return L[n - NS];
  }
  __device__ __forceinline__ double Lv(int n) const {
    if (n < NS) return Ls[n * TILE + ctid()];
    return L[n - NS];
  }
  double cz, ssq, dstrike, ff;
  __device__ void init(const ModelParams &mp_, Shared &s) {
    const double kz = libor_state_scale(mp_);
    for (int n = ctid(); n < S; n += TILE) s.l0[n] = kz * (mp_.delta * mp_.table[n]);
    sh = &s;
    cz = 1.0 / kz;
    dstrike = mp_.delta * mp_.strike;
    ff = mp_.front_factor;
    ssq = mp_.sigma * sqrt(mp_.delta);
  }
  __device__ void begin() {
#pragma unroll
    for (int n = 0; n < S; n++) Lr(n) = sh->l0[n];
  }
  // static step (S <= CHUNK: whole triangle unrolled, i compile-time)
  __device__ __forceinline__ void step(int i, double z) {
    double f = fma(ssq, z, 1.0);
#pragma unroll
    for (int n = 0; n < S; n++) {
      if (n >= i) {
        double r = rcp1(fma(cz, Lr(n), 1.0));
        f = fma(Lr(n), r, f);
        Lr(n) *= f;
      }
    }
  }
  // dynamic step (large S): the alive rates n >= i are walked in groups of
  // GRP with one uniform branch per group, so each group is straight-line
  // code whose GRP reciprocals overlap; only the first alive group is
  // partial and masks its dead rates with selects.
  static constexpr int GRP = S % 8 == 0 ? 8 : (S % 4 == 0 ? 4 : (S % 5 == 0 ? 5 : 1));
  __device__ __forceinline__ void group(int g, int i, double &f, bool partial) {
    double r[GRP];
#pragma unroll
    for (int k = 0; k < GRP; k++) r[k] = rcp1(fma(cz, Lr(g * GRP + k), 1.0));
#pragma unroll
    for (int k = 0; k < GRP; k++) {
      const int n = g * GRP + k;
      const double ln0 = Lr(n);
      const double fn = fma(ln0, r[k], f);
      const double ln = ln0 * fn;
      if (partial) {
        const bool alive = n >= i;
        f = alive ? fn : f;
        Lr(n) = alive ? ln : ln0;
      } else {
        f = fn;
        Lr(n) = ln;
      }
    }
  }
  __device__ __forceinline__ void step_dyn(int i, double z) {
    static_assert(S % GRP == 0, "S must be a multiple of the rate group");
    double f = fma(ssq, z, 1.0);
    const int first = i / GRP;
#pragma unroll
    for (int g = 0; g < S / GRP; g++) {
      if (g == first) group(g, i, f, true);
      else if (g > first) group(g, i, f, false);
    }
  }
  __device__ void chunk(int d0, int Dc, const double *zcol) {
    if (S <= CHUNK && S <= RQ_LIBOR_STATIC_MAX) {
#pragma unroll
      for (int i = 0; i < S; i++) step(i, zcol[i * TILE]);
    } else {
      for (int k = 0; k < Dc; k++) step_dyn(d0 + k, zcol[k * TILE]);
    }
  }
  __device__ double payoff() const {
    double prod = 1.0;
#pragma unroll
    for (int n = 0; n < S - 1; n++) prod *= fma(cz, Lv(n), 1.0);
    const double lt = Lv(S - 1);
    const double pay = fmax(fma(cz, lt, -dstrike), 0.0);
    return pay * ff * rcp2(fma(cz, lt, 1.0) * prod);
  }
};

// LIBOR with any number of steps S <= LIBOR_DYN_MAX (LiborConfig allows any
// integer maturity/accrual, models.py:172-193): the same operations per
// rate-step as ModelLibor<S> (models.py:271-293), the forward rates in
// dynamic shared memory Ls[S][TILE] and the rate loop dynamic.  The step
// counts of the benchmark configurations (10, 20, 40, 80) use the
// register-resident ModelLibor<S> instead.
struct ModelLiborDyn {
  static constexpr bool NORMALS = true;
  static constexpr bool SMALL_LIBOR = false;
  static constexpr int MINB = 2;
  struct Shared {
    double l0[LIBOR_DYN_MAX];
  };
  static __host__ __device__ int gen_dims(int dim) { return dim; }
  static __host__ __device__ size_t dyn_bytes(int dim) { return sizeof(double) * dim * TILE; }
  const Shared *sh;
  double *Ls;
  int S;
  double cz, ssq, dstrike, ff;
  __device__ void set_dyn(double *p) { Ls = p; }
  __device__ void init(const ModelParams &mp_, Shared &s) {
    S = mp_.dim;
    const double kz = libor_state_scale(mp_);
    for (int n = ctid(); n < S; n += TILE) s.l0[n] = kz * (mp_.delta * mp_.table[n]);
    sh = &s;
    cz = 1.0 / kz;
    dstrike = mp_.delta * mp_.strike;
    ff = mp_.front_factor;
    ssq = mp_.sigma * sqrt(mp_.delta);
  }
  __device__ void begin() {
    for (int n = 0; n < S; n++) Ls[n * TILE + ctid()] = sh->l0[n];
  }
  __device__ void chunk(int d0, int Dc, const double *zcol) {
    for (int k = 0; k < Dc; k++) {
      const int i = d0 + k;
      const double g1 = fma(ssq, zcol[k * TILE], 1.0);
      double f = g1;
      double *L = Ls + ctid();
#pragma unroll 4
      for (int n = i; n < S; n++) {
        const double ln = L[n * TILE];
        const double r = rcp1(fma(cz, ln, 1.0));
        f = fma(ln, r, f);
        L[n * TILE] = ln * f;
      }
    }
  }
  __device__ double payoff() const {
    const double *L = Ls + ctid();
    double prod = 1.0;
    for (int n = 0; n < S - 1; n++) prod *= fma(cz, L[n * TILE], 1.0);
    const double lt = L[(S - 1) * TILE];
    const double pay = fmax(fma(cz, lt, -dstrike), 0.0);
    return pay * ff * rcp2(fma(cz, lt, 1.0) * prod);
  }
};

// LIBOR with S > LIBOR_DYN_MAX steps (up to LIBOR_MAX): ModelLiborDyn's
// operations in the same order (bit-identical payoffs), the forward rates
// in a per-CTA slice of global memory, [S][TILE] doubles at
// mp.lstate + blockIdx.x * S * TILE (coalesced; the launcher sizes the grid
// to the slices it allocated), and L_n(0) formed from mp.table at begin().
struct ModelLiborBig {
  static constexpr bool NORMALS = true;
  static constexpr bool SMALL_LIBOR = false;
  static constexpr int MINB = 2;
  using Shared = NoShared;
  static __host__ __device__ int gen_dims(int dim) { return dim; }
  const double *tab;
  double *Ls;
  int S;
  double kz, delta, cz, ssq, dstrike, ff;
  __device__ void init(const ModelParams &mp_, Shared &) {
    S = mp_.dim;
    kz = libor_state_scale(mp_);
    delta = mp_.delta;
    tab = mp_.table;
    Ls = mp_.lstate + (size_t)blockIdx.x * S * TILE + ctid();
    cz = 1.0 / kz;
    dstrike = mp_.delta * mp_.strike;
    ff = mp_.front_factor;
    ssq = mp_.sigma * sqrt(mp_.delta);
  }
  __device__ void begin() {
    for (int n = 0; n < S; n++) Ls[(size_t)n * TILE] = kz * (delta * tab[n]);
  }
  __device__ void chunk(int d0, int Dc, const double *zcol) {
    for (int k = 0; k < Dc; k++) {
      const int i = d0 + k;
      const double g1 = fma(ssq, zcol[k * TILE], 1.0);
      double f = g1;
#pragma unroll 4
      for (int n = i; n < S; n++) {
        const double ln = Ls[(size_t)n * TILE];
        const double r = rcp1(fma(cz, ln, 1.0));
        f = fma(ln, r, f);
        Ls[(size_t)n * TILE] = ln * f;
      }
    }
  }
  __device__ double payoff() const {
    double prod = 1.0;
    for (int n = 0; n < S - 1; n++) prod *= fma(cz, Ls[(size_t)n * TILE], 1.0);
    const double lt = Ls[(size_t)(S - 1) * TILE];
    const double pay = fmax(fma(cz, lt, -dstrike), 0.0);
    return pay * ff * rcp2(fma(cz, lt, 1.0) * prod);
  }
};

// k0 * exp(sigma_xi * z) as one polynomial in z: the Taylor series of exp
// to x^9 with x = sigma_xi * z and k0 folded into the coefficients
// (ModelParams::ecoef, built on the host), valid for |x| <= 0.1 (truncation
// < 3.1e-17 relative).  The shocks stay there unless |z| > 5 at the
// reference's variance; beyond that (or for other variances) libdevice exp.
// atan(y) = atan(c) + atan(t), t = (y - c) / (1 + c y), c = 1/2 below 0.62
// and 3/4 above: |t| <= 0.1 for y in [0.381, 0.919] (MBS rates -1.2% ..
// 4.2% at k3 = 10, k4 = 0.5) and the odd series to t^13 is exact to 7e-17;
// other y: libdevice atan.
__constant__ double c_atan_ser[6] = {0.07692307692307693, -0.09090909090909091,
                                     0.1111111111111111,  -0.14285714285714285,
                                     0.2,                 -0.3333333333333333};
__constant__ double c_atan_ctr[4] = {0.5, 0.75, 0.4636476090008061, 0.6435011087932844};
// range tests on the high word (ALU pipe, not a DSETP on the FP64 pipe);
// they only choose between two valid evaluations, so they need not be exact
__device__ __forceinline__ uint32_t abs_hi(double x) {
  return (uint32_t)__double2hiint(x) & 0x7FFFFFFFu;
}
// out-of-range fallbacks: rare, kept out of line (instruction cache)
__device__ __noinline__ double atan_slow(double y) { return atan(y); }
__device__ __noinline__ double kexp_slow(double k0, double sxi, double z) {
  return k0 * exp(sxi * z);
}
__device__ __forceinline__ double atan_mbs(double y) {
  const bool hi = abs_hi(y) >= 0x3FE3D70Au;  // y >= ~0.62 (y > 0 here)
  const double c = hi ? c_atan_ctr[1] : c_atan_ctr[0];
  const double t = div2(y - c, fma(c, y, 1.0));
  if (abs_hi(t) > 0x3FB99999u || __double2hiint(y) < 0) return atan_slow(y);  // |t| > ~0.1
  const double t2 = t * t;
  double p = c_atan_ser[0];
#pragma unroll
  for (int k = 1; k < 6; k++) p = fma(p, t2, c_atan_ser[k]);
  return fma(t * t2, p, t) + (hi ? c_atan_ctr[3] : c_atan_ctr[2]);
}

// MBS present value (models.py:430-449), monthly steps.  State: R =
// payment * remaining (so the cash flow is one product), the rate, 1 - w of
// the previous month (1.0 before month 1: R * 1.0 is exact, as the
// reference's skipped update), and the present value as a fraction N / P:
// the reference's discount disc_k = 1 / P_k with P_k = prod_{j<=k} (1 +
// i_{j-1}), so pv_k = pv_{k-1} + a_k / P_k is N_k = N_{k-1} (1 + i_{k-1}) +
// a_k over P_k, and the 360 divisions become one per path.
struct ModelMbs {
  static constexpr bool NORMALS = true;
  static constexpr bool SMALL_LIBOR = false;
  static constexpr int MINB = 4;  // lower bound; 70 registers: 7 CTAs/SM run (measured best: 6 -2%, 5 -7%)
  static constexpr int MAXM = 1 << 20;
  using Shared = NoShared;
  static __host__ __device__ int gen_dims(int dim) { return dim; }
  const double *ck;
  double i0, sxi, k0, k1, k2, k3, k4, pay;
  uint32_t zlim_hi;  // high word of exp_zlim: |z| below it stays in the series range
  double ec[MBS_EXP_TERMS];
  double P, R, rate, omw, N;
  __device__ void init(const ModelParams &mp_, Shared &) {
    ck = mp_.table;  // annuity ratios: uniform across the warp, L1-resident
    i0 = mp_.i0;
    sxi = mp_.sigma_xi;
    k0 = mp_.k0;
    k1 = mp_.k1;
    k2 = mp_.k2;
    k3 = mp_.k3;
    k4 = mp_.k4;
    pay = mp_.payment;
    zlim_hi = abs_hi(mp_.exp_zlim);
#pragma unroll
    for (int k = 0; k < MBS_EXP_TERMS; k++) ec[k] = mp_.ecoef[k];
  }
  __device__ void begin() {
    P = 1.0;
    R = pay;
    rate = i0;
    omw = 1.0;
    N = 0.0;
  }
  __device__ __forceinline__ double kexp(double z) const {  // k0 * exp(sigma_xi z)
    if (abs_hi(z) >= zlim_hi) return kexp_slow(k0, sxi, z);
    double p = ec[MBS_EXP_TERMS - 1];
#pragma unroll
    for (int k = MBS_EXP_TERMS - 2; k >= 0; k--) p = fma(p, z, ec[k]);
    return p;
  }
  // Months in groups of MG: the shocks' exponentials, the discount
  // reciprocals and the prepayment arctangents of a group are independent
  // once the (cheap, serial) rate product is known, so they are issued
  // together; only P / R / N remain serial (models.py:437-448).
  static constexpr int MG = RQ_MBS_MG;
  __device__ void chunk(int d0, int Dc, const double *zcol) {
    int kk = 0;
    for (; kk + MG <= Dc; kk += MG) {
      double e[MG], u[MG], w[MG];
#pragma unroll
      for (int m = 0; m < MG; m++) e[m] = kexp(zcol[(kk + m) * TILE]);
      double r = rate;
#pragma unroll
      for (int m = 0; m < MG; m++) {
        u[m] = 1.0 + r;  // the discount uses the rate before this month's update
        r = e[m] * r;
        w[m] = r;
      }
#pragma unroll
      for (int m = 0; m < MG; m++) w[m] = fma(k2, atan_mbs(fma(k3, w[m], k4)), k1);
#pragma unroll
      for (int m = 0; m < MG; m++) {
        P *= u[m];
        R *= omw;
        omw = 1.0 - w[m];
        N = fma(N, u[m], R * fma(w[m], __ldg(ck + d0 + kk + m), omw));
      }
      rate = r;
      rescale();
    }
    for (; kk < Dc; kk++) {
      const double u = 1.0 + rate;
      P *= u;
      R *= omw;
      rate = kexp(zcol[kk * TILE]) * rate;
      const double w = fma(k2, atan_mbs(fma(k3, rate, k4)), k1);
      omw = 1.0 - w;
      N = fma(N, u, R * fma(w, __ldg(ck + d0 + kk), omw));
    }
    rescale();
  }
  // P = prod (1 + i) overflows for high-variance rates (the reference's
  // disc = 1/P underflows harmlessly instead): once P passes 2^512, scale
  // P, N and the undiscounted cash-flow factor R together by 2^-512 -- exact
  // (N_k = sum_j a_j P_k / P_j keeps its value over P), and the later cash
  // flows carry the same factor.  One integer compare per group of months.
  __device__ __forceinline__ void rescale() {
    if (__double2hiint(P) >= 0x5FF00000) {
      P *= 0x1p-512;
      N *= 0x1p-512;
      R *= 0x1p-512;
    }
  }
  __device__ double payoff() const { return N / P; }
};

// f = x_1 (FirstCoordinateModel, models.py:489-498) and f = 1 (ConstantModel).
template <bool CONST1>
struct ModelTest {
  static constexpr bool NORMALS = false;
  static constexpr bool SMALL_LIBOR = false;
  static constexpr int MINB = 4;
  using Shared = NoShared;
  static __host__ __device__ int gen_dims(int) { return CONST1 ? 0 : 1; }
  double f;
  __device__ void init(const ModelParams &, Shared &) {}
  __device__ void begin() { f = 1.0; }
  __device__ void chunk(int, int Dc, const double *zcol) {
    if (!CONST1 && Dc > 0) f = zcol[0];
  }
  __device__ double payoff() const { return f; }
};

// Test integrand with no reference counterpart: a 64-bit hash of the bit
// patterns of ALL coordinates in dimension order, payoff = its top 20 bits
// as a double.  Sums of such payoffs are exact (< 2^53), so theta pins every
// coordinate of every path bit for bit through the production path kernel
// (the x1 integrand only sees dimension 0).  Oracle: rqmc_oracle.c
// coord_hash (same constants).
constexpr uint64_t XHASH_INIT = 0x6A09E667F3BCC909ull;
constexpr uint64_t XHASH_MUL = 0x9E3779B97F4A7C15ull;
__device__ __forceinline__ uint64_t xhash_step(uint64_t h, double u) {
  h = (h ^ (uint64_t)__double_as_longlong(u)) * XHASH_MUL;
  return h ^ (h >> 32);
}
struct ModelHash {
  static constexpr bool NORMALS = false;
  static constexpr bool SMALL_LIBOR = false;
  static constexpr int MINB = 4;
  using Shared = NoShared;
  static __host__ __device__ int gen_dims(int dim) { return dim; }
  uint64_t h;
  __device__ void init(const ModelParams &, Shared &) {}
  __device__ void begin() { h = XHASH_INIT; }
  __device__ void chunk(int, int Dc, const double *zcol) {
    for (int k = 0; k < Dc; k++) h = xhash_step(h, zcol[k * TILE]);
  }
  __device__ double payoff() const { return (double)(h >> 44); }
};

// ======================================================================
// Fused, software-pipelined path kernel
// ======================================================================
struct PathArgs {
  RepTables t;
  ModelParams mp;
  int rep_local0, rep_n;
  int64_t p0;    // first path (a multiple of TILE; segments of long estimates)
  int64_t nmax;  // paths p0 .. p0 + nmax - 1
  int64_t tiles_per_rep;
  double *payoffs;  // [rep_n][nmax], path p0 + i at i
};

constexpr size_t ZT_BYTES = sizeof(double) * CHUNK * TILE;  // one uniform/normal tile

// CTAs/SM the launch bounds target: the model's choice, capped by the
// generator's, except that the persistent Rasrap tile (shared-memory heavy,
// generator phases latency bound) gains from a fifth CTA next to small LIBOR
// (measured +1.7% at C2; Philox loses 3% at 5, so it stays at 4).
template <class G, class Mdl>
struct PathsMinB;

template <class G>
struct MaxBlocks {  // optional per-generator cap on CTAs/SM (register budget)
  template <class T>
  static constexpr int get(decltype(T::MAXB) *) { return T::MAXB; }
  template <class T>
  static constexpr int get(...) { return 8; }
  static constexpr int value = get<G>(nullptr);
};
template <class G, class Mdl>
struct PathsMinB {
  static constexpr int base = Mdl::MINB < MaxBlocks<G>::value ? Mdl::MINB : MaxBlocks<G>::value;
  static constexpr int value =
      std::is_same<G, GenRasrapRecTile<true>>::value && Mdl::SMALL_LIBOR ? RQ_RASRAP_MINB : base;
};

template <class G, class Mdl>
__global__ void __launch_bounds__(TILE, PathsMinB<G, Mdl>::value) k_paths(PathArgs a) {
  extern __shared__ __align__(16) double z[];  // ZT_BYTES
  __shared__ PhaseShared phs;
  __shared__ typename G::Shared gsh;
  __shared__ typename Mdl::Shared msh;
  Mdl md;
  md.init(a.mp, msh);
  ModelDyn<Mdl>::give(md, z + CHUNK * TILE);
  const int warp = threadIdx.x >> 5;
  const int gdims = Mdl::gen_dims(a.mp.dim);
  G g;
  g.setup(a.t, gsh, gdims);
  give_phase(g, phs);
  __syncthreads();
  const int nchunk = gdims > 0 ? (gdims + CHUNK - 1) / CHUNK : 1;
  // tiles per launch <= (payoff batch 2^27 paths) / TILE: 32-bit counters
  const int total = a.rep_n * (int)a.tiles_per_rep;
  if ((int)blockIdx.x >= total) return;
  // Single-chunk models: CTA b owns the contiguous tiles [lo, hi) of the
  // batch (rep-major), so consecutive tiles of a replication stay on one CTA
  // and the generator advances a persistent state.  Multi-chunk models
  // (long paths, large per-replication tables): tiles are strided over the
  // CTAs so all CTAs work on the same replication's tables at a time (L2).
  const bool contiguous = nchunk == 1;
  const int nb = gridDim.x, b = blockIdx.x;
  const int lo = contiguous ? (int)((int64_t)total * b / nb) : b;
  const int ntile =
      contiguous ? (int)((int64_t)total * (b + 1) / nb) - lo : (total - b + nb - 1) / nb;
  const int nunit = ntile * nchunk;
  // unit cursor: (replication, tile, chunk) advanced incrementally
  struct Cursor {
    int rl, c, tile;
  };
  const int tpr = (int)a.tiles_per_rep;
  const int tstride = contiguous ? 1 : nb;
  auto advance = [&](Cursor &q) {
    if (++q.c == nchunk) {
      q.c = 0;
      q.tile += tstride;
      while (q.tile >= tpr) {
        q.tile -= tpr;
        q.rl++;
      }
    }
  };
  Cursor cur{a.rep_local0 + lo / tpr, 0, lo % tpr};
  auto dc_of = [&](int c) { return gdims - c * CHUNK < CHUNK ? gdims - c * CHUNK : CHUNK; };
  auto base_of = [&](const Cursor &q) { return a.p0 + (int64_t)q.tile * TILE; };
  for (int u = 0; u < nunit; u++) {
    const int rl = cur.rl, d0 = cur.c * CHUNK, Dc = dc_of(cur.c);
    const int64_t base = base_of(cur);
    if (gdims > 0) {
      g.unit(rl, (uint64_t)base, (uint64_t)(base + threadIdx.x), d0, Dc, z);
      __syncthreads();
    }
    if (d0 == 0) md.begin();
    if (Mdl::NORMALS)
      chunk_to_normals<FixedDims<Mdl>::value, std::is_same<G, GenRasrapRecTile<true>>::value>(
          z, Dc, phs.tq[warp]);
    md.chunk(d0, Dc, z + threadIdx.x);
    if (d0 + Dc >= gdims) {
      const int64_t i = base - a.p0 + threadIdx.x;
      if (i < a.nmax) a.payoffs[(int64_t)(rl - a.rep_local0) * a.nmax + i] = md.payoff();
    }
    __syncthreads();
    advance(cur);
  }
}

// ======================================================================
// Warp-specialised path kernel (RQ_WS): 2 x TILE threads.  The first TILE
// threads (warps 0..3, the "producer" warpgroup) run the generator and the
// inverse normal of unit u into buffer u & 1; the second TILE threads (the
// "consumer" warpgroup) run the model on unit u - 1 from the other buffer.
// The producer phases are integer / shared-memory / issue bound, the model
// is FP64-pipe bound, so each SM always holds both kinds of work instead of
// whatever mix the phases of independent CTAs happen to be in.  Hand-off
// through named barriers (FULL[b]: producers arrive, consumers wait; EMPTY[b]:
// the reverse); the producers' own phase barrier is a third, TILE-thread one.
// Same units, same generator and model code, same results as k_paths.
// ======================================================================
template <int ID, int N>
__device__ __forceinline__ void nbar_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(N) : "memory");
}
template <int ID, int N>
__device__ __forceinline__ void nbar_arrive() {
  asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(N) : "memory");
}
constexpr int BAR_PROD = 1, BAR_CONS = 2, BAR_FULL0 = 3, BAR_EMPTY0 = 5;  // FULL/EMPTY + b

#ifndef RQ_WS_MINB
#define RQ_WS_MINB 3
#endif

template <class G, class Mdl>
__global__ void __launch_bounds__(2 * TILE, RQ_WS_MINB) k_paths_ws(PathArgs a) {
  extern __shared__ __align__(16) double z[];  // 2 x ZT_BYTES (+ model dyn)
  __shared__ PhaseShared phs;
  __shared__ typename G::Shared gsh;
  __shared__ typename Mdl::Shared msh;
  const bool producer = threadIdx.x < TILE;
  const int gdims = Mdl::gen_dims(a.mp.dim);
  const int nchunk = gdims > 0 ? (gdims + CHUNK - 1) / CHUNK : 1;
  const int total = a.rep_n * (int)a.tiles_per_rep;
  if ((int)blockIdx.x >= total) return;
  const bool contiguous = nchunk == 1;
  const int nb = gridDim.x, b = blockIdx.x;
  const int lo = contiguous ? (int)((int64_t)total * b / nb) : b;
  const int ntile =
      contiguous ? (int)((int64_t)total * (b + 1) / nb) - lo : (total - b + nb - 1) / nb;
  const int nunit = ntile * nchunk;
  const int tpr = (int)a.tiles_per_rep;
  const int tstride = contiguous ? 1 : nb;
  struct Cursor {
    int rl, c, tile;
  };
  auto advance = [&](Cursor &q) {
    if (++q.c == nchunk) {
      q.c = 0;
      q.tile += tstride;
      while (q.tile >= tpr) {
        q.tile -= tpr;
        q.rl++;
      }
    }
  };
  Cursor cur{a.rep_local0 + lo / tpr, 0, lo % tpr};
  auto dc_of = [&](int c) { return gdims - c * CHUNK < CHUNK ? gdims - c * CHUNK : CHUNK; };
  if (producer) {
    const int warp = threadIdx.x >> 5;
    G g;
    g.setup(a.t, gsh, gdims);
    give_phase(g, phs);
    nbar_sync<BAR_PROD, TILE>();
    for (int u = 0; u < nunit; u++) {
      const int buf = u & 1;
      double *zb = z + buf * (CHUNK * TILE);
      const int rl = cur.rl, d0 = cur.c * CHUNK, Dc = dc_of(cur.c);
      const int64_t base = a.p0 + (int64_t)cur.tile * TILE;
      if (u >= 2) {  // the consumers are done with zb
        if (buf) nbar_sync<BAR_EMPTY0 + 1, 2 * TILE>();
        else nbar_sync<BAR_EMPTY0, 2 * TILE>();
      }
      if (gdims > 0) {
        g.unit(rl, (uint64_t)base, (uint64_t)(base + threadIdx.x), d0, Dc, zb);
        nbar_sync<BAR_PROD, TILE>();  // every dim of the unit is in zb
      }
      if (Mdl::NORMALS)
        chunk_to_normals<FixedDims<Mdl>::value, std::is_same<G, GenRasrapRecTile<true>>::value>(
            zb, Dc, phs.tq[warp]);
      if (buf) nbar_arrive<BAR_FULL0 + 1, 2 * TILE>();
      else nbar_arrive<BAR_FULL0, 2 * TILE>();
      advance(cur);
    }
  } else {
    Mdl md;
    md.init(a.mp, msh);
    ModelDyn<Mdl>::give(md, z + 2 * CHUNK * TILE);
    nbar_sync<BAR_CONS, TILE>();
    const int t = ctid();
    for (int u = 0; u < nunit; u++) {
      const int buf = u & 1;
      const double *zb = z + buf * (CHUNK * TILE);
      const int rl = cur.rl, d0 = cur.c * CHUNK, Dc = dc_of(cur.c);
      const int64_t base = a.p0 + (int64_t)cur.tile * TILE;
      if (buf) nbar_sync<BAR_FULL0 + 1, 2 * TILE>();  // the producers filled zb
      else nbar_sync<BAR_FULL0, 2 * TILE>();
      if (d0 == 0) md.begin();
      md.chunk(d0, Dc, zb + t);
      if (d0 + Dc >= gdims) {
        const int64_t i = base - a.p0 + t;
        if (i < a.nmax) a.payoffs[(int64_t)(rl - a.rep_local0) * a.nmax + i] = md.payoff();
      }
      if (buf) nbar_arrive<BAR_EMPTY0 + 1, 2 * TILE>();
      else nbar_arrive<BAR_EMPTY0, 2 * TILE>();
      advance(cur);
    }
  }
}

// ======================================================================
// Path kernel of the sequential word streams (MT19937 / XORWOW).  Units of
// work are (replication, segment of seg_len paths); a CTA walks its units
// grid-stride.  Per unit the generator is positioned once (snapshot load or
// per-thread jump) and then streams: XORWOW threads own runs of consecutive
// paths, MT19937 tiles are TILE consecutive paths.  The model side
// (inverse normal, path, payoff) is the same as k_paths.
// ======================================================================
struct ModelPoints {  // sampler.fill of a sequential stream: write the uniforms
  static constexpr bool NORMALS = false;
  static constexpr bool SMALL_LIBOR = false;
  static constexpr int MINB = 4;
  using Shared = NoShared;
  static __host__ __device__ int gen_dims(int dim) { return dim; }
  __device__ void init(const ModelParams &, Shared &) {}
  __device__ void begin() {}
  __device__ void chunk(int, int, const double *) {}
  __device__ double payoff() const { return 0.0; }
};

template <class G, class Mdl>
__global__ void __launch_bounds__(TILE, (Mdl::MINB < MaxBlocks<G>::value ? Mdl::MINB
                                                                          : MaxBlocks<G>::value))
    k_paths_seq(PathArgs a, SeqArgs q) {
  extern __shared__ __align__(16) double z[];  // ZT_BYTES
  __shared__ PhaseShared phs;
  __shared__ typename G::Shared gsh;
  __shared__ typename Mdl::Shared msh;
  constexpr bool POINTS = std::is_same<Mdl, ModelPoints>::value;
  Mdl md;
  md.init(a.mp, msh);
  const int warp = threadIdx.x >> 5;
  const int dim = a.mp.dim;
  const int gdims = Mdl::gen_dims(dim);
  G g;
  g.setup(a.t, gsh, q.scratch + (size_t)blockIdx.x * dim * TILE);
  if constexpr (!G::RUNS || std::is_same<G, GenKakutaniRuns>::value) g.set_seq(q, dim);
  g.set_dyn(z + CHUNK * TILE);
  ModelDyn<Mdl>::give(md, z + CHUNK * TILE + G::dyn_bytes(dim) / sizeof(double));
  __syncthreads();
  const int nchunk = gdims > 0 ? (gdims + CHUNK - 1) / CHUNK : 1;
  const int64_t nunits = (int64_t)a.rep_n * q.segs_per_rep;
#pragma unroll 1
  for (int64_t un = blockIdx.x; un < nunits; un += gridDim.x) {
    const int rl = a.rep_local0 + (int)(un / q.segs_per_rep);
    const int sg = (int)(un % q.segs_per_rep);
    const int64_t s0 = (int64_t)sg * q.seg_len;  // path offset in [0, nmax)
    const int slen = (int)min(q.seg_len, a.nmax - s0);
    const int ntile = (slen + TILE - 1) / TILE;
    const int64_t my0 = G::RUNS ? s0 + (int64_t)threadIdx.x * ntile : s0 + threadIdx.x;
    // the whole word stream is positioned even for path-free models (gdims
    // = 0 never reaches here for the sequential generators: no such model)
    g.begin_segment(rl, rl - a.rep_local0, sg, q.p0 + s0, q.p0 + my0, dim);
#pragma unroll 1
    for (int u = 0; u < ntile; u++) {
      const int rel = G::RUNS ? (int)threadIdx.x * ntile + u : u * TILE + (int)threadIdx.x;
      const bool ok = rel < slen;
      const int64_t off = s0 + rel;  // path offset of this thread in [0, nmax)
      const int npaths = min(TILE, slen - u * TILE);
#pragma unroll 1
      for (int c = 0; c < nchunk; c++) {
        const int d0 = c * CHUNK, Dc = gdims - d0 < CHUNK ? gdims - d0 : CHUNK;
        g.unit(rl, npaths, d0, Dc, z);
        if (d0 + Dc >= gdims) g.skip(dim - gdims);
        __syncthreads();
        if (d0 == 0) md.begin();
        if constexpr (POINTS) {
          if (ok)
            for (int dd = 0; dd < Dc; dd++)
              a.payoffs[off * dim + d0 + dd] = z[dd * TILE + threadIdx.x];
        } else {
          if (Mdl::NORMALS) chunk_to_normals<FixedDims<Mdl>::value>(z, Dc, phs.tq[warp]);
          md.chunk(d0, Dc, z + threadIdx.x);
          if (d0 + Dc >= gdims && ok)
            a.payoffs[(int64_t)(rl - a.rep_local0) * a.nmax + off] = md.payoff();
        }
        __syncthreads();
      }
    }
  }
}

// ======================================================================
// Point kernels (sampler.fill / sampler.at), out[count][dim] row-major.
// Consecutive rows use the tiled generators, explicit indices the direct.
// ======================================================================
template <class G>
__global__ void __launch_bounds__(TILE, 4) k_points(RepTables t, int rl, int64_t first,
                                                 const int64_t *idx, int64_t count,
                                                 double *out) {
  extern __shared__ __align__(16) double zt[];  // ZT_BYTES
  __shared__ PhaseShared phs;
  __shared__ typename G::Shared gsh;
  G g;
  g.setup(t, gsh, t.dim);
  give_phase(g, phs);
  __syncthreads();
  for (int64_t tb = (int64_t)blockIdx.x * TILE; tb < count; tb += (int64_t)gridDim.x * TILE) {
    const int64_t r = tb + threadIdx.x;
    const bool ok = r < count;
    const int64_t path = idx ? (ok ? idx[r] : 0) : first + r;
    for (int d0 = 0; d0 < t.dim; d0 += CHUNK) {
      const int Dc = t.dim - d0 < CHUNK ? t.dim - d0 : CHUNK;
      __syncthreads();
      g.unit(rl, (uint64_t)(first + tb), (uint64_t)path, d0, Dc, zt);
      __syncthreads();
      if (ok)
        for (int dd = 0; dd < Dc; dd++) out[r * t.dim + d0 + dd] = zt[dd * TILE + threadIdx.x];
    }
  }
}

// ======================================================================
// Stream throughput kernel (config 4): points [0, npoints) of dimension
// t.dim, fused inverse normal, consumed by a sum (and optionally stored).
// ======================================================================
template <class G>
__global__ void __launch_bounds__(TILE, 4) k_stream(RepTables t, int rl, int64_t npoints,
                                                 double *block_sums, double *store) {
  extern __shared__ __align__(16) double zt[];  // ZT_BYTES
  __shared__ PhaseShared phs;
  __shared__ typename G::Shared gsh;
  __shared__ double red[WARPS];
  G g;
  g.setup(t, gsh, t.dim);
  give_phase(g, phs);
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  double acc = 0.0;
  for (int64_t tb = (int64_t)blockIdx.x * TILE; tb < npoints;
       tb += (int64_t)gridDim.x * TILE) {
    const int64_t r = tb + threadIdx.x;
    const bool ok = r < npoints;
    for (int d0 = 0; d0 < t.dim; d0 += CHUNK) {
      const int Dc = t.dim - d0 < CHUNK ? t.dim - d0 : CHUNK;
      __syncthreads();
      g.unit(rl, (uint64_t)tb, (uint64_t)r, d0, Dc, zt);
      __syncthreads();
      chunk_to_normals(zt, Dc, phs.tq[warp]);
      if (ok) {
        for (int dd = 0; dd < Dc; dd++) {
          double z = zt[dd * TILE + threadIdx.x];
          acc += z;
          if (store) store[r * t.dim + d0 + dd] = z;
        }
      }
    }
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < WARPS; k++) s += red[k];
    block_sums[blockIdx.x] = s;
  }
}

// Chunk-major stream for the Rasrap tile (s > CHUNK): a CTA works on one
// chunk c of CHUNK dims -- c = its SM's id mod nchunk, so the CTAs sharing
// an SM (and its L1) read the same chunk's sigma tables -- and takes runs of
// STREAM_RUN consecutive tiles of that chunk from a per-chunk counter, over
// which its generator state advances tile to tile (odometer + re-chain)
// instead of being rebuilt from the digits of n0 + base per tile and dim.
// Same points, same normals; only which CTA sums which (point, chunk).
#ifndef RQ_STREAM_RUN
#define RQ_STREAM_RUN 32
#endif
constexpr int STREAM_RUN = RQ_STREAM_RUN;  // tiles per counter grab
template <class G, bool STORE = true>
#ifndef RQ_STREAM_MINB
#define RQ_STREAM_MINB 5  // (4: -2.3% C4 Rasrap, 6: -6.5%)
#endif
__global__ void __launch_bounds__(TILE, RQ_STREAM_MINB) k_stream_chunks(RepTables t, int rl, int64_t npoints,
                                                           double *block_sums, double *store,
                                                           unsigned long long *ctr) {
  extern __shared__ __align__(16) double zt[];  // ZT_BYTES
  __shared__ PhaseShared phs;
  __shared__ typename G::Shared gsh;
  __shared__ double red[WARPS];
  __shared__ unsigned long long run0;
  G g;
  give_phase(g, phs);
  const int warp = threadIdx.x >> 5;
  const int nchunk = (t.dim + CHUNK - 1) / CHUNK;
  uint32_t smid;
  asm("mov.u32 %0, %%smid;" : "=r"(smid));
  const int64_t ntile = (npoints + TILE - 1) / TILE;
  double acc = 0.0;
  // own chunk first, then help the others (an SM count that is not a
  // multiple of nchunk leaves some chunks with one SM fewer)
  for (int k = 0; k < nchunk; k++) {
  const int c = (int)((smid + (uint32_t)k) % (uint32_t)nchunk);
  const int d0 = c * CHUNK, Dc = t.dim - d0 < CHUNK ? t.dim - d0 : CHUNK;
  g.setup(t, gsh, t.dim);  // new dims: no state to advance
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) run0 = atomicAdd(ctr + c, (unsigned long long)STREAM_RUN);
    __syncthreads();
    const int64_t lo = (int64_t)run0;
    if (lo >= ntile) break;
    const int64_t hi = lo + STREAM_RUN < ntile ? lo + STREAM_RUN : ntile;
    for (int64_t tile = lo; tile < hi; tile++) {
      const int64_t tb = tile * TILE, r = tb + threadIdx.x;
      g.unit(rl, (uint64_t)tb, (uint64_t)r, d0, Dc, zt);
      __syncthreads();
      if constexpr (STORE) {
        chunk_to_normals(zt, Dc, phs.tq[warp]);
        if (r < npoints) {
          for (int dd = 0; dd < Dc; dd++) {
            const double z = zt[dd * TILE + threadIdx.x];
            acc += z;
            store[r * t.dim + d0 + dd] = z;
          }
        }
      } else {
        if (r >= npoints)  // points past the end: uniforms of 1/2 (normal 0)
          for (int dd = 0; dd < Dc; dd++) zt[dd * TILE + threadIdx.x] = 0.5;
        chunk_to_normals<0, false, true>(zt, Dc, phs.tq[warp], &acc);
      }
      __syncthreads();
    }
  }
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sm = 0.0;
    for (int k = 0; k < WARPS; k++) sm += red[k];
    block_sums[blockIdx.x] = sm;
  }
}

template <class G, class = void>
struct HasTileHook : std::false_type {};
template <class G>
struct HasTileHook<G, std::void_t<decltype(G::TILE_HOOK)>> : std::true_type {};

template <class G>
static size_t stream_reg_dyn(int dim) {
  if constexpr (HasTileHook<G>::value) return G::dyn_bytes(dim);
  else return 0;
}

// Register form of the stream for per-thread generators (Philox, SFC64):
// four coordinates at a time straight from the generator into the central
// inverse normal and the sum, no tile round trip through shared memory;
// only the ~9% tail inputs go to a per-warp queue (value, and the store slot
// when STORE), evaluated 32 at a time whenever 32 are waiting.
template <class G, bool STORE>
__global__ void __launch_bounds__(TILE) k_stream_reg(RepTables t, int rl, int64_t npoints,
                                                     double *block_sums, double *store) {
  constexpr int QCAP = 32 + 4 * 32;  // < 32 left over + one 4-coordinate group
  __shared__ double qv[WARPS][QCAP];
  __shared__ int64_t qs[STORE ? WARPS : 1][STORE ? QCAP : 1];
  __shared__ double red[WARPS];
  __shared__ typename G::Shared gsh;
  G g;
  g.setup(t, gsh, t.dim);
  if constexpr (HasTileHook<G>::value) g.rep(rl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  double acc = 0.0;
  int qn = 0;
  auto tail_one = [&](int i) {
    const double x = invn_queued(qv[warp][i]);  // tail candidates: exact test, then tail
    acc += x;
    if constexpr (STORE) store[qs[warp][i]] = x;
  };
  for (int64_t tb = (int64_t)blockIdx.x * TILE; tb < npoints; tb += (int64_t)gridDim.x * TILE) {
    if constexpr (HasTileHook<G>::value) g.tile((uint64_t)tb);
    const int64_t r = tb + threadIdx.x;
    const bool ok = r < npoints;
    for (int d0 = 0; d0 < t.dim; d0 += 4) {
      double u[4], x[4];
      bool tail[4], use[4];
      g.quad(rl, (uint64_t)r, d0, u);
      const bool whole = d0 + 4 <= t.dim;  // uniform
#pragma unroll
      for (int k = 0; k < 4; k++) {
        use[k] = ok && (whole || d0 + k < t.dim);
        tail[k] = use[k] && (RQ_TAIL_CAND ? invn_tail_cand(u[k]) : invn_tail_p(u[k]));
      }
#pragma unroll
      for (int k = 0; k < 4; k++) x[k] = invn_central_q(u[k] - 0.5);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (use[k] && !tail[k]) {
          acc += x[k];
          if constexpr (STORE) store[r * t.dim + d0 + k] = x[k];
        }
        const unsigned b = __ballot_sync(0xffffffffu, tail[k]);
        if (tail[k]) {
          const int i = qn + __popc(b & lt);
          qv[warp][i] = u[k];
          if constexpr (STORE) qs[warp][i] = r * t.dim + d0 + k;
        }
        qn += __popc(b);
      }
      if (qn >= 32) {
        __syncwarp();
        do {
          tail_one(qn - 32 + lane);
          qn -= 32;
        } while (qn >= 32);
        __syncwarp();
      }
    }
  }
  __syncwarp();
  if (lane < qn) tail_one(lane);
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sm = 0.0;
    for (int k = 0; k < WARPS; k++) sm += red[k];
    block_sums[blockIdx.x] = sm;
  }
}

// ======================================================================
// Model payoffs from caller uniforms (model.payoffs(u), models.py:311-322,
// 462-469): thread per path, scalar inverse normal.
// ======================================================================
template <class Mdl>
__global__ void __launch_bounds__(TILE) k_payoffs_u(ModelParams mp, const double *u,
                                                    int64_t npaths, double *out) {
  __shared__ typename Mdl::Shared msh;
  extern __shared__ __align__(16) double zt[];  // ZT_BYTES
  Mdl md;
  md.init(mp, msh);
  ModelDyn<Mdl>::give(md, zt + CHUNK * TILE);
  __syncthreads();
  // one tile per CTA; ModelLiborBig: grid-stride (the grid is its state slices)
  constexpr bool STRIDE = std::is_same<Mdl, ModelLiborBig>::value;
  for (int64_t p = (int64_t)blockIdx.x * TILE + threadIdx.x; p - threadIdx.x < npaths;
       p += (int64_t)gridDim.x * TILE) {
    const bool ok = p < npaths;
    md.begin();
    for (int d0 = 0; d0 < mp.dim; d0 += CHUNK) {
      const int Dc = mp.dim - d0 < CHUNK ? mp.dim - d0 : CHUNK;
      for (int k = 0; k < Dc; k++)
        zt[k * TILE + threadIdx.x] = ok ? inv_normal(u[p * mp.dim + d0 + k]) : 0.0;
      md.chunk(d0, Dc, zt + threadIdx.x);
    }
    if (ok) out[p] = md.payoff();
    if constexpr (!STRIDE) break;
  }
}

__global__ void k_inv_normal(const double *u, int64_t n, double *out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = inv_normal(u[i]);
}

// ======================================================================
// numpy pairwise reduction (np.sum of a contiguous float64 prefix)
// ======================================================================
__device__ double leaf_sum(const double *a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; i++) res = dadd(res, a[i]);
    return res;
  }
  double r0 = a[0], r1 = a[1], r2 = a[2], r3 = a[3], r4 = a[4], r5 = a[5], r6 = a[6], r7 = a[7];
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
    r0 = dadd(r0, a[i]);
    r1 = dadd(r1, a[i + 1]);
    r2 = dadd(r2, a[i + 2]);
    r3 = dadd(r3, a[i + 3]);
    r4 = dadd(r4, a[i + 4]);
    r5 = dadd(r5, a[i + 5]);
    r6 = dadd(r6, a[i + 6]);
    r7 = dadd(r7, a[i + 7]);
  }
  double res = dadd(dadd(dadd(r0, r1), dadd(r2, r3)), dadd(dadd(r4, r5), dadd(r6, r7)));
  for (; i < n; i++) res = dadd(res, a[i]);
  return res;
}

// grid = (leaf blocks, replications).  Every block sums up to blockDim
// leaves; the last block to finish a replication (atomic ticket) folds the
// internal nodes level by level and writes theta = root / N.
__global__ void k_reduce(SumPlan plan, const double *pay, int64_t pay_stride, double *theta,
                         int theta_stride, double *scratch, unsigned *tickets) {
  const int rep = blockIdx.y;
  const double *a = pay + (int64_t)rep * pay_stride;
  double *val = scratch + (int64_t)rep * plan.nnodes;
#if RQ_REDUCE_WARP
  {  // eight lanes per leaf: lane j carries numpy's accumulator r_j (elements
     // j, j+8, ... in order), the fold ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) by
     // xor shuffles (each sum formed by the same two operands), lane 0 adds
     // the n % 8 tail in order -- leaf_sum's arithmetic, coalesced loads
    const int j = threadIdx.x & 7;
    const int k = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 3);
    const bool has = k < plan.nleaves;
    const int n = has ? plan.leaf_len[k] : 0;
    const double *b = a + (has ? plan.leaf_start[k] : 0);
    const int m = n - n % 8;
    double r = n >= 8 ? b[j] : 0.0;
    for (int i = 8 + j; i < m; i += 8) r = dadd(r, b[i]);
    r = dadd(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = dadd(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = dadd(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (has && j == 0) {
      double res = n >= 8 ? r : 0.0;
      for (int i = m; i < n; i++) res = dadd(res, b[i]);
      val[k] = res;
    }
  }
#else
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < plan.nleaves) val[k] = leaf_sum(a + plan.leaf_start[k], plan.leaf_len[k]);
#endif
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&tickets[rep], 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int lv = 0; lv < plan.nlevels; lv++) {
    for (int e = plan.level_off[lv] + threadIdx.x; e < plan.level_off[lv + 1]; e += blockDim.x)
      val[plan.node_id[e]] = dadd(__ldcg(val + plan.node_l[e]), __ldcg(val + plan.node_r[e]));
    __threadfence_block();
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    theta[(int64_t)rep * theta_stride] = __ddiv_rn(__ldcg(val + plan.root), (double)plan.n);
    tickets[rep] = 0u;  // self-resetting for the next launch
  }
}

// ======================================================================
// FP64 pipe peak probe: independent DFMA chains, no memory traffic.
// ======================================================================
constexpr int PEAK_CHAINS = 8;
__global__ void __launch_bounds__(256) k_dfma_peak(int iters, double seed, double *sink) {
  double a[PEAK_CHAINS];
#pragma unroll
  for (int c = 0; c < PEAK_CHAINS; c++) a[c] = seed + threadIdx.x * 1e-9 + c;
  const double m = 0.9999999, k = 1e-7;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int u = 0; u < 16; u++)
#pragma unroll
      for (int c = 0; c < PEAK_CHAINS; c++) a[c] = fma(a[c], m, k);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < PEAK_CHAINS; c++) s += a[c];
  if (s == 12345.678) sink[threadIdx.x] = s;  // keep the chains alive
}

// ======================================================================
// Launchers
// ======================================================================
static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// every kernel taking dynamic shared memory opts in to the full carve-out
template <class K>
static size_t prep_dyn(K kernel, size_t dyn) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
  return dyn;
}

template <class K>
static int persistent_blocks(K kernel, int64_t work, size_t dyn = 0) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, TILE, dyn);
  // RQ_BLOCKS_PER_SM: optional cap on the persistent CTAs per SM (tuning)
  static const int cap = [] {
    const char *e = getenv("RQ_BLOCKS_PER_SM");
    return e ? atoi(e) : 0;
  }();
  if (cap > 0 && per_sm > cap) per_sm = cap;
  if (per_sm < 1) per_sm = 1;
  int64_t b = (int64_t)per_sm * sm_count();
  return (int)(work < b ? (work < 1 ? 1 : work) : b);
}

cudaError_t launch_dfma_peak(int blocks, int iters, double *sink, cudaStream_t s) {
  k_dfma_peak<<<blocks, 256, 0, s>>>(iters, 1.0, sink);
  return cudaGetLastError();
}

// Few (replication, dim) units with large bases (a single replication of a
// wide sampler, the config-4 stream): the setup is the latency of the
// longest shuffle chain, so those units get a warp each and shuffle in
// shared memory.  Many units (replication groups): one thread per unit
// keeps 32 chains in flight per warp, which wins on throughput.
constexpr int SETUP_WARP_P = 256, SETUP_WARP_PMAX = 8192, SETUP_WARP_UNITS = 16384;
cudaError_t launch_rasrap_setup(const RepTables &t, uint16_t *sigma, uint16_t *digits,
                                double *sums, uint64_t *start, cudaStream_t s,
                                const int *bases) {
  int dsplit = 0;
  while (dsplit < t.dim && bases[dsplit] <= SETUP_WARP_P) dsplit++;
  const int64_t big_units = (int64_t)t.rep_count * (t.dim - dsplit);
  if (big_units == 0 || big_units > SETUP_WARP_UNITS || bases[t.dim - 1] > SETUP_WARP_PMAX)
    dsplit = t.dim;
  {
    const int64_t n = (int64_t)t.rep_count * dsplit;
    if (n > 0)
      k_rasrap_setup<<<(int)((n + 127) / 128), 128, 0, s>>>(t, 0, dsplit, sigma, digits, sums,
                                                            start);
  }
  if (dsplit < t.dim) {
    const int smax = (bases[t.dim - 1] + 7) & ~7;  // u16 entries per warp (<= 16 KB)
    const int wpb = std::max(1, std::min(8, (48 << 10) / (2 * smax)));
    k_rasrap_setup_warp<<<(int)((big_units + wpb - 1) / wpb), 32 * wpb,
                          (size_t)wpb * smax * 2, s>>>(t, dsplit, t.dim, smax, sigma, digits, sums,
                                                       start);
  }
  return cudaGetLastError();
}

cudaError_t launch_sobol_setup(const RepTables &t, const uint32_t *v_dev, uint32_t *gen_v,
                               uint32_t *shift, cudaStream_t s) {
  int64_t n = (int64_t)t.rep_count * t.dim;
  int blocks = (int)((n + 127) / 128);
  k_sobol_setup<<<blocks, 128, 0, s>>>(t, v_dev, gen_v, shift);
  return cudaGetLastError();
}

template <class G>
static cudaError_t points_t(const RepTables &t, int rl, int64_t first, const int64_t *idx,
                            int64_t count, double *out, cudaStream_t s) {
  int64_t tiles = (count + TILE - 1) / TILE;
  size_t dyn = prep_dyn(k_points<G>, ZT_BYTES);
  int blocks = persistent_blocks(k_points<G>, tiles, dyn);
  k_points<G><<<blocks, TILE, dyn, s>>>(t, rl, first, idx, count, out);
  return cudaGetLastError();
}

cudaError_t launch_points(const RepTables &t, int rl, int64_t first, const int64_t *idx,
                          int64_t count, double *out, cudaStream_t s) {
  const bool at = idx != nullptr;
  switch (t.gen) {
    case GEN_RASRAP_RECURSIVE:
      if (at) return points_t<GenRasrapRecDirect>(t, rl, first, idx, count, out, s);
      return t.dim > CONST_DIMS
                 ? points_t<GenRasrapRecTile<false, false, true>>(t, rl, first, idx, count, out, s)
                 : points_t<GenRasrapRecTile<false>>(t, rl, first, idx, count, out, s);
    case GEN_RASRAP_COUNTER:
      if (at) return points_t<GenRasrapCounter>(t, rl, first, idx, count, out, s);
      return t.dim > CONST_DIMS
                 ? points_t<GenRasrapCounterTile<true>>(t, rl, first, idx, count, out, s)
                 : points_t<GenRasrapCounterTile<false>>(t, rl, first, idx, count, out, s);
    case GEN_PHILOX: return points_t<GenPhilox>(t, rl, first, idx, count, out, s);
    case GEN_SOBOL_GRAY:
      return at ? points_t<GenSobolDirect<true>>(t, rl, first, idx, count, out, s)
                : points_t<GenSobolTile<true>>(t, rl, first, idx, count, out, s);
    case GEN_SOBOL_COUNTER:
      return at ? points_t<GenSobolDirect<false>>(t, rl, first, idx, count, out, s)
                : points_t<GenSobolTile<false>>(t, rl, first, idx, count, out, s);
    case GEN_SFC64: return points_t<GenSfc64>(t, rl, first, idx, count, out, s);
  }
  return cudaErrorInvalidValue;
}

// ModelLiborBig: per-CTA forward-rate state in global memory, allocated in
// stream order around the launch; the grid is capped so it stays <= 1 GiB
// (and >= one CTA per SM).
template <class Mdl>
static constexpr bool big_libor = std::is_same<Mdl, ModelLiborBig>::value;
static size_t lstate_bytes(int S) { return sizeof(double) * (size_t)S * TILE; }
static int lstate_blocks(int64_t blocks, int S) {
  const int64_t cap = std::max<int64_t>(sm_count(), ((int64_t)1 << 30) / (int64_t)lstate_bytes(S));
  return (int)std::min<int64_t>(blocks, cap);
}
struct LState {
  double *p = nullptr;
  cudaStream_t s;
  explicit LState(cudaStream_t s_) : s(s_) {}
  cudaError_t alloc(int blocks, int S) {
    return cudaMallocAsync(reinterpret_cast<void **>(&p), lstate_bytes(S) * blocks, s);
  }
  ~LState() {
    if (p) cudaFreeAsync(p, s);
  }
};

template <class G, class Mdl>
static cudaError_t paths_gm(const PathArgs &a, int *launched, cudaStream_t s, bool probe,
                            int *blocks_out) {
  const int64_t work = (int64_t)a.rep_n * a.tiles_per_rep;
#if RQ_WS
  // generators whose unit has no CTA-wide barrier (the consumer warpgroup
  // never reaches one: GenRasrapCounterTile syncs the whole CTA); RQ_WS = 1:
  // only where it measured faster (the persistent Rasrap tile with LIBOR
  // S <= 20), 2: every eligible pair (experiments)
  constexpr bool ws_ok = !std::is_same<G, GenRasrapCounterTile<false>>::value &&
                        !std::is_same<G, GenRasrapCounterTile<true>>::value;
  // (the xhash test integrand takes the same kernel, so its bit-exact theta
  // pins the warp-specialised generator path the C2 headline runs)
  constexpr bool ws_pick = RQ_WS >= 2 || (std::is_same<G, GenRasrapRecTile<true>>::value &&
                                          (Mdl::SMALL_LIBOR || std::is_same<Mdl, ModelHash>::value));
  if constexpr (ws_ok && ws_pick) {
    size_t dyn = prep_dyn(k_paths_ws<G, Mdl>, 2 * ZT_BYTES + ModelDyn<Mdl>::bytes(a.mp.dim));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_paths_ws<G, Mdl>, 2 * TILE, dyn);
    if (per_sm < 1) per_sm = 1;
    const int64_t bmax = (int64_t)per_sm * sm_count();
    const int blocks = (int)(work < bmax ? (work < 1 ? 1 : work) : bmax);
    if (blocks_out) *blocks_out = blocks;
    if (probe) return cudaSuccess;
    k_paths_ws<G, Mdl><<<blocks, 2 * TILE, dyn, s>>>(a);
    if (launched) *launched += 1;
    return cudaGetLastError();
  }
#endif
  size_t dyn = prep_dyn(k_paths<G, Mdl>, ZT_BYTES + ModelDyn<Mdl>::bytes(a.mp.dim));
  int blocks = persistent_blocks(k_paths<G, Mdl>, work, dyn);
  if constexpr (big_libor<Mdl>) blocks = lstate_blocks(blocks, a.mp.dim);
  if (blocks_out) *blocks_out = blocks;
  if (probe) return cudaSuccess;
  if constexpr (big_libor<Mdl>) {
    LState ls(s);
    cudaError_t e = ls.alloc(blocks, a.mp.dim);
    if (e != cudaSuccess) return e;
    PathArgs b = a;
    b.mp.lstate = ls.p;
    k_paths<G, Mdl><<<blocks, TILE, dyn, s>>>(b);
  } else {
    k_paths<G, Mdl><<<blocks, TILE, dyn, s>>>(a);
  }
  if (launched) *launched += 1;
  return cudaGetLastError();
}

// LIBOR S = 80 in the fused kernel: 24 of the rates in shared memory (fewer
// shared-memory round trips than 40 at the same 3 CTAs/SM: +3.7% C5 Rasrap,
// +2.4% Philox); the counter-form tile needs more registers of its own and
// keeps 40 (24 spills there).
template <class G>
struct LiborSmemRates {
  static constexpr int value = 24;
};
template <bool W>
struct LiborSmemRates<GenRasrapCounterTile<W>> {
  static constexpr int value = RQ_LIBOR_SMEM_RATES;
};

template <class G>
static cudaError_t paths_g(const PathArgs &a, int *launched, cudaStream_t s, bool probe,
                           int *blocks) {
  switch (a.mp.kind) {
    case MODEL_LIBOR:
      switch (a.mp.dim) {
        case 10: return paths_gm<G, ModelLibor<10>>(a, launched, s, probe, blocks);
        case 20: return paths_gm<G, ModelLibor<20>>(a, launched, s, probe, blocks);
        case 40: return paths_gm<G, ModelLibor<40>>(a, launched, s, probe, blocks);
        case 80: return paths_gm<G, ModelLibor<80, LiborSmemRates<G>::value>>(a, launched, s, probe,
                                                                             blocks);
      }
      if (a.mp.dim >= 1 && a.mp.dim <= LIBOR_DYN_MAX)
        return paths_gm<G, ModelLiborDyn>(a, launched, s, probe, blocks);
      if (a.mp.dim > LIBOR_DYN_MAX && a.mp.dim <= LIBOR_MAX)
        return paths_gm<G, ModelLiborBig>(a, launched, s, probe, blocks);
      return cudaErrorInvalidValue;
    case MODEL_MBS:
      if (a.mp.dim > ModelMbs::MAXM) return cudaErrorInvalidValue;
      return paths_gm<G, ModelMbs>(a, launched, s, probe, blocks);
    case MODEL_X1: return paths_gm<G, ModelTest<false>>(a, launched, s, probe, blocks);
    case MODEL_CONST1: return paths_gm<G, ModelTest<true>>(a, launched, s, probe, blocks);
    case MODEL_XHASH: return paths_gm<G, ModelHash>(a, launched, s, probe, blocks);
  }
  return cudaErrorInvalidValue;
}

// generators of more than CONST_DIMS dims: only the models that take that
// many (LIBOR past the shared-memory model, MBS, the test integrands)
template <class G>
static cudaError_t paths_g_wide(const PathArgs &a, int *launched, cudaStream_t s, bool probe,
                                int *blocks) {
  switch (a.mp.kind) {
    case MODEL_LIBOR:
      if (a.mp.dim > LIBOR_DYN_MAX && a.mp.dim <= LIBOR_MAX)
        return paths_gm<G, ModelLiborBig>(a, launched, s, probe, blocks);
      return cudaErrorInvalidValue;
    case MODEL_MBS:
      if (a.mp.dim > ModelMbs::MAXM) return cudaErrorInvalidValue;
      return paths_gm<G, ModelMbs>(a, launched, s, probe, blocks);
    case MODEL_X1: return paths_gm<G, ModelTest<false>>(a, launched, s, probe, blocks);
    case MODEL_CONST1: return paths_gm<G, ModelTest<true>>(a, launched, s, probe, blocks);
    case MODEL_XHASH: return paths_gm<G, ModelHash>(a, launched, s, probe, blocks);
  }
  return cudaErrorInvalidValue;
}

static cudaError_t paths_dispatch(const PathArgs &a, int *launched, cudaStream_t s, bool probe,
                                  int *blocks) {
  switch (a.t.gen) {
    case GEN_RASRAP_RECURSIVE:
      if (a.t.dim > CONST_DIMS)
        return paths_g_wide<GenRasrapRecTile<false, false, true>>(a, launched, s, probe, blocks);
      return a.mp.kind == MODEL_MBS || a.mp.dim > CHUNK
                 ? paths_g<GenRasrapRecTile<false>>(a, launched, s, probe, blocks)
                 : paths_g<GenRasrapRecTile<true>>(a, launched, s, probe, blocks);
    case GEN_RASRAP_COUNTER:
      if (a.t.dim > CONST_DIMS)
        return paths_g_wide<GenRasrapCounterTile<true>>(a, launched, s, probe, blocks);
      return paths_g<GenRasrapCounterTile<false>>(a, launched, s, probe, blocks);
    case GEN_PHILOX: return paths_g<GenPhilox>(a, launched, s, probe, blocks);
#if RQ_SOBOL_PERSIST
    case GEN_SOBOL_GRAY:
      return a.mp.kind == MODEL_MBS || a.mp.dim > CHUNK
                 ? paths_g<GenSobolTile<true>>(a, launched, s, probe, blocks)
                 : paths_g<GenSobolTileP<true>>(a, launched, s, probe, blocks);
    case GEN_SOBOL_COUNTER:
      return a.mp.kind == MODEL_MBS || a.mp.dim > CHUNK
                 ? paths_g<GenSobolTile<false>>(a, launched, s, probe, blocks)
                 : paths_g<GenSobolTileP<false>>(a, launched, s, probe, blocks);
#else
    case GEN_SOBOL_GRAY: return paths_g<GenSobolTile<true>>(a, launched, s, probe, blocks);
    case GEN_SOBOL_COUNTER: return paths_g<GenSobolTile<false>>(a, launched, s, probe, blocks);
#endif
    case GEN_SFC64: return paths_g<GenSfc64>(a, launched, s, probe, blocks);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_paths(const RepTables &t, const ModelParams &mp, int rep_local0, int rep_n,
                         int64_t p0, int64_t nmax, double *payoffs, int *launched,
                         cudaStream_t s) {
  PathArgs a;
  a.t = t;
  a.mp = mp;
  a.rep_local0 = rep_local0;
  a.rep_n = rep_n;
  a.p0 = p0;
  a.nmax = nmax;
  a.tiles_per_rep = (nmax + TILE - 1) / TILE;
  a.payoffs = payoffs;
  return paths_dispatch(a, launched, s, false, nullptr);
}

int paths_grid_blocks(const RepTables &t, const ModelParams &mp) {
  PathArgs a{};
  a.t = t;
  a.mp = mp;
  a.rep_n = 1 << 20;
  a.tiles_per_rep = 1 << 20;
  int blocks = 0;
  paths_dispatch(a, nullptr, 0, true, &blocks);
  return blocks;
}

// ---------------------------------------------------------------- sequential streams
cudaError_t launch_xorwow_setup(const RepTables &t, uint32_t *state, cudaStream_t s) {
  k_xorwow_setup<<<(t.rep_count + 127) / 128, 128, 0, s>>>(t, state);
  return cudaGetLastError();
}

cudaError_t launch_kakutani_setup(const RepTables &t, double *x0, cudaStream_t s) {
  const int64_t n = (int64_t)t.rep_count * t.dim;
  k_kakutani_setup<<<(int)((n + 127) / 128), 128, 0, s>>>(t, x0);
  return cudaGetLastError();
}

cudaError_t launch_kak_snap(const RepTables &t, int rep_local0, int rep_n, const SeqArgs &q,
                            double *snap, cudaStream_t s) {
  const int64_t n = (int64_t)rep_n * t.dim;
  // latency-bound sequential walks: small CTAs spread them over all SMs
  const int64_t nthr = (n + KAK_KW - 1) / KAK_KW;
  if (kak_runs(t.dim))
    k_kak_walk<true><<<(int)((nthr + 31) / 32), 32, 0, s>>>(t, rep_local0, rep_n, q, snap);
  else
    k_kak_walk<false><<<(int)((nthr + 31) / 32), 32, 0, s>>>(t, rep_local0, rep_n, q, snap);
  return cudaGetLastError();
}

cudaError_t launch_mt_snap(const RepTables &t, int rep_local0, int rep_n, const SeqArgs &q,
                           uint32_t *snap, cudaStream_t s) {
  k_mt_snap<<<rep_n, 256, 0, s>>>(t, rep_local0, t.dim, q, snap);
  return cudaGetLastError();
}

template <class G, class Mdl>
static cudaError_t seq_gm(const PathArgs &a, const SeqArgs &q, int blocks, int *launched,
                          cudaStream_t s, int *occ) {
  size_t dyn =
      prep_dyn(k_paths_seq<G, Mdl>,
               ZT_BYTES + G::dyn_bytes(a.mp.dim) + ModelDyn<Mdl>::bytes(a.mp.dim));
  if (occ) {
    *occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k_paths_seq<G, Mdl>, TILE, dyn);
    if constexpr (big_libor<Mdl>)  // seq_layout's CTA count, capped to the rate-state slices
      *occ = std::max(1, std::min(*occ, lstate_blocks((int64_t)*occ * sm_count(), a.mp.dim) /
                                            sm_count()));
    return cudaSuccess;
  }
  if constexpr (big_libor<Mdl>) {
    LState ls(s);
    cudaError_t e = ls.alloc(blocks, a.mp.dim);
    if (e != cudaSuccess) return e;
    PathArgs b = a;
    b.mp.lstate = ls.p;
    k_paths_seq<G, Mdl><<<blocks, TILE, dyn, s>>>(b, q);
  } else {
    k_paths_seq<G, Mdl><<<blocks, TILE, dyn, s>>>(a, q);
  }
  if (launched) *launched += 1;
  return cudaGetLastError();
}

template <class G>
static cudaError_t seq_g(const PathArgs &a, const SeqArgs &q, int blocks, int *launched,
                         cudaStream_t s, int *occ) {
  switch (a.mp.kind) {
    case MODEL_LIBOR:
      switch (a.mp.dim) {
        case 10: return seq_gm<G, ModelLibor<10>>(a, q, blocks, launched, s, occ);
        case 20: return seq_gm<G, ModelLibor<20>>(a, q, blocks, launched, s, occ);
        case 40: return seq_gm<G, ModelLibor<40>>(a, q, blocks, launched, s, occ);
        case 80: return seq_gm<G, ModelLibor<80>>(a, q, blocks, launched, s, occ);
      }
      if (a.mp.dim >= 1 && a.mp.dim <= LIBOR_DYN_MAX)
        return seq_gm<G, ModelLiborDyn>(a, q, blocks, launched, s, occ);
      if (a.mp.dim > LIBOR_DYN_MAX && a.mp.dim <= LIBOR_MAX)
        return seq_gm<G, ModelLiborBig>(a, q, blocks, launched, s, occ);
      return cudaErrorInvalidValue;
    case MODEL_MBS:
      if (a.mp.dim > ModelMbs::MAXM) return cudaErrorInvalidValue;
      return seq_gm<G, ModelMbs>(a, q, blocks, launched, s, occ);
    case MODEL_X1: return seq_gm<G, ModelTest<false>>(a, q, blocks, launched, s, occ);
    case MODEL_CONST1: return seq_gm<G, ModelTest<true>>(a, q, blocks, launched, s, occ);
    case MODEL_XHASH: return seq_gm<G, ModelHash>(a, q, blocks, launched, s, occ);
    case MODEL_POINTS: return seq_gm<G, ModelPoints>(a, q, blocks, launched, s, occ);
  }
  return cudaErrorInvalidValue;
}

static cudaError_t seq_dispatch(const PathArgs &a, const SeqArgs &q, int blocks, int *launched,
                                cudaStream_t s, int *occ) {
  switch (a.t.gen) {
    case GEN_TWISTER: return seq_g<GenTwister>(a, q, blocks, launched, s, occ);
    case GEN_XORWOW: return seq_g<GenXorwow>(a, q, blocks, launched, s, occ);
    case GEN_KAKUTANI:
      return kak_runs(a.t.dim) ? seq_g<GenKakutaniRuns>(a, q, blocks, launched, s, occ)
                               : seq_g<GenKakutani>(a, q, blocks, launched, s, occ);
  }
  return cudaErrorInvalidValue;
}

// Segment length: long enough that positioning a segment (XORWOW: up to 48
// matrix-vector products per thread, ~30k instructions; MT19937: a 2.5 KB
// snapshot) is a few percent of its path work (~120 instructions per
// coordinate), short enough for >= 4 units per CTA.
void seq_layout(const RepTables &t, const ModelParams &mp, int rep_n, int64_t nmax,
                int64_t *seg_len, int *segs_per_rep, int *blocks) {
  PathArgs a{};
  a.t = t;
  a.mp = mp;
  int occ = 1;
  SeqArgs q{};
  seq_dispatch(a, q, 0, nullptr, 0, &occ);
  if (occ < 1) occ = 1;
  const int ctas = occ * sm_count();
  int64_t want = (int64_t)(128.0 * 1.5e6 / (120.0 * (mp.dim > 0 ? mp.dim : 1)));
  int64_t cap = ((int64_t)rep_n * nmax) / (4 * (int64_t)ctas);
  int64_t L = std::min(want, cap);
  L = std::max<int64_t>(L, 8 * TILE);
  L = (L + TILE - 1) / TILE * TILE;
  const int64_t nm = (nmax + TILE - 1) / TILE * TILE;
  if (L > nm) L = nm;
  *seg_len = L;
  *segs_per_rep = (int)((nmax + L - 1) / L);
  const int64_t units = (int64_t)rep_n * *segs_per_rep;
  *blocks = (int)std::min<int64_t>(units, ctas);
}

cudaError_t launch_paths_seq(const RepTables &t, const ModelParams &mp, int rep_local0,
                             int rep_n, int64_t nmax, const SeqArgs &q, int blocks,
                             double *payoffs, int *launched, cudaStream_t s) {
  PathArgs a{};
  a.t = t;
  a.mp = mp;
  a.rep_local0 = rep_local0;
  a.rep_n = rep_n;
  a.nmax = nmax;
  a.tiles_per_rep = (nmax + TILE - 1) / TILE;
  a.payoffs = payoffs;
  return seq_dispatch(a, q, blocks, launched, s, nullptr);
}

cudaError_t launch_reduce(const SumPlan &plan, const double *payoffs, int64_t pay_stride,
                          int reps, double *theta, int theta_stride, double *scratch,
                          unsigned *tickets, cudaStream_t s) {
  dim3 grid((plan.nleaves + (RQ_REDUCE_WARP ? 31 : 255)) / (RQ_REDUCE_WARP ? 32 : 256), reps);
  k_reduce<<<grid, 256, 0, s>>>(plan, payoffs, pay_stride, theta, theta_stride, scratch,
                                tickets);
  return cudaGetLastError();
}

cudaError_t launch_model_payoffs(const ModelParams &mp, const double *u, int64_t npaths,
                                 double *out, cudaStream_t s) {
  int blocks = (int)((npaths + TILE - 1) / TILE);
  if (blocks < 1) return cudaSuccess;
  if (mp.kind == MODEL_MBS) {
    if (mp.dim > ModelMbs::MAXM) return cudaErrorInvalidValue;
    k_payoffs_u<ModelMbs><<<blocks, TILE, ZT_BYTES, s>>>(mp, u, npaths, out);
    return cudaGetLastError();
  }
  if (mp.kind != MODEL_LIBOR) return cudaErrorInvalidValue;
  switch (mp.dim) {
    case 10: k_payoffs_u<ModelLibor<10>><<<blocks, TILE, ZT_BYTES, s>>>(mp, u, npaths, out); break;
    case 20: k_payoffs_u<ModelLibor<20>><<<blocks, TILE, ZT_BYTES, s>>>(mp, u, npaths, out); break;
    case 40: k_payoffs_u<ModelLibor<40>><<<blocks, TILE, ZT_BYTES, s>>>(mp, u, npaths, out); break;
    case 80: {
      const size_t dyn = prep_dyn(k_payoffs_u<ModelLibor<80>>,
                                  ZT_BYTES + ModelDyn<ModelLibor<80>>::bytes(80));
      k_payoffs_u<ModelLibor<80>><<<blocks, TILE, dyn, s>>>(mp, u, npaths, out);
      break;
    }
    default: {
      if (mp.dim > LIBOR_DYN_MAX && mp.dim <= LIBOR_MAX) {
        const int nb = lstate_blocks(blocks, mp.dim);
        LState ls(s);
        cudaError_t e = ls.alloc(nb, mp.dim);
        if (e != cudaSuccess) return e;
        ModelParams m2 = mp;
        m2.lstate = ls.p;
        k_payoffs_u<ModelLiborBig><<<nb, TILE, ZT_BYTES, s>>>(m2, u, npaths, out);
        break;
      }
      if (mp.dim < 1 || mp.dim > LIBOR_DYN_MAX) return cudaErrorInvalidValue;
      const size_t dyn =
          prep_dyn(k_payoffs_u<ModelLiborDyn>, ZT_BYTES + ModelDyn<ModelLiborDyn>::bytes(mp.dim));
      k_payoffs_u<ModelLiborDyn><<<blocks, TILE, dyn, s>>>(mp, u, npaths, out);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_inv_normal(const double *u, int64_t n, double *out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  k_inv_normal<<<blocks, 256, 0, s>>>(u, n, out);
  return cudaGetLastError();
}

template <class G>
static cudaError_t stream_t(const RepTables &t, int rl, int64_t npoints, double *sums,
                            int nblocks, double *store, cudaStream_t s) {
  size_t dyn = prep_dyn(k_stream<G>, ZT_BYTES);
  k_stream<G><<<nblocks, TILE, dyn, s>>>(t, rl, npoints, sums, store);
  return cudaGetLastError();
}

template <class G>
static cudaError_t stream_reg_t(const RepTables &t, int rl, int64_t npoints, double *sums,
                                int nblocks, double *store, cudaStream_t s) {
  const size_t dyn = stream_reg_dyn<G>(t.dim);
  if (store) {
    if (dyn) prep_dyn(k_stream_reg<G, true>, dyn);
    k_stream_reg<G, true><<<nblocks, TILE, dyn, s>>>(t, rl, npoints, sums, store);
  } else {
    if (dyn) prep_dyn(k_stream_reg<G, false>, dyn);
    k_stream_reg<G, false><<<nblocks, TILE, dyn, s>>>(t, rl, npoints, sums, nullptr);
  }
  return cudaGetLastError();
}

int stream_grid_blocks(const RepTables &t) {
  const int64_t big = (int64_t)1 << 30;
  switch (t.gen) {
    case GEN_PHILOX: return persistent_blocks(k_stream_reg<GenPhilox, true>, big);
    case GEN_SFC64: return persistent_blocks(k_stream_reg<GenSfc64, true>, big);
#if RQ_SOBOL_STREAM_REG
    case GEN_SOBOL_GRAY:
      return persistent_blocks(k_stream_reg<GenSobolStream<true>, true>, big,
                               prep_dyn(k_stream_reg<GenSobolStream<true>, true>,
                                        GenSobolStream<true>::dyn_bytes(t.dim)));
    case GEN_SOBOL_COUNTER:
      return persistent_blocks(k_stream_reg<GenSobolStream<false>, true>, big,
                               prep_dyn(k_stream_reg<GenSobolStream<false>, true>,
                                        GenSobolStream<false>::dyn_bytes(t.dim)));
#endif
    case GEN_RASRAP_RECURSIVE: {  // chunk-major
      using K = GenRasrapRecTile<true, false>;  // (the WIDE form has the same footprint)
      return persistent_blocks(k_stream_chunks<K>, big, prep_dyn(k_stream_chunks<K>, ZT_BYTES));
    }
  }
  ModelParams mp{};
  mp.kind = MODEL_X1;
  mp.dim = t.dim;
  return paths_grid_blocks(t, mp);
}

// chunk-major Rasrap stream (per-chunk run counters, zeroed in stream order)
template <class K>
static cudaError_t stream_chunks_t(const RepTables &t, int rl, int64_t npoints, double *block_sums,
                                   int nblocks, double *store, cudaStream_t s) {
  const int nchunk = (t.dim + CHUNK - 1) / CHUNK;
  unsigned long long *ctr = nullptr;
  cudaError_t e = cudaMallocAsync((void **)&ctr, sizeof(unsigned long long) * nchunk, s);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * nchunk, s);
  if (store) {
    prep_dyn(k_stream_chunks<K, true>, ZT_BYTES);
    k_stream_chunks<K, true><<<nblocks, TILE, ZT_BYTES, s>>>(t, rl, npoints, block_sums, store,
                                                             ctr);
  } else {
    prep_dyn(k_stream_chunks<K, false>, ZT_BYTES);
    k_stream_chunks<K, false><<<nblocks, TILE, ZT_BYTES, s>>>(t, rl, npoints, block_sums,
                                                              nullptr, ctr);
  }
  e = cudaGetLastError();
  cudaFreeAsync(ctr, s);
  return e;
}

cudaError_t launch_stream_normals(const RepTables &t, int rl, int64_t npoints,
                                  double *block_sums, int nblocks, double *store,
                                  cudaStream_t s) {
  switch (t.gen) {
    case GEN_RASRAP_RECURSIVE:
      return t.dim > CONST_DIMS
                 ? stream_chunks_t<GenRasrapRecTile<true, false, true>>(t, rl, npoints, block_sums,
                                                                        nblocks, store, s)
                 : stream_chunks_t<GenRasrapRecTile<true, false>>(t, rl, npoints, block_sums,
                                                                  nblocks, store, s);
    case GEN_RASRAP_COUNTER:
      return t.dim > CONST_DIMS
                 ? stream_t<GenRasrapCounterTile<true>>(t, rl, npoints, block_sums, nblocks, store, s)
                 : stream_t<GenRasrapCounterTile<false>>(t, rl, npoints, block_sums, nblocks, store,
                                                         s);
    case GEN_PHILOX: return stream_reg_t<GenPhilox>(t, rl, npoints, block_sums, nblocks, store, s);
#if RQ_SOBOL_STREAM_REG
    case GEN_SOBOL_GRAY:
      return stream_reg_t<GenSobolStream<true>>(t, rl, npoints, block_sums, nblocks, store, s);
    case GEN_SOBOL_COUNTER:
      return stream_reg_t<GenSobolStream<false>>(t, rl, npoints, block_sums, nblocks, store, s);
#else
    case GEN_SOBOL_GRAY:
      return stream_t<GenSobolTile<true>>(t, rl, npoints, block_sums, nblocks, store, s);
    case GEN_SOBOL_COUNTER:
      return stream_t<GenSobolTile<false>>(t, rl, npoints, block_sums, nblocks, store, s);
#endif
    case GEN_SFC64: return stream_reg_t<GenSfc64>(t, rl, npoints, block_sums, nblocks, store, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace rq
