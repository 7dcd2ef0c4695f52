// rq_kernels.cu -- sm_100a kernels of the RQMC estimator.
//
// Layout of the fused path kernel (one CTA = one tile of T consecutive
// paths of one replication, persistent over (replication, tile) work items):
//
//   for each chunk of D dimensions (Euler steps / months):
//     1. generator: every thread writes the D uniforms of ITS path into a
//        shared-memory column zt[dd][tid]            (no HBM traffic)
//     2. inverse normal, warp-cooperative: central branch inline, the ~9%
//        tail inputs are compacted into a per-warp queue and evaluated 32
//        at a time (no log/sqrt divergence in the common branch)
//     3. model: the thread advances its path state (forward rates / MBS
//        cash-flow state) in registers through the D steps
//   payoff -> payoffs[rep][path]  (8 B/path, the only HBM write)
//
// then k_reduce applies numpy's pairwise-summation tree to each
// replication's payoff prefix (bit-identical to the reference np.sum).
//
// Every warp only touches its own shared-memory columns, so the tile loop
// needs __syncwarp only -- no CTA barriers on the hot path.
#include <cuda_runtime.h>

#include <cstdint>

#include "rq_device.cuh"
#include "rq_internal.h"

namespace rq {

constexpr int TILE = 128;  // paths per CTA tile = threads per CTA
constexpr int CHUNK = CHUNK_DIMS;  // dimensions per generator chunk (multiple of 4 for Philox)
constexpr int WARPS = TILE / 32;

__constant__ HaltonDim c_hdim[MAX_DIM];
constexpr int WTS_CAP = 16384;
__device__ double g_wts[WTS_CAP];     // binpow(inv_p, j+1): numba `x ** int` (halton.py:409)
__device__ double g_cscale[WTS_CAP];  // counter-form scale chain (halton.py:436)

cudaError_t upload_halton_dims(const HaltonDim *dims, int n, const double *wts,
                               const double *cscale, int nw) {
  if (n > MAX_DIM || nw > WTS_CAP) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemcpyToSymbol(c_hdim, dims, sizeof(HaltonDim) * n);
  if (e != cudaSuccess) return e;
  e = cudaMemcpyToSymbol(g_wts, wts, sizeof(double) * nw);
  if (e != cudaSuccess) return e;
  return cudaMemcpyToSymbol(g_cscale, cscale, sizeof(double) * nw);
}

// floor(t / base) for t < 2^32 (round-up magic, 33-bit multiplier)
__device__ __forceinline__ uint32_t div_base(uint32_t t, const HaltonDim &h) {
  uint64_t x = (uint64_t)__umulhi(t, h.mlo) + t;
  return (uint32_t)(x >> h.ell);
}

// ======================================================================
// Setup kernels (per replication randomisation, on device)
// ======================================================================

// One thread per (replication, dimension): rasrap_config + RasrapStream
// init (halton.py:345-360, 256-278, 139-155; seeding.py:59-65).
__global__ void k_rasrap_setup(RepTables t, uint16_t *sigma, uint16_t *digits, double *sums,
                               uint64_t *start) {
  int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (int64_t)t.rep_count * t.dim) return;
  int rl = (int)(gid / t.dim), d = (int)(gid % t.dim);
  const HaltonDim h = c_hdim[d];
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
    sm[j] = dadd(sm[j + 1], dmul((double)sg[dg[j]], scale));
    scale = dmul(scale, (double)h.base);
  }
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
// Generators.  Every thread produces the uniforms of ITS point for dims
// [d0, d0+Dc) into a shared-memory column (stride TILE).  Interface:
//   begin(t, rl, base, path, sh, sig_dyn, sig_cap)  per thread
//   prepare(d0, Dc)   block-cooperative (all threads, may __syncthreads)
//   chunk(d0, Dc, zcol)
// "Tiled" generators assume path = base + threadIdx.x (consecutive points);
// "direct" ones take any path index (sampler.at).
// ======================================================================
constexpr int LEVBUF = 80;  // nodes per level buffer (>= TILE/2 + 2)

struct RasrapTileShared {
  uint16_t bd[CHUNK][MAX_CAP];     // base-p digits of the tile base B = n0 + base
  int16_t nn[CHUNK][MAX_CAP + 1];  // nodes per level: distinct prefixes floor(n / p^j)
  int32_t J[CHUNK];                // top level (one node shared by the whole tile)
  int32_t hB[CHUNK];               // highest digit where B differs from n0 (-1: B == n0)
  double sJ[CHUNK];                // stream partial sum S_J of the top node
  double lev[WARPS][2][LEVBUF];    // per-warp ping-pong level buffers
};
struct RasrapDirectShared {
  uint16_t scr[MAX_CAP][TILE];     // per-thread digits (direct path)
};
struct SobolTileShared {
  uint32_t lowtab[CHUNK][128];     // XOR of v_k over the set bits k < 7
  uint32_t xhi[CHUNK];             // shift ^ XOR of v_k over the tile's bits k >= 7
};
union GenShared {
  RasrapTileShared r;
  RasrapDirectShared rd;
  SobolTileShared s;
};

__device__ __forceinline__ double u16d(uint16_t v) { return (double)v; }

// floor(x / base) for x < 2^46 (64-bit round-up magic, see rq_capi.cu)
__device__ __forceinline__ uint64_t div_base64(uint64_t x, const HaltonDim &h) {
  return __umul64hi(x, h.m64);
}

// Recursive-form point at arbitrary index (Alg. 2, halton.py:392-416)
// evaluated without replaying the stream: for n = n0 + i let h be the
// highest digit where n and n0 differ (= highest carry the odometer
// reached).  The stream then holds sums[j] = init_sums[j] above h and the
// chain S_j = S_{j+1} + sigma(a_j) * binpow(1/p, j+1) below, so the point is
// that chain started from init_sums[h+1] -- bit-identical to the reference.
__device__ double rasrap_rec_direct(const RepTables &t, int rl, int d, uint32_t i,
                                    uint16_t *scr) {
  const HaltonDim &h = c_hdim[d];
  const uint16_t *d0 = t.digits + (int64_t)rl * t.dig_stride + h.dig_off;
  const uint16_t *sg = t.sigma + (int64_t)rl * t.sig_stride + h.sig_off;
  const double *sums = t.sums + (int64_t)rl * t.sum_stride + h.sum_off;
  uint32_t r = i, carry = 0;
  int hi = -1, j = 0;
  while (r != 0u || carry != 0u) {
    uint32_t q = div_base(r, h);
    uint32_t a0 = d0[j];
    uint32_t a = a0 + (r - q * (uint32_t)h.base) + carry;
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
  const RepTables *t;
  int rl;
  uint32_t i;
  uint16_t *scr;
  __device__ void begin(const RepTables &t_, int rl_, uint64_t, uint64_t path, GenShared &sh,
                        uint16_t *, int) {
    t = &t_;
    rl = rl_;
    i = (uint32_t)path;
    scr = &sh.rd.scr[0][0] + threadIdx.x;
  }
  __device__ void fill(int d0, int Dc, double *zt) {
    for (int dd = 0; dd < Dc; dd++)
      zt[dd * TILE + threadIdx.x] = rasrap_rec_direct(*t, rl, d0 + dd, i, scr);
  }
};

// Tiled recursive form, evaluated level by level over the digit tree of the
// tile's TILE consecutive indices n = B + k, B = n0 + base.
//
// With S_j(n) the stream's partial sum at position j for index n, the
// reference recursion (halton.py:402-414, init sums halton.py:273-278) is
//     S_j(n) = init_sums[j]                                if floor(n/p^j) == floor(n0/p^j)
//            = S_{j+1}(n) + sigma(n_j) * binpow(1/p, j+1)   otherwise
// and S_j only depends on the prefix u = floor(n/p^j).  The tile's indices
// have N_j distinct prefixes at level j (N_0 = TILE, N_{j+1} = floor((b_j +
// N_j - 1)/p) + 1 with b_j the digits of B), so the warp owning a dim
// evaluates the N_j nodes of each level from their parents, top (N_J = 1,
// whose S_J is the chain from init_sums[hB+1]) to level 0 = the points.
// That is ~TILE * p/(p-1) node updates per tile and dim instead of
// TILE * log_p(n) for independent per-point chains, with the same
// operations in the same order as the reference (bit-identical).
struct GenRasrapRecTile {
  const RepTables *t;
  int rl;
  uint64_t base;
  GenShared *sh;
  __device__ void begin(const RepTables &t_, int rl_, uint64_t base_, uint64_t, GenShared &s,
                        uint16_t *, int) {
    t = &t_;
    rl = rl_;
    base = base_;
    sh = &s;
  }
  __device__ void fill(int d0, int Dc, double *zt) {
    RasrapTileShared &R = sh->r;
    const uint16_t *gsig = t->sigma + (int64_t)rl * t->sig_stride;
    const uint16_t *gdig = t->digits + (int64_t)rl * t->dig_stride;
    const double *gsum = t->sums + (int64_t)rl * t->sum_stride;
    __syncthreads();  // previous users of the shared state are done
    if (threadIdx.x < Dc) {
      // ---- per-dim tile state: digits of B, hB, level sizes, S_J
      const int dd = threadIdx.x;
      const HaltonDim &h = c_hdim[d0 + dd];
      const uint32_t p = (uint32_t)h.base;
      const uint16_t *n0d = gdig + h.dig_off;
      const double *ini = gsum + h.sum_off;
      const uint16_t *sg = gsig + h.sig_off;
      const double *w = g_wts + h.sum_off;
      const uint64_t n0 = t->start[(int64_t)rl * t->dim + d0 + dd];
      uint64_t qb = n0 + base, qn = n0;
      int j = 0, hB = -1;
      while (qb != qn) {  // digits where B's prefix still differs from n0's
        uint64_t nb = div_base64(qb, h), nq = div_base64(qn, h);
        uint32_t db = (uint32_t)(qb - nb * p), dn = (uint32_t)(qn - nq * p);
        R.bd[dd][j] = (uint16_t)db;
        hB = db != dn ? j : hB;
        qb = nb;
        qn = nq;
        j++;
      }
      for (; j < h.cap; j++) R.bd[dd][j] = n0d[j];
      int N = TILE, J = 0;
      R.nn[dd][0] = (int16_t)N;
      while (N > 1) {
        N = (int)div_base((uint32_t)R.bd[dd][J] + (uint32_t)N - 1u, h) + 1;
        J++;
        R.nn[dd][J] = (int16_t)N;
      }
      double S = ini[hB + 1 > J ? hB + 1 : J];
      for (int k = hB; k >= J; k--) S = dadd(S, dmul(u16d(sg[R.bd[dd][k]]), w[k]));
      R.J[dd] = J;
      R.hB[dd] = hB;
      R.sJ[dd] = S;
    }
    __syncthreads();
    // ---- warp-cooperative descent of the digit tree, one dim at a time
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int dd = warp; dd < Dc; dd += WARPS) {
      const HaltonDim &h = c_hdim[d0 + dd];
      const uint32_t p = (uint32_t)h.base;
      const uint16_t *sg = gsig + h.sig_off;
      const double *ini = gsum + h.sum_off;
      const double *w = g_wts + h.sum_off;
      const int J = R.J[dd], hB = R.hB[dd];
      double *prev = R.lev[warp][0], *next = R.lev[warp][1];
      if (lane == 0) prev[0] = R.sJ[dd];
      __syncwarp();
      for (int j = J - 1; j >= 0; j--) {
        const int Nj = R.nn[dd][j];
        const uint32_t bj = R.bd[dd][j];
        const double wj = w[j], inij = ini[j];
        const bool at_n0 = j > hB;  // node 0 of this level has n0's prefix
        double *dst = j ? next : zt + dd * TILE;
        for (int k = lane; k < Nj; k += 32) {
          const uint32_t x = bj + (uint32_t)k;
          const uint32_t par = div_base(x, h);
          const uint32_t a = x - par * p;
          double v = dadd(prev[par], dmul(u16d(sg[a]), wj));
          dst[k] = (at_n0 && k == 0) ? inij : v;
        }
        __syncwarp();
        double *tmp = prev;
        prev = next;
        next = tmp;
      }
      if (J == 0 && lane == 0) zt[dd * TILE] = R.sJ[dd];  // unreachable: TILE > 1
    }
    __syncthreads();
  }
};

// Rasrap counter form (Alg. 3, halton.py:419-440): sum sigma(a_j)*scale_j
// from the least significant digit up, scale_j = (1/p)^(j+1) by repeated
// multiplication, over max(K, #digits) positions.
struct GenRasrapCounter {
  const uint16_t *sig, *dig;
  uint32_t i;
  __device__ void begin(const RepTables &t, int rl, uint64_t, uint64_t path, GenShared &,
                        uint16_t *, int) {
    sig = t.sigma + (int64_t)rl * t.sig_stride;
    dig = t.digits + (int64_t)rl * t.dig_stride;
    i = (uint32_t)path;
  }
  __device__ __forceinline__ double value(int d) const {
    const HaltonDim &h = c_hdim[d];
    const uint16_t *d0 = dig + h.dig_off;
    const uint16_t *sg = sig + h.sig_off;
    const double *cs = g_cscale + h.sum_off;
    uint32_t t = i, carry = 0;
    double x = 0.0;
    for (int j = 0; j < h.K || t != 0u || carry != 0u; j++) {
      uint32_t q = div_base(t, h);
      uint32_t a = d0[j] + (t - q * (uint32_t)h.base) + carry;
      carry = a >= (uint32_t)h.base;
      a = carry ? a - (uint32_t)h.base : a;
      x = dadd(x, dmul(u16d(sg[a]), cs[j]));
      t = q;
    }
    return x;
  }
  __device__ void fill(int d0, int Dc, double *zt) {
    for (int dd = 0; dd < Dc; dd++) zt[dd * TILE + threadIdx.x] = value(d0 + dd);
  }
};

// Philox-4x32-10, counter (b, path_lo, path_hi, 0), u = (w + 1/2) 2^-32
// (prng.py:180-231, harness.py:53-67).
struct GenPhilox {
  uint32_t k0, k1, plo, phi;
  __device__ void begin(const RepTables &t, int rl, uint64_t, uint64_t path, GenShared &,
                        uint16_t *, int) {
    uint64_t key = derive_key3(t.seed, 3, (uint64_t)(t.rep_first + rl));
    k0 = (uint32_t)key;
    k1 = (uint32_t)(key >> 32);
    plo = (uint32_t)path;
    phi = (uint32_t)(path >> 32);
  }
  __device__ void fill(int d0, int Dc, double *zt) {  // d0 % 4 == 0
    double *zcol = zt + threadIdx.x;
    for (int dd = 0; dd < Dc; dd += 4) {
      U4 w = philox4x32_10((uint32_t)((d0 + dd) >> 2), plo, phi, 0u, k0, k1);
      const double s = 2.3283064365386963e-10, hlf = 1.1641532182693481e-10;
      zcol[dd * TILE] = (double)w.x * s + hlf;
      if (dd + 1 < Dc) zcol[(dd + 1) * TILE] = (double)w.y * s + hlf;
      if (dd + 2 < Dc) zcol[(dd + 2) * TILE] = (double)w.z * s + hlf;
      if (dd + 3 < Dc) zcol[(dd + 3) * TILE] = (double)w.w * s + hlf;
    }
  }
};

// Scrambled Sobol' (sobol.py:313-372): point at index j is the XOR of the
// pre-scrambled direction words over the set bits of j, XOR the shift;
// the Gray-code sampler's point i is the counter point at i ^ (i >> 1).
template <bool GRAY>
struct GenSobolDirect {
  const uint32_t *v, *shift;
  uint64_t idx;
  __device__ void begin(const RepTables &t, int rl, uint64_t, uint64_t path, GenShared &,
                        uint16_t *, int) {
    v = t.sobol_v + (int64_t)rl * t.dim * SOBOL_BITS;
    shift = t.sobol_shift + (int64_t)rl * t.dim;
    idx = GRAY ? (path ^ (path >> 1)) : path;
  }
  __device__ void fill(int d0, int Dc, double *zt) {
    double *zcol = zt + threadIdx.x;
    for (int dd = 0; dd < Dc; dd++) {
      const uint32_t *vd = v + (d0 + dd) * SOBOL_BITS;
      uint32_t x = __ldg(shift + d0 + dd);
      uint32_t bits = (uint32_t)idx;
      while (bits) {
        int k = __ffs(bits) - 1;
        x ^= __ldg(vd + k);
        bits &= bits - 1u;
      }
      zcol[dd * TILE] = (double)x * 2.3283064365386963e-10;
    }
  }
};

// Tiled Sobol': the index bits >= 7 are shared by a 128-aligned tile, so
// prepare() folds them (and the shift) into one word per dim and tabulates
// the 128 low-bit XOR patterns; a point is then one table lookup.  Tiles
// that are not 128-aligned (sampler.fill from an odd start) take the
// direct loop.
template <bool GRAY>
struct GenSobolTile {
  const uint32_t *v, *shift;
  uint32_t idx, hi_key;
  bool aligned;
  GenShared *sh;
  __device__ void begin(const RepTables &t, int rl, uint64_t base, uint64_t path, GenShared &s,
                        uint16_t *, int) {
    v = t.sobol_v + (int64_t)rl * t.dim * SOBOL_BITS;
    shift = t.sobol_shift + (int64_t)rl * t.dim;
    uint32_t i = (uint32_t)path, b = (uint32_t)base;
    idx = GRAY ? (i ^ (i >> 1)) : i;
    uint32_t bidx = GRAY ? (b ^ (b >> 1)) : b;
    hi_key = bidx >> 7;
    aligned = (b & 127u) == 0u;
    sh = &s;
  }
  __device__ void prepare(int d0, int Dc) {
    SobolTileShared &S = sh->s;
    __syncthreads();
    if (aligned) {
      for (int e = threadIdx.x; e < Dc * 128; e += TILE) {
        int dd = e >> 7, x = e & 127;
        const uint32_t *vd = v + (d0 + dd) * SOBOL_BITS;
        uint32_t acc = 0;
        for (int k = 0; k < 7; k++)
          if (x & (1 << k)) acc ^= vd[k];
        S.lowtab[dd][x] = acc;
      }
      if (threadIdx.x < Dc) {
        const uint32_t *vd = v + (d0 + threadIdx.x) * SOBOL_BITS;
        uint32_t acc = shift[d0 + threadIdx.x], bits = hi_key;
        for (int k = 7; bits; k++, bits >>= 1)
          if (bits & 1u) acc ^= vd[k];
        S.xhi[threadIdx.x] = acc;
      }
    }
    __syncthreads();
  }
  __device__ void fill(int d0, int Dc, double *zt) {
    prepare(d0, Dc);
    double *zcol = zt + threadIdx.x;
    const SobolTileShared &S = sh->s;
    for (int dd = 0; dd < Dc; dd++) {
      uint32_t x;
      if (aligned) {
        x = S.xhi[dd] ^ S.lowtab[dd][idx & 127u];
      } else {
        const uint32_t *vd = v + (d0 + dd) * SOBOL_BITS;
        x = shift[d0 + dd];
        for (uint32_t bits = idx; bits; bits &= bits - 1u) x ^= vd[__ffs(bits) - 1];
      }
      zcol[dd * TILE] = (double)x * 2.3283064365386963e-10;
    }
  }
};

// SFC64 per-path stream (no reference counterpart; numpy SFC64 core):
// state from derive_words(derive_key(seed, 7, m, path), 6), 12 warm-up
// draws, u = (w >> 11) 2^-53 as numpy Generator.random().
struct GenSfc64 {
  Sfc64 s;
  __device__ void begin(const RepTables &t, int rl, uint64_t, uint64_t path, GenShared &,
                        uint16_t *, int) {
    uint64_t km = derive_key3(t.seed, 7, (uint64_t)(t.rep_first + rl));
    sfc_seed(s, splitmix64(km ^ path));
  }
  __device__ void fill(int d0, int Dc, double *zt) {
    for (int dd = 0; dd < Dc; dd++)
      zt[dd * TILE + threadIdx.x] = (double)(sfc_next(s) >> 11) * (1.0 / 9007199254740992.0);
  }
};

// ======================================================================
// Warp-cooperative inverse normal over a chunk (tail compaction)
// ======================================================================
__device__ __forceinline__ void chunk_to_normals(double *zt, int Dc, uint16_t *q) {
  const int lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  int qn = 0;
  for (int dd = 0; dd < Dc; dd++) {
    const int slot = dd * TILE + threadIdx.x;
    bool neg;
    double pl = invn_fold(zt[slot], &neg);
    bool tail = pl < InvNormal::PLOW;
    unsigned b = __ballot_sync(0xffffffffu, tail);
    if (tail) {
      q[qn + __popc(b & lt)] = (uint16_t)slot;
    } else {
      double x = invn_central(pl);
      zt[slot] = neg ? -x : x;
    }
    qn += __popc(b);
  }
  __syncwarp();
  for (int k = lane; k < qn; k += 32) {
    int slot = q[k];
    bool neg;
    double pl = invn_fold(zt[slot], &neg);
    double x = invn_tail(pl);
    zt[slot] = neg ? -x : x;
  }
  __syncwarp();
}

// ======================================================================
// Models (phase 2): thread-per-path state in registers
// ======================================================================

// LIBOR market-model caplet, one-factor Euler (models.py:271-293).  S static:
// forward rates live in registers; for S <= CHUNK the whole triangle is
// unrolled, above that the step loop is dynamic and the alive-rate loop is
// unrolled with uniform guards.  Division by (1 + delta L) uses a MUFU seed
// plus one Newton step in the drift (its weight in the path is ~1e-4, so
// the ~2^-44 relative error is far below the 1e-12 parity bar) and two
// steps everywhere else.
template <int S>
struct ModelLibor {
  static constexpr bool NORMALS = true;
  static constexpr int DIM = S;
  double L[S];
  double delta, s2d, ssq, g0;
  __device__ void begin(const ModelParams &mp, const double *l0s) {
#pragma unroll
    for (int n = 0; n < S; n++) L[n] = l0s[n];
    delta = mp.delta;
    s2d = mp.sigma * mp.sigma * mp.delta;
    ssq = mp.sigma * sqrt(mp.delta);
  }
  __device__ __forceinline__ void step(int i, double z) {
    const double g1 = 1.0 + ssq * z;
    double drift = 0.0;
#pragma unroll
    for (int n = 0; n < S; n++) {
      if (n >= i) {
        double r = rcp1(fma(delta, L[n], 1.0));
        drift = fma(s2d * L[n], r, drift);
        L[n] *= fma(drift, delta, g1);
      }
    }
  }
  __device__ void chunk(int d0, int Dc, const double *zcol, int stride) {
    if (S <= CHUNK) {
#pragma unroll
      for (int i = 0; i < S; i++) step(i, zcol[i * stride]);
    } else {
      for (int k = 0; k < Dc; k++) step(d0 + k, zcol[k * stride]);
    }
  }
  __device__ double payoff(const ModelParams &mp) const {
    // disc = front_factor / prod_{i<S-1} (1 + delta L_i(T_i)); L_i is frozen
    // after step i, so its final value is the fixing (models.py:289-290).
    double disc = mp.front_factor;
#pragma unroll
    for (int n = 0; n < S - 1; n++) disc *= rcp2(fma(delta, L[n], 1.0));
    double lt = L[S - 1];
    double pay = delta * fmax(lt - mp.strike, 0.0) * rcp2(fma(delta, lt, 1.0));
    return pay * disc;
  }
};

// MBS present value (models.py:430-449), 360 monthly steps.
struct ModelMbs {
  static constexpr bool NORMALS = true;
  double disc, rem, rate, prev_w, pv;
  const double *ck;
  __device__ void begin(const ModelParams &mp, const double *cks) {
    disc = 1.0;
    rem = 1.0;
    rate = mp.i0;
    prev_w = 0.0;
    pv = 0.0;
    ck = cks;
  }
  __device__ void chunk(int d0, int Dc, const double *zcol, int stride, const ModelParams &mp) {
    for (int kk = 0; kk < Dc; kk++) {
      const int k = d0 + kk;  // month k+1
      disc *= rcp2(1.0 + rate);
      if (k > 0) rem *= 1.0 - prev_w;
      double xi = mp.sigma_xi * zcol[kk * stride];
      rate = mp.k0 * exp(xi) * rate;
      double w = fma(mp.k2, atan(fma(mp.k3, rate, mp.k4)), mp.k1);
      pv = fma(disc * mp.payment * rem, fma(w, ck[k], 1.0 - w), pv);
      prev_w = w;
    }
  }
};

// ======================================================================
// Fused path kernel
// ======================================================================
struct PathArgs {
  RepTables t;
  ModelParams mp;
  int rep_local0, rep_n;
  int64_t nmax;
  int64_t tiles_per_rep;
  double *payoffs;  // [rep_n][nmax]
  int sig_cap;      // u16 sigma entries staged per chunk (0: read from global)
};

// dynamic shared memory: [model table doubles][staged sigma u16]
__device__ __forceinline__ uint16_t *dyn_sig(void *dyn, int table_doubles) {
  return reinterpret_cast<uint16_t *>(reinterpret_cast<double *>(dyn) + table_doubles);
}

template <class G, int S>
__global__ void __launch_bounds__(TILE) k_paths_libor(PathArgs a) {
  __shared__ double zt[CHUNK * TILE];
  __shared__ uint16_t tq[WARPS][CHUNK * 32];
  __shared__ GenShared gsh;
  __shared__ double l0s[S];
  extern __shared__ double dyn[];
  uint16_t *sig_dyn = dyn_sig(dyn, 0);
  for (int n = threadIdx.x; n < S; n += TILE) l0s[n] = a.mp.table[n];
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int64_t total = (int64_t)a.rep_n * a.tiles_per_rep;
  for (int64_t w = blockIdx.x; w < total; w += gridDim.x) {
    const int rl = a.rep_local0 + (int)(w / a.tiles_per_rep);
    const int64_t base = (w % a.tiles_per_rep) * TILE;
    const int64_t path = base + threadIdx.x;
    G g;
    g.begin(a.t, rl, (uint64_t)base, (uint64_t)path, gsh, sig_dyn, a.sig_cap);
    ModelLibor<S> md;
    md.begin(a.mp, l0s);
    for (int d0 = 0; d0 < S; d0 += CHUNK) {
      const int Dc = S - d0 < CHUNK ? S - d0 : CHUNK;
      g.fill(d0, Dc, zt);
      __syncwarp();
      chunk_to_normals(zt, Dc, tq[warp]);
      md.chunk(d0, Dc, zt + threadIdx.x, TILE);
      __syncwarp();
    }
    if (path < a.nmax)
      a.payoffs[(int64_t)(rl - a.rep_local0) * a.nmax + path] = md.payoff(a.mp);
  }
}

template <class G>
__global__ void __launch_bounds__(TILE) k_paths_mbs(PathArgs a) {
  __shared__ double zt[CHUNK * TILE];
  __shared__ uint16_t tq[WARPS][CHUNK * 32];
  __shared__ GenShared gsh;
  extern __shared__ double dyn[];
  double *cks = dyn;
  uint16_t *sig_dyn = dyn_sig(dyn, a.mp.dim);
  for (int n = threadIdx.x; n < a.mp.dim; n += TILE) cks[n] = a.mp.table[n];
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  const int64_t total = (int64_t)a.rep_n * a.tiles_per_rep;
  for (int64_t w = blockIdx.x; w < total; w += gridDim.x) {
    const int rl = a.rep_local0 + (int)(w / a.tiles_per_rep);
    const int64_t base = (w % a.tiles_per_rep) * TILE;
    const int64_t path = base + threadIdx.x;
    G g;
    g.begin(a.t, rl, (uint64_t)base, (uint64_t)path, gsh, sig_dyn, a.sig_cap);
    ModelMbs md;
    md.begin(a.mp, cks);
    for (int d0 = 0; d0 < a.mp.dim; d0 += CHUNK) {
      const int Dc = a.mp.dim - d0 < CHUNK ? a.mp.dim - d0 : CHUNK;
      g.fill(d0, Dc, zt);
      __syncwarp();
      chunk_to_normals(zt, Dc, tq[warp]);
      md.chunk(d0, Dc, zt + threadIdx.x, TILE, a.mp);
      __syncwarp();
    }
    if (path < a.nmax) a.payoffs[(int64_t)(rl - a.rep_local0) * a.nmax + path] = md.pv;
  }
}

// f = x_1 (FirstCoordinateModel, models.py:489-498) and f = 1 (ConstantModel).
template <class G, bool CONST1>
__global__ void __launch_bounds__(TILE) k_paths_test(PathArgs a) {
  __shared__ double zt[TILE];
  __shared__ GenShared gsh;
  extern __shared__ double dyn[];
  uint16_t *sig_dyn = dyn_sig(dyn, 0);
  const int64_t total = (int64_t)a.rep_n * a.tiles_per_rep;
  for (int64_t w = blockIdx.x; w < total; w += gridDim.x) {
    const int rl = a.rep_local0 + (int)(w / a.tiles_per_rep);
    const int64_t base = (w % a.tiles_per_rep) * TILE;
    const int64_t path = base + threadIdx.x;
    double f = 1.0;
    if (!CONST1) {
      G g;
      g.begin(a.t, rl, (uint64_t)base, (uint64_t)path, gsh, sig_dyn, a.sig_cap);
      g.fill(0, 1, zt);
      f = zt[threadIdx.x];
    }
    if (path < a.nmax) a.payoffs[(int64_t)(rl - a.rep_local0) * a.nmax + path] = f;
  }
}

// ======================================================================
// Point kernels (sampler.fill / sampler.at), out[count][dim] row-major.
// Consecutive rows use the tiled generators, explicit indices the direct.
// ======================================================================
template <class G>
__global__ void __launch_bounds__(TILE) k_points(RepTables t, int rl, int64_t first,
                                                 const int64_t *idx, int64_t count,
                                                 double *out, int sig_cap) {
  __shared__ double zt[CHUNK * TILE];
  __shared__ GenShared gsh;
  extern __shared__ double dyn[];
  uint16_t *sig_dyn = dyn_sig(dyn, 0);
  for (int64_t tb = (int64_t)blockIdx.x * TILE; tb < count; tb += (int64_t)gridDim.x * TILE) {
    const int64_t r = tb + threadIdx.x;
    const bool ok = r < count;
    const int64_t path = idx ? (ok ? idx[r] : 0) : first + r;
    G g;
    g.begin(t, rl, (uint64_t)(first + tb), (uint64_t)path, gsh, sig_dyn, sig_cap);
    for (int d0 = 0; d0 < t.dim; d0 += CHUNK) {
      const int Dc = t.dim - d0 < CHUNK ? t.dim - d0 : CHUNK;
      g.fill(d0, Dc, zt);
      if (ok)
        for (int dd = 0; dd < Dc; dd++) out[r * t.dim + d0 + dd] = zt[dd * TILE + threadIdx.x];
    }
  }
}

// ======================================================================
// Model payoffs from caller uniforms (model.payoffs(u), models.py:311-322,
// 462-469): thread per path, scalar inverse normal.
// ======================================================================
template <int S>
__global__ void k_libor_u(ModelParams mp, const double *u, int64_t npaths, double *out) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npaths) return;
  ModelLibor<S> md;
  md.begin(mp, mp.table);
  for (int i = 0; i < S; i++) md.step(i, inv_normal(u[p * S + i]));
  out[p] = md.payoff(mp);
}

__global__ void k_mbs_u(ModelParams mp, const double *u, int64_t npaths, double *out) {
  int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npaths) return;
  ModelMbs md;
  md.begin(mp, mp.table);
  double z[CHUNK];
  for (int d0 = 0; d0 < mp.dim; d0 += CHUNK) {
    int Dc = mp.dim - d0 < CHUNK ? mp.dim - d0 : CHUNK;
    for (int k = 0; k < Dc; k++) z[k] = inv_normal(u[p * mp.dim + d0 + k]);
    md.chunk(d0, Dc, z, 1, mp);
  }
  out[p] = md.pv;
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
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < plan.nleaves) val[k] = leaf_sum(a + plan.leaf_start[k], plan.leaf_len[k]);
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
// Stream throughput kernel (config 4): points [0, npoints) of dimension
// t.dim, fused inverse normal, consumed by a sum (and optionally stored).
// ======================================================================
template <class G>
__global__ void __launch_bounds__(TILE) k_stream(RepTables t, int rl, int64_t npoints,
                                                 double *block_sums, double *store, int sig_cap) {
  __shared__ double zt[CHUNK * TILE];
  __shared__ uint16_t tq[WARPS][CHUNK * 32];
  __shared__ GenShared gsh;
  __shared__ double red[WARPS];
  extern __shared__ double dyn[];
  uint16_t *sig_dyn = dyn_sig(dyn, 0);
  const int warp = threadIdx.x >> 5;
  double acc = 0.0;
  for (int64_t tb = (int64_t)blockIdx.x * TILE; tb < npoints; tb += (int64_t)gridDim.x * TILE) {
    const int64_t r = tb + threadIdx.x;
    const bool ok = r < npoints;
    G g;
    g.begin(t, rl, (uint64_t)tb, (uint64_t)r, gsh, sig_dyn, sig_cap);
    for (int d0 = 0; d0 < t.dim; d0 += CHUNK) {
      const int Dc = t.dim - d0 < CHUNK ? t.dim - d0 : CHUNK;
      g.fill(d0, Dc, zt);
      __syncwarp();
      chunk_to_normals(zt, Dc, tq[warp]);
      if (ok) {
        for (int dd = 0; dd < Dc; dd++) {
          double z = zt[dd * TILE + threadIdx.x];
          acc += z;
          if (store) store[r * t.dim + d0 + dd] = z;
        }
      }
      __syncwarp();
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

cudaError_t launch_dfma_peak(int blocks, int iters, double *sink, cudaStream_t s) {
  k_dfma_peak<<<blocks, 256, 0, s>>>(iters, 1.0, sink);
  return cudaGetLastError();
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

template <class K>
static int persistent_blocks(K kernel, size_t dyn_smem, int64_t work) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, TILE, dyn_smem);
  if (per_sm < 1) per_sm = 1;
  int64_t b = (int64_t)per_sm * sm_count();
  return (int)(work < b ? (work < 1 ? 1 : work) : b);
}

cudaError_t launch_rasrap_setup(const RepTables &t, uint16_t *sigma, uint16_t *digits,
                                double *sums, uint64_t *start, cudaStream_t s) {
  int64_t n = (int64_t)t.rep_count * t.dim;
  int blocks = (int)((n + 127) / 128);
  k_rasrap_setup<<<blocks, 128, 0, s>>>(t, sigma, digits, sums, start);
  return cudaGetLastError();
}

cudaError_t launch_sobol_setup(const RepTables &t, const uint32_t *v_dev, uint32_t *gen_v,
                               uint32_t *shift, cudaStream_t s) {
  int64_t n = (int64_t)t.rep_count * t.dim;
  int blocks = (int)((n + 127) / 128);
  k_sobol_setup<<<blocks, 128, 0, s>>>(t, v_dev, gen_v, shift);
  return cudaGetLastError();
}

// sigma tables are read from global (L1-resident); no staging
static int sig_cap_for(const RepTables &) { return 0; }
static size_t dyn_bytes(int table_doubles, int sig_cap) {
  return sizeof(double) * table_doubles + sizeof(uint16_t) * sig_cap;
}

template <class G>
static cudaError_t points_t(const RepTables &t, int rl, int64_t first, const int64_t *idx,
                            int64_t count, double *out, cudaStream_t s) {
  int64_t tiles = (count + TILE - 1) / TILE;
  int cap = idx ? 0 : sig_cap_for(t);
  size_t dyn = dyn_bytes(0, cap);
  int blocks = persistent_blocks(k_points<G>, dyn, tiles);
  k_points<G><<<blocks, TILE, dyn, s>>>(t, rl, first, idx, count, out, cap);
  return cudaGetLastError();
}

cudaError_t launch_points(const RepTables &t, int rl, int64_t first, const int64_t *idx,
                          int64_t count, double *out, cudaStream_t s) {
  const bool at = idx != nullptr;
  switch (t.gen) {
    case GEN_RASRAP_RECURSIVE:
      return at ? points_t<GenRasrapRecDirect>(t, rl, first, idx, count, out, s)
                : points_t<GenRasrapRecTile>(t, rl, first, idx, count, out, s);
    case GEN_RASRAP_COUNTER: return points_t<GenRasrapCounter>(t, rl, first, idx, count, out, s);
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

template <class G>
static cudaError_t paths_g(const PathArgs &a, int *launched, cudaStream_t s, bool probe,
                           int *blocks_out) {
  const int64_t work = (int64_t)a.rep_n * a.tiles_per_rep;
  int blocks = 0;
  switch (a.mp.kind) {
    case MODEL_LIBOR: {
      size_t dyn = dyn_bytes(0, a.sig_cap);
#define RQ_LIBOR_CASE(SS)                                              \
  case SS:                                                             \
    blocks = persistent_blocks(k_paths_libor<G, SS>, dyn, work);       \
    if (!probe) k_paths_libor<G, SS><<<blocks, TILE, dyn, s>>>(a);     \
    break;
      switch (a.mp.dim) {
        RQ_LIBOR_CASE(10)
        RQ_LIBOR_CASE(20)
        RQ_LIBOR_CASE(40)
        RQ_LIBOR_CASE(80)
        default: return cudaErrorInvalidValue;
      }
#undef RQ_LIBOR_CASE
      break;
    }
    case MODEL_MBS: {
      size_t dyn = dyn_bytes(a.mp.dim, a.sig_cap);
      blocks = persistent_blocks(k_paths_mbs<G>, dyn, work);
      if (!probe) k_paths_mbs<G><<<blocks, TILE, dyn, s>>>(a);
      break;
    }
    case MODEL_X1: {
      size_t dyn = dyn_bytes(0, a.sig_cap);
      blocks = persistent_blocks(k_paths_test<G, false>, dyn, work);
      if (!probe) k_paths_test<G, false><<<blocks, TILE, dyn, s>>>(a);
      break;
    }
    case MODEL_CONST1:
      blocks = persistent_blocks(k_paths_test<G, true>, 0, work);
      if (!probe) k_paths_test<G, true><<<blocks, TILE, 0, s>>>(a);
      break;
    default: return cudaErrorInvalidValue;
  }
  if (blocks_out) *blocks_out = blocks;
  if (launched && !probe) *launched += 1;
  return probe ? cudaSuccess : cudaGetLastError();
}

static cudaError_t paths_dispatch(const PathArgs &a, int *launched, cudaStream_t s, bool probe,
                                  int *blocks) {
  switch (a.t.gen) {
    case GEN_RASRAP_RECURSIVE: return paths_g<GenRasrapRecTile>(a, launched, s, probe, blocks);
    case GEN_RASRAP_COUNTER: return paths_g<GenRasrapCounter>(a, launched, s, probe, blocks);
    case GEN_PHILOX: return paths_g<GenPhilox>(a, launched, s, probe, blocks);
    case GEN_SOBOL_GRAY: return paths_g<GenSobolTile<true>>(a, launched, s, probe, blocks);
    case GEN_SOBOL_COUNTER: return paths_g<GenSobolTile<false>>(a, launched, s, probe, blocks);
    case GEN_SFC64: return paths_g<GenSfc64>(a, launched, s, probe, blocks);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_paths(const RepTables &t, const ModelParams &mp, int rep_local0, int rep_n,
                         int64_t nmax, double *payoffs, int *launched, cudaStream_t s) {
  PathArgs a;
  a.t = t;
  a.mp = mp;
  a.rep_local0 = rep_local0;
  a.rep_n = rep_n;
  a.nmax = nmax;
  a.tiles_per_rep = (nmax + TILE - 1) / TILE;
  a.payoffs = payoffs;
  a.sig_cap = sig_cap_for(t);
  return paths_dispatch(a, launched, s, false, nullptr);
}

int paths_grid_blocks(const RepTables &t, const ModelParams &mp) {
  PathArgs a{};
  a.t = t;
  a.mp = mp;
  a.rep_n = 1 << 20;
  a.tiles_per_rep = 1 << 20;
  a.sig_cap = sig_cap_for(t);
  int blocks = 0;
  paths_dispatch(a, nullptr, 0, true, &blocks);
  return blocks;
}

cudaError_t launch_reduce(const SumPlan &plan, const double *payoffs, int64_t pay_stride,
                          int reps, double *theta, int theta_stride, double *scratch,
                          unsigned *tickets, cudaStream_t s) {
  dim3 grid((plan.nleaves + 255) / 256, reps);
  k_reduce<<<grid, 256, 0, s>>>(plan, payoffs, pay_stride, theta, theta_stride, scratch,
                                tickets);
  return cudaGetLastError();
}

cudaError_t launch_model_payoffs(const ModelParams &mp, const double *u, int64_t npaths,
                                 double *out, cudaStream_t s) {
  int blocks = (int)((npaths + 127) / 128);
  if (blocks < 1) return cudaSuccess;
  if (mp.kind == MODEL_MBS) {
    k_mbs_u<<<blocks, 128, 0, s>>>(mp, u, npaths, out);
    return cudaGetLastError();
  }
  if (mp.kind != MODEL_LIBOR) return cudaErrorInvalidValue;
  switch (mp.dim) {
    case 10: k_libor_u<10><<<blocks, 128, 0, s>>>(mp, u, npaths, out); break;
    case 20: k_libor_u<20><<<blocks, 128, 0, s>>>(mp, u, npaths, out); break;
    case 40: k_libor_u<40><<<blocks, 128, 0, s>>>(mp, u, npaths, out); break;
    case 80: k_libor_u<80><<<blocks, 128, 0, s>>>(mp, u, npaths, out); break;
    default: return cudaErrorInvalidValue;
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
  int cap = sig_cap_for(t);
  k_stream<G><<<nblocks, TILE, dyn_bytes(0, cap), s>>>(t, rl, npoints, sums, store, cap);
  return cudaGetLastError();
}

cudaError_t launch_stream_normals(const RepTables &t, int rl, int64_t npoints,
                                  double *block_sums, int nblocks, double *store,
                                  cudaStream_t s) {
  switch (t.gen) {
    case GEN_RASRAP_RECURSIVE: return stream_t<GenRasrapRecTile>(t, rl, npoints, block_sums, nblocks, store, s);
    case GEN_RASRAP_COUNTER: return stream_t<GenRasrapCounter>(t, rl, npoints, block_sums, nblocks, store, s);
    case GEN_PHILOX: return stream_t<GenPhilox>(t, rl, npoints, block_sums, nblocks, store, s);
    case GEN_SOBOL_GRAY: return stream_t<GenSobolTile<true>>(t, rl, npoints, block_sums, nblocks, store, s);
    case GEN_SOBOL_COUNTER: return stream_t<GenSobolTile<false>>(t, rl, npoints, block_sums, nblocks, store, s);
    case GEN_SFC64: return stream_t<GenSfc64>(t, rl, npoints, block_sums, nblocks, store, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace rq
