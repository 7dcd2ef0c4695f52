// rq_device.cuh -- host/device building blocks of the B200 RQMC path.
//
// Everything here is compiled both for sm_100a (kernels) and for the host
// (table builders in rq_capi.cu), so the device and host table paths share
// one definition.  Bit-exact pieces (Halton chains) use __dadd_rn /
// __dmul_rn explicitly so nvcc can never contract them into FMAs.
#pragma once
#include <cstdint>
#include <cmath>

#if defined(__CUDACC__)
#define RQ_HD __host__ __device__ __forceinline__
#else
#define RQ_HD inline
#endif

namespace rq {

// ---------------------------------------------------------------- integers
RQ_HD uint64_t umulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}
RQ_HD uint32_t umulhi32(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

// Exact IEEE binary64 ops that are never fused (host: -ffp-contract=off TU).
RQ_HD double dadd(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
RQ_HD double dmul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}

// ---------------------------------------------------------------- seeding
// splitmix64 finaliser with the golden-ratio pre-add (seeding.py:27-32).
RQ_HD uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
// derive_key(a, b, ...) absorbs parts left to right from h = 0 (seeding.py:35-44).
RQ_HD uint64_t derive_key2(uint64_t a, uint64_t b) { return splitmix64(splitmix64(a) ^ b); }
RQ_HD uint64_t derive_key3(uint64_t a, uint64_t b, uint64_t c) {
  return splitmix64(derive_key2(a, b) ^ c);
}
RQ_HD uint64_t derive_key4(uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  return splitmix64(derive_key3(a, b, c) ^ d);
}

// ---------------------------------------------------------------- numpy PCG64
// numpy.random.PCG64(SeedSequence(key)): the generator behind derive_rng
// (seeding.py:59-65).  State/increment as (hi, lo) 64-bit halves.
struct Pcg64 {
  uint64_t sh, sl, ih, il;
  uint32_t spare;
  int has_spare;
};

RQ_HD void pcg_step(Pcg64 &g) {
  const uint64_t MH = 0x2360ED051FC65DA4ULL, ML = 0x4385DF649FCCF645ULL;
  uint64_t lo = g.sl * ML;
  uint64_t hi = umulhi64(g.sl, ML) + g.sl * MH + g.sh * ML;
  uint64_t nl = lo + g.il;
  hi += g.ih + (nl < lo ? 1u : 0u);
  g.sl = nl;
  g.sh = hi;
}

RQ_HD void pcg_seed(Pcg64 &g, uint64_t key) {
  // SeedSequence pool mixing (numpy bit_generator.pyx mix_entropy, pool 4).
  const uint32_t MULT_A = 0x931e8875u, MULT_B = 0x58f38dedu;
  const uint32_t ML = 0xca01f9ddu, MR = 0x4973f715u;
  uint32_t ent0 = (uint32_t)key, ent1 = (uint32_t)(key >> 32);
  int nent = (key >> 32) ? 2 : 1;
  uint32_t hc = 0x43b0d7e5u;
  uint32_t pool[4];
#define RQ_HASHMIX(val, out)  \
  {                           \
    uint32_t v_ = (val) ^ hc; \
    hc *= MULT_A;             \
    v_ *= hc;                 \
    out = v_ ^ (v_ >> 16);    \
  }
  for (int i = 0; i < 4; i++) {
    uint32_t e = (i == 0) ? ent0 : ((i == 1 && nent == 2) ? ent1 : 0u);
    RQ_HASHMIX(e, pool[i]);
  }
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) {
        uint32_t h;
        RQ_HASHMIX(pool[s], h);
        uint32_t r = ML * pool[d] - MR * h;
        pool[d] = r ^ (r >> 16);
      }
#undef RQ_HASHMIX
  uint32_t w[8];
  uint32_t hb = 0x8b51f9ddu;
  for (int i = 0; i < 8; i++) {
    uint32_t v = pool[i & 3] ^ hb;
    hb *= MULT_B;
    v *= hb;
    w[i] = v ^ (v >> 16);
  }
  uint64_t s0 = (uint64_t)w[0] | ((uint64_t)w[1] << 32);  // initstate hi
  uint64_t s1 = (uint64_t)w[2] | ((uint64_t)w[3] << 32);  // initstate lo
  uint64_t q0 = (uint64_t)w[4] | ((uint64_t)w[5] << 32);  // initseq hi
  uint64_t q1 = (uint64_t)w[6] | ((uint64_t)w[7] << 32);  // initseq lo
  g.ih = (q0 << 1) | (q1 >> 63);
  g.il = (q1 << 1) | 1u;
  g.sh = 0;
  g.sl = 0;
  pcg_step(g);
  uint64_t nl = g.sl + s1;
  g.sh = g.sh + s0 + (nl < s1 ? 1u : 0u);
  g.sl = nl;
  pcg_step(g);
  g.has_spare = 0;
  g.spare = 0;
}

RQ_HD uint64_t pcg_next64(Pcg64 &g) {
  pcg_step(g);
  uint64_t x = g.sh ^ g.sl;
  unsigned rot = (unsigned)(g.sh >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}
RQ_HD uint32_t pcg_next32(Pcg64 &g) {
  if (g.has_spare) {
    g.has_spare = 0;
    return g.spare;
  }
  uint64_t n = pcg_next64(g);
  g.has_spare = 1;
  g.spare = (uint32_t)(n >> 32);
  return (uint32_t)n;
}
// Generator.random(): 53 high bits
RQ_HD double pcg_random(Pcg64 &g) {
  return (double)(pcg_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}
// numpy random_interval(max) for max < 2^32: masked rejection on u32 halves.
RQ_HD uint32_t pcg_interval32(Pcg64 &g, uint32_t max) {
  if (max == 0) return 0;
  uint32_t mask = max;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  uint32_t v;
  do {
    v = pcg_next32(g) & mask;
  } while (v > max);
  return v;
}

// ---------------------------------------------------------------- Philox-4x32-10
// Counter (b, path_lo, path_hi, 0), key (k_lo, k_hi) (prng.py:180-212).
struct U4 {
  uint32_t x, y, z, w;
};
RQ_HD U4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                       uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; r++) {
    uint32_t hi0 = umulhi32(c0, 0xD2511F53u), lo0 = c0 * 0xD2511F53u;
    uint32_t hi1 = umulhi32(c2, 0xCD9E8D57u), lo1 = c2 * 0xCD9E8D57u;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  return U4{c0, c1, c2, c3};
}

// ---------------------------------------------------------------- SFC64
// numpy SFC64 core; per-path stream seeded from
// derive_words(derive_key(seed, 7, m, path), 6) + 12 discarded draws.
struct Sfc64 {
  uint64_t a, b, c, w;
};
RQ_HD uint64_t sfc_next(Sfc64 &s) {
  uint64_t tmp = s.a + s.b + s.w++;
  s.a = s.b ^ (s.b >> 11);
  s.b = s.c + (s.c << 3);
  s.c = ((s.c << 24) | (s.c >> 40)) + tmp;
  return tmp;
}
RQ_HD void sfc_seed(Sfc64 &s, uint64_t path_key) {
  // derive_words(key, 6) = low/high halves of 3 splitmix outputs
  uint64_t z1 = splitmix64(path_key), z2 = splitmix64(z1), z3 = splitmix64(z2);
  s.a = z1;
  s.b = z2;
  s.c = z3;
  s.w = 1;
  for (int i = 0; i < 12; i++) sfc_next(s);
}

// ---------------------------------------------------------------- division helpers
// Fast reciprocal: MUFU.RCP64H seed (~2^-20) + Newton.  One step leaves ~2^-40
// relative error, two steps ~1 ulp.
#if defined(__CUDACC__)
__device__ __forceinline__ double rcp_seed(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ double rcp1(double x) {
  double r = rcp_seed(x);
  double e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
// n / d by two residual corrections of the MUFU seed r0 (~2^-20):
// y1 = y0 + r0 (n - d y0) has relative error ~eps^2 ~ 1e-12, y2 ~eps^3.
__device__ __forceinline__ double div2(double n, double d) {
  const double r0 = rcp_seed(d), y0 = n * r0;
  const double y1 = fma(r0, fma(-d, y0, n), y0);
  return fma(r0, fma(-d, y1, n), y1);
}
__device__ __forceinline__ double rcp2(double x) {
  double r = rcp_seed(x);
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
#endif

// ---------------------------------------------------------------- inverse normal
// Coefficients of the reference's two-branch rational Phi^-1
// (models.py:23-64): central in u = (p - 1/2)^2 / R for p >= 0.0465, tail in
// w = (sqrt(-2 ln p) - V_LO) * V_SCALE; inputs clamped to >= 2^-53.
struct InvNormal {
  static constexpr double TINY = 1.1102230246251565e-16;
  static constexpr double PLOW = 0.0465;
  static constexpr double RMAX = 0.20566225000000002;
  static constexpr double VLO = 2.4772173769731336;
  static constexpr double VSCALE = 0.16408352781008756;
};

#if defined(__CUDACC__)
// Fold p into the lower half: returns pl, sets *neg for p > 1/2.
__device__ __forceinline__ double invn_fold(double p, bool *neg) {
  *neg = p > 0.5;
  double pl = *neg ? 1.0 - p : p;
  return pl < InvNormal::TINY ? InvNormal::TINY : pl;
}
// Tail test straight on the bit pattern of p in [0, 1): the reference takes
// the tail when fold(p) < PLOW (models.py:41-45), i.e. p < PLOW or
// 1 - p < PLOW; 1 - p is exact for p > 1/2, so the second is p > HI with
// HI = the largest double <= 1 - PLOW (real).  One unsigned range check.
constexpr uint64_t INVN_PLOW_BITS = 0x3fa7ced916872b02ULL;  // 0.0465
constexpr uint64_t INVN_HI_BITS = 0x3fee83126e978d4fULL;    // floor_double(1 - 0.0465)
__device__ __forceinline__ bool invn_tail_p(double p) {
  return (uint64_t)__double_as_longlong(p) - INVN_PLOW_BITS > INVN_HI_BITS - INVN_PLOW_BITS;
}
// The same test on the high word alone (two integer ops instead of a 64-bit
// range check): exact except for p sharing the high word of PLOW or HI,
// which it reports as tail CANDIDATES -- the tail queue re-tests them with
// invn_tail_p (inv_normal below), so the branch taken is the reference's.
constexpr uint32_t INVN_C_LO = (uint32_t)(INVN_PLOW_BITS >> 32) + 1u;  // first all-central high word
constexpr uint32_t INVN_C_HI = (uint32_t)(INVN_HI_BITS >> 32) - 1u;    // last all-central high word
__device__ __forceinline__ bool invn_tail_cand(double p) {
  return (uint32_t)__double2hiint(p) - INVN_C_LO > INVN_C_HI - INVN_C_LO;
}
// Central branch on Q = p - 1/2 without folding.  For p > 1/2 the
// reference computes q = (1 - p) - 1/2 = 1/2 - p exactly (Sterbenz) and
// returns -(q R(q^2)) = Q R(Q^2); for p <= 1/2, Q is the reference's own
// q = fl(p - 1/2).  R is the reference rational in u = q^2 / R_MAX
// (models.py:46-54) with the 1/R_MAX^k folded into the coefficients, so the
// polynomials run directly in Q^2.
// The coefficients live in the constant bank so every DFMA takes them as a
// c[][] operand; as immediates ptxas materialises each double with two UMOVs
// per use, which costs issue slots in the hot loops.
__constant__ double c_invn_num[8] = {-18758.264827117993, 121493.75753172635, -169742.25554056765,
                                     95028.92000917176,   -24309.66331940731, 2693.622228066229,
                                     -105.1488511356405,  3.8841077977297096};
__constant__ double c_invn_den[8] = {-27571.106587154845, 92106.19422816113, -98233.8844955836,
                                     46868.23917353603,   -10776.85973982955, 1116.658786813825,
                                     -43.57099147618938,  1.5495348220676615};
__device__ __forceinline__ double invn_central_q(double Q) {
  const double s = Q * Q;
  double num = c_invn_num[0], den = c_invn_den[0];
#pragma unroll
  for (int k = 1; k < 8; k++) {
    num = fma(num, s, c_invn_num[k]);
    den = fma(den, s, c_invn_den[k]);
  }
  return div2(Q * num, den);
}
__device__ __forceinline__ double invn_central(double pl) { return invn_central_q(pl - 0.5); }
__constant__ double c_invn_tnum[8] = {49.41588603624166,  34.09554370467819,  -120.62391569766385,
                                      -36.11819081101896, 77.35661807857605,  12.678668433221901,
                                      -15.636790505919562, -3.141967925161121};
__constant__ double c_invn_tden[8] = {-0.0005317355830972598, -8.101041244986659, -2.3666362350675305,
                                      19.91298298968798,       -1.4094956335739925, -10.941521790794202,
                                      1.2762506234112334,      1.8704632131064214};
// ln(pl) for the tail's pl in [2^-53, 0.0465] (normal doubles): pl = m 2^e
// with m in [sqrt(1/2), sqrt(2)), ln m = 2 atanh(s), s = (m - 1)/(m + 1),
// |s| <= 0.1716, odd series to s^21 (truncation < 1e-17 absolute), and
// e ln2 split hi/lo (e * ln2_hi exact).  Absolute error ~1e-16 against
// |ln pl| >= 3.07: a few ulp, far inside the 2e-13 parity bar, at a third of
// the instructions of the general libdevice log.
__constant__ double c_log_ser[10] = {0.047619047619047616, 0.05263157894736842,
                                     0.058823529411764705, 0.06666666666666667,
                                     0.07692307692307693,  0.09090909090909091,
                                     0.1111111111111111,   0.14285714285714285,
                                     0.2,                  0.3333333333333333};
__device__ __forceinline__ double log_tail(double pl) {
  if (pl != pl) return pl;  // NaN in, NaN out (the reference's math.log)
  int hi = __double2hiint(pl);
  int e = (hi >> 20) - 1023;
  hi = (hi & 0x000FFFFF) | 0x3FF00000;  // m in [1, 2)
  if (hi >= 0x3FF6A09E) {                // m >= ~sqrt(2): use m / 2
    hi -= 0x00100000;
    e += 1;
  }
  const double m = __hiloint2double(hi, __double2loint(pl));
  const double f = m - 1.0;  // exact (Sterbenz)
  const double sv = div2(f, 2.0 + f), s2 = sv * sv;
  double p = c_log_ser[0];
#pragma unroll
  for (int k = 1; k < 10; k++) p = fma(p, s2, c_log_ser[k]);
  const double t = 2.0 * sv;
  const double lnm = fma(t * s2, p, t);
  const double de = (double)e;
  return fma(de, 0x1.62e42fee00000p-1, fma(de, 1.9082149292705877e-10, lnm));
}
__device__ __forceinline__ double invn_tail(double pl) {
  const double w = (sqrt(-2.0 * log_tail(pl)) - InvNormal::VLO) * InvNormal::VSCALE;
  double num = c_invn_tnum[0], den = c_invn_tden[0];
#pragma unroll
  for (int k = 1; k < 8; k++) {
    num = fma(num, w, c_invn_tnum[k]);
    den = fma(den, w, c_invn_tden[k]);
  }
  return num * rcp2(den);
}
// A queued tail candidate (invn_tail_cand): the tail, or -- for the rare p
// that only shares PLOW's / HI's high word -- the central branch, out of
// line so the tail loops keep their register budget.
static __device__ __noinline__ double invn_central_rare(double p) { return invn_central_q(p - 0.5); }
__device__ __forceinline__ double invn_queued(double p) {
  if (!invn_tail_p(p)) return invn_central_rare(p);
  bool neg;
  const double x = invn_tail(invn_fold(p, &neg));
  return neg ? -x : x;
}
// Scalar Phi^-1 (divergent tail); the tile filler uses a compacted tail.
__device__ __forceinline__ double inv_normal(double p) {
  if (!invn_tail_p(p)) return invn_central_q(p - 0.5);
  bool neg;
  double x = invn_tail(invn_fold(p, &neg));
  return neg ? -x : x;
}
#endif

}  // namespace rq
