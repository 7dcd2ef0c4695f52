/* rqmc_oracle.c -- CPU restatement of the reference RQMC hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see rqmc_oracle.h).  Compiled with
 * -ffp-contract=off so every a*b+c is two roundings, as in the numba
 * kernels of the reference.  Citations are to
 * /root/reference/pkg/src/rqmcbench/<file>:<line>.
 */
#include "rqmc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ */
/* seeding.py                                                          */
/* ------------------------------------------------------------------ */

/* seeding.py:27-32 */
uint64_t orc_splitmix64(uint64_t z) {
  z = z + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

/* seeding.py:35-44 */
uint64_t orc_derive_key(const uint64_t *parts, int nparts) {
  uint64_t h = 0;
  for (int i = 0; i < nparts; i++) h = orc_splitmix64(h ^ parts[i]);
  return h;
}

/* seeding.py:47-56 */
void orc_derive_words(uint64_t key, int count, uint32_t *out) {
  uint64_t z = key;
  int n = 0;
  while (n < count) {
    z = orc_splitmix64(z);
    out[n++] = (uint32_t)z;
    if (n < count) out[n++] = (uint32_t)(z >> 32);
  }
}

/* ------------------------------------------------------------------ */
/* numpy SeedSequence + PCG64 (numpy/random/bit_generator.pyx,          */
/* numpy/random/src/pcg64/pcg64.h, distributions.c random_interval,     */
/* _generator.pyx shuffle / random_bounded_uint32_fill)                 */
/* ------------------------------------------------------------------ */

#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

static uint32_t ss_hashmix(uint32_t v, uint32_t *hc) {
  v ^= *hc;
  *hc *= SS_MULT_A;
  v *= *hc;
  v ^= v >> 16;
  return v;
}
static uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  return r ^ (r >> 16);
}

/* SeedSequence(entropy=key).generate_state(4, uint64) */
static void seedseq_state4(uint64_t key, uint64_t out[4]) {
  uint32_t ent[2];
  int nent;
  ent[0] = (uint32_t)key;
  ent[1] = (uint32_t)(key >> 32);
  nent = (key >> 32) ? 2 : 1; /* _int_to_uint32_array */
  uint32_t pool[4];
  uint32_t hc = SS_INIT_A;
  for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < nent ? ent[i] : 0u, &hc);
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
  uint32_t w[8];
  uint32_t hb = SS_INIT_B;
  for (int i = 0; i < 8; i++) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= SS_MULT_B;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  for (int i = 0; i < 4; i++) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

static const u128 PCG_MULT = (((u128)0x2360ED051FC65DA4ULL) << 64) | 0x4385DF649FCCF645ULL;

static u128 pcg_get(uint64_t hi, uint64_t lo) { return (((u128)hi) << 64) | lo; }

void orc_pcg64_seed(orc_pcg64 *g, uint64_t key) {
  uint64_t v[4];
  seedseq_state4(key, v);
  u128 initstate = pcg_get(v[0], v[1]);
  u128 initseq = pcg_get(v[2], v[3]);
  u128 inc = (initseq << 1) | 1u;
  u128 st = 0;
  st = st * PCG_MULT + inc;
  st += initstate;
  st = st * PCG_MULT + inc;
  g->st_hi = (uint64_t)(st >> 64);
  g->st_lo = (uint64_t)st;
  g->inc_hi = (uint64_t)(inc >> 64);
  g->inc_lo = (uint64_t)inc;
  g->has_u32 = 0;
  g->u32 = 0;
}

uint64_t orc_pcg64_next64(orc_pcg64 *g) {
  u128 st = pcg_get(g->st_hi, g->st_lo);
  st = st * PCG_MULT + pcg_get(g->inc_hi, g->inc_lo);
  g->st_hi = (uint64_t)(st >> 64);
  g->st_lo = (uint64_t)st;
  uint64_t x = g->st_hi ^ g->st_lo;
  unsigned rot = (unsigned)(g->st_hi >> 58);
  return (x >> rot) | (x << ((64 - rot) & 63));
}

uint32_t orc_pcg64_next32(orc_pcg64 *g) {
  if (g->has_u32) {
    g->has_u32 = 0;
    return g->u32;
  }
  uint64_t n = orc_pcg64_next64(g);
  g->has_u32 = 1;
  g->u32 = (uint32_t)(n >> 32);
  return (uint32_t)n;
}

double orc_pcg64_random(orc_pcg64 *g) {
  return (double)(orc_pcg64_next64(g) >> 11) * (1.0 / 9007199254740992.0);
}

static uint64_t random_interval(orc_pcg64 *g, uint64_t max) {
  if (max == 0) return 0;
  uint64_t mask = max, v;
  mask |= mask >> 1;
  mask |= mask >> 2;
  mask |= mask >> 4;
  mask |= mask >> 8;
  mask |= mask >> 16;
  mask |= mask >> 32;
  if (max <= 0xffffffffULL) {
    while ((v = (orc_pcg64_next32(g) & mask)) > max) {
    }
  } else {
    while ((v = (orc_pcg64_next64(g) & mask)) > max) {
    }
  }
  return v;
}

/* Generator.permutation(n) = shuffle(arange(n)), Fisher-Yates from the top */
void orc_pcg64_permutation(orc_pcg64 *g, int64_t n, int64_t *out) {
  for (int64_t i = 0; i < n; i++) out[i] = i;
  for (int64_t i = n - 1; i >= 1; i--) {
    int64_t j = (int64_t)random_interval(g, (uint64_t)i);
    int64_t t = out[j];
    out[j] = out[i];
    out[i] = t;
  }
}

/* Generator.integers(0, 2**32, size=n, dtype=uint32): raw buffered u32 */
void orc_pcg64_u32_stream(uint64_t key, int n, uint32_t *out) {
  orc_pcg64 g;
  orc_pcg64_seed(&g, key);
  for (int i = 0; i < n; i++) out[i] = orc_pcg64_next32(&g);
}

/* ------------------------------------------------------------------ */
/* halton.py                                                           */
/* ------------------------------------------------------------------ */

/* halton.py:40-56 (plain trial division gives the same list) */
int orc_primes(int count, int64_t *out) {
  int n = 0;
  for (int64_t c = 2; n < count; c++) {
    int ok = 1;
    for (int k = 0; k < n && out[k] * out[k] <= c; k++)
      if (c % out[k] == 0) {
        ok = 0;
        break;
      }
    if (ok) out[n++] = c;
  }
  return n;
}

/* halton.py:59-66 */
int orc_digit_capacity(int64_t base) {
  int k = 1;
  u128 v = (u128)base;
  while (v < ((u128)1 << 32)) {
    v *= (u128)base;
    k++;
  }
  return k;
}

/* halton.py:139-155.  omega is a double in [0,1): omega = mant * 2^e
 * exactly; floor(omega * base^k) computed in 128-bit integers. */
uint64_t orc_invert_radical(double omega, int64_t base, int k) {
  int e;
  double fr = frexp(omega, &e); /* omega = fr * 2^e, fr in [0.5,1) */
  uint64_t mant = (uint64_t)ldexp(fr, 53);
  int shift = 53 - e; /* omega = mant / 2^shift */
  u128 pk = 1;
  for (int i = 0; i < k; i++) pk *= (u128)base;
  u128 scaled;
  if (omega == 0.0) {
    scaled = 0;
  } else if (shift >= 128) {
    scaled = 0;
  } else {
    /* mant < 2^53, pk < 2^32 * base: product < 2^97 for base < 2^12 */
    u128 prod = (u128)mant * pk;
    scaled = prod >> shift;
  }
  uint64_t n = 0;
  for (int i = 0; i < k; i++) {
    uint64_t d = (uint64_t)(scaled % (u128)base);
    scaled /= (u128)base;
    n = n * (uint64_t)base + d;
  }
  return n;
}

/* halton.py:345-360 (+ derive_rng seeding.py:59-65) */
int orc_rasrap_config(int dim, uint64_t key, int64_t *start, double *omega, int64_t *sigma,
                      int maxbase) {
  int64_t *bases = (int64_t *)malloc(sizeof(int64_t) * dim);
  orc_primes(dim, bases);
  int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)bases[dim - 1]);
  for (int i = 0; i < dim; i++) {
    uint64_t parts[2] = {key, (uint64_t)i};
    orc_pcg64 g;
    orc_pcg64_seed(&g, orc_derive_key(parts, 2));
    double w = orc_pcg64_random(&g);
    orc_pcg64_permutation(&g, bases[i], perm);
    if (omega) omega[i] = w;
    start[i] = (int64_t)orc_invert_radical(w, bases[i], orc_digit_capacity(bases[i]));
    if (sigma) {
      for (int a = 0; a < maxbase; a++) sigma[(int64_t)i * maxbase + a] = 0;
      for (int a = 0; a < bases[i]; a++) sigma[(int64_t)i * maxbase + a] = perm[a];
    }
  }
  int mb = (int)bases[dim - 1];
  free(perm);
  free(bases);
  return mb;
}

/* numba `float ** int` (numba/cpython/numbers.py int_power): binary
 * exponentiation starting from r = 1. */
static double nb_ipow(double a, int64_t e) {
  double r = 1.0;
  while (e != 0) {
    if (e & 1) r *= a;
    e >>= 1;
    a *= a;
  }
  return r;
}

typedef struct {
  int64_t base, cap;
  int64_t *digits; /* cap */
  double *sums;    /* cap + 1 */
  int64_t *sig;    /* base */
  int64_t active;
  double first;
} rasrap_stream;

/* RasrapStream.__init__ halton.py:256-278 */
static void stream_init(rasrap_stream *s, int64_t base, const int64_t *sig, int64_t n0) {
  int K = orc_digit_capacity(base);
  s->base = base;
  s->cap = K + 8;
  s->digits = (int64_t *)calloc((size_t)s->cap, sizeof(int64_t));
  s->sums = (double *)calloc((size_t)s->cap + 1, sizeof(double));
  s->sig = (int64_t *)malloc(sizeof(int64_t) * (size_t)base);
  memcpy(s->sig, sig, sizeof(int64_t) * (size_t)base);
  int64_t n = n0, hi = -1;
  for (int64_t i = 0; i < s->cap; i++) {
    s->digits[i] = n % base;
    n /= base;
    if (s->digits[i]) hi = i;
  }
  s->active = K > hi + 1 ? K : hi + 1;
  if (hi < 0 && s->active < 1) s->active = 1;
  double inv_p = 1.0 / (double)base;
  double scale = pow(inv_p, (double)s->active); /* Python float ** int */
  for (int64_t j = s->active - 1; j >= 0; j--) {
    s->sums[j] = s->sums[j + 1] + (double)s->sig[s->digits[j]] * scale;
    scale *= (double)base;
  }
  s->first = s->sums[0];
}

static void stream_free(rasrap_stream *s) {
  free(s->digits);
  free(s->sums);
  free(s->sig);
}

/* _rasrap_fill_recursive, one dimension, one step (halton.py:402-414) */
static double stream_next(rasrap_stream *s) {
  int64_t base = s->base;
  double inv_p = 1.0 / (double)base;
  int64_t m = 0;
  while (s->digits[m] + 1 == base) m++;
  if (m >= s->active) s->active = m + 1;
  s->sums[m] = s->sums[m + 1] + (double)s->sig[s->digits[m] + 1] * nb_ipow(inv_p, m + 1);
  s->digits[m] += 1;
  double s0 = (double)s->sig[0];
  for (int64_t j = m - 1; j >= 0; j--) {
    s->digits[j] = 0;
    s->sums[j] = s->sums[j + 1] + s0 * nb_ipow(inv_p, j + 1);
  }
  return s->sums[0];
}

typedef struct {
  int dim;
  int maxbase;
  int64_t *bases;
  int64_t *start;
  int64_t *sigma; /* dim x maxbase */
} rasrap_cfg;

static void cfg_make(rasrap_cfg *c, int dim, uint64_t key) {
  c->dim = dim;
  c->bases = (int64_t *)malloc(sizeof(int64_t) * dim);
  orc_primes(dim, c->bases);
  c->maxbase = (int)c->bases[dim - 1];
  c->start = (int64_t *)malloc(sizeof(int64_t) * dim);
  c->sigma = (int64_t *)malloc(sizeof(int64_t) * (size_t)dim * c->maxbase);
  orc_rasrap_config(dim, key, c->start, NULL, c->sigma, c->maxbase);
}
static void cfg_free(rasrap_cfg *c) {
  free(c->bases);
  free(c->start);
  free(c->sigma);
}

/* RasrapRecursive.fill (halton.py:451-490): row 0 is the start point */
typedef struct {
  rasrap_cfg cfg;
  rasrap_stream *st;
  int64_t emitted;
} rasrap_rec;

static void rec_init(rasrap_rec *r, int dim, uint64_t key) {
  cfg_make(&r->cfg, dim, key);
  r->st = (rasrap_stream *)malloc(sizeof(rasrap_stream) * dim);
  for (int d = 0; d < dim; d++)
    stream_init(&r->st[d], r->cfg.bases[d], r->cfg.sigma + (int64_t)d * r->cfg.maxbase,
                r->cfg.start[d]);
  r->emitted = 0;
}
static void rec_fill(rasrap_rec *r, int64_t n, double *out) {
  int dim = r->cfg.dim;
  for (int64_t i = 0; i < n; i++) {
    for (int d = 0; d < dim; d++)
      out[i * dim + d] = r->emitted == 0 ? r->st[d].first : stream_next(&r->st[d]);
    r->emitted++;
  }
}
static void rec_free(rasrap_rec *r) {
  for (int d = 0; d < r->cfg.dim; d++) stream_free(&r->st[d]);
  free(r->st);
  cfg_free(&r->cfg);
}

void orc_rasrap_recursive_points(int dim, uint64_t key, int64_t count, double *out) {
  rasrap_rec r;
  rec_init(&r, dim, key);
  rec_fill(&r, count, out);
  rec_free(&r);
}

/* _rasrap_fill_counter halton.py:419-440 */
static void counter_points(const rasrap_cfg *c, const int64_t *idx, int64_t n, double *out) {
  for (int d = 0; d < c->dim; d++) {
    int64_t base = c->bases[d];
    int cap = orc_digit_capacity(base);
    const int64_t *sg = c->sigma + (int64_t)d * c->maxbase;
    double inv_p = 1.0 / (double)base;
    for (int64_t i = 0; i < n; i++) {
      int64_t v = c->start[d] + idx[i];
      double x = 0.0, scale = 1.0;
      int j = 0;
      while (v > 0 || j < cap) {
        scale *= inv_p;
        x += (double)sg[v % base] * scale;
        v /= base;
        j++;
      }
      out[i * c->dim + d] = x;
    }
  }
}

void orc_rasrap_counter_points(int dim, uint64_t key, const int64_t *idx, int64_t n,
                               double *out) {
  rasrap_cfg c;
  cfg_make(&c, dim, key);
  counter_points(&c, idx, n, out);
  cfg_free(&c);
}

/* ------------------------------------------------------------------ */
/* prng.py Philox-4x32-10                                               */
/* ------------------------------------------------------------------ */

/* prng.py:157-177 */
void orc_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; r++) {
    uint64_t p0 = (uint64_t)c0 * 0xD2511F53u;
    uint64_t p1 = (uint64_t)c2 * 0xCD9E8D57u;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0;
    c1 = n1;
    c2 = n2;
    c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* _philox_fill_indexed prng.py:234-246 / PhiloxPaths prng.py:249-267 */
void orc_philox_words(uint64_t key, const int64_t *paths, int64_t npaths, int nwords,
                      uint32_t *out) {
  uint32_t k[2] = {(uint32_t)key, (uint32_t)(key >> 32)};
  int nblocks = (nwords + 3) / 4;
  for (int64_t p = 0; p < npaths; p++) {
    uint64_t path = (uint64_t)paths[p];
    for (int b = 0; b < nblocks; b++) {
      uint32_t c[4] = {(uint32_t)b, (uint32_t)path, (uint32_t)(path >> 32), 0}, w[4];
      orc_philox_block(c, k, w);
      for (int j = 0; j < 4 && 4 * b + j < nwords; j++) out[p * nwords + 4 * b + j] = w[j];
    }
  }
}

/* ------------------------------------------------------------------ */
/* sobol.py                                                             */
/* ------------------------------------------------------------------ */

/* random_scramble sobol.py:259-270 + scramble_words_matrix sobol.py:236-248 */
void orc_sobol_scramble(int dim, const uint32_t *v, uint64_t key, int64_t replication,
                        uint32_t *gen_v, uint32_t *shift) {
  for (int d = 0; d < dim; d++) {
    uint64_t parts[3] = {key, (uint64_t)replication, (uint64_t)d};
    orc_pcg64 g;
    orc_pcg64_seed(&g, orc_derive_key(parts, 3));
    uint32_t cols[32];
    for (int c = 0; c < 32; c++) {
      uint32_t bits = orc_pcg64_next32(&g);
      uint32_t diag = 1u << (31 - c);
      cols[c] = diag | (bits & (diag - 1u));
    }
    shift[d] = orc_pcg64_next32(&g);
    for (int k = 0; k < 32; k++) {
      uint32_t y = v[d * 32 + k], z = 0;
      for (int c = 0; c < 32; c++)
        if (y & (1u << (31 - c))) z ^= cols[c];
      gen_v[d * 32 + k] = z;
    }
  }
}

/* _counter_fill_words sobol.py:313-327 */
void orc_sobol_counter_words(int dim, const uint32_t *gen_v, const uint32_t *shift,
                             const int64_t *idx, int64_t n, uint32_t *out) {
  for (int64_t p = 0; p < n; p++) {
    for (int d = 0; d < dim; d++) {
      uint32_t x = shift[d];
      uint64_t ii = (uint64_t)idx[p];
      int k = 0;
      while (ii) {
        if (ii & 1) x ^= gen_v[d * 32 + k];
        ii >>= 1;
        k++;
      }
      out[p * dim + d] = x;
    }
  }
}

/* ------------------------------------------------------------------ */
/* models.py                                                            */
/* ------------------------------------------------------------------ */

#define INV_TINY 1.1102230246251565e-16 /* 2**-53 */
#define INV_PLOW 0.0465
#define INV_RMAX 0.20566225000000002
#define INV_VLO 2.4772173769731336
#define INV_VSCALE 0.16408352781008756

/* models.py:39-64 */
double orc_inv_normal(double p) {
  int flip = p > 0.5;
  double pl = flip ? 1.0 - p : p;
  if (pl < INV_TINY) pl = INV_TINY;
  double x;
  if (pl >= INV_PLOW) {
    double q = pl - 0.5;
    double u = q * q / INV_RMAX;
    double num = ((((((-0.2919273214264852 * u + 9.193512285907598) * u + -62.454377324061355) * u +
                     170.0098658859532) * u + -211.46704297849197) * u + 113.93203453144044) * u +
                  -21.62514930947088) * u + 3.8841077977297096;
    double den = ((((((-0.4290780287479735 * u + 6.969736103714354) * u + -36.143835067804716) * u +
                     83.84882260510376) * u + -93.74669783914054) * u + 47.23127323999088) * u +
                  -8.96090814172393) * u + 1.5495348220676615;
    x = q * num / den;
  } else {
    double w = (sqrt(-2.0 * log(pl)) - INV_VLO) * INV_VSCALE;
    double num = ((((((49.41588603624166 * w + 34.09554370467819) * w + -120.62391569766385) * w +
                     -36.11819081101896) * w + 77.35661807857605) * w + 12.678668433221901) * w +
                  -15.636790505919562) * w + -3.141967925161121;
    double den = ((((((-0.0005317355830972598 * w + -8.101041244986659) * w + -2.3666362350675305) * w +
                     19.91298298968798) * w + -1.4094956335739925) * w + -10.941521790794202) * w +
                  1.2762506234112334) * w + 1.8704632131064214;
    x = num / den;
  }
  return flip ? -x : x;
}

void orc_inv_normal_n(const double *p, int64_t n, double *out) {
  for (int64_t i = 0; i < n; i++) out[i] = orc_inv_normal(p[i]);
}

/* _libor_payoffs models.py:271-293 */
void orc_libor_payoffs(const double *u, int64_t npaths, int steps, const double *l0,
                       double delta, double sigma, double strike, double front_factor,
                       double *out) {
  double sig2 = sigma * sigma;
  double sqdt = sqrt(delta);
  double *rates = (double *)malloc(sizeof(double) * steps);
  for (int64_t p = 0; p < npaths; p++) {
    for (int n = 0; n < steps; n++) rates[n] = l0[n];
    double disc = front_factor;
    for (int i = 0; i < steps; i++) {
      double shock = sigma * sqdt * orc_inv_normal(u[p * steps + i]);
      double drift = 0.0;
      for (int n = i; n < steps; n++) {
        double dl = delta * rates[n];
        drift += sig2 * dl / (1.0 + dl);
        rates[n] = rates[n] * (1.0 + drift * delta + shock);
      }
      if (i < steps - 1) disc /= 1.0 + delta * rates[i];
    }
    double lt = rates[steps - 1];
    double payoff = delta * fmax(lt - strike, 0.0) / (1.0 + delta * lt);
    out[p] = payoff * disc;
  }
  free(rates);
}

/* _mbs_payoffs models.py:430-449 */
void orc_mbs_payoffs(const double *u, int64_t npaths, int months, double i0, double k0,
                     double k1, double k2, double k3, double k4, double sigma_xi,
                     double payment, const double *ck, double *out) {
  for (int64_t p = 0; p < npaths; p++) {
    double disc = 1.0, remaining = 1.0, rate = i0, prev_w = 0.0, pv = 0.0;
    for (int k = 1; k <= months; k++) {
      disc /= 1.0 + rate;
      if (k > 1) remaining *= 1.0 - prev_w;
      double xi = sigma_xi * orc_inv_normal(u[p * months + k - 1]);
      rate = k0 * exp(xi) * rate;
      double w = k1 + k2 * atan(k3 * rate + k4);
      pv += disc * payment * remaining * ((1.0 - w) + w * ck[k - 1]);
      prev_w = w;
    }
    out[p] = pv;
  }
}

/* numpy DOUBLE_pairwise_sum (numpy/_core/src/umath/loops_utils.h.src),
 * PW_BLOCKSIZE 128, unroll 8. */
double orc_pairwise_sum(const double *a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; i++) res += a[i];
    return res;
  } else if (n <= 128) {
    double r[8];
    int64_t i;
    for (int j = 0; j < 8; j++) r[j] = a[j];
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return orc_pairwise_sum(a, n2) + orc_pairwise_sum(a + n2, n - n2);
  }
}

/* ------------------------------------------------------------------ */
/* SFC64 per-path streams (builder-defined layout, numpy SFC64 core)   */
/* ------------------------------------------------------------------ */

typedef struct {
  uint64_t a, b, c, w;
} sfc64;

static uint64_t sfc64_next(sfc64 *s) {
  uint64_t tmp = s->a + s->b + s->w++;
  s->a = s->b ^ (s->b >> 11);
  s->b = s->c + (s->c << 3);
  s->c = ((s->c << 24) | (s->c >> 40)) + tmp;
  return tmp;
}

static void sfc64_path_seed(sfc64 *s, uint64_t seed, int64_t m, int64_t path) {
  uint64_t parts[4] = {seed, 7, (uint64_t)m, (uint64_t)path};
  uint32_t w[6];
  orc_derive_words(orc_derive_key(parts, 4), 6, w);
  s->a = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  s->b = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
  s->c = (uint64_t)w[4] | ((uint64_t)w[5] << 32);
  s->w = 1;
  for (int i = 0; i < 12; i++) sfc64_next(s);
}

void orc_sfc64_path_uniforms(uint64_t seed, int64_t m, const int64_t *paths, int64_t n,
                             int dim, double *out) {
  for (int64_t p = 0; p < n; p++) {
    sfc64 s;
    sfc64_path_seed(&s, seed, m, paths[p]);
    for (int d = 0; d < dim; d++)
      out[p * dim + d] = (double)(sfc64_next(&s) >> 11) * (1.0 / 9007199254740992.0);
  }
}

/* ------------------------------------------------------------------ */
/* MT19937 and XORWOW word streams (prng.py:40-149)                     */
/* ------------------------------------------------------------------ */

/* MT19937 with the classic 32-bit seeding (prng.py:63-72); cursor starts at
 * 624 so the first word triggers a twist (prng.py:43-52). */
void orc_mt19937_init(orc_mt19937 *g, uint32_t seed) {
  g->state[0] = seed;
  for (int i = 1; i < 624; i++) {
    uint32_t prev = g->state[i - 1];
    g->state[i] = 1812433253u * (prev ^ (prev >> 30)) + (uint32_t)i;
  }
  g->cursor = 624;
}

/* _mt_fill (prng.py:40-60): in-place twist, then tempering. */
void orc_mt19937_words(orc_mt19937 *g, int64_t n, uint32_t *out) {
  uint32_t *st = g->state;
  for (int64_t i = 0; i < n; i++) {
    if (g->cursor >= 624) {
      for (int j = 0; j < 624; j++) {
        uint32_t y = (st[j] & 0x80000000u) | (st[(j + 1) % 624] & 0x7FFFFFFFu);
        uint32_t val = st[(j + 397) % 624] ^ (y >> 1);
        if (y & 1u) val ^= 0x9908B0DFu;
        st[j] = val;
      }
      g->cursor = 0;
    }
    uint32_t y = st[g->cursor++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9D2C5680u;
    y ^= (y << 15) & 0xEFC60000u;
    y ^= y >> 18;
    out[i] = y;
  }
}

/* Xorwow(seed) (prng.py:128-134): derive_words(seed, 6), re-derived from
 * seed + 1, + 2, ... while the five xorshift words are all zero. */
void orc_xorwow_init(orc_xorwow *g, uint64_t seed) {
  for (;;) {
    orc_derive_words(seed, 6, g->s);
    if (g->s[0] | g->s[1] | g->s[2] | g->s[3] | g->s[4]) break;
    seed = seed + 1;
  }
}

/* _xorwow_fill (prng.py:90-115), 32-bit wraparound. */
void orc_xorwow_words(orc_xorwow *g, int64_t n, uint32_t *out) {
  uint32_t x = g->s[0], y = g->s[1], z = g->s[2], w = g->s[3], v = g->s[4], d = g->s[5];
  for (int64_t i = 0; i < n; i++) {
    uint32_t t = x ^ (x >> 2);
    x = y;
    y = z;
    z = w;
    w = v;
    v = (v ^ (v << 4)) ^ (t ^ (t << 1));
    d += 362437u;
    out[i] = d + v;
  }
  g->s[0] = x;
  g->s[1] = y;
  g->s[2] = z;
  g->s[3] = w;
  g->s[4] = v;
  g->s[5] = d;
}

/* ------------------------------------------------------------------ */
/* Kakutani orbits (halton.py:163-239, 521-542)                          */
/* ------------------------------------------------------------------ */

/* Bracket tables per dimension, [dims][64] (KakutaniState._grow_tables,
 * halton.py:178-193): exact rationals rounded by Python; set by oracle.py. */
static const double *KK_THR = NULL, *KK_B = NULL;
static int KK_DIMS = 0;
#define KK_TAB 64

void orc_kakutani_set_tables(const double *thr, const double *b, int dims) {
  KK_THR = thr;
  KK_B = b;
  KK_DIMS = dims;
}

/* kakutani_next (halton.py:208-239): log guess, then the two bracket loops */
static int kak_next(double *x, int d, int64_t p) {
  const double *thr = KK_THR + (size_t)d * KK_TAB, *b = KK_B + (size_t)d * KK_TAB;
  double one_minus = 1.0 - *x;
  int k = (int)(-log(one_minus) / log((double)p)) + 1;
  if (k < 1) k = 1;
  if (k + 1 > KK_TAB) return -1;
  while (one_minus <= thr[k - 1]) {
    k++;
    if (k + 1 > KK_TAB) return -1;
  }
  while (k > 1 && one_minus > thr[k - 2]) k--;
  double v = *x + b[k - 1];
  if (v >= 1.0) v -= 1.0;
  *x = v;
  return 0;
}

typedef struct {
  int dim, emitted;
  double *x;
  int64_t *base;
} kak_sampler;

static int kak_init(kak_sampler *s, int dim, uint64_t key) {
  if (!KK_THR || dim > KK_DIMS) return -1;
  s->dim = dim;
  s->emitted = 0;
  s->x = (double *)malloc(sizeof(double) * dim);
  s->base = (int64_t *)malloc(sizeof(int64_t) * dim);
  orc_primes(dim, s->base);
  for (int d = 0; d < dim; d++) { /* derive_rng(seed, i).random() (halton.py:532-534) */
    uint64_t parts[2] = {key, (uint64_t)d};
    orc_pcg64 g;
    orc_pcg64_seed(&g, orc_derive_key(parts, 2));
    s->x[d] = orc_pcg64_random(&g);
  }
  return 0;
}

/* KakutaniSampler.fill (halton.py:536-542) */
static int kak_fill(kak_sampler *s, int64_t n, double *out) {
  for (int64_t i = 0; i < n; i++) {
    if (!s->emitted) {
      s->emitted = 1;
    } else {
      for (int d = 0; d < s->dim; d++)
        if (kak_next(&s->x[d], d, s->base[d])) return -1;
    }
    for (int d = 0; d < s->dim; d++) out[i * s->dim + d] = s->x[d];
  }
  return 0;
}

static void kak_free(kak_sampler *s) {
  free(s->x);
  free(s->base);
}

int orc_kakutani_points(int dim, uint64_t key, int64_t count, double *out) {
  kak_sampler s;
  if (kak_init(&s, dim, key)) return -1;
  int rc = kak_fill(&s, count, out);
  kak_free(&s);
  return rc;
}

/* ------------------------------------------------------------------ */
/* harness.py replication loop                                          */
/* ------------------------------------------------------------------ */

#define CHUNK_PATHS 8192 /* harness.py:25 */

/* Test integrand with no reference counterpart (RQ_MODEL_XHASH,
 * include/rqmc_b200.h): top 20 bits of a 64-bit hash of the coordinates'
 * bit patterns in dimension order.  Exact sums, so theta pins every
 * coordinate of every path of the device stream. */
double orc_coord_hash(const double *u, int dim) {
  uint64_t h = 0x6A09E667F3BCC909ull;
  for (int d = 0; d < dim; d++) {
    uint64_t b;
    memcpy(&b, &u[d], 8);
    h = (h ^ b) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 32;
  }
  return (double)(h >> 44);
}

/* seeding.py:17-24 (twister 1, xorwow 2, philox 3, rasrap 4, sobol 5, kakutani 6);
 * 7 = sfc64 */
static const uint64_t FAMILY_ID[9] = {4, 4, 3, 5, 5, 7, 1, 2, 6};

int orc_run_replication(int gen, int model, int dim, const double *mparams, uint64_t seed,
                        int64_t m, const int64_t *grid, int ngrid, const uint32_t *sobol_v,
                        double *theta) {
  if (gen < 0 || gen > 8 || model < 0 || model > 5 || model == 4 || ngrid < 1) return -1;
  int64_t nmax = grid[ngrid - 1];
  uint64_t parts[3] = {seed, FAMILY_ID[gen], (uint64_t)m};
  uint64_t key = orc_derive_key(parts, 3); /* harness.py:113 */
  double *payoffs = (double *)malloc(sizeof(double) * (size_t)nmax);
  double *buf = (double *)malloc(sizeof(double) * (size_t)CHUNK_PATHS * dim);
  int64_t *idx = (int64_t *)malloc(sizeof(int64_t) * CHUNK_PATHS);
  uint32_t *words = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)CHUNK_PATHS * dim);
  uint32_t *gen_v = NULL, *shift = NULL;
  rasrap_rec rec;
  rasrap_cfg cfg;
  orc_mt19937 mt;
  orc_xorwow xw;
  kak_sampler kk;
  if (gen == 8 && kak_init(&kk, dim, key)) return -1;
  if (gen == 6) orc_mt19937_init(&mt, (uint32_t)key); /* harness.py:111 key & 0xFFFFFFFF */
  if (gen == 7) orc_xorwow_init(&xw, key);             /* harness.py:113 */
  if (gen == 0) rec_init(&rec, dim, key);
  if (gen == 1) cfg_make(&cfg, dim, key);
  if (gen == 3 || gen == 4) {
    gen_v = (uint32_t *)malloc(sizeof(uint32_t) * 32 * dim);
    shift = (uint32_t *)malloc(sizeof(uint32_t) * dim);
    orc_sobol_scramble(dim, sobol_v, key, m, gen_v, shift); /* harness.py:122 */
  }
  int rc = 0;
  for (int64_t done = 0; done < nmax;) {
    int64_t cnt = nmax - done < CHUNK_PATHS ? nmax - done : CHUNK_PATHS;
    for (int64_t i = 0; i < cnt; i++) idx[i] = done + i;
    if (gen == 0) {
      rec_fill(&rec, cnt, buf);
    } else if (gen == 8) {
      if (kak_fill(&kk, cnt, buf)) {
        rc = -1;
        break;
      }
    } else if (gen == 1) {
      counter_points(&cfg, idx, cnt, buf);
    } else if (gen == 5) {
      orc_sfc64_path_uniforms(seed, m, idx, cnt, dim, buf);
    } else if (gen == 2 || gen == 6 || gen == 7) {
      /* _WordSampler.fill (harness.py:46-50): the next cnt*dim words, row-major */
      if (gen == 2) orc_philox_words(key, idx, cnt, dim, words);
      if (gen == 6) orc_mt19937_words(&mt, cnt * dim, words);
      if (gen == 7) orc_xorwow_words(&xw, cnt * dim, words);
      for (int64_t i = 0; i < cnt * dim; i++)
        buf[i] = (double)words[i] * 2.3283064365386963e-10 + 1.1641532182693481e-10;
    } else {
      /* sobol-gray: Gray-order point i is the counter point at i ^ (i >> 1)
       * (sobol.py:290-310); sobol-counter: the counter point at i. */
      if (gen == 3)
        for (int64_t i = 0; i < cnt; i++) idx[i] = idx[i] ^ (idx[i] >> 1);
      orc_sobol_counter_words(dim, gen_v, shift, idx, cnt, words);
      for (int64_t i = 0; i < cnt * dim; i++) buf[i] = (double)words[i] * 2.3283064365386963e-10;
    }
    double *out = payoffs + done;
    if (model == 0) {
      orc_libor_payoffs(buf, cnt, dim, mparams + 4, mparams[0], mparams[1], mparams[2],
                        mparams[3], out);
    } else if (model == 1) {
      orc_mbs_payoffs(buf, cnt, dim, mparams[0], mparams[1], mparams[2], mparams[3],
                      mparams[4], mparams[5], mparams[6], mparams[7], mparams + 8, out);
    } else if (model == 2) {
      for (int64_t i = 0; i < cnt; i++) out[i] = buf[i * dim];
    } else if (model == 5) {
      for (int64_t i = 0; i < cnt; i++) out[i] = orc_coord_hash(buf + i * dim, dim);
    } else {
      for (int64_t i = 0; i < cnt; i++) out[i] = 1.0;
    }
    done += cnt;
  }
  for (int g = 0; rc == 0 && g < ngrid; g++)
    theta[g] = orc_pairwise_sum(payoffs, grid[g]) / (double)grid[g]; /* harness.py:314 */
  if (gen == 8) kak_free(&kk);
  if (gen == 0) rec_free(&rec);
  if (gen == 1) cfg_free(&cfg);
  free(gen_v);
  free(shift);
  free(words);
  free(idx);
  free(buf);
  free(payoffs);
  return rc;
}

typedef struct {
  int gen, model, dim, ngrid;
  const double *mparams;
  uint64_t seed;
  int64_t first, count;
  const int64_t *grid;
  const uint32_t *sobol_v;
  double *theta;
  int64_t next; /* shared work counter (guarded by lock) */
  pthread_mutex_t lock;
  int rc;
} rep_job;

static void *rep_worker(void *arg) {
  rep_job *j = (rep_job *)arg;
  for (;;) {
    pthread_mutex_lock(&j->lock);
    int64_t r = j->next++;
    pthread_mutex_unlock(&j->lock);
    if (r >= j->count) break;
    int rc = orc_run_replication(j->gen, j->model, j->dim, j->mparams, j->seed, j->first + r,
                                 j->grid, j->ngrid, j->sobol_v, j->theta + r * j->ngrid);
    if (rc) {
      pthread_mutex_lock(&j->lock);
      j->rc = rc;
      pthread_mutex_unlock(&j->lock);
    }
  }
  return NULL;
}

/* run_experiment replication-parallel loop (harness.py:349-358): each
 * worker owns whole replications; results land in fixed slots, so theta is
 * independent of the thread count. */
int orc_run_replications(int gen, int model, int dim, const double *mparams, uint64_t seed,
                         int64_t first, int64_t count, const int64_t *grid, int ngrid,
                         const uint32_t *sobol_v, int threads, double *theta) {
  rep_job j = {gen, model, dim, ngrid, mparams, seed, first, count, grid, sobol_v, theta, 0,
               PTHREAD_MUTEX_INITIALIZER, 0};
  if (threads < 1) threads = 1;
  if (threads > 1024) threads = 1024;
  pthread_t tid[1024];
  for (int t = 1; t < threads; t++) pthread_create(&tid[t], NULL, rep_worker, &j);
  rep_worker(&j);
  for (int t = 1; t < threads; t++) pthread_join(tid[t], NULL);
  return j.rc;
}
