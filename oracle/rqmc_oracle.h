/* rqmc_oracle.h -- CPU restatement of the reference RQMC hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker the CUDA path is
 * compared against (tests/, __graft_entry__.smoke(), bench.py's
 * cpu_baseline / --impl reference arm).  Nothing in paper_1408_5526_b200/
 * links, imports or calls it.
 *
 * Every function restates one reference function (file:line under
 * /root/reference/pkg/src/rqmcbench/) in sequential C with the same
 * operation order and no FMA contraction (-ffp-contract=off), so that it is
 * bit-identical to the numba kernels.  Third-party algorithms the reference
 * calls (numpy SeedSequence / PCG64 / Generator.random / .permutation /
 * .integers, numpy pairwise np.sum) are restated from numpy 2.3 sources and
 * pinned against numpy itself in tests/test_oracle.py.
 *
 * Pinning: tests/test_oracle.py checks every function here against the
 * golden fixtures in tests/golden/ written by tests/golden/make_golden.py
 * from the unmodified reference package.
 */
#ifndef RQMC_ORACLE_H
#define RQMC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* seeding.py:27-56 */
uint64_t orc_splitmix64(uint64_t z);
uint64_t orc_derive_key(const uint64_t *parts, int nparts);
void orc_derive_words(uint64_t key, int count, uint32_t *out);

/* numpy PCG64(SeedSequence(key)) -- seeding.py:59-65 */
typedef struct {
  uint64_t st_hi, st_lo, inc_hi, inc_lo;
  int has_u32;
  uint32_t u32;
} orc_pcg64;
void orc_pcg64_seed(orc_pcg64 *g, uint64_t key);
uint64_t orc_pcg64_next64(orc_pcg64 *g);
uint32_t orc_pcg64_next32(orc_pcg64 *g);
double orc_pcg64_random(orc_pcg64 *g);
void orc_pcg64_permutation(orc_pcg64 *g, int64_t n, int64_t *out);
void orc_pcg64_u32_stream(uint64_t key, int n, uint32_t *out);

/* halton.py */
int orc_primes(int count, int64_t *out);
int orc_digit_capacity(int64_t base);
uint64_t orc_invert_radical(double omega, int64_t base, int k);
/* rasrap_config (halton.py:345-360): start indices, omega, packed sigmas
 * [dim x maxbase] (maxbase = largest base); returns maxbase. */
int orc_rasrap_config(int dim, uint64_t key, int64_t *start, double *omega, int64_t *sigma,
                      int maxbase);
/* RasrapRecursive.fill over rows 0..count-1 (halton.py:392-416, 451-490) */
void orc_rasrap_recursive_points(int dim, uint64_t key, int64_t count, double *out);
/* RasrapCounter.at (halton.py:419-440, 493-518) */
void orc_rasrap_counter_points(int dim, uint64_t key, const int64_t *idx, int64_t n,
                               double *out);

/* prng.py:157-246 */
void orc_philox_block(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
void orc_philox_words(uint64_t key, const int64_t *paths, int64_t npaths, int nwords,
                      uint32_t *out);

/* sobol.py: scramble (259-275) and Gray / counter words (290-327).
 * v: unscrambled direction words [dim x 32]. */
void orc_sobol_scramble(int dim, const uint32_t *v, uint64_t key, int64_t replication,
                        uint32_t *gen_v, uint32_t *shift);
void orc_sobol_counter_words(int dim, const uint32_t *gen_v, const uint32_t *shift,
                             const int64_t *idx, int64_t n, uint32_t *out);

/* models.py:39-64 */
double orc_inv_normal(double p);
void orc_inv_normal_n(const double *p, int64_t n, double *out);
/* models.py:271-293 */
void orc_libor_payoffs(const double *u, int64_t npaths, int steps, const double *l0,
                       double delta, double sigma, double strike, double front_factor,
                       double *out);
/* models.py:430-449 */
void orc_mbs_payoffs(const double *u, int64_t npaths, int months, double i0, double k0,
                     double k1, double k2, double k3, double k4, double sigma_xi,
                     double payment, const double *ck, double *out);

/* numpy pairwise sum of a contiguous float64 vector (np.sum) */
double orc_pairwise_sum(const double *a, int64_t n);
double orc_coord_hash(const double *u, int dim); /* xhash test integrand (no reference counterpart) */

/* One full replication (harness.py:291-315): generator -> model -> prefix
 * estimates theta[g] = np.sum(payoffs[:grid[g]]) / grid[g].
 * gen: 0 rasrap-recursive, 1 rasrap-counter, 2 philox, 3 sobol-gray,
 *      4 sobol-counter, 5 sfc64 (builder-defined per-path streams), 6 twister,
 *      7 xorwow, 8 kakutani (needs orc_kakutani_set_tables).  model: 0 libor, 1 mbs, 2 x1, 3 const1.
 * mparams: libor {delta, sigma, strike, front_factor, l0[steps]...};
 *          mbs {i0,k0,k1,k2,k3,k4,sigma_xi,payment, ck[months]...}.
 * sobol_v: unscrambled direction words [dim x 32] (gen 3/4 only). */
int orc_run_replication(int gen, int model, int dim, const double *mparams, uint64_t seed,
                        int64_t m, const int64_t *grid, int ngrid, const uint32_t *sobol_v,
                        double *theta);
/* run_experiment's replication loop for reps first..first+count-1 with
 * `threads` OpenMP threads; theta[count x ngrid]. */
int orc_run_replications(int gen, int model, int dim, const double *mparams, uint64_t seed,
                         int64_t first, int64_t count, const int64_t *grid, int ngrid,
                         const uint32_t *sobol_v, int threads, double *theta);

/* MT19937 (prng.py:40-82) and XORWOW (prng.py:90-149) word streams. */
typedef struct {
  uint32_t state[624];
  int cursor;
} orc_mt19937;
void orc_mt19937_init(orc_mt19937 *g, uint32_t seed);
void orc_mt19937_words(orc_mt19937 *g, int64_t n, uint32_t *out);
typedef struct {
  uint32_t s[6]; /* x, y, z, w, v, d */
} orc_xorwow;
void orc_xorwow_init(orc_xorwow *g, uint64_t seed);
void orc_xorwow_words(orc_xorwow *g, int64_t n, uint32_t *out);

/* Kakutani orbits (halton.py:163-239, 521-542).  The bracket tables
 * [dims][64] (thr = float(1/p^k) + 1e-11, b = float((p+1-p^k)/p^k)) come
 * from oracle.py, computed with fractions.Fraction as the reference does. */
void orc_kakutani_set_tables(const double *thr, const double *b, int dims);
int orc_kakutani_points(int dim, uint64_t key, int64_t count, double *out);

/* SFC64 (no reference counterpart; numpy.random.SFC64 is the oracle).
 * Per-path stream seeded from derive_words(derive_key(seed, 7, m, path), 6). */
void orc_sfc64_path_uniforms(uint64_t seed, int64_t m, const int64_t *paths, int64_t n,
                             int dim, double *out);

#ifdef __cplusplus
}
#endif
#endif
