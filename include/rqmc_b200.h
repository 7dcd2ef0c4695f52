/* rqmc_b200.h -- C ABI of the B200-native RQMC estimator (librqmc_b200.so).
 *
 * Drop-in boundary for the reference package `rqmcbench`
 * (/root/reference/pkg/src/rqmcbench).  Each entry point replaces one piece
 * of the reference's hot path; the reference interface it stands in for is
 * cited as file:line.  All functions return 0 on success and a negative
 * RQ_ERR_* code on failure (rq_last_error() gives the message); none of them
 * throws, and none falls back to the CPU.
 *
 * Pointers named *_dev are device pointers (e.g. torch.Tensor.data_ptr()),
 * *_host are host pointers.  `stream` is a cudaStream_t (NULL = the legacy
 * default stream).  Plain C types only -- no torch types cross this ABI.
 */
#ifndef RQMC_B200_H
#define RQMC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RQ_ABI_VERSION 1

/* error codes (mapped by the Python shim: VALUE -> ValueError /
 * ConfigurationError (harness.py:28-29), CUDA -> RuntimeError,
 * NONFINITE -> ArithmeticError (harness.py:222-226)) */
#define RQ_OK 0
#define RQ_ERR_VALUE (-1)
#define RQ_ERR_CUDA (-2)
#define RQ_ERR_RANGE (-3)
#define RQ_ERR_NONFINITE (-4)

/* Generator ids: the names of harness.GENERATOR_NAMES (harness.py:84-93)
 * that have a device implementation, plus SFC64 (north-star addition, no
 * reference counterpart).  Family ids for key derivation follow
 * seeding.GENERATOR_IDS (seeding.py:17-24); SFC64 uses family 7. */
enum rq_generator {
  RQ_GEN_RASRAP_RECURSIVE = 0, /* halton.RasrapRecursive  halton.py:451-490 */
  RQ_GEN_RASRAP_COUNTER = 1,   /* halton.RasrapCounter    halton.py:493-518 */
  RQ_GEN_PHILOX = 2,           /* harness._PhiloxSampler  harness.py:53-72  */
  RQ_GEN_SOBOL_GRAY = 3,       /* sobol.SobolGray         sobol.py:330-346  */
  RQ_GEN_SOBOL_COUNTER = 4,    /* sobol.SobolCounter      sobol.py:349-372  */
  RQ_GEN_SFC64 = 5,            /* per-path SFC64 streams (numpy SFC64 core) */
  RQ_GEN_TWISTER = 6,          /* prng.MT19937 word stream  prng.py:40-82, harness.py:110-111 */
  RQ_GEN_XORWOW = 7,           /* prng.Xorwow word stream   prng.py:90-149, harness.py:112-113 */
  RQ_GEN_KAKUTANI = 8          /* halton.KakutaniSampler     halton.py:521-542, harness.py:118-119 */
};

/* Model kinds: models.LiborModel (models.py:296-329), models.MbsModel
 * (models.py:452-469), models.FirstCoordinateModel / ConstantModel
 * (models.py:477-498).  RQ_MODEL_XHASH is a test integrand with no
 * reference counterpart: payoff = top 20 bits of a 64-bit hash of every
 * coordinate's bit pattern in dimension order (h = 0x6A09E667F3BCC909;
 * per coordinate h = (h ^ bits(u)) * 0x9E3779B97F4A7C15, h ^= h >> 32),
 * so an exact theta pins all coordinates of all paths. */
enum rq_model_kind {
  RQ_MODEL_LIBOR = 0,
  RQ_MODEL_MBS = 1,
  RQ_MODEL_X1 = 2,
  RQ_MODEL_CONST1 = 3,
  RQ_MODEL_XHASH = 5
};

/* Model description = the arguments of the reference's payoff kernels
 * (_libor_payoffs models.py:271, _mbs_payoffs models.py:430).
 * LIBOR: dim = steps (1..6542; 10/20/40/80 register-resident, <= 160 in
 *        shared memory, longer in global memory), delta = accrual, sigma, strike,
 *        front_factor = 1/(1 + delta*L_0(0)), table = l0[dim] (HOST).
 * MBS:   dim = months, i0..payment as MbsConfig, table = ck[dim] (HOST).
 * X1 / CONST1 / XHASH: dim only. */
typedef struct rq_model {
  int32_t kind;
  int32_t dim;
  double delta, sigma, strike, front_factor;
  double i0, k0, k1, k2, k3, k4, sigma_xi, payment;
  const double *table;
} rq_model;

/* Opaque device-resident randomisation for replications
 * rep_first .. rep_first+rep_count-1 of one (generator, dim, seed):
 * Rasrap starts/permutations/init sums, Sobol scrambles, PRNG keys. */
typedef struct rq_sampler rq_sampler;

const char *rq_last_error(void);
int rq_abi_version(void);

/* make_sampler(name, dim, seed, replication) for a range of replications
 * (harness.py:99-125; rasrap_config halton.py:345-360; random_scramble
 * sobol.py:259-270).  The randomisation is generated ON THE DEVICE (numpy
 * SeedSequence/PCG64 restated), bit-identical to the reference.
 * Dimensions: Rasrap and Kakutani 1..6542 (the first 6542 primes, every base
 * below 2^16), Sobol' 1..421 (the direction table), the PRNGs any. */
int rq_sampler_create(rq_sampler **out, int generator, int dim, uint64_t seed,
                      int64_t rep_first, int32_t rep_count, void *stream);
void rq_sampler_destroy(rq_sampler *s);

/* Exclusive upper bound on point indices the device evaluates for a
 * generator (the reference takes int64 indices: RasrapCounter.at
 * halton.py:506-512, the Philox counter's path_hi prng.py:180-246):
 * 2^62 for Philox and SFC64, 2^39 for both Rasrap forms (n0 + i stays inside
 * the digit window, >= 2^40 for every base), 2^32 for Sobol' (32-bit
 * direction numbers: sobol.py:181-193 raises beyond) and for the sequential
 * word streams / Kakutani orbits.  Larger indices return RQ_ERR_RANGE. */
int64_t rq_index_limit(int generator);

/* sampler.fill(out) for rows first..first+count-1 of replication
 * rep_first+rep_local (halton.py:479, sobol.py:341, harness.py:63):
 * out_dev[count][dim] row-major float64. */
int rq_sampler_points(rq_sampler *s, int32_t rep_local, int64_t first, int64_t count,
                      double *out_dev, void *stream);
/* sampler.at(indices) (halton.py:507, sobol.py:359, harness.py:69).  The
 * sequential word streams (twister, xorwow) have no at() in the reference
 * (_WordSampler, harness.py:37-50): RQ_ERR_VALUE. */
int rq_sampler_points_at(rq_sampler *s, int32_t rep_local, const int64_t *idx_dev,
                         int64_t count, double *out_dev, void *stream);
/* Rasrap tables of one replication, for inspection/tests (strides padded
 * to multiples of 4): start digits [sum of (K+8)] uint16, digit
 * permutations [sum of bases] uint16, init partial sums [sum of (K+9)]. */
int rq_sampler_rasrap_tables(rq_sampler *s, int32_t rep_local, uint16_t *digits_host,
                             uint16_t *sigma_host, double *sums_host);

/* The fused replication engine: for every replication of the sampler and
 * every N in grid (strictly increasing), theta[r][g] = np.sum(payoffs[:N])/N
 * (harness.py:291-315, with numpy's pairwise summation order).
 * theta_dev[rep_count][ngrid].  kernel_launches (nullable) += kernels run.
 * N <= min(2^40, rq_index_limit(generator)); marks above RQ_SEG_PATHS
 * (env, default 2^31) run as pairwise-tree segments (same result). */
int rq_estimate(rq_sampler *s, const rq_model *model, const int64_t *grid_host, int32_t ngrid,
                double *theta_dev, int32_t *kernel_launches, void *stream);

/* End to end: run_experiment's replication loop (harness.py:342-358) for
 * replications rep_first..rep_first+rep_count-1, host in / host out.
 * Randomisation setup, paths and reduction all run on the device. */
int rq_run_replications(int generator, const rq_model *model, uint64_t seed, int64_t rep_first,
                        int64_t rep_count, const int64_t *grid_host, int32_t ngrid,
                        double *theta_host, int32_t *kernel_launches);

/* model.payoffs(u) (models.py:311-322 / 462-469): u_dev[npaths][dim]. */
int rq_model_payoffs(const rq_model *model, const double *u_dev, int64_t npaths,
                     double *out_dev, void *stream);
/* models.inv_normal (models.py:73-82) */
int rq_inv_normal(const double *u_dev, int64_t n, double *out_dev, void *stream);
/* Config-4 stream: points 0..npoints-1 of replication rep_local, Phi^-1
 * fused, summed into *sum_dev (and stored to store_dev[npoints][dim] if
 * non-NULL).  bench_throughput analogue (harness.py:401-429). */
int rq_stream_normals(rq_sampler *s, int32_t rep_local, int64_t npoints, double *sum_dev,
                      double *store_dev, void *stream);
/* np.sum of a contiguous float64 device vector (numpy pairwise order). */
int rq_pairwise_sum(const double *a_dev, int64_t n, double *out_dev, void *stream);

/* Same reduction on the host through the same plan (tests the plan
 * without a GPU; not used on the device path). */
int rq_pairwise_sum_host(const double *a_host, int64_t n, double *out_host);

/* Measurement hooks (bench.py): host<->device bytes moved by the ABI and,
 * with timing on, CUDA-event durations of the setup / path / reduce
 * kernels on their launching stream. */
void rq_stats_reset(int timing);
void rq_stats_get(uint64_t *h2d, uint64_t *d2h, double *setup_ms, double *paths_ms,
                  double *reduce_ms, int64_t *paths_launches);
/* FP64 pipe peak probe: DFMA slots per second over all SMs (best of 5). */
int rq_fp64_peak(double *slots_per_s, double *ms);

/* Host-side constant tables (for tests and the Python shim). */
int rq_sobol_directions(int dim, uint32_t *v_host); /* default_table(dim).v sobol.py:170 */
int rq_halton_constants(int dim, int32_t *base, int32_t *K, double *scale0);
/* Kakutani bracket tables of dims 0..dim-1 (KakutaniState._grow_tables,
 * halton.py:178-193): thr[d][k] = float(1/p^(k+1)) + 1e-11 and
 * b[d][k] = float((p + 1 - p^(k+1)) / p^(k+1)), 64 entries per dim. */
int rq_kakutani_tables(int dim, double *thr_host, double *b_host);
/* The device's division-by-base magic for dimension d, evaluated on the
 * host: q64 = floor(x / p) for x < 2^46, q32 = floor((uint32)x / p). */
int rq_halton_divide(int d, uint64_t x, uint64_t *q64, uint32_t *q32);

#ifdef __cplusplus
}
#endif
#endif
