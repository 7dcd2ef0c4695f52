// rq_internal.h -- structures shared by the C-ABI layer (rq_capi.cu) and the
// kernels (rq_kernels.cu).  Not part of the public ABI (include/rqmc_b200.h).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace rq {

// Halton/Rasrap/Kakutani dimensions: the first 6542 primes, i.e. every base
// below 2^16 (digits and sigma entries are uint16; the reference takes any
// count, halton.py:40-56, but its packed sigma table, halton.py:443-448, is
// dim x max(base) int64 = 3.4 GB per sampler here).  The HaltonDim entries
// of the first CONST_DIMS dims are in the constant bank, the rest in global
// memory (see hdim in rq_kernels.cu).
constexpr int MAX_DIM = 6542;
constexpr int CONST_DIMS = 512;
constexpr int MAX_CAP = 40;     // K + 8 for base 2 (largest digit window)
constexpr int SOBOL_BITS = 32;  // sobol.py:30
constexpr int TILE_PATHS = 128;  // paths per CTA tile (rq_kernels.cu TILE)
constexpr int CHUNK_DIMS = 20;  // dimensions per generator chunk in the fused kernels
constexpr int LIBOR_DYN_MAX = 160;  // LIBOR steps of the generic shared-memory model
constexpr int LIBOR_MAX = MAX_DIM;  // longer: forward rates in global memory (ModelLiborBig)
constexpr int MBS_EXP_TERMS = 10;  // k0 exp(sigma_xi z) polynomial: z^0 .. z^9

enum Gen : int {
  GEN_RASRAP_RECURSIVE = 0,
  GEN_RASRAP_COUNTER = 1,
  GEN_PHILOX = 2,
  GEN_SOBOL_GRAY = 3,
  GEN_SOBOL_COUNTER = 4,
  GEN_SFC64 = 5,
  GEN_TWISTER = 6,  // MT19937 word stream (prng.py:40-82), one per replication
  GEN_XORWOW = 7,   // XORWOW word stream (prng.py:90-149), one per replication
  GEN_KAKUTANI = 8, // Kakutani orbits (halton.py:163-239, 521-542), one per (replication, dim)
};
constexpr int GEN_LAST = GEN_KAKUTANI;
__host__ __device__ constexpr bool gen_sequential(int g) {
  return g == GEN_TWISTER || g == GEN_XORWOW || g == GEN_KAKUTANI;
}
constexpr int KK_TAB = 64;  // Kakutani bracket table entries per base (halton.py:182, 64)
constexpr int MT_N = 624;       // MT19937 state words
constexpr int XW_JUMPS = 48;    // XORWOW jump matrices A^(2^k), k < XW_JUMPS
constexpr int XW_COLW = 8;      // words per matrix column (5 used, padded for 128-bit loads)
enum ModelKind : int {
  MODEL_LIBOR = 0,
  MODEL_MBS = 1,
  MODEL_X1 = 2,
  MODEL_CONST1 = 3,
  MODEL_POINTS = 4,  // internal: write the uniforms (sampler.fill of a sequential stream)
  MODEL_XHASH = 5,   // test integrand: hash of every coordinate's bits (rq_kernels.cu ModelHash)
};

// Per-dimension Halton constants (depend only on the d-th prime).  Offsets
// are prefix sums over dimensions 0..d-1, identical for every replication.
struct HaltonDim {
  int32_t base;     // d-th prime (halton.py:345-350)
  int32_t K;        // digit_capacity(base) (halton.py:59-66)
  int32_t cap;      // K + _CAP_PAD (halton.py:38, 262)
  int32_t ell;      // ceil(log2 base): division by base = (umulhi(t,mlo)+t) >> ell
  uint32_t mlo;     // low 32 bits of ceil(2^(32+ell)/base)
  int32_t sig_off;  // offset of sigma_d in a replication's sigma block (sum of bases)
  int32_t dig_off;  // offset of the start digits (sum of caps)
  int32_t sum_off;  // offset of partial sums / weight tables (sum of cap+1)
  uint64_t m64;     // floor(x / base) = umulhi64(x, m64) for x < 2^46
  uint32_t m16;     // floor(x / base) = umulhi(x, m16) for x < 2^16
  int32_t tdig;     // highest nonzero base-p digit position of the tile size (128)
  double inv_p;     // 1.0 / base
  double scale0;    // Python pow(inv_p, K): first init-sum weight (halton.py:274)
};

// Device view of one replication batch's randomisation tables.
struct RepTables {
  int gen;
  int dim;
  uint64_t seed;
  int64_t rep_first;   // replication id of local replication 0 (ids start at 1)
  int32_t rep_count;
  // Rasrap
  const uint16_t *sigma;   // [rep][sig_stride] digit permutations sigma_d
  const uint16_t *digits;  // [rep][dig_stride] base-p digits of the start index n0
  const double *sums;      // [rep][sum_stride] init partial sums (halton.py:273-278)
  const uint64_t *start;   // [rep][dim] start indices n0 (invert_radical, halton.py:139-155)
  int64_t sig_stride, dig_stride, sum_stride;
  int32_t sig_chunk_max;   // max over CHUNK-dim groups of the sigma entries they need
  // Sobol
  const uint32_t *sobol_v;     // [rep][dim][32] scrambled direction words
  const uint32_t *sobol_shift; // [rep][dim]
  // XORWOW: per-replication initial state (x, y, z, w, v, d) (prng.py:128-134)
  const uint32_t *xw_state;    // [rep][6]
  // Kakutani: random starts x0 (halton.py:532-534)
  const double *kk_x0;         // [rep][dim]
};

// Segments of the sequential word streams (MT19937 / XORWOW).  A
// replication's paths [p0, p0 + nmax) are cut into segments of seg_len paths;
// a segment is one unit of work for one CTA.  MT19937: the CTA shares one
// generator state, loaded from a snapshot taken by k_mt_snap at the
// segment's first word; XORWOW: every thread owns a run of consecutive
// paths and jumps its own state there with precomputed matrix powers.
struct SeqArgs {
  int64_t p0;          // first path of the range (sampler.fill cursor; 0 for estimates)
  int64_t nmax;        // paths in the range
  int64_t seg_len;     // paths per segment (multiple of the tile)
  int32_t segs_per_rep;
  const uint32_t *mt_snap;  // [rep - rep_local0][seg][MT_N] raw MT state after the twist that
                            // produced the segment's first word
  const double *kk_snap;    // Kakutani orbit points at segment starts, [rep - rep_local0][seg][dim]
                            // (tile layout) or at run starts, [rep - rep_local0][seg][TILE][dim]
  uint32_t *scratch;        // [gridDim][dim][TILE] tempered MT words (Kakutani: doubles) of a tile
};

struct ModelParams {
  int kind;
  int dim;
  double delta, sigma, strike, front_factor;          // LIBOR (models.py:301-322)
  double i0, k0, k1, k2, k3, k4, sigma_xi, payment;   // MBS (models.py:337-370)
  const double *table;  // device: LIBOR l0[dim] / MBS ck[dim]
  // MBS: k0 sigma_xi^k / k!, k < MBS_EXP_TERMS (the kernel's k0 exp(sigma_xi z)
  // for |z| <= exp_zlim = 0.1 / sigma_xi)
  double ecoef[MBS_EXP_TERMS];
  double exp_zlim;
  // LIBOR S > LIBOR_DYN_MAX: per-CTA forward-rate state [block][S][TILE]
  // (allocated by the launcher, stream-ordered)
  double *lstate;
};

// numpy pairwise-sum plan for one N (see rq_capi.cu build_plan).
struct SumPlan {
  int64_t n;
  int32_t nleaves, nnodes, nlevels;
  const int64_t *leaf_start;   // [nleaves]
  const int32_t *leaf_len;     // [nleaves]  (node id of leaf k is k)
  const int32_t *level_off;    // [nlevels+1] offsets into the internal-node arrays
  const int32_t *node_id, *node_l, *node_r;  // internal nodes grouped by height
  int32_t root;
};

// ---------------------------------------------------------------- launchers
cudaError_t upload_halton_dims(const HaltonDim *dims, int n, const double *wts,
                               const double *cscale, int nw);
cudaError_t launch_rasrap_setup(const RepTables &t, uint16_t *sigma, uint16_t *digits,
                                double *sums, uint64_t *start, cudaStream_t s,
                                const int *bases);  // host: the dims' bases
cudaError_t launch_sobol_setup(const RepTables &t, const uint32_t *v_dev, uint32_t *gen_v,
                               uint32_t *shift, cudaStream_t s);
cudaError_t launch_points(const RepTables &t, int rep_local, int64_t first,
                          const int64_t *idx, int64_t count, double *out, cudaStream_t s);
cudaError_t launch_paths(const RepTables &t, const ModelParams &mp, int rep_local0,
                         int rep_n, int64_t p0, int64_t nmax, double *payoffs, int *launched,
                         cudaStream_t s);
cudaError_t upload_xorwow_jumps(const uint32_t *cols, size_t words);
cudaError_t upload_kakutani_tables(const double *thr, const double *b, int dims);
cudaError_t launch_kakutani_setup(const RepTables &t, double *x0, cudaStream_t s);
cudaError_t launch_kak_snap(const RepTables &t, int rep_local0, int rep_n, const SeqArgs &q,
                            double *snap, cudaStream_t s);
constexpr int KK_RUNS_MAXDIM = 40;  // Kakutani: per-thread runs (orbit state in smem) up to this dim
__host__ __device__ constexpr bool kak_runs(int dim) { return dim <= KK_RUNS_MAXDIM; }
cudaError_t launch_xorwow_setup(const RepTables &t, uint32_t *state, cudaStream_t s);
// choose the segment length / grid of the sequential-stream path kernel
void seq_layout(const RepTables &t, const ModelParams &mp, int rep_n, int64_t nmax,
                int64_t *seg_len, int *segs_per_rep, int *blocks);
cudaError_t launch_mt_snap(const RepTables &t, int rep_local0, int rep_n, const SeqArgs &q,
                           uint32_t *snap, cudaStream_t s);
cudaError_t launch_paths_seq(const RepTables &t, const ModelParams &mp, int rep_local0,
                             int rep_n, int64_t nmax, const SeqArgs &q, int blocks,
                             double *payoffs, int *launched, cudaStream_t s);
cudaError_t launch_reduce(const SumPlan &plan, const double *payoffs, int64_t pay_stride,
                          int reps, double *theta, int theta_stride, double *scratch,
                          unsigned *tickets, cudaStream_t s);
cudaError_t launch_model_payoffs(const ModelParams &mp, const double *u, int64_t npaths,
                                 double *out, cudaStream_t s);
cudaError_t launch_inv_normal(const double *u, int64_t n, double *out, cudaStream_t s);
cudaError_t launch_stream_normals(const RepTables &t, int rep_local, int64_t npoints,
                                  double *block_sums, int nblocks, double *store,
                                  cudaStream_t s);
cudaError_t launch_dfma_peak(int blocks, int iters, double *sink, cudaStream_t s);
constexpr int PEAK_SLOTS_PER_ITER = 16 * 8;  // DFMA per thread per iteration of k_dfma_peak
int paths_grid_blocks(const RepTables &t, const ModelParams &mp);
int stream_grid_blocks(const RepTables &t);

}  // namespace rq
