/*
 * pcs_oracle.h -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement, in plain C11, of the reference PC-stable skeleton path
 * (/root/reference/proj/include/pcstable/{rng,datagen,comb,stats,core,skeleton}.hpp).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load the shared library built from this file.
 *
 * Parity status: the reference cannot be built in this container (Eigen3,
 * GoogleTest and CLI11 are absent).  This restatement is
 * pinned against every known-answer test and golden value the reference's
 * own test-suite holds for the path (tests/test_oracle_*.py), and the
 * decisions that involve only exact or commutative arithmetic (level 0 and
 * level 1, which cover the bulk of all tests) are bit-identical to the
 * reference by construction.  Eigen-internal summation order inside the
 * |S| >= 3 small products is NOT pinned (documented in DESIGN.md).
 *
 * Two additions serve the whole-run fixtures (tests/golden, tools/make_golden.py):
 *  - ORC_FAST: Strategy::Serial's result computed set-shared (one pseudo-inverse
 *    per (row, set), lanes over the row's targets, the same per-test operation
 *    sequence); result-identical to ORC_SERIAL (tests/test_oracle_fast.py);
 *  - orc_compute_correlation_fma: compute_correlation in the device's pinned
 *    order (tree column means, FMA-chain Gram over k), the order the reference
 *    leaves to Eigen; the device's matrix equals it bit for bit.
 */
#ifndef PCS_ORACLE_H
#define PCS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: mirror the reference's exception classes */
enum {
    ORC_OK = 0,
    ORC_EINVAL = 1,        /* std::invalid_argument */
    ORC_EZEROVAR = 2,      /* pcstable::ZeroVarianceError */
    ORC_EOVERFLOW = 3,     /* std::overflow_error (binomial) */
    ORC_ENAN = 4,          /* std::invalid_argument thrown by fisher_z on NaN rho */
    ORC_ELEVEL = 5,        /* pcstable::LevelUnreachableError (internal) */
    ORC_ENOMEM = 6
};

/* ORC_KEYS: serial-rule keys, one pseudo-inverse per test (test_edge_over_sets order).
 * ORC_FAST: the same keys by set-shared evaluation (one pseudo-inverse per (row, set),
 *           lane-parallel over targets); result-identical to ORC_SERIAL. */
enum { ORC_SERIAL = 0, ORC_EDGE = 1, ORC_SET = 2, ORC_KEYS = 3, ORC_FAST = 4 };
enum { ORC_STOP_MAX_DEGREE = 0, ORC_STOP_LEVEL_CAP = 1, ORC_STOP_SAMPLE_SIZE = 2 };

const char* orc_last_error(void);

/* ---- rng.hpp ---- */
typedef struct {
    uint64_t s[4];
    double spare;
    int has_spare;
} orc_xoshiro;
void orc_xo_seed(orc_xoshiro* g, uint64_t seed);
uint64_t orc_xo_next(orc_xoshiro* g);
double orc_xo_uniform01(orc_xoshiro* g);
double orc_xo_normal(orc_xoshiro* g);
/* fill out[n] with successive normal() draws of a fresh generator */
void orc_normals(uint64_t seed, double* out, int64_t n);
void orc_raw(uint64_t seed, uint64_t* out, int64_t n);

/* ---- datagen.hpp ---- weights row-major n*n (weights[i*n+j] : j causes i, j<i) */
int orc_random_dag(int n, double density, uint64_t seed, double* weights);
/* data column-major m x n (x[j*m + r]) like Eigen::MatrixXd */
int orc_sample_linear_gaussian(const double* weights, int n, int m, uint64_t seed, double* x);

/* ---- comb.hpp ---- */
int orc_binomial(int n, int k, uint64_t* out);
int orc_unrank_positions(int width, int ell, uint64_t t, int32_t* out);
int orc_unrank_positions_excluding(int reduced_width, int ell, uint64_t t, int skip, int32_t* out);
int orc_next_combination(int32_t* positions, int ell, int width);

/* ---- stats.hpp ---- */
int orc_normal_quantile(double p, double* out);
int orc_fisher_z(double rho, double* out);
int orc_threshold_tau(double alpha, int m, int ell, double* out);
/* x column-major m x p; c_out row-major p x p; *zero_col set on ORC_EZEROVAR */
int orc_compute_correlation(const double* x, int m, int p, double* c_out, int* zero_col, int threads);
/* the same in the device's pinned order: tree column means, FMA-chain Gram over k, k extent padded
 * to a multiple of kpad (0: none) -- see pcs_oracle.c */
int orc_compute_correlation_fma(const double* x, int m, int p, int kpad, double* c, int* zero_col, int threads);
/* CorrelationMatrix constructor: validate + symmetrise + clamp in place (core.hpp:73-95) */
int orc_correlation_normalize(double* c, int p);
/* a, out row-major n x n */
int orc_pseudo_inverse(const double* a, int n, double* out);
int orc_partial_correlation(const double* c, int p, int i, int j, const int32_t* set, int ell,
                            double* rho, int* degenerate);
int orc_ci_test(const double* c, int p, int i, int j, const int32_t* set, int ell, double tau,
                int* independent, double* z, double* rho, int* degenerate);

/* ---- skeleton.hpp ---- */
typedef struct {
    double alpha;
    int max_level;         /* -1: none */
    int strategy;          /* ORC_SERIAL / ORC_EDGE / ORC_SET / ORC_KEYS */
    int edges_per_unit;    /* beta */
    int workers_per_edge;  /* gamma (inert) */
    int set_groups;        /* delta */
    int unit_width;        /* theta */
    int worker_count;
    int has_schedule_seed;
    uint64_t schedule_seed;
} orc_config;

typedef struct {
    int32_t level;
    int32_t pad;
    uint64_t ci_tests;
    uint64_t pseudo_inverses;
    uint64_t edges_removed;
    double elapsed_s;
} orc_level_stats;

typedef struct orc_result orc_result;

void orc_config_default(orc_config* cfg);
int orc_run_pc_stable(const double* c, int p, int m, const orc_config* cfg, orc_result** out);
int orc_result_p(const orc_result* r);
int orc_result_levels(const orc_result* r, orc_level_stats* out, int cap);
int orc_result_stop_reason(const orc_result* r);
void orc_result_adjacency(const orc_result* r, uint8_t* out);
int64_t orc_result_member_total(const orc_result* r);
/* per unordered pair slot (triangular index, core.hpp:329-335): level (-1 none), offset into members */
void orc_result_sepsets(const orc_result* r, int32_t* level, int64_t* offset, int32_t* members);
void orc_result_free(orc_result* r);

/*
 * Serial-rule keys for one level (Appendix B of SURVEY.md): for every
 * undirected snapshot edge e (a<b, CSR order) with index in [e_begin, e_end):
 *   key = (dir << 62) | reduced_rank of the first separating set, or INT64_MAX.
 * Snapshot: offsets[p+1], indices[] ascending rows (core.hpp:200-239).
 */
int orc_level_keys(const double* c, int p, const int32_t* offsets, const int32_t* indices, int ell,
                   double tau, int64_t e_begin, int64_t e_end, int64_t* keys, int threads);

/* the same keys as orc_level_keys over ALL edges of the snapshot, by set-shared evaluation */
int orc_level_keys_fast(const double* c, int p, const int32_t* offsets, const int32_t* indices, int ell,
                        double tau, int64_t* keys, int threads);

/* one level on a given snapshot, rows [row_begin, row_end) only (bounded CPU sample) */
int orc_run_level(const double* c, int p, const int32_t* offsets, const int32_t* indices, int ell, double tau,
                  const orc_config* cfg, int row_begin, int row_end, orc_level_stats* out);

/* the SET level on rows [row_begin, row_end) running only every keep_stride-th unit chunk (a spread
 * 1/keep_stride of each row's sets): bench.py's reference-arm sampler of rows too heavy to run whole */
int orc_run_level_sampled(const double* c, int p, const int32_t* offsets, const int32_t* indices, int ell, double tau,
                          const orc_config* cfg, int row_begin, int row_end, int keep_stride, orc_level_stats* out);

/* ---- orient.hpp (pcs_orient_oracle.c) ----
 * stage bit 1: find_v_structures, bit 2: apply_meek_rules (3 = orient_skeleton).  With bit 1 clear
 * the input mixed graph is directed_in + every other skeleton edge undirected.  Outputs ascending
 * pairs; buffers hold n*(n-1)/2 pairs.  ORC_EINVAL: a consulted nonadjacent pair has no sepset. */
int orc_orient(int n, const uint8_t* skeleton, const int32_t* sep_level, const int64_t* sep_offset,
               const int32_t* members, int stage, const int32_t* directed_in, int64_t n_directed_in,
               int32_t* dir_out, int64_t* n_dir, int32_t* und_out, int64_t* n_und);

#ifdef __cplusplus
}
#endif
#endif
