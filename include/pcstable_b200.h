/*
 * pcstable_b200.h -- C ABI of the B200-native PC-stable skeleton library
 * (libpcstable_b200.so, built from paper_1812_08491_b200/csrc/).
 *
 * This is the drop-in boundary for the reference's hot path
 *   stats::compute_correlation  (proj/include/pcstable/stats.hpp:132)
 *   stats::threshold_tau        (proj/include/pcstable/stats.hpp:120)
 *   run_pc_stable               (proj/include/pcstable/skeleton.hpp:341)
 *   stats::ci_test / pseudo_inverse (stats.hpp:366, :172)  -- batch parity helpers
 * Plain pointers and sizes only.  Buffers are caller-allocated; calls are
 * synchronous; the library owns device memory for the duration of a call or
 * session.  include/pcstable_b200.hpp re-creates the reference's C++ names
 * (pcstable::run_pc_stable, SkeletonResult, ...) on top of this ABI, and maps
 * the status codes back to the reference's exception classes.
 *
 * Matrices: correlation matrices are p x p row-major (symmetric, so identical
 * to the reference's Eigen column-major storage); data matrices are m x p
 * column-major exactly like Eigen::MatrixXd in DataMatrix (core.hpp:48-67),
 * i.e. x[j*m + r] is sample r of variable j.
 */
#ifndef PCSTABLE_B200_H
#define PCSTABLE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCS_ABI_VERSION 1

typedef enum {
    PCS_OK = 0,
    PCS_EINVAL = 1,       /* std::invalid_argument: config (core.hpp:370-383), m < 4 (skeleton.hpp:344),
                             DataMatrix / CorrelationMatrix validation (core.hpp:50-95) */
    PCS_EZEROVAR = 2,     /* pcstable::ZeroVarianceError (core.hpp:23-31); column via zero_var_col */
    PCS_EOVERFLOW = 3,    /* std::overflow_error from comb::binomial (comb.hpp:43) */
    PCS_ENAN = 4,         /* std::invalid_argument thrown by stats::fisher_z on NaN (stats.hpp:112) */
    PCS_ECUDA = 5,        /* CUDA runtime failure or no device */
    PCS_ENOMEM = 6,
    PCS_EUNSUPPORTED = 7, /* conditioning level beyond the device path */
    PCS_ELEVEL = 8        /* pcstable::LevelUnreachableError (core.hpp:41-44): m - ell - 3 < 1 */
} pcs_status;

/* device variants of the level >= 1 CI-test kernels (both give identical results) */
enum { PCS_VARIANT_SET = 0 /* cuPC-S, paper Alg. 4 */, PCS_VARIANT_EDGE = 1 /* cuPC-E, paper Alg. 3 */ };
/* StopReason (skeleton.hpp:22) */
enum { PCS_STOP_MAX_DEGREE = 0, PCS_STOP_LEVEL_CAP = 1, PCS_STOP_SAMPLE_SIZE = 2 };

/* SkeletonConfig (core.hpp:357-384) + device fields */
typedef struct {
    double alpha;              /* (0, 1) */
    int32_t max_level;         /* -1: no cap */
    int32_t variant;           /* PCS_VARIANT_* (replaces Strategy) */
    int32_t edges_per_unit;    /* beta: tuning hint, results never depend on it */
    int32_t workers_per_edge;  /* gamma: tuning hint */
    int32_t set_groups;        /* delta: tuning hint */
    int32_t unit_width;        /* theta: tuning hint */
    int32_t device;            /* CUDA device ordinal */
    int32_t shard_index;       /* multi-GPU session: this rank (0 for single GPU) */
    int32_t shard_count;       /* multi-GPU session: world size (1 for single GPU) */
    int32_t reserved0;
    uint64_t stream;           /* cudaStream_t to run on (0: the library creates its own) */
    int32_t reserved[4];
} pcs_config;

/* LevelStats (core.hpp:387-393) + device counters */
typedef struct {
    int32_t level;
    int32_t pad;
    uint64_t ci_tests;                /* == Strategy::Serial's LevelStats::ci_tests */
    uint64_t pseudo_inverses;         /* == Strategy::Serial's LevelStats::pseudo_inverses */
    uint64_t edges_removed;
    double elapsed_s;                 /* host wall time of the level (includes compaction) */
    uint64_t device_ci_tests;         /* CI tests the device actually executed */
    uint64_t device_pseudo_inverses;  /* (row, set) pseudo-inverses the device's CI tests used (computed per
                                         set, or read from the level's l = 2, 3 table) */
    double kernel_ms;                 /* CUDA-event time of the level's CI-test kernels */
    uint64_t device_exact_tests;      /* tests whose statistic the device evaluated (in the reference's
                                         operation order); the rest of device_ci_tests were decided
                                         without arithmetic (set with h00 == 0: degenerate) */
    uint64_t device_near_threshold;   /* tests whose statistic fell inside the +-1e-9 band around the
                                         threshold (or was tiny) and were decided by the exact
                                         fisher_z comparison (stats.hpp:345-351) -- listed, not hidden */
} pcs_level_stats;

typedef struct pcs_result pcs_result;
typedef struct pcs_session pcs_session;

const char* pcs_version(void);
const char* pcs_last_error(void); /* thread-local message of the last failure */
unsigned long long pcs_kernel_launches(void); /* kernels launched by this library so far */
/* measured FP64 FMA peak of the current device in TFLOP/s (roofline denominator of the CI kernels) */
int pcs_probe_fp64_tflops(double* tflops);
void pcs_config_default(pcs_config* cfg);

/* stats::threshold_tau (stats.hpp:120-129); PCS_EINVAL for bad alpha/ell, PCS_ELEVEL for m - ell - 3 < 1 */
pcs_status pcs_threshold_tau(double alpha, int32_t m, int32_t ell, double* tau);

/* stats::compute_correlation (stats.hpp:132-156) on the device.  x: m x p column-major host buffer. */
pcs_status pcs_correlation(const double* x, int32_t m, int32_t p, double* c_out, int32_t* zero_var_col);

/* run_pc_stable (skeleton.hpp:341-391).  c: p x p host correlation matrix, validated and normalised
   exactly like the CorrelationMatrix constructor (core.hpp:73-95). */
pcs_status pcs_run_pc_stable(const double* c, int32_t p, int32_t m, const pcs_config* cfg, pcs_result** out);
/* One level on a given live graph (skeleton.hpp:262-333: run_level_zero for ell = 0, run_level_serial /
   run_level_edge_parallel / run_level_set_shared for ell >= 1 by cfg->variant): graph_cells is the p x p
   symmetric 0/1 adjacency (core.hpp:109-194) and doubles as the level-start snapshot (compact(),
   core.hpp:227-239); tau is the caller's threshold; graph_cells is updated in place and *out holds the
   level's LevelStats (one entry) and the sepsets of the pairs it removed.  Counters follow
   Strategy::Serial's definition for every variant (include/pcstable_b200.hpp). */
pcs_status pcs_run_level(const double* c, int32_t p, int32_t ell, double tau, const pcs_config* cfg,
                         uint8_t* graph_cells, pcs_result** out);
/* compute_correlation from device-resident m x p column-major data into a device p x ldc buffer,
   enqueued on `stream` (0 = legacy default stream); synchronous */
pcs_status pcs_correlation_device(const double* d_x, int32_t m, int32_t p, double* d_c, int64_t ldc, uint64_t stream,
                                  int32_t* zero_var_col);
/* rows [row_begin, row_end) of the same matrix only (the other rows of d_c are not written): the
   multi-GPU split of stats.hpp:132-156 -- each rank builds its row band, the bands are all-gathered;
   bit-identical to the rows pcs_correlation_device writes */
pcs_status pcs_correlation_device_rows(const double* d_x, int32_t m, int32_t p, int32_t row_begin, int32_t row_end,
                                       double* d_c, int64_t ldc, uint64_t stream, int32_t* zero_var_col);
/* compute_correlation + run_pc_stable from m x p column-major host data (one device pipeline) */
pcs_status pcs_run_pc_stable_data(const double* x, int32_t m, int32_t p, const pcs_config* cfg, pcs_result** out,
                                  int32_t* zero_var_col);
/* same, with the m x p column-major data already in device memory */
pcs_status pcs_run_pc_stable_data_device(const double* d_x, int32_t m, int32_t p, const pcs_config* cfg,
                                         pcs_result** out, int32_t* zero_var_col);
/* same as pcs_run_pc_stable with the correlation matrix already in device memory (row stride ldc) */
pcs_status pcs_run_pc_stable_device(const double* d_c, int64_t ldc, int32_t p, int32_t m, const pcs_config* cfg,
                                    pcs_result** out);

/* SkeletonResult accessors (skeleton.hpp:33-40) */
int32_t pcs_result_p(const pcs_result* r);
int32_t pcs_result_levels(const pcs_result* r, pcs_level_stats* out, int32_t cap);
int32_t pcs_result_stop_reason(const pcs_result* r);
void pcs_result_adjacency(const pcs_result* r, uint8_t* out /* p*p, row-major */);
int64_t pcs_result_edge_count(const pcs_result* r);
void pcs_result_edge_list(const pcs_result* r, int32_t* out /* 2*edge_count, (i<j) ascending */);
int64_t pcs_result_member_total(const pcs_result* r);
/* per unordered pair, triangular slot index of core.hpp:329-335: level (-1 = kept), offset into members */
void pcs_result_sepsets(const pcs_result* r, int32_t* level, int64_t* offset, int32_t* members);
double pcs_result_device_seconds(const pcs_result* r); /* CUDA-event time of the whole device pipeline */
/* Near-threshold tests (BASELINE parity protocol: "listed, not hidden"): every CI decision whose
   statistic fell inside the +-1e-9 band around the threshold and was taken by the exact fisher_z
   comparison (stats.hpp:345-351).  These are the only decisions that could differ from the reference's
   if a libm log differed in the last ulp.  count = all of the run, records = the first 4096. */
typedef struct {
    int32_t level, i, j;     /* level, tested row i and target j (unordered pair for level 0) */
    int32_t independent;     /* the decision */
    double rho, z;           /* the partial correlation and fisher_z(rho); tau is threshold_tau(level) */
} pcs_near_record;
int64_t pcs_result_near_count(const pcs_result* r);
int64_t pcs_result_near_records(const pcs_result* r, pcs_near_record* out, int64_t cap);
/* compact forms: live bitmask p x ceil(p/32) uint32 (bit j of word i*W + j/32), and the removal records
   of levels >= 1 as consecutive (a, b, ell, members[ell]) int32 tuples (level-0 removals are implied) */
void pcs_result_bitmask(const pcs_result* r, uint32_t* out);
int64_t pcs_result_record_ints(const pcs_result* r);
void pcs_result_records(const pcs_result* r, int32_t* out);
void pcs_result_free(pcs_result* r);

/* stats::ci_test for n tests of one level ell on the device (parity helper).
   ij: 2n ints, sets: n*ell ints (ascending members).  Outputs per test. */
pcs_status pcs_ci_test_batch(const double* c, int32_t p, int32_t ell, int64_t n, const int32_t* ij,
                             const int32_t* sets, double tau, uint8_t* independent, double* z, double* rho,
                             uint8_t* degenerate);
/* stats::pseudo_inverse for n row-major ell x ell blocks on the device (parity helper) */
pcs_status pcs_pseudo_inverse_batch(const double* a, int32_t ell, int64_t n, double* out);

/* Benchmark-input generation, bit-identical to the reference generator (host, sequential by
   construction): random_dag (datagen.hpp:42-56) -> weights n x n row-major (weights[i*n+j] != 0:
   j causes i, j < i); sample_linear_gaussian (datagen.hpp:62-82) -> x m x n column-major. */
pcs_status pcs_random_dag(int32_t n, double density, uint64_t seed, double* weights);
pcs_status pcs_sample_linear_gaussian(const double* weights, int32_t n, int32_t m, uint64_t seed, double* x);
/* The reference generator's noise stream (rng.hpp: xoshiro256++ / Marsaglia polar, one normal per
   (sample, variable) in sample-major order): the first `count` normals of Xoshiro256PlusPlus(seed),
   normal n stored at out[(n % p) * m + n / p], generated in jump-ahead chunks on the host threads
   (GF(2) jump matrix; bit-identical to the sequential stream) */
pcs_status pcs_noise_stream(uint64_t seed, int64_t count, int32_t p, int32_t m, double* out);
/* sample_linear_gaussian (datagen.hpp:62-82) into device memory d_x (m x n column-major): the noise
   stream above, then the structural equations on the device (thread per sample, parents ascending);
   rescaled != 0: pcs_sample_linear_gaussian_rescaled's overflow-safe variant (cooperative grid;
   log_scale: host array of n, may be null).  Bit-identical to the host generators. */
pcs_status pcs_sample_linear_gaussian_device(const double* weights, int32_t n, int32_t m, uint64_t seed,
                                             int32_t rescaled, double* d_x, double* log_scale, uint64_t stream);
/* Overflow-safe sample_linear_gaussian for the scaling shapes (no reference counterpart):
 * same noise stream, every variable scaled to unit RMS, log_scale[n] = log of the reference variable's RMS,
 * so x_ref[i] = x[i] * exp(log_scale[i]) and the correlation matrix is the reference generator's. */
pcs_status pcs_sample_linear_gaussian_rescaled(const double* weights, int32_t n, int32_t m, uint64_t seed, double* x,
                                               double* log_scale);

/* Level-stepped session: the building block of multi-GPU runs (one process per GPU, the caller
   all-reduces the per-level key array with MIN between passes).  pcs_run_pc_stable is a session
   with shard_count = 1. */
pcs_status pcs_session_create(const double* c, int32_t p, int32_t m, const pcs_config* cfg, pcs_session** out);
pcs_status pcs_session_create_device(const double* d_c, int64_t ldc, int32_t p, int32_t m, const pcs_config* cfg,
                                     pcs_session** out);
/* starts the next level; *running = 0 once the loop has stopped (stop reason recorded) */
pcs_status pcs_session_level_begin(pcs_session* s, int32_t* running, int32_t* ell, int64_t* num_keys);
/* pass 0: edges tested from their lower endpoint's row; pass 1: from the upper endpoint's row.
   cuPC-S levels >= 2 (register-template kernel) test both directions in pass 0 and pass 1 is empty. */
pcs_status pcs_session_level_pass(pcs_session* s, int32_t pass);
/* number of passes the current level needs (1 when pass 0 covers both directions, else 2): a
   multi-GPU caller MIN-reduces the keys after each of them */
pcs_status pcs_session_level_passes(pcs_session* s, int32_t* passes);
/* device pointer to the level's int64 key array (num_keys entries; MIN-reduce across ranks) */
pcs_status pcs_session_keys(pcs_session* s, void** device_ptr, int64_t* count);
pcs_status pcs_session_level_end(pcs_session* s);
/* re-shard subsequent passes (multi-GPU rebalancing, profiling of a slice) */
pcs_status pcs_session_set_shard(pcs_session* s, int32_t shard_index, int32_t shard_count);
/* CSR snapshot of the current level (compact(), core.hpp:227-239): offsets[p+1], indices[offsets[p]] */
pcs_status pcs_session_snapshot(pcs_session* s, int32_t* offsets, int32_t* indices);
pcs_status pcs_session_finish(pcs_session* s, pcs_result** out);
void pcs_session_free(pcs_session* s);

/* ---- orientation (orient.hpp) ----
 * MixedGraph (orient.hpp:15-32): directed (from, to) pairs and undirected (a < b) pairs, both ascending
 * (the reference's std::set order).  stage 1 = find_v_structures (orient.hpp:40-89, device kernel),
 * 2 = apply_meek_rules (orient.hpp:147-167, host fixed point in the reference's visiting order),
 * 3 = orient_skeleton (orient.hpp:170-173).  PCS_EINVAL when a consulted nonadjacent pair has no
 * separating set (the reference's std::invalid_argument, orient.hpp:60-63). */
typedef struct pcs_mixed_graph pcs_mixed_graph;
/* on a device result (its skeleton and sepsets; level-0 removals carry S = {}) */
pcs_status pcs_orient_result(const pcs_result* r, int32_t stage, pcs_mixed_graph** out);
/* on the compact result form: live bitmask p x ceil(p/32) and the (a, b, ell, members) records */
pcs_status pcs_orient_records(int32_t p, const uint32_t* bitmask, const int32_t* records, int64_t record_ints,
                              int32_t stage, pcs_mixed_graph** out);
/* on caller data: skeleton p*p uint8 (symmetric) and sepsets in pcs_result_sepsets' triangular layout
 * (level -1 = no separating set).  With stage 2 the input mixed graph is directed_in (pairs) plus every
 * other skeleton edge undirected. */
pcs_status pcs_orient_skeleton(int32_t p, const uint8_t* adj, const int32_t* sep_level, const int64_t* sep_offset,
                               const int32_t* members, int32_t stage, const int32_t* directed_in,
                               int64_t n_directed_in, pcs_mixed_graph** out);
int64_t pcs_mixed_directed_count(const pcs_mixed_graph* g);
int64_t pcs_mixed_undirected_count(const pcs_mixed_graph* g);
void pcs_mixed_directed(const pcs_mixed_graph* g, int32_t* pairs /* 2 * count */);
void pcs_mixed_undirected(const pcs_mixed_graph* g, int32_t* pairs /* 2 * count */);
void pcs_mixed_free(pcs_mixed_graph* g);

#ifdef __cplusplus
}
#endif
#endif /* PCSTABLE_B200_H */
