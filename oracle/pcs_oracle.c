/*
 * pcs_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the reference
 * PC-stable skeleton path; see pcs_oracle.h for scope and parity status.
 *
 * Every function cites the reference lines it restates.  Floating point is
 * evaluated in the reference's operation order with no FMA contraction (the
 * Makefile builds with -ffp-contract=off and no -march, like the reference's
 * Release build, proj/CMakeLists.txt:7-9).  For the Eigen library calls the
 * reference makes (GEMM, GEMV, LLT, triangular solve) the order is the
 * straightforward left-to-right order documented in DESIGN.md section
 * "Oracle canonical order"; the device kernels follow the same order.
 */
#define _GNU_SOURCE
#include "pcs_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static _Thread_local char g_err[256];
static void set_err(const char* msg) {
    strncpy(g_err, msg, sizeof g_err - 1);
    g_err[sizeof g_err - 1] = 0;
}
const char* orc_last_error(void) { return g_err; }

#define NONE_KEY INT64_MAX
static double now_s(void);

/* ===================================================== rng.hpp:10-81 ===== */
static uint64_t splitmix_next(uint64_t* st) { /* rng.hpp:14-19 */
    uint64_t z = (*st += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
static inline uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

void orc_xo_seed(orc_xoshiro* g, uint64_t seed) { /* rng.hpp:31-34 */
    uint64_t st = seed;
    for (int w = 0; w < 4; ++w) g->s[w] = splitmix_next(&st);
    g->spare = 0.0;
    g->has_spare = 0;
}
uint64_t orc_xo_next(orc_xoshiro* g) { /* rng.hpp:36-46 */
    uint64_t* s = g->s;
    const uint64_t result = rotl64(s[0] + s[3], 23) + s[0];
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}
double orc_xo_uniform01(orc_xoshiro* g) { /* rng.hpp:49 */
    return (double)(orc_xo_next(g) >> 11) * 0x1.0p-53;
}
static double xo_uniform(orc_xoshiro* g, double lo, double hi) { /* rng.hpp:52 */
    return lo + (hi - lo) * orc_xo_uniform01(g);
}
double orc_xo_normal(orc_xoshiro* g) { /* rng.hpp:58-73, Marsaglia polar */
    if (g->has_spare) {
        g->has_spare = 0;
        return g->spare;
    }
    double u, v, s;
    do {
        u = 2.0 * orc_xo_uniform01(g) - 1.0;
        v = 2.0 * orc_xo_uniform01(g) - 1.0;
        s = u * u + v * v;
    } while (s >= 1.0 || s == 0.0);
    const double scale = sqrt(-2.0 * log(s) / s);
    g->spare = v * scale;
    g->has_spare = 1;
    return u * scale;
}
void orc_normals(uint64_t seed, double* out, int64_t n) {
    orc_xoshiro g;
    orc_xo_seed(&g, seed);
    for (int64_t k = 0; k < n; ++k) out[k] = orc_xo_normal(&g);
}
void orc_raw(uint64_t seed, uint64_t* out, int64_t n) {
    orc_xoshiro g;
    orc_xo_seed(&g, seed);
    for (int64_t k = 0; k < n; ++k) out[k] = orc_xo_next(&g);
}

/* ================================================= datagen.hpp:42-82 ===== */
int orc_random_dag(int n, double density, uint64_t seed, double* w) {
    if (n < 2) { set_err("random_dag: need n >= 2"); return ORC_EINVAL; }
    if (!(density > 0.0 && density < 1.0)) {
        set_err("random_dag: density must lie in (0, 1)");
        return ORC_EINVAL;
    }
    memset(w, 0, sizeof(double) * (size_t)n * n);
    orc_xoshiro g;
    orc_xo_seed(&g, seed);
    for (int i = 1; i < n; ++i)         /* datagen.hpp:51-53: row by row */
        for (int j = 0; j < i; ++j)
            if (orc_xo_uniform01(&g) < density) w[(size_t)i * n + j] = xo_uniform(&g, 0.1, 1.0);
    return ORC_OK;
}

int orc_sample_linear_gaussian(const double* w, int n, int m, uint64_t seed, double* x) {
    if (m < 4) { set_err("sample_linear_gaussian: need m >= 4"); return ORC_EINVAL; }
    if (n < 2) { set_err("sample_linear_gaussian: malformed dag"); return ORC_EINVAL; }
    for (int i = 0; i < n; ++i)
        for (int j = i; j < n; ++j)
            if (w[(size_t)i * n + j] != 0.0) {
                set_err("sample_linear_gaussian: weights must be strictly lower triangular");
                return ORC_EINVAL;
            }
    /* parent lists in ascending cause order: same additions as datagen.hpp:75-78 */
    int64_t* start = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
    int64_t nnz = 0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < i; ++j) nnz += w[(size_t)i * n + j] != 0.0;
    int32_t* par = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nnz + 1));
    double* pw = (double*)malloc(sizeof(double) * (size_t)(nnz + 1));
    if (!start || !par || !pw) { free(start); free(par); free(pw); set_err("oom"); return ORC_ENOMEM; }
    nnz = 0;
    for (int i = 0; i < n; ++i) {
        start[i] = nnz;
        for (int j = 0; j < i; ++j)
            if (w[(size_t)i * n + j] != 0.0) { par[nnz] = j; pw[nnz] = w[(size_t)i * n + j]; ++nnz; }
    }
    start[n] = nnz;
    orc_xoshiro g;
    orc_xo_seed(&g, seed);
    for (int r = 0; r < m; ++r) {
        for (int i = 0; i < n; ++i) {
            double value = orc_xo_normal(&g);
            for (int64_t e = start[i]; e < start[i + 1]; ++e)
                value += pw[e] * x[(size_t)par[e] * m + r];
            x[(size_t)i * m + r] = value;
        }
    }
    free(start); free(par); free(pw);
    return ORC_OK;
}

/* ===================================================== comb.hpp:18-118 ==== */
static uint64_t g_pascal[65][65];
static pthread_once_t g_pascal_once = PTHREAD_ONCE_INIT;
static void pascal_init(void) { /* comb.hpp:18-28 */
    for (int n = 0; n < 65; ++n) {
        g_pascal[n][0] = 1;
        for (int k = 1; k <= n; ++k) g_pascal[n][k] = g_pascal[n - 1][k - 1] + (k <= n - 1 ? g_pascal[n - 1][k] : 0);
    }
}

int orc_binomial(int n, int k, uint64_t* out) { /* comb.hpp:35-46 */
    pthread_once(&g_pascal_once, pascal_init);
    if (n < 0 || k < 0 || k > n) { set_err("binomial: need 0 <= k <= n"); return ORC_EINVAL; }
    if (n < 65) { *out = g_pascal[n][k]; return ORC_OK; }
    if (n - k < k) k = n - k;
    unsigned __int128 result = 1;
    for (int i = 1; i <= k; ++i) {
        result = result * (unsigned)(n - k + i) / (unsigned)i;
        if (result > (unsigned __int128)UINT64_MAX) {
            set_err("binomial: C(n, k) exceeds 64 bits");
            return ORC_EOVERFLOW;
        }
    }
    *out = (uint64_t)result;
    return ORC_OK;
}

int orc_unrank_positions(int width, int ell, uint64_t t, int32_t* out) { /* comb.hpp:50-67 */
    if (width < ell || ell < 0) { set_err("unrank: need width >= k >= 0"); return ORC_EINVAL; }
    uint64_t total;
    int rc = orc_binomial(width, ell, &total);
    if (rc) return rc;
    if (t >= total) { set_err("unrank: rank out of range"); return ORC_EINVAL; }
    uint64_t covered = 0;
    int value = 0;
    for (int c = 0; c < ell; ++c) {
        uint64_t block;
        if ((rc = orc_binomial(width - value - 1, ell - c - 1, &block))) return rc;
        while (covered + block <= t) {
            covered += block;
            ++value;
            if ((rc = orc_binomial(width - value - 1, ell - c - 1, &block))) return rc;
        }
        out[c] = value;
        ++value;
    }
    return ORC_OK;
}

int orc_unrank_positions_excluding(int reduced_width, int ell, uint64_t t, int skip, int32_t* out) {
    /* comb.hpp:87-94 */
    if (skip < 0 || skip > reduced_width) { set_err("unrank: skip position out of range"); return ORC_EINVAL; }
    int rc = orc_unrank_positions(reduced_width, ell, t, out);
    if (rc) return rc;
    for (int k = 0; k < ell; ++k)
        if (out[k] >= skip) ++out[k];
    return ORC_OK;
}

int orc_next_combination(int32_t* pos, int ell, int width) { /* comb.hpp:108-118 */
    for (int idx = ell - 1; idx >= 0; --idx) {
        if (pos[idx] < width - (ell - idx)) {
            ++pos[idx];
            for (int k = idx + 1; k < ell; ++k) pos[k] = pos[k - 1] + 1;
            return 1;
        }
    }
    return 0;
}

/* ================================================== stats.hpp:19-129 ===== */
/* Wichura AS 241 (PPND16): published coefficients, Horner order as stats.hpp:25-106 */
static const double AS241_A[8] = {3.3871328727963666080e0, 1.3314166789178437745e2, 1.9715909503065514427e3,
                                  1.3731693765509461125e4, 4.5921953931549871457e4, 6.7265770927008700853e4,
                                  3.3430575583588128105e4, 2.5090809287301226727e3};
static const double AS241_B[8] = {1.0, 4.2313330701600911252e1, 6.8718700749205790830e2,
                                  5.3941960214247511077e3, 2.1213794301586595867e4, 3.9307895800092710610e4,
                                  2.8729085735721942674e4, 5.2264952788528545610e3};
static const double AS241_C[8] = {1.42343711074968357734e0, 4.63033784615654529590e0, 5.76949722146069140550e0,
                                  3.64784832476320460504e0, 1.27045825245236838258e0, 2.41780725177450611770e-1,
                                  2.27238449892691845833e-2, 7.74545014278341407640e-4};
static const double AS241_D[8] = {1.0, 2.05319162663775882187e0, 1.67638483018380384940e0,
                                  6.89767334985100004550e-1, 1.48103976427480074590e-1, 1.51986665636164571966e-2,
                                  5.47593808499534494600e-4, 1.05075007164441684324e-9};
static const double AS241_E[8] = {6.65790464350110377720e0, 5.46378491116411436990e0, 1.78482653991729133580e0,
                                  2.96560571828504891230e-1, 2.65321895265761230930e-2, 1.24266094738807843860e-3,
                                  2.71155556874348757815e-5, 2.01033439929228813265e-7};
static const double AS241_F[8] = {1.0, 5.99832206555887937690e-1, 1.36929880922735805310e-1,
                                  1.48753612908506148525e-2, 7.86869131145613259100e-4, 1.84631831751005468180e-5,
                                  1.42151175831644588870e-7, 2.04426310338993978564e-15};
static double horner7(const double* k, double r) { /* (((((((k7 r + k6) r + k5) ... ) r + k0 */
    double acc = k[7] * r + k[6];
    for (int d = 5; d >= 0; --d) acc = acc * r + k[d];
    return acc;
}

int orc_normal_quantile(double p, double* out) { /* stats.hpp:19-108 */
    if (!(p > 0.0 && p < 1.0)) { set_err("normal_quantile: p must lie in (0, 1)"); return ORC_EINVAL; }
    const double q = p - 0.5;
    if (fabs(q) <= 0.425) {
        const double r = 0.180625 - q * q;
        *out = q * horner7(AS241_A, r) / horner7(AS241_B, r);
        return ORC_OK;
    }
    double r = q < 0.0 ? p : 1.0 - p;
    r = sqrt(-log(r));
    double z;
    if (r <= 5.0) {
        r -= 1.6;
        z = horner7(AS241_C, r) / horner7(AS241_D, r);
    } else {
        r -= 5.0;
        z = horner7(AS241_E, r) / horner7(AS241_F, r);
    }
    *out = q < 0.0 ? -z : z;
    return ORC_OK;
}

int orc_fisher_z(double rho, double* out) { /* stats.hpp:111-115 */
    if (!(rho > -1.0 && rho < 1.0)) { set_err("fisher_z: rho must lie in (-1, 1)"); return ORC_ENAN; }
    *out = fabs(0.5 * log((1.0 + rho) / (1.0 - rho)));
    return ORC_OK;
}

int orc_threshold_tau(double alpha, int m, int ell, double* out) { /* stats.hpp:120-129 */
    if (!(alpha > 0.0 && alpha <= 1.0)) { set_err("threshold_tau: alpha must lie in (0, 1]"); return ORC_EINVAL; }
    if (ell < 0) { set_err("threshold_tau: ell must be >= 0"); return ORC_EINVAL; }
    const double dof = (double)m - ell - 3;
    if (dof < 1.0) { set_err("threshold_tau: need m - ell - 3 >= 1"); return ORC_ELEVEL; }
    double q;
    int rc = orc_normal_quantile(1.0 - alpha / 2.0, &q);
    if (rc) return rc;
    *out = q / sqrt(dof);
    return ORC_OK;
}

/* ---- compute_correlation (stats.hpp:132-156), row-parallel (results thread-count independent) */
typedef struct {
    const double* xc;
    int m, p;
    double* gram;
    atomic_int next;
} corr_job;
static void* corr_worker(void* arg) {
    corr_job* J = (corr_job*)arg;
    const int m = J->m, p = J->p;
    for (;;) {
        const int i = atomic_fetch_add(&J->next, 1);
        if (i >= p) break;
        const double* a = J->xc + (size_t)i * m;
        for (int j = i; j < p; ++j) {
            const double* b = J->xc + (size_t)j * m;
            double s = a[0] * b[0];
            for (int r = 1; r < m; ++r) s += a[r] * b[r];
            J->gram[(size_t)i * p + j] = s;
        }
    }
    return NULL;
}

int orc_compute_correlation(const double* x, int m, int p, double* c, int* zero_col, int threads) {
    if (m < 4 || p < 2) { set_err("DataMatrix: need m >= 4 samples and n >= 2 variables"); return ORC_EINVAL; }
    for (size_t k = 0; k < (size_t)m * p; ++k)
        if (!isfinite(x[k])) { set_err("DataMatrix: values must be finite"); return ORC_EINVAL; }
    double* xc = (double*)malloc(sizeof(double) * (size_t)m * p);
    double* gram = (double*)malloc(sizeof(double) * (size_t)p * p);
    if (!xc || !gram) { free(xc); free(gram); set_err("oom"); return ORC_ENOMEM; }
    for (int j = 0; j < p; ++j) { /* colwise mean (:135) and centring (:136) */
        const double* col = x + (size_t)j * m;
        double s = col[0];
        for (int r = 1; r < m; ++r) s += col[r];
        const double mean = s / m;
        for (int r = 0; r < m; ++r) xc[(size_t)j * m + r] = col[r] - mean;
    }
    corr_job J = {xc, m, p, gram, 0};
    if (threads < 1) threads = 1;
    pthread_t th[256];
    if (threads > 256) threads = 256;
    for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, corr_worker, &J);
    corr_worker(&J);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
    free(xc);
    double* sd = (double*)malloc(sizeof(double) * (size_t)p);
    for (int i = 0; i < p; ++i) { /* :139-145 */
        const double ss = gram[(size_t)i * p + i];
        if (!(ss > 0.0)) {
            if (zero_col) *zero_col = i;
            free(gram); free(sd);
            set_err("compute_correlation: column has zero variance");
            return ORC_EZEROVAR;
        }
        sd[i] = sqrt(ss);
    }
    for (int i = 0; i < p; ++i) { /* :147-154 */
        c[(size_t)i * p + i] = 1.0;
        for (int j = i + 1; j < p; ++j) {
            double v = gram[(size_t)i * p + j] / (sd[i] * sd[j]);
            v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
            c[(size_t)i * p + j] = v;
            c[(size_t)j * p + i] = v;
        }
    }
    free(gram); free(sd);
    return orc_correlation_normalize(c, p); /* CorrelationMatrix ctor (:155) */
}

/* ---- compute_correlation in the device's pinned order (FMA Gram) --------------------------
 * stats.hpp:132-156 leaves the Gram's summation order to Eigen (unpinned by the reference's
 * tests, which are all tolerance-based).  The device fixes it, and this restates it exactly:
 *   mean_j : 256 strided partial sums (lane t adds rows t, t+256, ... in order, from +0.0), then a
 *            halving tree (lane t += lane t+d, d = 128 .. 1); mean = sum / m        (:135)
 *   xc     : x - mean                                                              (:136)
 *   G(i,j) : i <= j, g = +0.0; for r = 0 .. m-1: g = fma(xc_i[r], xc_j[r], g); then, if the
 *            device pads the k extent (m not a multiple of kpad), g = g + 0.0     (:137)
 *            (the FP64 tensor-core MMA is a correctly rounded FMA chain over k: measured,
 *            tools/micro/dmma_semantics.cu, 12.8M/12.8M outputs)
 *   sd, c  : as compute_correlation below (:139-154)
 * G rows are computed lane-parallel over j (independent FMA chains; bit-identical to scalar). */
typedef struct {
    const double* xc;   /* p x m, variable-major */
    const double* xt;   /* m x p, sample-major (xt[r*p + j]) */
    int m, p, pad;
    double* gram;
    atomic_int next;
} fcorr_job;

__attribute__((target_clones("avx512f", "fma", "default")))
static void fcorr_row(const fcorr_job* J, int i) {
    const int m = J->m, p = J->p;
    const double* a = J->xc + (size_t)i * m;
    double acc[64];
    for (int j0 = i; j0 < p; j0 += 64) {
        const int nj = p - j0 < 64 ? p - j0 : 64;
        for (int jj = 0; jj < 64; ++jj) acc[jj] = 0.0;
        for (int r = 0; r < m; ++r) {
            const double ar = a[r];
            const double* b = J->xt + (size_t)r * p + j0;
            if (nj == 64) {
                for (int jj = 0; jj < 64; ++jj) acc[jj] = __builtin_fma(ar, b[jj], acc[jj]);
            } else {
                for (int jj = 0; jj < nj; ++jj) acc[jj] = __builtin_fma(ar, b[jj], acc[jj]);
            }
        }
        for (int jj = 0; jj < nj; ++jj) J->gram[(size_t)i * p + j0 + jj] = J->pad ? acc[jj] + 0.0 : acc[jj];
    }
}
static void* fcorr_worker(void* arg) {
    fcorr_job* J = (fcorr_job*)arg;
    for (;;) {
        const int i = atomic_fetch_add(&J->next, 1);
        if (i >= J->p) break;
        fcorr_row(J, i);
    }
    return NULL;
}

int orc_compute_correlation_fma(const double* x, int m, int p, int kpad, double* c, int* zero_col, int threads) {
    if (m < 4 || p < 2) { set_err("DataMatrix: need m >= 4 samples and n >= 2 variables"); return ORC_EINVAL; }
    for (size_t k = 0; k < (size_t)m * p; ++k)
        if (!isfinite(x[k])) { set_err("DataMatrix: values must be finite"); return ORC_EINVAL; }
    double* xc = (double*)malloc(sizeof(double) * (size_t)m * p);
    double* xt = (double*)malloc(sizeof(double) * (size_t)m * p);
    double* gram = (double*)malloc(sizeof(double) * (size_t)p * p);
    if (!xc || !xt || !gram) { free(xc); free(xt); free(gram); set_err("oom"); return ORC_ENOMEM; }
    for (int j = 0; j < p; ++j) {
        const double* col = x + (size_t)j * m;
        double red[256];
        for (int t = 0; t < 256; ++t) {
            double s = 0.0;
            for (int r = t; r < m; r += 256) s += col[r];
            red[t] = s;
        }
        for (int d = 128; d > 0; d >>= 1)
            for (int t = 0; t < d; ++t) red[t] += red[t + d];
        const double mean = red[0] / m;
        for (int r = 0; r < m; ++r) {
            const double v = col[r] - mean;
            xc[(size_t)j * m + r] = v;
            xt[(size_t)r * p + j] = v;
        }
    }
    fcorr_job J = {xc, xt, m, p, kpad > 0 && m % kpad != 0, gram, 0};
    if (threads < 1) threads = 1;
    pthread_t th[256];
    if (threads > 256) threads = 256;
    for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, fcorr_worker, &J);
    fcorr_worker(&J);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
    free(xc); free(xt);
    double* sd = (double*)malloc(sizeof(double) * (size_t)p);
    for (int i = 0; i < p; ++i) {
        const double ss = gram[(size_t)i * p + i];
        if (!(ss > 0.0)) {
            if (zero_col) *zero_col = i;
            free(gram); free(sd);
            set_err("compute_correlation: column has zero variance");
            return ORC_EZEROVAR;
        }
        sd[i] = sqrt(ss);
    }
    for (int i = 0; i < p; ++i) {
        c[(size_t)i * p + i] = 1.0;
        for (int j = i + 1; j < p; ++j) {
            double v = gram[(size_t)i * p + j] / (sd[i] * sd[j]);
            v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
            c[(size_t)i * p + j] = v;
            c[(size_t)j * p + i] = v;
        }
    }
    free(gram); free(sd);
    return orc_correlation_normalize(c, p);
}

int orc_correlation_normalize(double* c, int p) { /* core.hpp:73-95 */
    const double tol = 1e-12;
    if (p < 2) { set_err("CorrelationMatrix: need a square matrix, n >= 2"); return ORC_EINVAL; }
    for (int i = 0; i < p; ++i) {
        if (fabs(c[(size_t)i * p + i] - 1.0) > tol) { set_err("CorrelationMatrix: diagonal must be 1"); return ORC_EINVAL; }
        c[(size_t)i * p + i] = 1.0;
        for (int j = i + 1; j < p; ++j) {
            const double a = c[(size_t)i * p + j], b = c[(size_t)j * p + i];
            if (!isfinite(a) || !isfinite(b) || fabs(a - b) > tol) {
                set_err("CorrelationMatrix: matrix must be symmetric");
                return ORC_EINVAL;
            }
            double v = 0.5 * (a + b);
            if (fabs(v) > 1.0 + tol) { set_err("CorrelationMatrix: entries must lie in [-1, 1]"); return ORC_EINVAL; }
            v = v < -1.0 ? -1.0 : (v > 1.0 ? 1.0 : v);
            c[(size_t)i * p + j] = v;
            c[(size_t)j * p + i] = v;
        }
    }
    return ORC_OK;
}

/* ---- pseudo_inverse_into (stats.hpp:172-208); all matrices row-major n x n scratch ---- */
typedef struct {
    int cap;
    double *g, *l, *k, *rinv, *lr, *t;
} pinv_ws;
static int ws_reserve(pinv_ws* w, int n) {
    if (n <= w->cap) return 0;
    free(w->g); free(w->l); free(w->k); free(w->rinv); free(w->lr); free(w->t);
    size_t sz = sizeof(double) * (size_t)n * n;
    w->g = malloc(sz); w->l = malloc(sz); w->k = malloc(sz); w->rinv = malloc(sz); w->lr = malloc(sz); w->t = malloc(sz);
    w->cap = n;
    return (w->g && w->l && w->k && w->rinv && w->lr && w->t) ? 0 : -1;
}
static void ws_free(pinv_ws* w) {
    free(w->g); free(w->l); free(w->k); free(w->rinv); free(w->lr); free(w->t);
    memset(w, 0, sizeof *w);
}

/* returns 0 ok, ORC_EINVAL on non-finite input */
static int pinv_core(const double* a, int n, double* out, pinv_ws* w) {
    for (int q = 0; q < n * n; ++q)
        if (!isfinite(a[q])) { set_err("pseudo_inverse: entries must be finite"); return ORC_EINVAL; }
    double *G = w->g, *L = w->l, *K = w->k, *R = w->rinv, *LR = w->lr, *T = w->t;
#define AT(M, i, j) (M)[(i) * n + (j)]
    /* gram = a' a (:177) */
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = AT(a, 0, i) * AT(a, 0, j);
            for (int q = 1; q < n; ++q) s += AT(a, q, i) * AT(a, q, j);
            AT(G, i, j) = s;
        }
    double mx = AT(G, 0, 0); /* diagonal().maxCoeff() (:178) */
    for (int i = 1; i < n; ++i)
        if (AT(G, i, i) > mx) mx = AT(G, i, i);
    const double tol = 1e-10 * mx;
    if (!(tol > 0.0)) { /* :180-183 */
        for (int q = 0; q < n * n; ++q) out[q] = 0.0;
        return 0;
    }
    /* column-dropping Cholesky (:184-198) */
    int r = 0;
    for (int k = 0; k < n; ++k) {
        for (int i = 0; i < n; ++i) AT(L, i, r) = 0.0;
        for (int i = k; i < n; ++i) {
            double v = AT(G, i, k);
            if (r > 0) {
                double s = AT(L, i, 0) * AT(L, k, 0);
                for (int c = 1; c < r; ++c) s += AT(L, i, c) * AT(L, k, c);
                v = v - s;
            }
            AT(L, i, r) = v;
        }
        const double pivot = AT(L, k, r);
        if (pivot > tol) {
            const double root = sqrt(pivot);
            AT(L, k, r) = root;
            for (int i = k + 1; i < n; ++i) AT(L, i, r) = AT(L, i, r) / root;
            ++r;
        }
    }
    if (r == 0) { /* :199-202 */
        for (int q = 0; q < n * n; ++q) out[q] = 0.0;
        return 0;
    }
    /* K = L' L  (r x r) (:204) */
    for (int x = 0; x < r; ++x)
        for (int y = 0; y < r; ++y) {
            double s = AT(L, 0, x) * AT(L, 0, y);
            for (int i = 1; i < n; ++i) s += AT(L, i, x) * AT(L, i, y);
            AT(K, x, y) = s;
        }
    /* K.llt() (:205): unblocked lower LLT, stops at the first non-positive pivot */
    for (int k = 0; k < r; ++k) {
        double x = AT(K, k, k);
        if (k > 0) {
            double s = AT(K, k, 0) * AT(K, k, 0);
            for (int c = 1; c < k; ++c) s += AT(K, k, c) * AT(K, k, c);
            x = x - s;
        }
        if (x <= 0.0) break;
        x = sqrt(x);
        AT(K, k, k) = x;
        if (k > 0)
            for (int i = k + 1; i < r; ++i) {
                double s = AT(K, i, 0) * AT(K, k, 0);
                for (int c = 1; c < k; ++c) s += AT(K, i, c) * AT(K, k, c);
                AT(K, i, k) = AT(K, i, k) - s;
            }
        for (int i = k + 1; i < r; ++i) AT(K, i, k) = AT(K, i, k) / x;
    }
    /* .solve(I): forward with lower(K), backward with lower(K)' (:205) */
    for (int col = 0; col < r; ++col) {
        for (int k = 0; k < r; ++k) {
            double y = (k == col) ? 1.0 : 0.0;
            for (int c = 0; c < k; ++c) y = y - AT(K, k, c) * AT(R, c, col);
            AT(R, k, col) = y / AT(K, k, k);
        }
        for (int k = r - 1; k >= 0; --k) {
            double y = AT(R, k, col);
            for (int c = k + 1; c < r; ++c) y = y - AT(K, c, k) * AT(R, c, col);
            AT(R, k, col) = y / AT(K, k, k);
        }
    }
    /* lr = L R (n x r) (:206) */
    for (int i = 0; i < n; ++i)
        for (int y = 0; y < r; ++y) {
            double s = AT(L, i, 0) * AT(R, 0, y);
            for (int x = 1; x < r; ++x) s += AT(L, i, x) * AT(R, x, y);
            AT(LR, i, y) = s;
        }
    /* T = lr lr' (n x n), out = T a' (:207) */
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = AT(LR, i, 0) * AT(LR, j, 0);
            for (int y = 1; y < r; ++y) s += AT(LR, i, y) * AT(LR, j, y);
            AT(T, i, j) = s;
        }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = AT(T, i, 0) * AT(a, j, 0);
            for (int q = 1; q < n; ++q) s += AT(T, i, q) * AT(a, j, q);
            out[i * n + j] = s;
        }
#undef AT
    return 0;
}

int orc_pseudo_inverse(const double* a, int n, double* out) {
    if (n < 1) { set_err("pseudo_inverse: need n >= 1"); return ORC_EINVAL; }
    pinv_ws w = {0};
    if (ws_reserve(&w, n)) { ws_free(&w); set_err("oom"); return ORC_ENOMEM; }
    int rc = pinv_core(a, n, out, &w);
    ws_free(&w);
    return rc;
}

/* ---- CI test (stats.hpp:228-395) ---- */
typedef struct {
    pinv_ws pw;
    int cap;
    double *m2, *m2inv;
    int32_t *set, *pos;
} ci_ws;
static int ci_reserve(ci_ws* w, int ell) {
    if (ell < 1) ell = 1;
    if (ws_reserve(&w->pw, ell)) return -1;
    if (ell <= w->cap) return 0;
    free(w->m2); free(w->m2inv); free(w->set); free(w->pos);
    w->m2 = malloc(sizeof(double) * (size_t)ell * ell);
    w->m2inv = malloc(sizeof(double) * (size_t)ell * ell);
    w->set = malloc(sizeof(int32_t) * (size_t)ell);
    w->pos = malloc(sizeof(int32_t) * (size_t)ell);
    w->cap = ell;
    return (w->m2 && w->m2inv && w->set && w->pos) ? 0 : -1;
}
static void ci_free(ci_ws* w) {
    ws_free(&w->pw);
    free(w->m2); free(w->m2inv); free(w->set); free(w->pos);
    memset(w, 0, sizeof *w);
}

static const double RHO_CLAMP = 1.0 - 1e-12; /* stats.hpp:284 */

static void fill_m2(const double* c, int p, const int32_t* set, int ell, double* m2) { /* :253-258 */
    for (int a = 0; a < ell; ++a)
        for (int b = 0; b < ell; ++b) m2[a * ell + b] = c[(size_t)set[a] * p + set[b]];
}

/* partial_correlation_with_inverse (:292-307).  returns 1 if degenerate */
static int pcor_with_inverse(const double* c, int p, int i, int j, const int32_t* set, int ell,
                             const double* minv, double* rho) {
    double P0[64], P1[64], *P0d = P0, *P1d = P1;
    double* heap = NULL;
    if (ell > 64) { heap = malloc(sizeof(double) * 2 * ell); P0d = heap; P1d = heap + ell; }
    const double* ci = c + (size_t)i * p;
    const double* cj = c + (size_t)j * p;
    for (int col = 0; col < ell; ++col) { /* P = m1 * m2_inv (:296) */
        double s0 = ci[set[0]] * minv[0 * ell + col];
        double s1 = cj[set[0]] * minv[0 * ell + col];
        for (int k = 1; k < ell; ++k) {
            s0 += ci[set[k]] * minv[k * ell + col];
            s1 += cj[set[k]] * minv[k * ell + col];
        }
        P0d[col] = s0;
        P1d[col] = s1;
    }
    double d00 = P0d[0] * ci[set[0]], d11 = P1d[0] * cj[set[0]];
    double d01 = P0d[0] * cj[set[0]], d10 = P1d[0] * ci[set[0]];
    for (int k = 1; k < ell; ++k) {
        d00 += P0d[k] * ci[set[k]];
        d11 += P1d[k] * cj[set[k]];
        d01 += P0d[k] * cj[set[k]];
        d10 += P1d[k] * ci[set[k]];
    }
    free(heap);
    const double h00 = 1.0 - d00;                   /* :297 */
    const double h11 = 1.0 - d11;                   /* :298 */
    const double h01 = ci[j] - 0.5 * (d01 + d10);   /* :299-300 */
    const double denom = h00 * h11;                 /* :301 */
    if (!(denom > 0.0)) return 1;                   /* :302-305 */
    double v = h01 / sqrt(denom);                   /* :306 */
    *rho = v < -RHO_CLAMP ? -RHO_CLAMP : (v > RHO_CLAMP ? RHO_CLAMP : v);
    return 0;
}

static int validate_args(int p, int i, int j, const int32_t* set, int ell) { /* :228-241 */
    if (i == j || i < 0 || j < 0 || i >= p || j >= p) { set_err("ci arguments: i and j must be distinct vertices"); return ORC_EINVAL; }
    for (int a = 0; a < ell; ++a) {
        const int s = set[a];
        if (s < 0 || s >= p) { set_err("ci arguments: set member out of range"); return ORC_EINVAL; }
        if (s == i || s == j) { set_err("ci arguments: set must not contain i or j"); return ORC_EINVAL; }
        for (int b = a + 1; b < ell; ++b)
            if (set[b] == s) { set_err("ci arguments: set members must be distinct"); return ORC_EINVAL; }
    }
    return ORC_OK;
}

/* the decision given rho (stats.hpp:345-351); NaN rho -> ORC_ENAN like fisher_z's throw */
static int decide(double rho, double tau, int* indep, double* z) {
    double zz;
    int rc = orc_fisher_z(rho, &zz);
    if (rc) return rc;
    *z = zz;
    *indep = zz <= tau;
    return ORC_OK;
}

/* ci_test with scratch (stats.hpp:366-373); set may be empty */
static int ci_test_ws(const double* c, int p, int i, int j, const int32_t* set, int ell, double tau,
                      ci_ws* w, int* indep, double* z, double* rho_out, int* degen) {
    double rho;
    *degen = 0;
    if (ell == 0) {
        const double v = c[(size_t)i * p + j]; /* :312 */
        rho = v < -RHO_CLAMP ? -RHO_CLAMP : (v > RHO_CLAMP ? RHO_CLAMP : v);
    } else {
        fill_m2(c, p, set, ell, w->m2);
        int rc = pinv_core(w->m2, ell, w->m2inv, &w->pw);
        if (rc) return rc;
        if (pcor_with_inverse(c, p, i, j, set, ell, w->m2inv, &rho)) { /* degenerate_decision :353-360 */
            *degen = 1;
            *indep = 0;
            *z = INFINITY;
            if (rho_out) *rho_out = 0.0;
            return ORC_OK;
        }
    }
    if (rho_out) *rho_out = rho;
    return decide(rho, tau, indep, z);
}

int orc_partial_correlation(const double* c, int p, int i, int j, const int32_t* set, int ell, double* rho,
                            int* degenerate) {
    int rc = validate_args(p, i, j, set, ell);
    if (rc) return rc;
    *degenerate = 0;
    if (ell == 0) {
        const double v = c[(size_t)i * p + j];
        *rho = v < -RHO_CLAMP ? -RHO_CLAMP : (v > RHO_CLAMP ? RHO_CLAMP : v);
        return ORC_OK;
    }
    ci_ws w = {0};
    if (ci_reserve(&w, ell)) { ci_free(&w); return ORC_ENOMEM; }
    fill_m2(c, p, set, ell, w.m2);
    rc = pinv_core(w.m2, ell, w.m2inv, &w.pw);
    if (!rc) *degenerate = pcor_with_inverse(c, p, i, j, set, ell, w.m2inv, rho);
    ci_free(&w);
    return rc;
}

int orc_ci_test(const double* c, int p, int i, int j, const int32_t* set, int ell, double tau, int* independent,
                double* z, double* rho, int* degenerate) {
    int rc = validate_args(p, i, j, set, ell);
    if (rc) return rc;
    ci_ws w = {0};
    if (ci_reserve(&w, ell)) { ci_free(&w); return ORC_ENOMEM; }
    rc = ci_test_ws(c, p, i, j, set, ell, tau, &w, independent, z, rho, degenerate);
    ci_free(&w);
    return rc;
}

/* ============================================ core.hpp + skeleton.hpp ===== */
typedef struct {
    int len;
    int32_t m[];
} sepset_t;

struct orc_result {
    int p;
    int stop_reason;
    int nlevels;
    orc_level_stats levels[128];
    atomic_uchar* adj;           /* p*p cells (core.hpp:109-194) */
    _Atomic(sepset_t*)* slots;   /* p(p-1)/2 (core.hpp:267-339) */
};

static inline size_t slot_of(int p, int i, int j) { /* core.hpp:329-335 */
    if (i > j) { int t = i; i = j; j = t; }
    return (size_t)i * (2 * (size_t)p - i - 1) / 2 + (size_t)(j - i - 1);
}
static inline int adj_at(const orc_result* R, int i, int j) {
    return atomic_load_explicit(&R->adj[(size_t)i * R->p + j], memory_order_relaxed);
}
static int clear_edge(orc_result* R, int i, int j) { /* core.hpp:155-161 */
    if (i > j) { int t = i; i = j; j = t; }
    const int was = atomic_exchange_explicit(&R->adj[(size_t)i * R->p + j], 0, memory_order_acq_rel);
    atomic_store_explicit(&R->adj[(size_t)j * R->p + i], 0, memory_order_release);
    return was;
}
static void sep_store(orc_result* R, int i, int j, const int32_t* set, int ell) { /* core.hpp:302-306 */
    sepset_t* s = (sepset_t*)malloc(sizeof(sepset_t) + sizeof(int32_t) * (size_t)(ell > 0 ? ell : 1));
    s->len = ell;
    for (int k = 0; k < ell; ++k) s->m[k] = set[k];
    sepset_t* old = atomic_exchange_explicit(&R->slots[slot_of(R->p, i, j)], s, memory_order_acq_rel);
    free(old);
}

typedef struct { uint64_t ci, pinv, removed; } tally_t;

static void claim_removal(orc_result* R, int i, int j, const int32_t* set, int ell, tally_t* t) {
    if (!clear_edge(R, i, j)) return; /* skeleton.hpp:123-129 */
    sep_store(R, i, j, set, ell);
    ++t->removed;
}

typedef struct { /* CompactedAdjacency (core.hpp:200-239) */
    int p;
    int32_t* off;
    int32_t* idx;
    int max_width;
} snapshot_t;

static int compact(const orc_result* R, snapshot_t* S) { /* core.hpp:227-239 */
    const int p = R->p;
    S->p = p;
    S->off = (int32_t*)malloc(sizeof(int32_t) * (size_t)(p + 1));
    int64_t cnt = 0;
    for (size_t k = 0; k < (size_t)p * p; ++k) cnt += atomic_load_explicit(&R->adj[k], memory_order_relaxed);
    S->idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cnt + 1));
    if (!S->off || !S->idx) return ORC_ENOMEM;
    int64_t n = 0;
    S->max_width = 0;
    for (int i = 0; i < p; ++i) {
        S->off[i] = (int32_t)n;
        for (int j = 0; j < p; ++j)
            if (adj_at(R, i, j)) S->idx[n++] = j;
        if ((int)(n - S->off[i]) > S->max_width) S->max_width = (int)(n - S->off[i]);
    }
    S->off[p] = (int32_t)n;
    return ORC_OK;
}
static void snap_free(snapshot_t* S) { free(S->off); free(S->idx); }

typedef struct {
    const double* c;
    int p;
    const snapshot_t* snap;
    orc_result* R;
    double tau;
    int ell;
    const orc_config* cfg;
} level_ctx;

/* test_edge_over_sets (skeleton.hpp:135-160) */
static int test_edge_over_sets(level_ctx* X, int i, const int32_t* row, int width, int pidx, ci_ws* w, tally_t* t) {
    const int j = row[pidx];
    const int ell = X->ell;
    uint64_t total;
    int rc = orc_binomial(width - 1, ell, &total);
    if (rc) return rc;
    if ((rc = orc_unrank_positions(width - 1, ell, 0, w->pos))) return rc;
    for (uint64_t tt = 0;;) {
        if (!adj_at(X->R, i, j)) return ORC_OK;
        for (int k = 0; k < ell; ++k) {
            const int pos = w->pos[k];
            w->set[k] = row[pos >= pidx ? pos + 1 : pos];
        }
        int indep, degen;
        double z;
        if ((rc = ci_test_ws(X->c, X->p, i, j, w->set, ell, X->tau, w, &indep, &z, NULL, &degen))) return rc;
        ++t->ci;
        ++t->pinv;
        if (indep) {
            claim_removal(X->R, i, j, w->set, ell, t);
            return ORC_OK;
        }
        if (++tt >= total) return ORC_OK;
        orc_next_combination(w->pos, ell, width - 1);
    }
}

/* should_skip_unit (skeleton.hpp:54-70) */
static int should_skip(int width, int ell, int chunk, int strategy, const orc_config* cfg, int* skip) {
    if (width < ell + 1) { *skip = 1; return ORC_OK; }
    if (strategy == ORC_EDGE) { *skip = (uint64_t)chunk * cfg->edges_per_unit >= (uint64_t)width; return ORC_OK; }
    if (strategy == ORC_SET) {
        uint64_t b;
        int rc = orc_binomial(width, ell, &b);
        if (rc) return rc;
        *skip = (uint64_t)chunk * cfg->unit_width >= b;
        return ORC_OK;
    }
    *skip = 0;
    return ORC_OK;
}

/* run_edge_parallel_unit (skeleton.hpp:162-170) */
static int edge_unit(level_ctx* X, int row_i, int chunk, ci_ws* w, tally_t* t) {
    const int32_t* row = X->snap->idx + X->snap->off[row_i];
    const int width = X->snap->off[row_i + 1] - X->snap->off[row_i];
    int skip, rc;
    if ((rc = should_skip(width, X->ell, chunk, ORC_EDGE, X->cfg, &skip))) return rc;
    if (skip) return ORC_OK;
    const int begin = chunk * X->cfg->edges_per_unit;
    int end = begin + X->cfg->edges_per_unit;
    if (end > width) end = width;
    for (int pp = begin; pp < end; ++pp)
        if ((rc = test_edge_over_sets(X, row_i, row, width, pp, w, t))) return rc;
    return ORC_OK;
}

/* test_set_over_row (skeleton.hpp:175-200) */
static int test_set_over_row(level_ctx* X, int i, const int32_t* row, int width, ci_ws* w, tally_t* t) {
    const int ell = X->ell;
    int have_inverse = 0, next_member = 0, rc;
    for (int pp = 0; pp < width; ++pp) {
        if (next_member < ell && w->pos[next_member] == pp) { ++next_member; continue; }
        const int j = row[pp];
        if (!adj_at(X->R, i, j)) continue;
        if (!have_inverse) {
            for (int k = 0; k < ell; ++k) w->set[k] = row[w->pos[k]];
            fill_m2(X->c, X->p, w->set, ell, w->m2);
            if ((rc = pinv_core(w->m2, ell, w->m2inv, &w->pw))) return rc;
            ++t->pinv;
            have_inverse = 1;
        }
        /* ci_test_with_inverse (stats.hpp:383-395) */
        double rho, z;
        int indep = 0;
        if (pcor_with_inverse(X->c, X->p, i, j, w->set, ell, w->m2inv, &rho)) indep = 0;
        else if ((rc = decide(rho, X->tau, &indep, &z))) return rc;
        ++t->ci;
        if (indep) claim_removal(X->R, i, j, w->set, ell, t);
    }
    return ORC_OK;
}

/* run_set_shared_unit (skeleton.hpp:202-222) */
static int set_unit(level_ctx* X, int row_i, int chunk, ci_ws* w, tally_t* t) {
    const int32_t* row = X->snap->idx + X->snap->off[row_i];
    const int width = X->snap->off[row_i + 1] - X->snap->off[row_i];
    int skip, rc;
    if ((rc = should_skip(width, X->ell, chunk, ORC_SET, X->cfg, &skip))) return rc;
    if (skip) return ORC_OK;
    uint64_t total;
    if ((rc = orc_binomial(width, X->ell, &total))) return rc;
    const uint64_t band = (uint64_t)X->cfg->unit_width;
    const uint64_t stride = band * (uint64_t)X->cfg->set_groups;
    for (uint64_t bs = (uint64_t)chunk * band; bs < total; bs += stride) {
        const uint64_t be = bs + band < total ? bs + band : total;
        if ((rc = orc_unrank_positions(width, X->ell, bs, w->pos))) return rc;
        for (uint64_t tt = bs;;) {
            if ((rc = test_set_over_row(X, row_i, row, width, w, t))) return rc;
            if (++tt >= be) break;
            orc_next_combination(w->pos, X->ell, width);
        }
    }
    return ORC_OK;
}

/* ---- run_units (skeleton.hpp:90-118): atomic cursor over units, first error wins */
typedef struct { int row, chunk; } unit_t;
typedef struct {
    level_ctx* X;
    const unit_t* units;
    size_t n;
    atomic_size_t cursor;
    atomic_int failed;
    int first_error;
    char first_msg[256];
    pthread_mutex_t mu;
    int strategy;
    tally_t* tallies;
} units_job;
typedef struct { units_job* J; int wid; } worker_arg;

static void* units_worker(void* arg) {
    worker_arg* A = (worker_arg*)arg;
    units_job* J = A->J;
    ci_ws w = {0};
    if (ci_reserve(&w, J->X->ell)) {
        pthread_mutex_lock(&J->mu);
        if (!J->first_error) { J->first_error = ORC_ENOMEM; strcpy(J->first_msg, "oom"); }
        pthread_mutex_unlock(&J->mu);
        atomic_store(&J->failed, 1);
        return NULL;
    }
    tally_t* t = &J->tallies[A->wid];
    while (!atomic_load_explicit(&J->failed, memory_order_relaxed)) {
        const size_t idx = atomic_fetch_add_explicit(&J->cursor, 1, memory_order_relaxed);
        if (idx >= J->n) break;
        const unit_t u = J->units[idx];
        int rc = J->strategy == ORC_EDGE ? edge_unit(J->X, u.row, u.chunk, &w, t) : set_unit(J->X, u.row, u.chunk, &w, t);
        if (rc) {
            pthread_mutex_lock(&J->mu);
            if (!J->first_error) { J->first_error = rc; strcpy(J->first_msg, g_err); }
            pthread_mutex_unlock(&J->mu);
            atomic_store(&J->failed, 1);
            break;
        }
    }
    ci_free(&w);
    return NULL;
}

static int run_units(units_job* J, int workers) {
    pthread_mutex_init(&J->mu, NULL);
    atomic_init(&J->cursor, 0);
    atomic_init(&J->failed, 0);
    J->first_error = 0;
    worker_arg args[512];
    pthread_t th[512];
    if (workers > 512) workers = 512;
    for (int wdx = 0; wdx < workers; ++wdx) args[wdx] = (worker_arg){J, wdx};
    for (int wdx = 1; wdx < workers; ++wdx) pthread_create(&th[wdx], NULL, units_worker, &args[wdx]);
    units_worker(&args[0]);
    for (int wdx = 1; wdx < workers; ++wdx) pthread_join(th[wdx], NULL);
    pthread_mutex_destroy(&J->mu);
    if (J->first_error) set_err(J->first_msg);
    return J->first_error;
}

static void shuffle_units(unit_t* u, size_t n, uint64_t seed) { /* skeleton.hpp:224-228 */
    orc_xoshiro g;
    orc_xo_seed(&g, seed);
    for (size_t a = n; a > 1; --a) {
        const size_t b = (size_t)(orc_xo_next(&g) % a);
        unit_t tmp = u[a - 1];
        u[a - 1] = u[b];
        u[b] = tmp;
    }
}

/* run_level_units (skeleton.hpp:232-256) */
/* keep_stride > 1 (bench sampling only): run just the units whose chunk is a multiple of keep_stride */
static int g_keep_stride = 1;
static int run_level_units(level_ctx* X, int chunks_per_row, int strategy, orc_level_stats* st) {
    const int p = X->p;
    size_t n = (size_t)p * (size_t)chunks_per_row;
    unit_t* units = (unit_t*)malloc(sizeof(unit_t) * (n ? n : 1));
    if (!units) return ORC_ENOMEM;
    size_t k = 0;
    for (int i = 0; i < p; ++i)
        for (int ch = 0; ch < chunks_per_row; ++ch)
            if (ch % g_keep_stride == 0) units[k++] = (unit_t){i, ch};
    n = k;
    if (X->cfg->has_schedule_seed) shuffle_units(units, n, X->cfg->schedule_seed + (uint64_t)X->ell);
    const int workers = X->cfg->worker_count;
    units_job J;
    memset(&J, 0, sizeof J);
    J.X = X;
    J.units = units;
    J.n = n;
    J.strategy = strategy;
    J.tallies = (tally_t*)calloc((size_t)workers, sizeof(tally_t));
    int rc = run_units(&J, workers);
    st->ci_tests = st->pseudo_inverses = st->edges_removed = 0;
    for (int wdx = 0; wdx < workers; ++wdx) {
        st->ci_tests += J.tallies[wdx].ci;
        st->pseudo_inverses += J.tallies[wdx].pinv;
        st->edges_removed += J.tallies[wdx].removed;
    }
    free(J.tallies);
    free(units);
    return rc;
}

/* ---- run_level_zero (skeleton.hpp:262-288): rows are independent; counts are order free */
typedef struct {
    const double* c;
    orc_result* R;
    double tau;
    atomic_int next;
    atomic_ullong removed;
    atomic_int err;
} l0_job;
static void* l0_worker(void* arg) {
    l0_job* J = (l0_job*)arg;
    const int p = J->R->p;
    uint64_t removed = 0;
    for (;;) {
        const int i = atomic_fetch_add(&J->next, 1);
        if (i >= p) break;
        for (int j = i + 1; j < p; ++j) {
            const double v = J->c[(size_t)i * p + j];
            const double rho = v < -RHO_CLAMP ? -RHO_CLAMP : (v > RHO_CLAMP ? RHO_CLAMP : v);
            double z;
            if (orc_fisher_z(rho, &z)) { atomic_store(&J->err, ORC_ENAN); continue; }
            if (z <= J->tau && clear_edge(J->R, i, j)) {
                sep_store(J->R, i, j, NULL, 0);
                ++removed;
            }
        }
    }
    atomic_fetch_add(&J->removed, removed);
    return NULL;
}
static int run_level_zero(const double* c, orc_result* R, double tau, int workers, orc_level_stats* st) {
    l0_job J = {c, R, tau, 0, 0, 0};
    pthread_t th[512];
    if (workers > 512) workers = 512;
    for (int w = 1; w < workers; ++w) pthread_create(&th[w], NULL, l0_worker, &J);
    l0_worker(&J);
    for (int w = 1; w < workers; ++w) pthread_join(th[w], NULL);
    if (atomic_load(&J.err)) { set_err("fisher_z: rho must lie in (-1, 1)"); return ORC_ENAN; }
    const uint64_t p = (uint64_t)R->p;
    st->ci_tests = p * (p - 1) / 2;
    st->pseudo_inverses = 0;
    st->edges_removed = atomic_load(&J.removed);
    return ORC_OK;
}

/* run_level_serial (skeleton.hpp:292-307) */
static int run_level_serial(level_ctx* X, orc_level_stats* st) {
    ci_ws w = {0};
    if (ci_reserve(&w, X->ell)) { ci_free(&w); return ORC_ENOMEM; }
    tally_t t = {0, 0, 0};
    int rc = ORC_OK;
    for (int i = 0; i < X->p && !rc; ++i) {
        const int32_t* row = X->snap->idx + X->snap->off[i];
        const int width = X->snap->off[i + 1] - X->snap->off[i];
        if (width < X->ell + 1) continue;
        for (int pp = 0; pp < width && !rc; ++pp) rc = test_edge_over_sets(X, i, row, width, pp, &w, &t);
    }
    ci_free(&w);
    st->ci_tests = t.ci;
    st->pseudo_inverses = t.pinv;
    st->edges_removed = t.removed;
    return rc;
}

/* ---- serial-rule keys, one level ---- */
typedef struct {
    const double* c;
    int p;
    const int32_t* off;
    const int32_t* idx;
    int ell;
    double tau;
    const int64_t* edge_row;  /* per undirected edge: row a */
    const int32_t* edge_pos;  /* position of b in row a */
    int64_t e_begin, e_end;
    int64_t* keys;
    atomic_llong next;
    atomic_int err;
    char msg[256];
    pthread_mutex_t mu;
} keys_job;

static int bsearch_row(const int32_t* row, int w, int v) {
    int lo = 0, hi = w - 1;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        if (row[mid] == v) return mid;
        if (row[mid] < v) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* first separating reduced rank over row r minus position q; -1 if none */
static int first_pass(keys_job* J, int r, int q, ci_ws* w, int64_t* rank_out) {
    const int32_t* row = J->idx + J->off[r];
    const int width = J->off[r + 1] - J->off[r];
    const int ell = J->ell;
    *rank_out = -1;
    if (width < ell + 1) return ORC_OK;
    uint64_t total;
    int rc = orc_binomial(width - 1, ell, &total);
    if (rc) return rc;
    if ((rc = orc_unrank_positions(width - 1, ell, 0, w->pos))) return rc;
    const int j = row[q];
    for (uint64_t t = 0;;) {
        for (int k = 0; k < ell; ++k) {
            const int pos = w->pos[k];
            w->set[k] = row[pos >= q ? pos + 1 : pos];
        }
        int indep, degen;
        double z;
        if ((rc = ci_test_ws(J->c, J->p, r, j, w->set, ell, J->tau, w, &indep, &z, NULL, &degen))) return rc;
        if (indep) { *rank_out = (int64_t)t; return ORC_OK; }
        if (++t >= total) return ORC_OK;
        orc_next_combination(w->pos, ell, width - 1);
    }
}

static void* keys_worker(void* arg) {
    keys_job* J = (keys_job*)arg;
    ci_ws w = {0};
    if (ci_reserve(&w, J->ell)) { atomic_store(&J->err, ORC_ENOMEM); ci_free(&w); return NULL; }
    for (;;) {
        if (atomic_load_explicit(&J->err, memory_order_relaxed)) break;
        const int64_t e = atomic_fetch_add(&J->next, 1);
        if (e >= J->e_end) break;
        const int a = (int)J->edge_row[e];
        const int qa = J->edge_pos[e];
        const int b = J->idx[J->off[a] + qa];
        int64_t rk;
        int rc = first_pass(J, a, qa, &w, &rk);
        int64_t key = NONE_KEY;
        if (!rc && rk >= 0) key = rk;
        if (!rc && rk < 0) {
            const int qb = bsearch_row(J->idx + J->off[b], J->off[b + 1] - J->off[b], a);
            rc = first_pass(J, b, qb, &w, &rk);
            if (!rc && rk >= 0) key = ((int64_t)1 << 62) | rk;
        }
        if (rc) {
            pthread_mutex_lock(&J->mu);
            if (!atomic_load(&J->err)) { strcpy(J->msg, g_err); atomic_store(&J->err, rc); }
            pthread_mutex_unlock(&J->mu);
            break;
        }
        J->keys[e - J->e_begin] = key;
    }
    ci_free(&w);
    return NULL;
}

static int level_keys_impl(const double* c, int p, const int32_t* off, const int32_t* idx, int ell, double tau,
                           int64_t e_begin, int64_t e_end, int64_t* keys, int threads) {
    /* undirected edge list in CSR order: rows ascending, b > a ascending */
    int64_t ne = 0;
    for (int a = 0; a < p; ++a)
        for (int q = off[a]; q < off[a + 1]; ++q) ne += idx[q] > a;
    if (e_end > ne) e_end = ne;
    if (e_begin < 0) e_begin = 0;
    int64_t* er = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ne + 1));
    int32_t* ep = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ne + 1));
    if (!er || !ep) { free(er); free(ep); return ORC_ENOMEM; }
    int64_t e = 0;
    for (int a = 0; a < p; ++a)
        for (int q = off[a]; q < off[a + 1]; ++q)
            if (idx[q] > a) { er[e] = a; ep[e] = q - off[a]; ++e; }
    keys_job J;
    memset(&J, 0, sizeof J);
    J.c = c; J.p = p; J.off = off; J.idx = idx; J.ell = ell; J.tau = tau;
    J.edge_row = er; J.edge_pos = ep; J.e_begin = e_begin; J.e_end = e_end; J.keys = keys;
    atomic_init(&J.next, e_begin);
    atomic_init(&J.err, 0);
    pthread_mutex_init(&J.mu, NULL);
    if (threads < 1) threads = 1;
    if (threads > 512) threads = 512;
    pthread_t th[512];
    for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, keys_worker, &J);
    keys_worker(&J);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&J.mu);
    free(er); free(ep);
    const int rc = atomic_load(&J.err);
    if (rc) set_err(J.msg);
    return rc;
}

int orc_level_keys(const double* c, int p, const int32_t* offsets, const int32_t* indices, int ell, double tau,
                   int64_t e_begin, int64_t e_end, int64_t* keys, int threads) {
    if (ell < 1) { set_err("level_keys: need ell >= 1"); return ORC_EINVAL; }
    return level_keys_impl(c, p, offsets, indices, ell, tau, e_begin, e_end, keys, threads);
}

/* ---- fast serial-rule keys: set-shared evaluation, one pseudo-inverse per (row, set) ----
 *
 * Result-identical to run_level_serial (skeleton.hpp:292-307): for every row r and target
 * position q the first set, in the order test_edge_over_sets walks (lexicographic over the
 * positions of row r minus q, skeleton.hpp:140-160), whose CI test is independent -- or whose
 * statistic is NaN, where the serial strategy throws (stats.hpp:112).  The sets of row r are
 * walked ONCE in lexicographic order of full-row positions (the run_set_shared_unit order,
 * skeleton.hpp:175-222): the sets that avoid q appear in the same relative order, so the first
 * hit per target is the serial one.  Each test runs pcor_with_inverse's exact operation
 * sequence (stats.hpp:292-307), lane-parallel over the row's live targets with IEEE
 * elementwise operations only (no FMA: -ffp-contract=off; correctly rounded div/sqrt), so every
 * statistic is bit-identical to the scalar path.  The decision z <= tau is taken on |rho|
 * against tanh(tau) widened by 1e-9 relative; tests inside that band call decide() exactly.
 */
#define FAST_FIRST_NONE INT64_C(-1)
#define FAST_FIRST_NAN INT64_C(-2)

typedef struct {
    int cap;
    int32_t *lst, *tcol, *where;
    double *cij, *cjs, *rho;
    uint8_t *live, *indm, *exm;
} fast_ws;

static void fast_ws_free(fast_ws* W) {
    free(W->lst); free(W->tcol); free(W->where); free(W->cij); free(W->cjs); free(W->rho);
    free(W->live); free(W->indm); free(W->exm);
    memset(W, 0, sizeof *W);
}
static int fast_ws_reserve(fast_ws* W, int w, int ell) {
    if (w <= W->cap) return 0;
    fast_ws_free(W);
    const size_t n = (size_t)w + 16;
    W->lst = malloc(sizeof(int32_t) * n);
    W->tcol = malloc(sizeof(int32_t) * n);
    W->where = malloc(sizeof(int32_t) * n);
    W->cij = calloc(n, sizeof(double));
    W->cjs = calloc(n * (size_t)(ell > 4 ? 4 : ell), sizeof(double));
    W->rho = calloc(n, sizeof(double));
    W->live = calloc(n, 1);
    W->indm = calloc(n / 8 + 2, 1);
    W->exm = calloc(n / 8 + 2, 1);
    W->cap = w;
    return (W->lst && W->tcol && W->where && W->cij && W->cjs && W->rho && W->live && W->indm && W->exm) ? 0 : -1;
}

/* Per block of 8 lanes: indm bit = live, non-degenerate and surely independent; exm bit = live,
 * non-degenerate and inside the decision band (or NaN): decide() exactly.  Everything else is
 * dependent (degenerate H, stats.hpp:302-305, or |rho| above the band).  n is a multiple of 8;
 * lanes past the live targets have live = 0.  Returns nonzero if any bit is set.
 * Portable version: the per-test body of pcor_with_inverse (stats.hpp:292-307) verbatim. */
static int fast_lanes_c(const int L, const int n, const double* cjs, const double* cij, const uint8_t* live,
                        const double* minv, const double* P0, const double* ciS, const double h00,
                        const double rlo, const double rhi, uint8_t* indm, uint8_t* exm, double* rho_out) {
    int any = 0;
    for (int blk = 0; blk < n / 8; ++blk) {
        unsigned im = 0, em = 0;
        for (int l8 = 0; l8 < 8; ++l8) {
            const int t = blk * 8 + l8;
            if (!live[t]) continue;
            double cj[64], P1[64];
            for (int k = 0; k < L; ++k) cj[k] = cjs[(size_t)k * n + t];
            for (int col = 0; col < L; ++col) {
                double s1 = cj[0] * minv[0 * L + col];
                for (int k = 1; k < L; ++k) s1 += cj[k] * minv[k * L + col];
                P1[col] = s1;
            }
            double d11 = P1[0] * cj[0], d01 = P0[0] * cj[0], d10 = P1[0] * ciS[0];
            for (int k = 1; k < L; ++k) {
                d11 += P1[k] * cj[k];
                d01 += P0[k] * cj[k];
                d10 += P1[k] * ciS[k];
            }
            const double h11 = 1.0 - d11;
            const double h01 = cij[t] - 0.5 * (d01 + d10);
            const double denom = h00 * h11;
            if (!(denom > 0.0)) continue;
            const double v = h01 / sqrt(denom);
            const double rho = v < -RHO_CLAMP ? -RHO_CLAMP : (v > RHO_CLAMP ? RHO_CLAMP : v);
            const double a = fabs(rho);
            rho_out[t] = rho;
            if (a < rlo) im |= 1u << l8;
            else if (!(a > rhi)) em |= 1u << l8;
        }
        indm[blk] = (uint8_t)im;
        exm[blk] = (uint8_t)em;
        any |= (int)(im | em);
    }
    return any;
}

#if defined(__x86_64__)
#include <immintrin.h>
/* The same operation sequence, 8 lanes per AVX-512 instruction (IEEE mul/add/sub/div/sqrt,
 * correctly rounded, no FMA): bit-identical to fast_lanes_c. */
static inline __attribute__((always_inline, target("avx512f"))) int fast_lanes_avx512(
    const int L, const int n, const double* cjs, const double* cij, const uint8_t* live, const double* minv,
    const double* P0, const double* ciS, const double h00, const double rlo, const double rhi, uint8_t* indm,
    uint8_t* exm, double* rho_out) {
    __m512d mv[16], p0[4], cs[4];
    for (int q = 0; q < L * L; ++q) mv[q] = _mm512_set1_pd(minv[q]);
    for (int k = 0; k < L; ++k) { p0[k] = _mm512_set1_pd(P0[k]); cs[k] = _mm512_set1_pd(ciS[k]); }
    const __m512d one = _mm512_set1_pd(1.0), half = _mm512_set1_pd(0.5), zero = _mm512_setzero_pd();
    const __m512d pcl = _mm512_set1_pd(RHO_CLAMP), ncl = _mm512_set1_pd(-RHO_CLAMP);
    const __m512d vlo = _mm512_set1_pd(rlo), vhi = _mm512_set1_pd(rhi), vh00 = _mm512_set1_pd(h00);
    int any = 0;
    for (int t = 0; t < n; t += 8) {
        const __mmask8 lm = _mm512_cmpneq_epi64_mask(
            _mm512_cvtepu8_epi64(_mm_loadl_epi64((const __m128i*)(live + t))), _mm512_setzero_si512());
        if (!lm) { indm[t / 8] = 0; exm[t / 8] = 0; continue; }
        __m512d cj[4], P1[4];
        for (int k = 0; k < L; ++k) cj[k] = _mm512_loadu_pd(cjs + (size_t)k * n + t);
        for (int col = 0; col < L; ++col) {
            __m512d s1 = _mm512_mul_pd(cj[0], mv[0 * L + col]);
            for (int k = 1; k < L; ++k) s1 = _mm512_add_pd(s1, _mm512_mul_pd(cj[k], mv[k * L + col]));
            P1[col] = s1;
        }
        __m512d d11 = _mm512_mul_pd(P1[0], cj[0]), d01 = _mm512_mul_pd(p0[0], cj[0]), d10 = _mm512_mul_pd(P1[0], cs[0]);
        for (int k = 1; k < L; ++k) {
            d11 = _mm512_add_pd(d11, _mm512_mul_pd(P1[k], cj[k]));
            d01 = _mm512_add_pd(d01, _mm512_mul_pd(p0[k], cj[k]));
            d10 = _mm512_add_pd(d10, _mm512_mul_pd(P1[k], cs[k]));
        }
        const __m512d h11 = _mm512_sub_pd(one, d11);
        const __m512d h01 = _mm512_sub_pd(_mm512_loadu_pd(cij + t), _mm512_mul_pd(half, _mm512_add_pd(d01, d10)));
        const __m512d denom = _mm512_mul_pd(vh00, h11);
        const __mmask8 ok = _mm512_cmp_pd_mask(denom, zero, _CMP_GT_OQ) & lm;
        const __m512d v = _mm512_div_pd(h01, _mm512_sqrt_pd(_mm512_mask_blend_pd(ok, one, denom)));
        __m512d rho = _mm512_mask_blend_pd(_mm512_cmp_pd_mask(v, ncl, _CMP_LT_OQ), v, ncl);
        rho = _mm512_mask_blend_pd(_mm512_cmp_pd_mask(rho, pcl, _CMP_GT_OQ), rho, pcl);
        const __m512d a = _mm512_abs_pd(rho);
        const __mmask8 im = _mm512_cmp_pd_mask(a, vlo, _CMP_LT_OQ) & ok;
        const __mmask8 em = (__mmask8)(ok & ~im & ~_mm512_cmp_pd_mask(a, vhi, _CMP_GT_OQ));
        _mm512_storeu_pd(rho_out + t, rho);
        indm[t / 8] = (uint8_t)im;
        exm[t / 8] = (uint8_t)em;
        any |= (int)(im | em);
    }
    return any;
}
#define FAST_AVX(LL)                                                                                        \
    static __attribute__((target("avx512f"))) int fast_lanes_avx512_##LL(                                  \
        int n, const double* cjs, const double* cij, const uint8_t* live, const double* minv, const double* P0, \
        const double* ciS, double h00, double rlo, double rhi, uint8_t* indm, uint8_t* exm, double* rho) {     \
        return fast_lanes_avx512(LL, n, cjs, cij, live, minv, P0, ciS, h00, rlo, rhi, indm, exm, rho);        \
    }
FAST_AVX(1)
FAST_AVX(2)
FAST_AVX(3)
FAST_AVX(4)
static int g_have_avx512 = -1;
#endif

static int fast_lanes(int L, int n, const double* cjs, const double* cij, const uint8_t* live, const double* minv,
                      const double* P0, const double* ciS, double h00, double rlo, double rhi, uint8_t* indm,
                      uint8_t* exm, double* rho) {
#if defined(__x86_64__)
    if (g_have_avx512 < 0) g_have_avx512 = __builtin_cpu_supports("avx512f") ? 1 : 0;
    if (g_have_avx512 && !getenv("ORC_NO_AVX512")) {
        switch (L) {
            case 1: return fast_lanes_avx512_1(n, cjs, cij, live, minv, P0, ciS, h00, rlo, rhi, indm, exm, rho);
            case 2: return fast_lanes_avx512_2(n, cjs, cij, live, minv, P0, ciS, h00, rlo, rhi, indm, exm, rho);
            case 3: return fast_lanes_avx512_3(n, cjs, cij, live, minv, P0, ciS, h00, rlo, rhi, indm, exm, rho);
            case 4: return fast_lanes_avx512_4(n, cjs, cij, live, minv, P0, ciS, h00, rlo, rhi, indm, exm, rho);
            default: break;
        }
    }
#endif
    return fast_lanes_c(L, n, cjs, cij, live, minv, P0, ciS, h00, rlo, rhi, indm, exm, rho);
}

typedef struct {
    const double* c;
    int p;
    const int32_t* off;
    const int32_t* idx;
    int ell;
    double tau, rlo, rhi;
    int64_t* first;          /* per directed CSR entry: full-row rank of the first event */
    const int32_t* order;    /* rows, widest first */
    atomic_int next;
    atomic_int err;
    char msg[256];
    pthread_mutex_t mu;
} fast_job;

static int fast_row(fast_job* J, int r, ci_ws* cw, fast_ws* W) {
    const int ell = J->ell, p = J->p;
    const int32_t* row = J->idx + J->off[r];
    const int w = J->off[r + 1] - J->off[r];
    int64_t* first = J->first + J->off[r];
    for (int q = 0; q < w; ++q) first[q] = FAST_FIRST_NONE;
    if (w < ell + 1) return ORC_OK; /* no target of this row has an ell-subset of the others */
    if (fast_ws_reserve(W, w, ell)) return ORC_ENOMEM;
    const double* cr = J->c + (size_t)r * p;
    int n = w; /* live targets, compacted (lst: row position, tcol: vertex) */
    for (int q = 0; q < w; ++q) {
        W->lst[q] = q;
        W->tcol[q] = row[q];
        W->where[q] = q;
        W->cij[q] = cr[row[q]];
        W->live[q] = 1;
    }
    for (int t = n; t < n + 8; ++t) { W->live[t] = 0; W->cij[t] = 0.0; }
    int alive = w;
    int32_t* pos = cw->pos;
    int32_t* set = cw->set;
    for (int k = 0; k < ell; ++k) pos[k] = k;
    double P0[64], ciS[64];
    for (int64_t rank = 0;; ++rank) {
        int members_alive = 0;
        for (int k = 0; k < ell; ++k) {
            const int li = W->where[pos[k]];
            members_alive += li >= 0 && W->live[li];
        }
        if (alive - members_alive > 0) { /* some live target outside this set */
            for (int k = 0; k < ell; ++k) set[k] = row[pos[k]];
            fill_m2(J->c, p, set, ell, cw->m2);
            int rc = pinv_core(cw->m2, ell, cw->m2inv, &cw->pw);
            if (rc) return rc;
            const double* minv = cw->m2inv;
            for (int k = 0; k < ell; ++k) ciS[k] = cr[set[k]];
            for (int col = 0; col < ell; ++col) { /* P0 = m1 row i times m2_inv, pcor_with_inverse order */
                double s0 = ciS[0] * minv[0 * ell + col];
                for (int k = 1; k < ell; ++k) s0 += ciS[k] * minv[k * ell + col];
                P0[col] = s0;
            }
            double d00 = P0[0] * ciS[0];
            for (int k = 1; k < ell; ++k) d00 += P0[k] * ciS[k];
            const double h00 = 1.0 - d00;
            uint8_t saved[64];
            for (int k = 0; k < ell; ++k) { /* members are not targets of this set */
                const int li = W->where[pos[k]];
                saved[k] = li >= 0 ? W->live[li] : 0;
                if (li >= 0) W->live[li] = 0;
            }
            const int np = (n + 7) & ~7;
            int any;
            if (ell <= 4) {
                for (int k = 0; k < ell; ++k) {
                    const double* csk = J->c + (size_t)set[k] * p; /* C symmetric: C(j, s) = C(s, j) */
                    double* dst = W->cjs + (size_t)k * np;
                    for (int t = 0; t < n; ++t) dst[t] = csk[W->tcol[t]];
                    for (int t = n; t < np; ++t) dst[t] = 0.0;
                }
                any = fast_lanes(ell, np, W->cjs, W->cij, W->live, minv, P0, ciS, h00, J->rlo, J->rhi, W->indm,
                                 W->exm, W->rho);
            } else { /* deep levels: few tests, scalar pcor_with_inverse per live target */
                any = 0;
                for (int blk = 0; blk < np / 8; ++blk) { W->indm[blk] = 0; W->exm[blk] = 0; }
                for (int t = 0; t < n; ++t) {
                    if (!W->live[t]) continue;
                    double rho;
                    if (pcor_with_inverse(J->c, p, r, W->tcol[t], set, ell, minv, &rho)) continue;
                    W->rho[t] = rho;
                    W->exm[t / 8] |= (uint8_t)(1u << (t % 8));
                    any = 1;
                }
            }
            for (int k = 0; k < ell; ++k) {
                const int li = W->where[pos[k]];
                if (li >= 0) W->live[li] = saved[k];
            }
            if (any) {
                for (int blk = 0; blk < np / 8; ++blk) {
                    unsigned bits = (unsigned)W->indm[blk] | (unsigned)W->exm[blk];
                    while (bits) {
                        const int l8 = __builtin_ctz(bits);
                        bits &= bits - 1;
                        const int t = blk * 8 + l8;
                        int64_t ev = rank;
                        if ((W->exm[blk] >> l8) & 1) {
                            int indep;
                            double z;
                            const int rc2 = decide(W->rho[t], J->tau, &indep, &z);
                            if (rc2 == ORC_ENAN) ev = FAST_FIRST_NAN - rank; /* the serial run throws here */
                            else if (rc2) return rc2;
                            else if (!indep) continue;
                        }
                        first[W->lst[t]] = ev;
                        W->live[t] = 0;
                        --alive;
                    }
                }
                if (alive == 0) break;
                if (alive * 4 < n * 3 && n > 32) { /* re-compact the live targets */
                    int m2 = 0;
                    for (int t = 0; t < n; ++t) {
                        if (!W->live[t]) { W->where[W->lst[t]] = -1; continue; }
                        W->lst[m2] = W->lst[t];
                        W->tcol[m2] = W->tcol[t];
                        W->cij[m2] = W->cij[t];
                        W->live[m2] = 1;
                        W->where[W->lst[m2]] = m2;
                        ++m2;
                    }
                    for (int t = m2; t < n + 8; ++t) { W->live[t] = 0; W->cij[t] = 0.0; }
                    n = m2;
                }
            }
        }
        if (!orc_next_combination(pos, ell, w)) break;
    }
    return ORC_OK;
}

static void* fast_worker(void* arg) {
    fast_job* J = (fast_job*)arg;
    ci_ws cw = {0};
    fast_ws W = {0};
    if (ci_reserve(&cw, J->ell)) { atomic_store(&J->err, ORC_ENOMEM); ci_free(&cw); return NULL; }
    for (;;) {
        if (atomic_load_explicit(&J->err, memory_order_relaxed)) break;
        const int k = atomic_fetch_add(&J->next, 1);
        if (k >= J->p) break;
        int rc = fast_row(J, J->order[k], &cw, &W);
        if (rc) {
            pthread_mutex_lock(&J->mu);
            if (!atomic_load(&J->err)) { strcpy(J->msg, rc == ORC_ENOMEM ? "oom" : g_err); atomic_store(&J->err, rc); }
            pthread_mutex_unlock(&J->mu);
            break;
        }
    }
    fast_ws_free(&W);
    ci_free(&cw);
    return NULL;
}

/* Binomials C(n, k) for n < nmax, k <= ell (values checked against orc_binomial's overflow rule
 * by the caller's run_level_keys; saturate otherwise). */
typedef struct { int nmax, ell; uint64_t* v; } bin_tab;
static uint64_t bt(const bin_tab* T, int n, int k) {
    if (n < 0 || k < 0 || k > n) return 0;
    return T->v[(size_t)n * (T->ell + 1) + k];
}
static int bin_tab_init(bin_tab* T, int nmax, int ell) {
    T->nmax = nmax; T->ell = ell;
    T->v = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(nmax + 1) * (ell + 1));
    if (!T->v) return ORC_ENOMEM;
    for (int n = 0; n <= nmax; ++n)
        for (int k = 0; k <= ell; ++k) {
            uint64_t b = 0;
            if (k <= n && orc_binomial(n, k, &b)) b = UINT64_MAX;
            T->v[(size_t)n * (ell + 1) + k] = b;
        }
    return ORC_OK;
}

/* unrank (comb.hpp:50-67) with a binary search per position: the number of ell-subsets of
 * [0, width) whose c-th element precedes x (given the earlier elements) is
 * C(width - start, ell - c) - C(width - x, ell - c). */
static void unrank_fast(const bin_tab* T, int width, int ell, uint64_t t, int32_t* pos) {
    int start = 0;
    for (int c = 0; c < ell; ++c) {
        const uint64_t all = bt(T, width - start, ell - c);
        int lo = start, hi = width - (ell - c); /* largest x in [lo, hi] with covered(x) <= t */
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (all - bt(T, width - mid, ell - c) <= t) lo = mid; else hi = mid - 1;
        }
        t -= all - bt(T, width - lo, ell - c);
        pos[c] = lo;
        start = lo + 1;
    }
}

/* rank of ascending positions among the ell-subsets of [0, width), lexicographic */
static uint64_t rank_fast(const bin_tab* T, int width, int ell, const int32_t* pos) {
    uint64_t rk = 0;
    int start = 0;
    for (int c = 0; c < ell; ++c) {
        rk += bt(T, width - start, ell - c) - bt(T, width - pos[c], ell - c);
        start = pos[c] + 1;
    }
    return rk;
}

/* full-row rank of row r's set -> rank among the sets of row r minus position q */
static int64_t reduced_rank(const bin_tab* T, int w, int ell, int64_t full, int q, int32_t* pos) {
    unrank_fast(T, w, ell, (uint64_t)full, pos);
    for (int k = 0; k < ell; ++k) pos[k] -= pos[k] > q;
    return (int64_t)rank_fast(T, w - 1, ell, pos);
}

static int level_keys_fast(const double* c, int p, const int32_t* off, const int32_t* idx, int ell, double tau,
                           int64_t* keys, int threads) {
    fast_job J;
    memset(&J, 0, sizeof J);
    J.c = c; J.p = p; J.off = off; J.idx = idx; J.ell = ell; J.tau = tau;
    const long double rt = tanhl((long double)tau);
    J.rlo = (double)(rt * (1.0L - 1e-9L));
    J.rhi = (double)(rt * (1.0L + 1e-9L));
    J.first = (int64_t*)malloc(sizeof(int64_t) * (size_t)(off[p] + 1));
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)p);
    if (!J.first || !order) { free(J.first); free(order); return ORC_ENOMEM; }
    /* widest rows first (counting sort on width) */
    int maxw = 0;
    for (int r = 0; r < p; ++r) if (off[r + 1] - off[r] > maxw) maxw = off[r + 1] - off[r];
    int n = 0;
    for (int wd = maxw; wd >= 0; --wd)
        for (int r = 0; r < p; ++r) if (off[r + 1] - off[r] == wd) order[n++] = r;
    J.order = order;
    atomic_init(&J.next, 0);
    atomic_init(&J.err, 0);
    pthread_mutex_init(&J.mu, NULL);
    if (threads < 1) threads = 1;
    if (threads > 512) threads = 512;
    pthread_t th[512];
    for (int t = 1; t < threads; ++t) pthread_create(&th[t], NULL, fast_worker, &J);
    fast_worker(&J);
    for (int t = 1; t < threads; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&J.mu);
    free(order);
    int rc = atomic_load(&J.err);
    if (rc) { set_err(J.msg); free(J.first); return rc; }
    /* per undirected edge (a < b, CSR order): direction 0 = row a, then row b (Appendix B) */
    int32_t pos[65];
    bin_tab T;
    if (bin_tab_init(&T, maxw + 1, ell)) { free(J.first); return ORC_ENOMEM; }
    int64_t e = 0;
    for (int a = 0; a < p && !rc; ++a) {
        const int wa = off[a + 1] - off[a];
        for (int qa = 0; qa < wa; ++qa) {
            const int b = idx[off[a] + qa];
            if (b <= a) continue;
            int64_t key = NONE_KEY;
            int64_t ev = J.first[off[a] + qa];
            int dir = 0, wr = wa, q = qa;
            if (ev == FAST_FIRST_NONE) {
                const int wb = off[b + 1] - off[b];
                q = bsearch_row(idx + off[b], wb, a);
                ev = J.first[off[b] + q];
                dir = 1;
                wr = wb;
            }
            if (ev <= FAST_FIRST_NAN) { set_err("fisher_z: rho must lie in (-1, 1)"); rc = ORC_ENAN; break; }
            if (ev >= 0) key = ((int64_t)dir << 62) | reduced_rank(&T, wr, ell, ev, q, pos);
            keys[e++] = key;
        }
    }
    free(T.v);
    free(J.first);
    return rc;
}

int orc_level_keys_fast(const double* c, int p, const int32_t* offsets, const int32_t* indices, int ell, double tau,
                        int64_t* keys, int threads) {
    if (ell < 1) { set_err("level_keys: need ell >= 1"); return ORC_EINVAL; }
    return level_keys_fast(c, p, offsets, indices, ell, tau, keys, threads);
}

/* a whole level in key mode: identical skeleton/sepsets/counters to Serial */
static int run_level_keys(level_ctx* X, orc_level_stats* st) {
    const snapshot_t* S = X->snap;
    const int p = X->p, ell = X->ell;
    int64_t ne = 0;
    for (int a = 0; a < p; ++a)
        for (int q = S->off[a]; q < S->off[a + 1]; ++q) ne += S->idx[q] > a;
    /* the serial strategy evaluates binomial(w-1, ell) for every edge of every row with w >= ell+1 */
    for (int a = 0; a < p; ++a) {
        const int w = S->off[a + 1] - S->off[a];
        uint64_t b;
        if (w >= ell + 1) {
            int rc = orc_binomial(w - 1, ell, &b);
            if (rc) return rc;
        }
    }
    int64_t* keys = (int64_t*)malloc(sizeof(int64_t) * (size_t)(ne + 1));
    if (!keys) return ORC_ENOMEM;
    int rc = X->cfg->strategy == ORC_FAST
                 ? level_keys_fast(X->c, p, S->off, S->idx, ell, X->tau, keys, X->cfg->worker_count)
                 : level_keys_impl(X->c, p, S->off, S->idx, ell, X->tau, 0, ne, keys, X->cfg->worker_count);
    if (rc) { free(keys); return rc; }
    uint64_t tests = 0, removed = 0;
    int64_t e = 0;
    bin_tab T;
    if (bin_tab_init(&T, S->max_width + 1, ell)) { free(keys); return ORC_ENOMEM; }
    int32_t* set = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ell + 1));
    int32_t* pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ell + 1));
    for (int a = 0; a < p; ++a) {
        const int wa = S->off[a + 1] - S->off[a];
        for (int q = S->off[a]; q < S->off[a + 1]; ++q) {
            const int b = S->idx[q];
            if (b <= a) continue;
            const int wb = S->off[b + 1] - S->off[b];
            const uint64_t t0 = wa >= ell + 1 ? bt(&T, wa - 1, ell) : 0;
            const uint64_t t1 = wb >= ell + 1 ? bt(&T, wb - 1, ell) : 0;
            const int64_t key = keys[e++];
            if (key == NONE_KEY) { tests += t0 + t1; continue; }
            const int dir = (int)(key >> 62);
            const uint64_t rk = (uint64_t)(key & (((int64_t)1 << 62) - 1));
            tests += dir == 0 ? rk + 1 : t0 + rk + 1;
            const int r = dir == 0 ? a : b;
            const int32_t* row = S->idx + S->off[r];
            const int wr = S->off[r + 1] - S->off[r];
            const int qq = dir == 0 ? q - S->off[a] : bsearch_row(row, wr, a);
            unrank_fast(&T, wr - 1, ell, rk, pos); /* comb.hpp:87-94 */
            for (int k = 0; k < ell; ++k) set[k] = row[pos[k] >= qq ? pos[k] + 1 : pos[k]];
            clear_edge(X->R, a, b);
            sep_store(X->R, a, b, set, ell);
            ++removed;
        }
    }
    free(set); free(pos); free(keys); free(T.v);
    st->ci_tests = tests;
    st->pseudo_inverses = tests;
    st->edges_removed = removed;
    return ORC_OK;
}

/* One level (ell >= 1) of a strategy on a given snapshot, restricted to rows
 * [row_begin, row_end) -- the bounded CPU sample bench.py times.  The live graph
 * starts as the snapshot (run_level_* of skeleton.hpp:292-333). */
int orc_run_level(const double* c, int p, const int32_t* offsets, const int32_t* indices, int ell, double tau,
                  const orc_config* cfg, int row_begin, int row_end, orc_level_stats* out) {
    if (ell < 1) { set_err("run_level: need ell >= 1"); return ORC_EINVAL; }
    orc_result* R = (orc_result*)calloc(1, sizeof(orc_result));
    if (!R) return ORC_ENOMEM;
    R->p = p;
    R->adj = (atomic_uchar*)malloc(sizeof(atomic_uchar) * (size_t)p * p);
    const size_t ns = (size_t)p * (p - 1) / 2;
    R->slots = (_Atomic(sepset_t*)*)malloc(sizeof(*R->slots) * (ns ? ns : 1));
    if (!R->adj || !R->slots) { orc_result_free(R); return ORC_ENOMEM; }
    for (size_t q = 0; q < ns; ++q) atomic_init(&R->slots[q], NULL);
    for (size_t q = 0; q < (size_t)p * p; ++q) atomic_init(&R->adj[q], 0);
    snapshot_t S;
    S.p = p;
    S.off = (int32_t*)malloc(sizeof(int32_t) * (size_t)(p + 1));
    S.idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)(offsets[p] + 1));
    S.max_width = 0;
    if (row_begin < 0) row_begin = 0;
    if (row_end > p) row_end = p;
    /* restrict the snapshot rows outside the range to empty (their units skip) */
    int32_t n = 0;
    for (int i = 0; i < p; ++i) {
        S.off[i] = n;
        for (int q = offsets[i]; q < offsets[i + 1]; ++q) {
            const int j = indices[q];
            atomic_store(&R->adj[(size_t)i * p + j], 1);
            atomic_store(&R->adj[(size_t)j * p + i], 1);
            if (i >= row_begin && i < row_end) S.idx[n++] = j;
        }
        if ((int)(n - S.off[i]) > S.max_width) S.max_width = (int)(n - S.off[i]);
    }
    S.off[p] = n;
    orc_config cfg2 = *cfg;
    level_ctx X = {c, p, &S, R, tau, ell, &cfg2};
    orc_level_stats st;
    memset(&st, 0, sizeof st);
    const double t0 = now_s();
    int rc;
    switch (cfg->strategy) {
        case ORC_SERIAL: rc = run_level_serial(&X, &st); break;
        case ORC_EDGE: {
            const int chunks = (S.max_width + cfg->edges_per_unit - 1) / cfg->edges_per_unit;
            rc = run_level_units(&X, chunks, ORC_EDGE, &st);
            break;
        }
        case ORC_SET: rc = run_level_units(&X, cfg->set_groups, ORC_SET, &st); break;
        default: rc = run_level_keys(&X, &st); break;
    }
    st.elapsed_s = now_s() - t0;
    st.level = ell;
    snap_free(&S);
    orc_result_free(R);
    if (!rc) *out = st;
    return rc;
}

/* A sample of one SetShared level (bench.py's reference arm): rows [row_begin, row_end) of the snapshot,
 * with set_groups = G units per row of which only chunks 0, keep_stride, 2 keep_stride, ... run -- every
 * (G)th band of 64 sets from those chunks, i.e. 1/keep_stride of each row's sets, spread over the whole
 * rank range.  Not thread-safe against concurrent orc_run_level calls (test infrastructure). */
int orc_run_level_sampled(const double* c, int p, const int32_t* offsets, const int32_t* indices, int ell, double tau,
                          const orc_config* cfg, int row_begin, int row_end, int keep_stride, orc_level_stats* out) {
    if (cfg->strategy != ORC_SET || keep_stride < 1) { set_err("run_level_sampled: SET strategy only"); return ORC_EINVAL; }
    g_keep_stride = keep_stride;
    const int rc = orc_run_level(c, p, offsets, indices, ell, tau, cfg, row_begin, row_end, out);
    g_keep_stride = 1;
    return rc;
}

void orc_config_default(orc_config* cfg) { /* core.hpp:357-368 */
    memset(cfg, 0, sizeof *cfg);
    cfg->alpha = 0.05;
    cfg->max_level = -1;
    cfg->strategy = ORC_SERIAL;
    cfg->edges_per_unit = 2;
    cfg->workers_per_edge = 32;
    cfg->set_groups = 2;
    cfg->unit_width = 64;
    cfg->worker_count = 1;
}

static int validate_cfg(const orc_config* cfg) { /* core.hpp:370-383 */
    if (!(cfg->alpha > 0.0 && cfg->alpha < 1.0)) { set_err("SkeletonConfig: alpha must lie in (0, 1)"); return ORC_EINVAL; }
    if (cfg->max_level < -1) { set_err("SkeletonConfig: max_level must be >= 0"); return ORC_EINVAL; }
    if (cfg->edges_per_unit < 1) { set_err("SkeletonConfig: edges_per_unit must be >= 1"); return ORC_EINVAL; }
    if (cfg->workers_per_edge < 1) { set_err("SkeletonConfig: workers_per_edge must be >= 1"); return ORC_EINVAL; }
    if (cfg->set_groups < 1) { set_err("SkeletonConfig: set_groups must be >= 1"); return ORC_EINVAL; }
    if (cfg->unit_width < 1) { set_err("SkeletonConfig: unit_width must be >= 1"); return ORC_EINVAL; }
    if (cfg->worker_count < 1) { set_err("SkeletonConfig: worker_count must be >= 1"); return ORC_EINVAL; }
    if (cfg->strategy < ORC_SERIAL || cfg->strategy > ORC_FAST) { set_err("SkeletonConfig: bad strategy"); return ORC_EINVAL; }
    return ORC_OK;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

void orc_result_free(orc_result* R) {
    if (!R) return;
    if (R->slots) {
        const size_t ns = (size_t)R->p * (R->p - 1) / 2;
        for (size_t s = 0; s < ns; ++s) free(atomic_load(&R->slots[s]));
        free(R->slots);
    }
    free(R->adj);
    free(R);
}

/* run_pc_stable (skeleton.hpp:341-391) */
int orc_run_pc_stable(const double* c, int p, int m, const orc_config* cfg, orc_result** out) {
    *out = NULL;
    int rc = validate_cfg(cfg);
    if (rc) return rc;
    if (m < 4) { set_err("run_pc_stable: need at least 4 samples"); return ORC_EINVAL; }
    if (p < 2) { set_err("AdjacencyMatrix: need n >= 2"); return ORC_EINVAL; }
    orc_result* R = (orc_result*)calloc(1, sizeof(orc_result));
    if (!R) return ORC_ENOMEM;
    R->p = p;
    R->adj = (atomic_uchar*)malloc(sizeof(atomic_uchar) * (size_t)p * p);
    const size_t ns = (size_t)p * (p - 1) / 2;
    R->slots = (_Atomic(sepset_t*)*)malloc(sizeof(*R->slots) * (ns ? ns : 1));
    if (!R->adj || !R->slots) { orc_result_free(R); return ORC_ENOMEM; }
    for (size_t s = 0; s < ns; ++s) atomic_init(&R->slots[s], NULL);
    for (int i = 0; i < p; ++i) /* AdjacencyMatrix::complete (core.hpp:116-121) */
        for (int j = 0; j < p; ++j) atomic_init(&R->adj[(size_t)i * p + j], (unsigned char)(i != j));
    const int workers = cfg->strategy == ORC_SERIAL ? 1 : cfg->worker_count;
    R->stop_reason = ORC_STOP_MAX_DEGREE;
    for (int ell = 0;; ++ell) {
        if (cfg->max_level >= 0 && ell > cfg->max_level) { R->stop_reason = ORC_STOP_LEVEL_CAP; break; }
        double tau;
        rc = orc_threshold_tau(cfg->alpha, m, ell, &tau);
        if (rc == ORC_ELEVEL) { R->stop_reason = ORC_STOP_SAMPLE_SIZE; rc = ORC_OK; break; }
        if (rc) break;
        const double t0 = now_s();
        orc_level_stats st;
        memset(&st, 0, sizeof st);
        if (ell == 0) {
            rc = run_level_zero(c, R, tau, workers, &st);
        } else {
            snapshot_t S;
            memset(&S, 0, sizeof S);
            rc = compact(R, &S);
            if (rc) { snap_free(&S); break; }
            if (S.max_width - 1 < ell) { snap_free(&S); R->stop_reason = ORC_STOP_MAX_DEGREE; break; }
            level_ctx X = {c, p, &S, R, tau, ell, cfg};
            switch (cfg->strategy) {
                case ORC_SERIAL: rc = run_level_serial(&X, &st); break;
                case ORC_EDGE: {
                    const int chunks = (S.max_width + cfg->edges_per_unit - 1) / cfg->edges_per_unit;
                    rc = run_level_units(&X, chunks, ORC_EDGE, &st);
                    break;
                }
                case ORC_SET: rc = run_level_units(&X, cfg->set_groups, ORC_SET, &st); break;
                default: rc = run_level_keys(&X, &st); break;
            }
            snap_free(&S);
        }
        if (rc) break;
        st.level = ell;
        st.elapsed_s = now_s() - t0;
        if (R->nlevels < 128) R->levels[R->nlevels++] = st;
    }
    if (rc) { orc_result_free(R); return rc; }
    *out = R;
    return ORC_OK;
}

int orc_result_p(const orc_result* R) { return R->p; }
int orc_result_levels(const orc_result* R, orc_level_stats* out, int cap) {
    for (int k = 0; k < R->nlevels && k < cap; ++k) out[k] = R->levels[k];
    return R->nlevels;
}
int orc_result_stop_reason(const orc_result* R) { return R->stop_reason; }
void orc_result_adjacency(const orc_result* R, uint8_t* out) {
    for (size_t k = 0; k < (size_t)R->p * R->p; ++k) out[k] = atomic_load_explicit(&R->adj[k], memory_order_relaxed);
}
int64_t orc_result_member_total(const orc_result* R) {
    const size_t ns = (size_t)R->p * (R->p - 1) / 2;
    int64_t tot = 0;
    for (size_t s = 0; s < ns; ++s) {
        sepset_t* x = atomic_load(&R->slots[s]);
        if (x) tot += x->len;
    }
    return tot;
}
void orc_result_sepsets(const orc_result* R, int32_t* level, int64_t* offset, int32_t* members) {
    const size_t ns = (size_t)R->p * (R->p - 1) / 2;
    int64_t at = 0;
    for (size_t s = 0; s < ns; ++s) {
        sepset_t* x = atomic_load(&R->slots[s]);
        offset[s] = at;
        if (!x) { level[s] = -1; continue; }
        level[s] = x->len;
        for (int k = 0; k < x->len; ++k) members[at + k] = x->m[k];
        at += x->len;
    }
}
