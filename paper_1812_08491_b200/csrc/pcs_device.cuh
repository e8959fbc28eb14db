// pcs_device.cuh -- device-side building blocks of the B200 PC-stable path.
//
// Every floating-point expression here follows the operation order of the
// reference (/root/reference/proj/include/pcstable/stats.hpp) and of the CPU
// oracle (oracle/pcs_oracle.c); the translation units that include this file
// are compiled with -fmad=false so no a*b+c is contracted into one rounding.
// Together with correctly rounded IEEE sqrt/div this makes every CI decision
// bit-identical to the oracle (only log() may differ by an ulp, and log is
// evaluated only inside the +-1e-9 band around the threshold; see
// decide_fast()).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pcs {

constexpr int64_t kNoneKey = INT64_MAX;              // "no separating set found"
constexpr int kDirShift = 62;                         // key = dir << 62 | full-row rank
constexpr uint64_t kRankMask = (1ull << 62) - 1;
constexpr double kRhoClamp = 1.0 - 1e-12;             // stats.hpp:284

// Per-level decision constants (host computes them in long double).
struct Thresholds {
    double tau;      // threshold_tau(alpha, m, ell)          (stats.hpp:120-129)
    double lo;       // |rho| <= lo  => z <= tau for certain (level 0)
    double hi;       // |rho| >= hi  => z >  tau for certain (level 0)
    double lo2;      // rho^2 <= lo2 => independent for certain
    double hi2;      // rho^2 >= hi2 => dependent for certain
    double hi2x4;    // 4 hi2 (the cuPC-S step loop's scaled filter; a kernel-parameter load, no DMUL per step)
};

// ---------------------------------------------------------------- binomials
// Table T[k * stride + n] = C(n, k) for 0 <= k <= ell, 0 <= n < stride,
// saturated at UINT64_MAX (host-built per level, comb.hpp:35-46).
struct BinomTable {
    const unsigned long long* t;
    int stride;
    __device__ __forceinline__ unsigned long long operator()(int n, int k) const {
        if (k < 0 || n < k) return 0ull;
        return __ldg(t + (size_t)k * stride + n);
    }
};

// Lexicographic unrank of rank t among the ell-subsets of {0..w-1}
// (same map as comb.hpp:50-67, computed by binary search over the table).
template <int L>
__device__ __forceinline__ void unrank(const BinomTable& C, int w, unsigned long long t, int (&pos)[L]) {
    int start = 0;
#pragma unroll
    for (int c = 0; c < L; ++c) {
        const int k = L - c;
        const unsigned long long total = C(w - start, k);
        const unsigned long long need = total - t;  // largest v with C(w-v,k) >= need
        int lo = start, hi = w - k;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (C(w - mid, k) >= need) lo = mid; else hi = mid - 1;
        }
        pos[c] = lo;
        t -= total - C(w - lo, k);
        start = lo + 1;
    }
}

// Same map, with each member's binary search replaced by a closed-form estimate and a local fix-up:
// the largest v with C(w - v, k) >= need has x = w - v with C(x, k) ~ need, and C(x, k) ~ (x - (k-1)/2)^k / k!
// gives x ~ (k! need)^(1/k) + (k-1)/2 (FP32, MUFU); the exact table entries around the estimate then
// settle v (usually one round of two independent loads instead of ~log2(w) dependent ones).
template <int L>
__device__ __forceinline__ void unrank_est(const BinomTable& C, int w, unsigned long long t, int (&pos)[L]) {
    int start = 0;
#pragma unroll
    for (int c = 0; c < L; ++c) {
        const int k = L - c;
        const unsigned long long total = C(w - start, k);
        const unsigned long long need = total - t;  // >= 1
        float fk = 1.0f;
#pragma unroll
        for (int q = 2; q <= L; ++q)
            if (q <= k) fk *= (float)q;
        const float xf = k == 1 ? (float)need : exp2f(__log2f(fk * (float)need) / (float)k) + 0.5f * (float)(k - 1);
        int v = w - (int)floorf(xf);
        v = v < start ? start : (v > w - k ? w - k : v);
        for (;;) {
            const unsigned long long a = C(w - v, k);
            const unsigned long long b = v < w - k ? C(w - v - 1, k) : 0ull;
            if (a < need) { --v; continue; }
            if (b >= need) { ++v; continue; }
            break;
        }
        pos[c] = v;
        t -= total - C(w - v, k);
        start = v + 1;
    }
}

// Advance a lexicographic L-subset {pos[0] < ... < pos[L-1]} of {0..n-1} by k ranks (L = 2, 3): the last
// member absorbs k, and each overflow past n - 1 carries into the next block of the member before it
// (block (a, b) holds c in [b + 1, n - 1]).  The same map as comb.hpp:50-67's unrank of rank t + k;
// past the last subset the positions are left unspecified (callers check the rank).
template <int L>
__host__ __device__ __forceinline__ void advance_lex(int (&pos)[L], int n, int k) {
    if constexpr (L == 2) {
        int a = pos[0], b = pos[1] + k;
        while (b >= n && a < n - 2) {
            a += 1;
            b = b - n + a + 1;
        }
        pos[0] = a;
        pos[1] = b;
    } else {
        int a = pos[0], b = pos[1], c = pos[2] + k;
        while (c >= n) {
            const int o = c - n;
            b += 1;
            if (b > n - 2) {
                a += 1;
                b = a + 1;
                if (a > n - 3) break;
            }
            c = b + 1 + o;
        }
        pos[0] = a;
        pos[1] = b;
        pos[2] = c;
    }
}

// Inverse map: lexicographic rank of ascending positions in width w.
template <int L>
__device__ __forceinline__ unsigned long long rank_of(const BinomTable& C, int w, const int (&pos)[L]) {
    unsigned long long s = 0;
#pragma unroll
    for (int a = 0; a < L; ++a) s += C(w - 1 - pos[a], L - a);
    return C(w, L) - 1ull - s;
}

// ------------------------------------------------------- pseudo-inverse
// pseudo_inverse_into (stats.hpp:172-208) for an L x L row-major block.
// Kept Cholesky columns stay at their static index k (flag kept[k]) instead of
// being compacted, so every loop bound is a compile-time constant and the
// arrays live in registers; the sums visit exactly the same terms in the same
// order as the compacted form (a sum starts from its first term, never 0.0).
template <int L>
__device__ __forceinline__ void pinv(const double (&a)[L * L], double (&out)[L * L]) {
    double G[L * L];
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int j = 0; j < L; ++j) {
            double s = a[0 * L + i] * a[0 * L + j];
#pragma unroll
            for (int q = 1; q < L; ++q) s = s + a[q * L + i] * a[q * L + j];
            G[i * L + j] = s;
        }
    double mx = G[0];
#pragma unroll
    for (int i = 1; i < L; ++i) mx = G[i * L + i] > mx ? G[i * L + i] : mx;
    const double tol = 1e-10 * mx;
#pragma unroll
    for (int q = 0; q < L * L; ++q) out[q] = 0.0;
    if (!(tol > 0.0)) return;

    double Lm[L * L];  // Lm[i*L + k]: column stored at static index k
    bool kept[L];
#pragma unroll
    for (int k = 0; k < L; ++k) {
#pragma unroll
        for (int i = 0; i < L; ++i) {
            if (i < k) { Lm[i * L + k] = 0.0; continue; }
            double v = G[i * L + k];
            bool have = false;
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < k; ++c)
                if (kept[c]) { const double pr = Lm[i * L + c] * Lm[k * L + c]; s = have ? s + pr : pr; have = true; }
            if (have) v = v - s;
            Lm[i * L + k] = v;
        }
        const double pivot = Lm[k * L + k];
        kept[k] = pivot > tol;
        if (kept[k]) {
            const double root = sqrt(pivot);
            Lm[k * L + k] = root;
#pragma unroll
            for (int i = k + 1; i < L; ++i) Lm[i * L + k] = Lm[i * L + k] / root;
        }
    }
    bool any = false;
#pragma unroll
    for (int k = 0; k < L; ++k) any |= kept[k];
    if (!any) return;

    // K = L'L over kept columns (stats.hpp:204)
    double K[L * L];
#pragma unroll
    for (int x = 0; x < L; ++x)
#pragma unroll
        for (int y = 0; y < L; ++y) {
            double s = Lm[0 * L + x] * Lm[0 * L + y];
#pragma unroll
            for (int i = 1; i < L; ++i) s = s + Lm[i * L + x] * Lm[i * L + y];
            K[x * L + y] = s;
        }
    // in-place lower LLT over the kept index set (stats.hpp:205, Eigen unblocked LLT)
    bool failed = false;
#pragma unroll
    for (int k = 0; k < L; ++k) {
        if (!kept[k] || failed) continue;
        double x = K[k * L + k];
        {
            bool have = false;
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < k; ++c)
                if (kept[c]) { const double pr = K[k * L + c] * K[k * L + c]; s = have ? s + pr : pr; have = true; }
            if (have) x = x - s;
        }
        if (x <= 0.0) { failed = true; continue; }
        x = sqrt(x);
        K[k * L + k] = x;
#pragma unroll
        for (int i = k + 1; i < L; ++i) {
            if (!kept[i]) continue;
            bool have = false;
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < k; ++c)
                if (kept[c]) { const double pr = K[i * L + c] * K[k * L + c]; s = have ? s + pr : pr; have = true; }
            if (have) K[i * L + k] = K[i * L + k] - s;
        }
#pragma unroll
        for (int i = k + 1; i < L; ++i)
            if (kept[i]) K[i * L + k] = K[i * L + k] / x;
    }
    // R = (L'L)^-1 by forward/backward substitution on lower(K)
    double R[L * L];
#pragma unroll
    for (int col = 0; col < L; ++col) {
        if (!kept[col]) continue;
#pragma unroll
        for (int k = 0; k < L; ++k) {
            if (!kept[k]) continue;
            double y = (k == col) ? 1.0 : 0.0;
#pragma unroll
            for (int c = 0; c < k; ++c)
                if (kept[c]) y = y - K[k * L + c] * R[c * L + col];
            R[k * L + col] = y / K[k * L + k];
        }
#pragma unroll
        for (int k = L - 1; k >= 0; --k) {
            if (!kept[k]) continue;
            double y = R[k * L + col];
#pragma unroll
            for (int c = k + 1; c < L; ++c)
                if (kept[c]) y = y - K[c * L + k] * R[c * L + col];
            R[k * L + col] = y / K[k * L + k];
        }
    }
    // LR = L R  (n x r)
    double LR[L * L];
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int y = 0; y < L; ++y) {
            if (!kept[y]) continue;
            bool have = false;
            double s = 0.0;
#pragma unroll
            for (int x = 0; x < L; ++x)
                if (kept[x]) { const double pr = Lm[i * L + x] * R[x * L + y]; s = have ? s + pr : pr; have = true; }
            LR[i * L + y] = s;
        }
    // T = LR LR'; out = T a'  (stats.hpp:207)
    double T[L * L];
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int j = 0; j < L; ++j) {
            bool have = false;
            double s = 0.0;
#pragma unroll
            for (int y = 0; y < L; ++y)
                if (kept[y]) { const double pr = LR[i * L + y] * LR[j * L + y]; s = have ? s + pr : pr; have = true; }
            T[i * L + j] = s;
        }
#pragma unroll
    for (int i = 0; i < L; ++i)
#pragma unroll
        for (int j = 0; j < L; ++j) {
            double s = T[i * L + 0] * a[j * L + 0];
#pragma unroll
            for (int q = 1; q < L; ++q) s = s + T[i * L + q] * a[j * L + q];
            out[i * L + j] = s;
        }
}

// --------------------------------------------------------- decision
// Outcome codes of one CI test.
enum : int { kDependent = 0, kIndependent = 1, kNanError = 2 };
// decide_fast / decide0 set this bit when the outcome came from the exact comparison inside the
// +-1e-9 band around the threshold (the near-threshold tests the parity protocol lists)
constexpr int kNearBit = 8;

// Exact reference decision from (h01, denom) (stats.hpp:301-306 + 345-351).
__device__ __forceinline__ int decide_exact(double h01, double denom, double tau, double* z_out = nullptr,
                                            double* rho_out = nullptr) {
    if (!(denom > 0.0)) {  // degenerate -> dependent, z = +inf
        if (z_out) *z_out = __longlong_as_double(0x7ff0000000000000ll);
        if (rho_out) *rho_out = 0.0;
        return kDependent;
    }
    double v = h01 / sqrt(denom);
    v = v < -kRhoClamp ? -kRhoClamp : (v > kRhoClamp ? kRhoClamp : v);
    if (rho_out) *rho_out = v;
    if (!(v > -1.0 && v < 1.0)) return kNanError;  // fisher_z throws (stats.hpp:112)
    const double z = fabs(0.5 * log((1.0 + v) / (1.0 - v)));
    if (z_out) *z_out = z;
    return z <= tau ? kIndependent : kDependent;
}

// Same decision; the log is skipped when rho^2 is provably outside the
// +-1e-9 band around tanh(tau)^2 (host-computed lo2 / hi2 in long double).
__device__ __forceinline__ int decide_fast(double h01, double denom, const Thresholds& th) {
    if (!(denom > 0.0)) return kDependent;
    const double A = h01 * h01;
    if (denom >= 1e-250 && A >= 1e-250) {
        if (A <= denom * th.lo2) return kIndependent;
        if (A >= denom * th.hi2) return kDependent;
        return decide_exact(h01, denom, th.tau) | kNearBit;  // inside the +-1e-9 band
    }
    return decide_exact(h01, denom, th.tau);  // tiny h01 or denom (e.g. an exactly zero statistic)
}

// Branch-free common-case filter: true only when decide_fast() is certainly
// kDependent.  If denom <= 0 (or NaN) decide_fast() returns kDependent anyway.
// Otherwise g = RN(denom*hi2 + 1e-240) >= RN(denom*hi2) (monotone rounding), so
// h01^2 >= g gives decide_fast()'s "A >= denom*hi2" branch when denom >= 1e-250;
// when 0 < denom < 1e-250, A >= 1e-240 makes |rho| = |h01|/sqrt(denom) >= 1e5,
// clamped to 1-1e-12, whose z exceeds every tau with a finite hi2 (hi2 is +inf
// when tau reaches the clamp's z: then g = +inf and nothing is certified).
// NaN h01 -> false.  denom <= 0 is the degenerate branch (stats.hpp:301-305),
// dependent whatever h01 is -- frequent on rank-truncated inputs (C2), so it is
// certified here rather than in the divergent slow path.
__device__ __forceinline__ bool surely_dependent(double h01, double denom, double hi2) {
    return (h01 * h01 >= fma(denom, hi2, 1e-240)) | (denom <= 0.0);
}

// surely_dependent with h01 and the threshold scaled by 2 (h2 = 2 h01, hi2x4 = 4 hi2) and the
// degenerate test on the bit pattern (ALU pipe instead of a DSETP): (int64)bits(denom) <= 0 holds
// exactly for +0, -0, negative denominators and negative-signed NaNs, all of which the reference
// treats as degenerate -> dependent (!(denom > 0), stats.hpp:301); a positive NaN falls through to
// the comparison, which is false, so it takes the exact path.  Soundness of the scaled
// comparison: when it holds, h2^2 >= 4e-240 so |h2| >= 2e-120 is normal; then h2 = RN(2c - s) =
// 2 RN(c - s/2) = 2 h01 exactly (if s/2 is inexact, s is subnormal and both sides round to c),
// h2^2 = 4 RN(h01^2) and RN(denom * 4hi2 + 4e-240) = 4 RN(denom * hi2 + 1e-240), so the
// unscaled filter holds as well.
// (The integer test only needs the sign bit: a negative / -0 / negative-NaN denom is degenerate; +0
// falls to the comparison, whose right-hand side is then 4e-240, or to the exact path.)
__device__ __forceinline__ bool surely_dependent2(double h2, double denom, double hi2x4) {
    constexpr double kTiny4 = 4.0 * 1e-240;
    return (h2 * h2 >= fma(denom, hi2x4, kTiny4)) | (__double2hiint(denom) < 0);
}

// surely_dependent2 with one FP64 instruction less: the sign of the exactly rounded difference
// RN(h2 * h2 - g) (one FMA; a zero difference is +0) decides h2^2 >= g on the real numbers, which implies
// RN(h2^2) >= g and so surely_dependent2's comparison (more conservative by at most the rounding of h2^2);
// the sign is read as an integer (ALU), like the degenerate-denominator test.  A NaN h2 cannot occur
// (finite, validated C); it would read as "certified".
__device__ __forceinline__ bool surely_dependent2f(double h2, double denom, double hi2x4) {
    constexpr double kTiny4 = 4.0 * 1e-240;
    const double g = fma(denom, hi2x4, kTiny4);
    return (__double2hiint(fma(h2, h2, -g)) >= 0) | (__double2hiint(denom) < 0);
}

// The comparison alone (3 FP64 ops, no integer test): a degenerate denom <= 0 makes the right-hand
// side <= 4e-240, so it is certified too unless |h2| < 2e-120 (then the exact path decides it).
__device__ __forceinline__ bool surely_dependent3(double h2, double denom, double hi2x4) {
    constexpr double kTiny4 = 4.0 * 1e-240;
    return h2 * h2 >= fma(denom, hi2x4, kTiny4);
}

// Level-0 decision on rho = clamp(c_ij) (stats.hpp:309-312).
__device__ __forceinline__ int decide0(double c, const Thresholds& th) {
    const double ac = fabs(c);
    if (ac <= th.lo) return kIndependent;
    if (ac >= th.hi) return kDependent;
    double v = c < -kRhoClamp ? -kRhoClamp : (c > kRhoClamp ? kRhoClamp : c);
    if (!(v > -1.0 && v < 1.0)) return kNanError;
    const double z = fabs(0.5 * log((1.0 + v) / (1.0 - v)));
    return (z <= th.tau ? kIndependent : kDependent) | kNearBit;
}

// Partial-correlation pieces with a shared inverse (stats.hpp:292-307):
// given ciS (M1 row 0), P0 = ciS * Minv, h00 = 1 - P0.ciS (all per set)
// and the target's cjS (M1 row 1) and c_ij, return (h01, denom).
template <int L>
__device__ __forceinline__ void h_terms(const double* Minv, const double* ciS, const double* P0, double h00,
                                        const double (&cjS)[L], double cij, double& h01, double& denom) {
    double P1[L];
#pragma unroll
    for (int col = 0; col < L; ++col) {
        double s = cjS[0] * Minv[0 * L + col];
#pragma unroll
        for (int k = 1; k < L; ++k) s = s + cjS[k] * Minv[k * L + col];
        P1[col] = s;
    }
    double d11 = P1[0] * cjS[0], d01 = P0[0] * cjS[0], d10 = P1[0] * ciS[0];
#pragma unroll
    for (int k = 1; k < L; ++k) {
        d11 = d11 + P1[k] * cjS[k];
        d01 = d01 + P0[k] * cjS[k];
        d10 = d10 + P1[k] * ciS[k];
    }
    const double h11 = 1.0 - d11;
    h01 = cij - 0.5 * (d01 + d10);
    denom = h00 * h11;
}

// P0 = ciS * Minv and h00 = 1 - P0.ciS (row 0 of stats.hpp:296-297).
template <int L>
__device__ __forceinline__ void p0_terms(const double (&Minv)[L * L], const double (&ciS)[L], double (&P0)[L],
                                         double& h00) {
#pragma unroll
    for (int col = 0; col < L; ++col) {
        double s = ciS[0] * Minv[0 * L + col];
#pragma unroll
        for (int k = 1; k < L; ++k) s = s + ciS[k] * Minv[k * L + col];
        P0[col] = s;
    }
    double d00 = P0[0] * ciS[0];
#pragma unroll
    for (int k = 1; k < L; ++k) d00 = d00 + P0[k] * ciS[k];
    h00 = 1.0 - d00;
}

// ------------------------------------------------------- runtime-ell variants
// Same operation order as pinv<L> / p0_terms<L> / h_terms<L>; matrices live in
// caller-provided (global) scratch.  Used for ell > kMaxTemplLevel.
constexpr int kMaxRtLevel = 64;

// ws: 5*n*n doubles
__device__ inline void pinv_rt(const double* a, int n, double* out, double* ws) {
    double* G = ws;
    double* Lm = ws + n * n;
    double* K = ws + 2 * n * n;
    double* R = ws + 3 * n * n;
    double* LR = ws + 4 * n * n;
    double* T = G;  // G is dead once the Cholesky is done
    bool kept[kMaxRtLevel];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = a[0 * n + i] * a[0 * n + j];
            for (int q = 1; q < n; ++q) s = s + a[q * n + i] * a[q * n + j];
            G[i * n + j] = s;
        }
    double mx = G[0];
    for (int i = 1; i < n; ++i) mx = G[i * n + i] > mx ? G[i * n + i] : mx;
    const double tol = 1e-10 * mx;
    for (int q = 0; q < n * n; ++q) out[q] = 0.0;
    if (!(tol > 0.0)) return;
    for (int k = 0; k < n; ++k) {
        for (int i = 0; i < n; ++i) {
            if (i < k) { Lm[i * n + k] = 0.0; continue; }
            double v = G[i * n + k];
            bool have = false;
            double s = 0.0;
            for (int c = 0; c < k; ++c)
                if (kept[c]) { const double pr = Lm[i * n + c] * Lm[k * n + c]; s = have ? s + pr : pr; have = true; }
            if (have) v = v - s;
            Lm[i * n + k] = v;
        }
        const double pivot = Lm[k * n + k];
        kept[k] = pivot > tol;
        if (kept[k]) {
            const double root = sqrt(pivot);
            Lm[k * n + k] = root;
            for (int i = k + 1; i < n; ++i) Lm[i * n + k] = Lm[i * n + k] / root;
        }
    }
    bool any = false;
    for (int k = 0; k < n; ++k) any |= kept[k];
    if (!any) return;
    for (int x = 0; x < n; ++x)
        for (int y = 0; y < n; ++y) {
            if (!kept[x] || !kept[y]) continue;
            double s = Lm[0 * n + x] * Lm[0 * n + y];
            for (int i = 1; i < n; ++i) s = s + Lm[i * n + x] * Lm[i * n + y];
            K[x * n + y] = s;
        }
    bool failed = false;
    for (int k = 0; k < n; ++k) {
        if (!kept[k] || failed) continue;
        double x = K[k * n + k];
        {
            bool have = false;
            double s = 0.0;
            for (int c = 0; c < k; ++c)
                if (kept[c]) { const double pr = K[k * n + c] * K[k * n + c]; s = have ? s + pr : pr; have = true; }
            if (have) x = x - s;
        }
        if (x <= 0.0) { failed = true; continue; }
        x = sqrt(x);
        K[k * n + k] = x;
        for (int i = k + 1; i < n; ++i) {
            if (!kept[i]) continue;
            bool have = false;
            double s = 0.0;
            for (int c = 0; c < k; ++c)
                if (kept[c]) { const double pr = K[i * n + c] * K[k * n + c]; s = have ? s + pr : pr; have = true; }
            if (have) K[i * n + k] = K[i * n + k] - s;
        }
        for (int i = k + 1; i < n; ++i)
            if (kept[i]) K[i * n + k] = K[i * n + k] / x;
    }
    for (int col = 0; col < n; ++col) {
        if (!kept[col]) continue;
        for (int k = 0; k < n; ++k) {
            if (!kept[k]) continue;
            double y = (k == col) ? 1.0 : 0.0;
            for (int c = 0; c < k; ++c)
                if (kept[c]) y = y - K[k * n + c] * R[c * n + col];
            R[k * n + col] = y / K[k * n + k];
        }
        for (int k = n - 1; k >= 0; --k) {
            if (!kept[k]) continue;
            double y = R[k * n + col];
            for (int c = k + 1; c < n; ++c)
                if (kept[c]) y = y - K[c * n + k] * R[c * n + col];
            R[k * n + col] = y / K[k * n + k];
        }
    }
    for (int i = 0; i < n; ++i)
        for (int y = 0; y < n; ++y) {
            if (!kept[y]) continue;
            bool have = false;
            double s = 0.0;
            for (int x = 0; x < n; ++x)
                if (kept[x]) { const double pr = Lm[i * n + x] * R[x * n + y]; s = have ? s + pr : pr; have = true; }
            LR[i * n + y] = s;
        }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            bool have = false;
            double s = 0.0;
            for (int y = 0; y < n; ++y)
                if (kept[y]) { const double pr = LR[i * n + y] * LR[j * n + y]; s = have ? s + pr : pr; have = true; }
            T[i * n + j] = s;
        }
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = T[i * n + 0] * a[j * n + 0];
            for (int q = 1; q < n; ++q) s = s + T[i * n + q] * a[j * n + q];
            out[i * n + j] = s;
        }
}

__device__ inline void p0_terms_rt(const double* Minv, const double* ciS, int n, double* P0, double& h00) {
    for (int col = 0; col < n; ++col) {
        double s = ciS[0] * Minv[0 * n + col];
        for (int k = 1; k < n; ++k) s = s + ciS[k] * Minv[k * n + col];
        P0[col] = s;
    }
    double d00 = P0[0] * ciS[0];
    for (int k = 1; k < n; ++k) d00 = d00 + P0[k] * ciS[k];
    h00 = 1.0 - d00;
}

// P1 scratch of n doubles
__device__ inline void h_terms_rt(const double* Minv, const double* ciS, const double* P0, double h00,
                                  const double* cjS, int n, double cij, double* P1, double& h01, double& denom) {
    for (int col = 0; col < n; ++col) {
        double s = cjS[0] * Minv[0 * n + col];
        for (int k = 1; k < n; ++k) s = s + cjS[k] * Minv[k * n + col];
        P1[col] = s;
    }
    double d11 = P1[0] * cjS[0], d01 = P0[0] * cjS[0], d10 = P1[0] * ciS[0];
    for (int k = 1; k < n; ++k) {
        d11 = d11 + P1[k] * cjS[k];
        d01 = d01 + P0[k] * cjS[k];
        d10 = d10 + P1[k] * ciS[k];
    }
    const double h11 = 1.0 - d11;
    h01 = cij - 0.5 * (d01 + d10);
    denom = h00 * h11;
}

}  // namespace pcs
