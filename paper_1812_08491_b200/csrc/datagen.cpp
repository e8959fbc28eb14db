// datagen.cpp -- benchmark-input generation of the reference:
//   xoshiro256++ seeded by splitmix64, Marsaglia polar normals   rng.hpp:10-81
//   random_dag(n, density, seed)                                  datagen.hpp:42-56
//   sample_linear_gaussian(dag, m, seed)                          datagen.hpp:62-82
// The reference draws one normal per (sample, variable) from a single stream in
// sample-major order and its polar method consumes a data-dependent number of
// uniforms, so a bit-exact generator is inherently sequential per dataset; it
// runs on the host.  Parents are visited in ascending cause order exactly like
// the dense inner loop of datagen.hpp:75-78, so the sums round identically.
// Built with -ffp-contract=off (no FMA), like the reference's Release build.
#include <algorithm>
#include <array>
#include <atomic>
#include <mutex>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/pcstable_b200.h"

namespace {

struct Xoshiro {
    uint64_t s[4];
    double spare = 0.0;
    bool has_spare = false;
    static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    explicit Xoshiro(uint64_t seed) {
        uint64_t st = seed;
        for (auto& w : s) {  // splitmix64 (rng.hpp:14-19)
            uint64_t z = (st += 0x9e3779b97f4a7c15ULL);
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
            w = z ^ (z >> 31);
        }
    }
    uint64_t next() {
        const uint64_t r = rotl(s[0] + s[3], 23) + s[0];
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = rotl(s[3], 45);
        return r;
    }
    double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
    double normal() {
        if (has_spare) { has_spare = false; return spare; }
        double u, v, q;
        do {
            u = 2.0 * uniform01() - 1.0;
            v = 2.0 * uniform01() - 1.0;
            q = u * u + v * v;
        } while (q >= 1.0 || q == 0.0);
        const double scale = std::sqrt(-2.0 * std::log(q) / q);
        spare = v * scale;
        has_spare = true;
        return u * scale;
    }
};

// ---- the noise stream in parallel ("jump-ahead per block keeps seed
// determinism").  xoshiro256++'s state update is linear over GF(2): one step is a 256 x 256 bit matrix
// M, and J = M^(2^kChunkLog) jumps a whole chunk of outputs.  The polar method consumes exactly two
// uniforms per attempt, so attempts sit at fixed even offsets of the raw stream; chunks (an even number
// of outputs) are generated independently, their accepted attempts counted, prefix-summed, and
// regenerated into place: normal 2a / 2a+1 of the stream = u / v times the scale of the a-th accepted
// attempt, exactly the sequential generator's values (same uniforms, same sqrt(-2 log(s) / s) with
// this host's libm, as the reference).
constexpr int kChunkLog = 16;  // 65536 outputs = 32768 attempts per chunk

struct M256 {
    uint64_t c[256][4];  // column k = M e_k
};

void xo_advance(uint64_t s[4]) {
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = Xoshiro::rotl(s[3], 45);
}

void mat_vec(const M256& M, const uint64_t in[4], uint64_t out[4]) {
    uint64_t o[4] = {0, 0, 0, 0};
    for (int k = 0; k < 256; ++k)
        if ((in[k >> 6] >> (k & 63)) & 1u)
            for (int w = 0; w < 4; ++w) o[w] ^= M.c[k][w];
    std::memcpy(out, o, sizeof o);
}

const M256& chunk_jump() {
    static M256 J;
    static bool built = false;
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    if (built) return J;
    M256 A, B;
    for (int k = 0; k < 256; ++k) {
        uint64_t e[4] = {0, 0, 0, 0};
        e[k >> 6] = 1ull << (k & 63);
        xo_advance(e);
        std::memcpy(A.c[k], e, sizeof e);
    }
    for (int sq = 0; sq < kChunkLog; ++sq) {  // A <- A^2
        for (int k = 0; k < 256; ++k) mat_vec(A, A.c[k], B.c[k]);
        A = B;
    }
    J = A;
    built = true;
    return J;
}

// the first `count` normals of Xoshiro(seed).normal(), normal n written to out[(n % p) * m + n / p]
// (variable-major: the n-th draw is sample n / p, variable n % p), on up to 16 host threads
void noise_stream(uint64_t seed, int64_t count, int p, int m, double* out) {
    const int64_t attempts_needed = (count + 1) / 2;
    const int64_t per_chunk = 1ll << (kChunkLog - 1);
    const M256& J = chunk_jump();
    std::vector<std::array<uint64_t, 4>> state;
    std::vector<int64_t> accepted;
    Xoshiro g0(seed);
    std::array<uint64_t, 4> cur{g0.s[0], g0.s[1], g0.s[2], g0.s[3]};
    unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    auto run = [&](size_t c0, size_t c1, auto&& body) {
        std::vector<std::thread> th;
        std::atomic<size_t> next{c0};
        for (unsigned t = 0; t < nt; ++t)
            th.emplace_back([&] {
                for (size_t c; (c = next.fetch_add(1)) < c1;) body(c);
            });
        for (auto& x : th) x.join();
    };
    int64_t total = 0;
    while (total < attempts_needed) {  // extend the chunk list until enough attempts are accepted
        const size_t c0 = state.size();
        const int64_t more = (int64_t)((double)(attempts_needed - total) / 0.78 / per_chunk) + 1;
        for (int64_t k = 0; k < more; ++k) {
            state.push_back(cur);
            uint64_t nx[4];
            mat_vec(J, cur.data(), nx);
            cur = {nx[0], nx[1], nx[2], nx[3]};
        }
        accepted.resize(state.size());
        run(c0, state.size(), [&](size_t c) {
            Xoshiro g(0);
            std::memcpy(g.s, state[c].data(), sizeof g.s);
            int64_t n = 0;
            for (int64_t a = 0; a < per_chunk; ++a) {
                const double u = 2.0 * g.uniform01() - 1.0, v = 2.0 * g.uniform01() - 1.0;
                const double q = u * u + v * v;
                n += !(q >= 1.0 || q == 0.0);
            }
            accepted[c] = n;
        });
        for (size_t c = c0; c < state.size(); ++c) total += accepted[c];
    }
    std::vector<int64_t> base(state.size() + 1, 0);
    for (size_t c = 0; c < state.size(); ++c) base[c + 1] = base[c] + accepted[c];
    run(0, state.size(), [&](size_t c) {
        if (base[c] >= attempts_needed) return;
        Xoshiro g(0);
        std::memcpy(g.s, state[c].data(), sizeof g.s);
        int64_t a = base[c];
        for (int64_t k = 0; k < per_chunk && a < attempts_needed; ++k) {
            const double u = 2.0 * g.uniform01() - 1.0, v = 2.0 * g.uniform01() - 1.0;
            const double q = u * u + v * v;
            if (q >= 1.0 || q == 0.0) continue;
            const double scale = std::sqrt(-2.0 * std::log(q) / q);  // rng.hpp:68
            const int64_t n0 = 2 * a;
            out[(size_t)(n0 % p) * m + (size_t)(n0 / p)] = u * scale;
            if (n0 + 1 < count) out[(size_t)((n0 + 1) % p) * m + (size_t)((n0 + 1) / p)] = v * scale;
            ++a;
        }
    });
}

}  // namespace

extern "C" {

pcs_status pcs_noise_stream(uint64_t seed, int64_t count, int32_t p, int32_t m, double* out) {
    if (count < 0 || p < 1 || m < 1 || (int64_t)p * m < count) return PCS_EINVAL;
    noise_stream(seed, count, p, m, out);
    return PCS_OK;
}

pcs_status pcs_random_dag(int32_t n, double density, uint64_t seed, double* weights) {
    if (n < 2 || !(density > 0.0 && density < 1.0)) return PCS_EINVAL;
    std::memset(weights, 0, sizeof(double) * (size_t)n * n);
    Xoshiro g(seed);
    for (int i = 1; i < n; ++i)
        for (int j = 0; j < i; ++j)
            if (g.uniform01() < density) weights[(size_t)i * n + j] = g.uniform(0.1, 1.0);
    return PCS_OK;
}

pcs_status pcs_sample_linear_gaussian(const double* weights, int32_t n, int32_t m, uint64_t seed, double* x) {
    if (m < 4 || n < 2) return PCS_EINVAL;
    std::vector<int64_t> start((size_t)n + 1);
    std::vector<int32_t> par;
    std::vector<double> pw;
    for (int i = 0; i < n; ++i) {
        start[i] = (int64_t)par.size();
        for (int j = 0; j < n; ++j) {
            const double w = weights[(size_t)i * n + j];
            if (w == 0.0) continue;
            if (j >= i) return PCS_EINVAL;  // strictly lower triangular (datagen.hpp:66-69)
            par.push_back(j);
            pw.push_back(w);
        }
    }
    start[n] = (int64_t)par.size();
    // the noise draws first (the stream's sample-major order, jump-ahead parallel), then the equations
    // sample by sample in the reference's order (datagen.hpp:72-78): the same values as interleaving
    noise_stream(seed, (int64_t)n * m, n, m, x);
    for (int r = 0; r < m; ++r)
        for (int i = 0; i < n; ++i) {
            double value = x[(size_t)i * m + r];
            for (int64_t e = start[i]; e < start[i + 1]; ++e) value += pw[e] * x[(size_t)par[e] * m + r];
            x[(size_t)i * m + r] = value;
        }
    return PCS_OK;
}

// Overflow-safe variant for the BASELINE scaling shapes ("C5 needs the per-column-
// rescaled generator"): the same noise draws in the same (sample-major) stream order, but every
// variable is kept at unit RMS and its scale is carried as a logarithm.  With x_i the reference's
// variable (x_i = sum_j w_ij x_j + n_i) and s_i its RMS over the m samples, this computes
// x'_i = x_i / s_i through x'_i = (sum_j w_ij (s_j / F) x'_j + n_i / F) / rms(.) with F = the largest of
// the parents' scales and the noise's, so no intermediate overflows.  Correlations are scale-invariant:
// corr(x') = corr(x) in exact arithmetic (equal to rounding where the reference stays finite, finite
// where the reference overflows).  Variable-major, the m samples of one variable in parallel chunks.
pcs_status pcs_sample_linear_gaussian_rescaled(const double* weights, int32_t n, int32_t m, uint64_t seed, double* x,
                                               double* log_scale) {
    if (m < 4 || n < 2) return PCS_EINVAL;
    std::vector<int64_t> start((size_t)n + 1);
    std::vector<int32_t> par;
    std::vector<double> pw;
    for (int i = 0; i < n; ++i) {
        start[i] = (int64_t)par.size();
        for (int j = 0; j < n; ++j) {
            const double w = weights[(size_t)i * n + j];
            if (w == 0.0) continue;
            if (j >= i) return PCS_EINVAL;
            par.push_back(j);
            pw.push_back(w);
        }
    }
    start[n] = (int64_t)par.size();
    {  // the reference's noise stream, one normal per (sample, variable) in sample-major order
        noise_stream(seed, (int64_t)n * m, n, m, x);
    }
    // Scales are carried as mant * 2^exp (mant in [0.5, 1), frexp) and combined with ldexp and IEEE
    // mul/div/sqrt only -- no exp/log, whose last bits differ between libm builds -- and the sum of
    // squares over fixed sample chunks added in chunk order (not per thread), so the output is the same
    // bits on every host whatever its core count.
    constexpr int kChunks = 16;
    std::vector<double> smant((size_t)n);
    std::vector<long long> sexp((size_t)n);
    unsigned nt = std::max(1u, std::min((unsigned)kChunks, std::thread::hardware_concurrency()));
    if ((long long)m * (long long)(start[n] / std::max(1, n) + 1) < 200000) nt = 1;
    std::vector<double> coef, part(kChunks);
    for (int i = 0; i < n; ++i) {
        const int64_t b = start[i], e = start[i + 1];
        double Fm = 0.5;  // largest contributing scale (noise: 1 = 0.5 * 2^1)
        long long Fe = 1;
        for (int64_t k = b; k < e; ++k) {
            const int j = par[k];
            if (sexp[j] > Fe || (sexp[j] == Fe && smant[j] > Fm)) { Fm = smant[j]; Fe = sexp[j]; }
        }
        auto ratio = [&](double mant, long long ex) {  // (mant * 2^ex) / (Fm * 2^Fe), in (0, 2]
            const long long d = ex - Fe;
            return d < -2200 ? 0.0 : std::ldexp(mant / Fm, (int)d);
        };
        coef.resize((size_t)(e - b));
        for (int64_t k = b; k < e; ++k) coef[(size_t)(k - b)] = pw[k] * ratio(smant[par[k]], sexp[par[k]]);
        const double nz = ratio(0.5, 1);
        double* xi = x + (size_t)i * m;
        auto work = [&](unsigned t) {
            for (int c = (int)t; c < kChunks; c += (int)nt) {
                const int r0 = (int)((long long)m * c / kChunks), r1 = (int)((long long)m * (c + 1) / kChunks);
                double ss = 0.0;
                for (int r = r0; r < r1; ++r) {
                    double v = xi[r] * nz;
                    for (int64_t k = b; k < e; ++k) v += coef[(size_t)(k - b)] * x[(size_t)par[k] * m + r];
                    xi[r] = v;
                    ss += v * v;
                }
                part[(size_t)c] = ss;
            }
        };
        if (nt == 1) {
            work(0);
        } else {
            std::vector<std::thread> th;
            for (unsigned t = 0; t < nt; ++t) th.emplace_back(work, t);
            for (auto& t : th) t.join();
        }
        double ss = 0.0;
        for (int c = 0; c < kChunks; ++c) ss += part[(size_t)c];
        const double rms = std::sqrt(ss / m);
        if (!(rms > 0.0) || !std::isfinite(rms)) return PCS_EINVAL;
        const double inv = 1.0 / rms;
        for (int r = 0; r < m; ++r) xi[r] *= inv;
        int ex = 0;
        smant[(size_t)i] = std::frexp(Fm * rms, &ex);  // scale_i = F * rms
        sexp[(size_t)i] = Fe + ex;
        log_scale[i] = std::log(smant[(size_t)i]) + (double)sexp[(size_t)i] * 0.69314718055994530942;  // output only
    }
    return PCS_OK;
}

}  // extern "C"
