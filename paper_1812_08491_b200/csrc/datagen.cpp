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
#include <cmath>
#include <cstdint>
#include <cstring>
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

}  // namespace

extern "C" {

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
    Xoshiro g(seed);
    for (int r = 0; r < m; ++r)
        for (int i = 0; i < n; ++i) {
            double value = g.normal();
            for (int64_t e = start[i]; e < start[i + 1]; ++e) value += pw[e] * x[(size_t)par[e] * m + r];
            x[(size_t)i * m + r] = value;
        }
    return PCS_OK;
}

}  // extern "C"
