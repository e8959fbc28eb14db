// Host-side check of the device set stepper advance_lex<L> (pcs_device.cuh; used by the staged cuPC-E
// kernel): from every starting rank t < k, stepping by k ranks must visit exactly the lexicographic
// L-subsets t, t + k, t + 2k, ... of {0..n-1} (comb.hpp:50-67's order), for L = 2, 3.
#include <cstdio>
#include <vector>

#include "pcs_device.cuh"

template <int L>
static std::vector<std::vector<int>> all_subsets(int n) {
    std::vector<std::vector<int>> out;
    std::vector<int> c(L);
    for (int a = 0; a < L; ++a) c[a] = a;
    if (n < L) return out;
    for (;;) {
        out.push_back(c);
        int x = L - 1;
        while (x >= 0 && c[x] == n - L + x) --x;
        if (x < 0) break;
        ++c[x];
        for (int y = x + 1; y < L; ++y) c[y] = c[y - 1] + 1;
    }
    return out;
}

template <int L>
static int check(int n, int k) {
    const auto subs = all_subsets<L>(n);
    const long long total = (long long)subs.size();
    for (int start = 0; start < k && start < total; ++start) {
        int pos[L];
        for (int a = 0; a < L; ++a) pos[a] = subs[start][a];
        for (long long t = start; t < total; t += k) {
            for (int a = 0; a < L; ++a)
                if (pos[a] != subs[t][a]) {
                    std::printf("FAIL L=%d n=%d k=%d start=%d rank=%lld\n", L, n, k, start, t);
                    return 1;
                }
            if (t + k < total) pcs::advance_lex<L>(pos, n, k);
        }
    }
    return 0;
}

int main() {
    int bad = 0;
    long long cases = 0;
    for (int n = 2; n <= 60; ++n)
        for (int k : {1, 2, 3, 7, 31, 32, 33, 64}) {
            bad |= check<2>(n, k);
            if (n >= 3) bad |= check<3>(n, k);
            ++cases;
        }
    std::printf("%s: %lld (n, k) cases for L = 2, 3\n", bad ? "FAILED" : "ok", cases);
    return bad;
}
