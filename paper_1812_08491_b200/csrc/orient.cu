// orient.cu -- orientation of the skeleton into a CPDAG (
// /root/reference/proj/include/pcstable/orient.hpp).
//
//   vstruct_kernel   find_v_structures (orient.hpp:40-89): every unshielded triple
//                    i - k - j votes i -> k and j -> k iff k is not in sepset(i, j).
//                    One warp per skeleton entry (k, i) with lanes over the later
//                    neighbours j of k: sum_k deg(k)^2 / 2 triples, each a bitmask
//                    probe plus (for nonadjacent pairs) a binary search in the sorted
//                    sepset index.  Votes are atomicOr'ed into a p x W bitmask.
//   meek (host)      apply_meek_rules (orient.hpp:147-167) is a Gauss-Seidel fixed point
//                    whose outcome depends on the visiting order (edges ascending, (x,y)
//                    before (y,x), orientations visible to later edges of the same pass),
//                    so it runs on the host with bitset adjacency and in/out lists: every
//                    rule premise is an O(deg) or O(deg^2) probe instead of the reference's
//                    scan over all directed edges.
#include <algorithm>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/pcstable_b200.h"
#include "pcs_internal.h"

struct pcs_mixed_graph {
    int p = 0;
    std::vector<int32_t> dir;  // (from, to) pairs, ascending
    std::vector<int32_t> und;  // (a, b) pairs, a < b, ascending
};

namespace pcs {

struct SepIndex {
    const long long* key;   // sorted a * p + b (a < b) of pairs with a non-empty recorded sepset
    const long long* off;   // offset of the pair's members
    const int32_t* len;     // |S|
    const int32_t* mem;     // members
    long long n;
    const uint32_t* has;    // p x W bit (a, b): the pair has a separating set; null = every nonadjacent pair
};

namespace {

__device__ __forceinline__ bool bit(const uint32_t* m, int W, int i, int j) {
    return (__ldg(m + (size_t)i * W + (j >> 5)) >> (j & 31)) & 1u;
}

__global__ void vstruct_kernel(const int32_t* __restrict__ off, const int32_t* __restrict__ nbr,
                               const uint32_t* __restrict__ adj, int p, int W, SepIndex S, uint32_t* votes,
                               int* err) {
    const int lane = threadIdx.x & 31;
    const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long e_total = off[p];
    for (long long e = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < e_total; e += nwarps) {
        int lo = 0, hi = p - 1;  // row k of entry e
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (__ldg(off + mid) <= e) lo = mid; else hi = mid - 1;
        }
        const int k = lo;
        const int i = __ldg(nbr + e);
        const int end = __ldg(off + k + 1);
        for (long long f = e + 1 + lane; f < end; f += 32) {
            const int j = __ldg(nbr + f);  // i < j (rows ascending)
            if (bit(adj, W, i, j)) continue;  // shielded triple
            if (S.has && !bit(S.has, W, i, j)) {
                atomicOr(err, 1);  // nonadjacent pair without a separating set (orient.hpp:60-63)
                continue;
            }
            const long long key = (long long)i * p + j;
            long long a = 0, b = S.n;
            while (a < b) {
                const long long mid = (a + b) >> 1;
                if (__ldg(S.key + mid) < key) a = mid + 1; else b = mid;
            }
            bool contains = false;
            if (a < S.n && __ldg(S.key + a) == key) {
                const long long o = __ldg(S.off + a);
                const int len = __ldg(S.len + a);
                for (int q = 0; q < len; ++q) contains |= __ldg(S.mem + o + q) == k;
            }
            if (!contains) {
                atomicOr(votes + (size_t)i * W + (k >> 5), 1u << (k & 31));
                atomicOr(votes + (size_t)j * W + (k >> 5), 1u << (k & 31));
            }
        }
    }
}

pcs_status orient_fail(pcs_status st, const std::string& msg) {
    set_last_error(msg);
    return st;
}

#define ORIENT_CUDA(expr)                                                                       \
    do {                                                                                        \
        cudaError_t e_ = (expr);                                                                \
        if (e_ != cudaSuccess) {                                                                \
            st = orient_fail(PCS_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));    \
            goto done;                                                                          \
        }                                                                                       \
    } while (0)

// find_v_structures on the device; votes_out: p x W host bitmask (bit (x, k): vote x -> k)
pcs_status device_votes(int p, int W, const std::vector<uint32_t>& adj, const std::vector<long long>& key,
                        const std::vector<long long>& off, const std::vector<int32_t>& len,
                        const std::vector<int32_t>& mem, const std::vector<uint32_t>* has,
                        std::vector<uint32_t>& votes_out) {
    pcs_status st = PCS_OK;
    cudaStream_t s = nullptr;
    uint32_t *dAdj = nullptr, *dVotes = nullptr, *dHas = nullptr;
    int32_t *dDeg = nullptr, *dLow = nullptr, *dOff = nullptr, *dUp = nullptr, *dNbr = nullptr, *dLen = nullptr,
            *dMem = nullptr;
    long long *dKey = nullptr, *dSOff = nullptr;
    SnapInfo* dInfo = nullptr;
    SnapInfo info{};
    int* dErr = nullptr;
    int herr = 0;
    const size_t words = (size_t)p * W;
    ORIENT_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    ORIENT_CUDA(cudaMalloc(&dAdj, sizeof(uint32_t) * words));
    ORIENT_CUDA(cudaMalloc(&dVotes, sizeof(uint32_t) * words));
    ORIENT_CUDA(cudaMalloc(&dDeg, sizeof(int32_t) * p));
    ORIENT_CUDA(cudaMalloc(&dLow, sizeof(int32_t) * p));
    ORIENT_CUDA(cudaMalloc(&dOff, sizeof(int32_t) * (p + 1)));
    ORIENT_CUDA(cudaMalloc(&dUp, sizeof(int32_t) * (p + 1)));
    ORIENT_CUDA(cudaMalloc(&dInfo, sizeof(SnapInfo)));
    ORIENT_CUDA(cudaMalloc(&dErr, sizeof(int)));
    ORIENT_CUDA(cudaMalloc(&dKey, sizeof(long long) * std::max<size_t>(key.size(), 1)));
    ORIENT_CUDA(cudaMalloc(&dSOff, sizeof(long long) * std::max<size_t>(off.size(), 1)));
    ORIENT_CUDA(cudaMalloc(&dLen, sizeof(int32_t) * std::max<size_t>(len.size(), 1)));
    ORIENT_CUDA(cudaMalloc(&dMem, sizeof(int32_t) * std::max<size_t>(mem.size(), 1)));
    ORIENT_CUDA(cudaMemcpyAsync(dAdj, adj.data(), sizeof(uint32_t) * words, cudaMemcpyHostToDevice, s));
    if (!key.empty()) {
        ORIENT_CUDA(cudaMemcpyAsync(dKey, key.data(), sizeof(long long) * key.size(), cudaMemcpyHostToDevice, s));
        ORIENT_CUDA(cudaMemcpyAsync(dSOff, off.data(), sizeof(long long) * off.size(), cudaMemcpyHostToDevice, s));
        ORIENT_CUDA(cudaMemcpyAsync(dLen, len.data(), sizeof(int32_t) * len.size(), cudaMemcpyHostToDevice, s));
    }
    if (!mem.empty())
        ORIENT_CUDA(cudaMemcpyAsync(dMem, mem.data(), sizeof(int32_t) * mem.size(), cudaMemcpyHostToDevice, s));
    if (has) {
        ORIENT_CUDA(cudaMalloc(&dHas, sizeof(uint32_t) * words));
        ORIENT_CUDA(cudaMemcpyAsync(dHas, has->data(), sizeof(uint32_t) * words, cudaMemcpyHostToDevice, s));
    }
    ORIENT_CUDA(cudaMemsetAsync(dVotes, 0, sizeof(uint32_t) * words, s));
    ORIENT_CUDA(cudaMemsetAsync(dErr, 0, sizeof(int), s));
    // CSR of the skeleton with the snapshot kernels (compact(), core.hpp:227-239)
    launch_snapshot_degrees(dAdj, p, W, dDeg, dLow, s);
    launch_snapshot_scan(dDeg, dLow, p, dOff, dUp, dInfo, s);
    ORIENT_CUDA(cudaMemcpyAsync(&info, dInfo, sizeof(SnapInfo), cudaMemcpyDeviceToHost, s));
    ORIENT_CUDA(cudaStreamSynchronize(s));
    if (info.e_dir > 0) {
        ORIENT_CUDA(cudaMalloc(&dNbr, sizeof(int32_t) * (size_t)info.e_dir));
        launch_snapshot_fill(dAdj, p, W, dOff, dNbr, s);
        SepIndex S{dKey, dSOff, dLen, dMem, (long long)key.size(), dHas};
        long long blocks = (info.e_dir * 32 + 255) / 256;
        if (blocks > 148 * 16) blocks = 148 * 16;
        ++g_kernel_launches;
        vstruct_kernel<<<(int)blocks, 256, 0, s>>>(dOff, dNbr, dAdj, p, W, S, dVotes, dErr);
        ORIENT_CUDA(cudaGetLastError());
    }
    votes_out.assign(words, 0u);
    ORIENT_CUDA(cudaMemcpyAsync(votes_out.data(), dVotes, sizeof(uint32_t) * words, cudaMemcpyDeviceToHost, s));
    ORIENT_CUDA(cudaMemcpyAsync(&herr, dErr, sizeof(int), cudaMemcpyDeviceToHost, s));
    ORIENT_CUDA(cudaStreamSynchronize(s));
    if (herr) st = orient_fail(PCS_EINVAL, "find_v_structures: a nonadjacent pair has no separating set");
done:
    cudaFree(dAdj); cudaFree(dVotes); cudaFree(dHas); cudaFree(dDeg); cudaFree(dLow); cudaFree(dOff);
    cudaFree(dUp); cudaFree(dNbr); cudaFree(dLen); cudaFree(dMem); cudaFree(dKey); cudaFree(dSOff);
    cudaFree(dInfo); cudaFree(dErr);
    if (s) cudaStreamDestroy(s);
    return st;
}

// ---------------------------------------------------------------- Meek rules (host)
struct Mixed {
    int p, W;
    std::vector<uint32_t> A, D, U;  // skeleton adjacency, directed a->b, undirected (symmetric)
    std::vector<std::vector<int>> in, out;
    Mixed(int p_, const std::vector<uint32_t>& adj) : p(p_), W((p_ + 31) / 32), A(adj), D(adj.size(), 0u),
                                                      U(adj.size(), 0u), in(p_), out(p_) {}
    static bool get(const std::vector<uint32_t>& m, int W, int i, int j) {
        return (m[(size_t)i * W + (j >> 5)] >> (j & 31)) & 1u;
    }
    static void put(std::vector<uint32_t>& m, int W, int i, int j, bool v) {
        uint32_t& w = m[(size_t)i * W + (j >> 5)];
        w = v ? (w | (1u << (j & 31))) : (w & ~(1u << (j & 31)));
    }
    bool adjacent(int a, int b) const { return get(A, W, a, b); }
    bool directed(int a, int b) const { return get(D, W, a, b); }
    bool undirected(int a, int b) const { return get(U, W, a, b); }
    void set_directed(int a, int b) {
        put(D, W, a, b, true);
        out[a].push_back(b);
        in[b].push_back(a);
    }
    void set_undirected(int a, int b, bool v) {
        put(U, W, a, b, v);
        put(U, W, b, a, v);
    }
    // orient.hpp:95-101: some c -> a with c != b and c, b nonadjacent
    bool rule1(int a, int b) const {
        for (int c : in[a])
            if (c != b && !adjacent(c, b)) return true;
        return false;
    }
    // orient.hpp:105-111: a -> c -> b
    bool rule2(int a, int b) const {
        for (int c : out[a])
            if (directed(c, b)) return true;
        return false;
    }
    // orient.hpp:116-124: two nonadjacent c, d with c -> b, d -> b, a - c, a - d
    bool rule3(int a, int b, std::vector<int>& buf) const {
        buf.clear();
        for (int c : in[b])
            if (undirected(a, c)) buf.push_back(c);
        for (size_t x = 0; x < buf.size(); ++x)
            for (size_t y = x + 1; y < buf.size(); ++y)
                if (!adjacent(buf[x], buf[y])) return true;
        return false;
    }
    // orient.hpp:129-138: c -> d -> b, d != a, c != a, b, c adjacent to a, c and b nonadjacent
    bool rule4(int a, int b) const {
        for (int d : in[b]) {
            if (d == a) continue;
            for (int c : in[d]) {
                if (c == a || c == b) continue;
                if (adjacent(a, c) && !adjacent(c, b)) return true;
            }
        }
        return false;
    }
    void meek() {  // apply_meek_rules, orient.hpp:147-167
        std::vector<std::pair<int, int>> edges;
        std::vector<int> buf;
        for (int x = 0; x < p; ++x)
            for (int y = x + 1; y < p; ++y)
                if (undirected(x, y)) edges.emplace_back(x, y);
        bool changed = true;
        while (changed) {
            changed = false;
            std::vector<std::pair<int, int>> next;
            next.reserve(edges.size());
            for (const auto& [x, y] : edges) {
                bool oriented = false;
                for (int d = 0; d < 2 && !oriented; ++d) {
                    const int a = d ? y : x, b = d ? x : y;
                    if (rule1(a, b) || rule2(a, b) || rule3(a, b, buf) || rule4(a, b)) {
                        set_undirected(x, y, false);
                        set_directed(a, b);
                        changed = true;
                        oriented = true;
                    }
                }
                if (!oriented) next.push_back({x, y});
            }
            edges.swap(next);  // still ascending: the next pass's snapshot of g.undirected
        }
    }
    void emit(pcs_mixed_graph* g) const {
        g->p = p;
        for (int a = 0; a < p; ++a)
            for (int b = 0; b < p; ++b) {
                if (directed(a, b)) { g->dir.push_back(a); g->dir.push_back(b); }
                if (a < b && undirected(a, b)) { g->und.push_back(a); g->und.push_back(b); }
            }
    }
};

// votes -> MixedGraph (orient.hpp:73-87)
void apply_votes(Mixed& g, const std::vector<uint32_t>& votes) {
    for (int i = 0; i < g.p; ++i)
        for (int j = i + 1; j < g.p; ++j) {
            if (!g.adjacent(i, j)) continue;
            const bool fwd = Mixed::get(votes, g.W, i, j), rev = Mixed::get(votes, g.W, j, i);
            if (fwd && !rev) g.set_directed(i, j);
            else if (rev && !fwd) g.set_directed(j, i);
            else g.set_undirected(i, j, true);
        }
}

pcs_status orient_common(int p, std::vector<uint32_t>& adj, const std::vector<long long>& key,
                         const std::vector<long long>& off, const std::vector<int32_t>& len,
                         const std::vector<int32_t>& mem, const std::vector<uint32_t>* has, int stage,
                         const int32_t* directed_in, int64_t n_directed_in, pcs_mixed_graph** out) {
    if (stage < 1 || stage > 3) return orient_fail(PCS_EINVAL, "orient: stage must be 1, 2 or 3");
    const int W = (p + 31) / 32;
    for (int i = 0; i < p; ++i) Mixed::put(adj, W, i, i, false);
    Mixed g(p, adj);
    if (stage & 1) {
        std::vector<uint32_t> votes;
        pcs_status st = device_votes(p, W, adj, key, off, len, mem, has, votes);
        if (st) return st;
        apply_votes(g, votes);
    } else {
        for (int64_t e = 0; e < n_directed_in; ++e) {
            const int a = directed_in[2 * e], b = directed_in[2 * e + 1];
            if (a < 0 || b < 0 || a >= p || b >= p || !g.adjacent(a, b))
                return orient_fail(PCS_EINVAL, "apply_meek_rules: directed pair is not a skeleton edge");
            if (!g.directed(a, b)) g.set_directed(a, b);
        }
        for (int i = 0; i < p; ++i)
            for (int j = i + 1; j < p; ++j)
                if (g.adjacent(i, j) && !g.directed(i, j) && !g.directed(j, i)) g.set_undirected(i, j, true);
    }
    if (stage & 2) g.meek();
    auto* res = new pcs_mixed_graph;
    g.emit(res);
    *out = res;
    return PCS_OK;
}

}  // namespace
}  // namespace pcs

using namespace pcs;

extern "C" {

pcs_status pcs_orient_records(int32_t p, const uint32_t* bitmask, const int32_t* records, int64_t record_ints,
                              int32_t stage, pcs_mixed_graph** out) {
    if (!out || p < 0 || (p > 0 && !bitmask)) return orient_fail(PCS_EINVAL, "orient: bad arguments");
    const int W = (p + 31) / 32;
    std::vector<uint32_t> adj(bitmask, bitmask + (size_t)p * W);
    // sepset index of the level >= 1 removals; level-0 removals (every other nonadjacent pair) have S = {}
    std::vector<std::pair<long long, long long>> order;
    for (int64_t k = 0; k + 2 < record_ints;) {
        int a = records[k], b = records[k + 1];
        const int ell = records[k + 2];
        if (a > b) std::swap(a, b);
        if (ell > 0) order.emplace_back((long long)a * p + b, k);
        k += 3 + ell;
    }
    std::sort(order.begin(), order.end());
    std::vector<long long> key, off;
    std::vector<int32_t> len, mem;
    for (const auto& [kk, at] : order) {
        key.push_back(kk);
        off.push_back((long long)mem.size());
        const int ell = records[at + 2];
        len.push_back(ell);
        for (int q = 0; q < ell; ++q) mem.push_back(records[at + 3 + q]);
    }
    return orient_common(p, adj, key, off, len, mem, nullptr, stage, nullptr, 0, out);
}

pcs_status pcs_orient_result(const pcs_result* r, int32_t stage, pcs_mixed_graph** out) {
    if (!r) return orient_fail(PCS_EINVAL, "orient: null result");
    const int p = pcs_result_p(r);
    std::vector<uint32_t> bits((size_t)p * ((p + 31) / 32));
    pcs_result_bitmask(r, bits.data());
    std::vector<int32_t> recs((size_t)pcs_result_record_ints(r));
    pcs_result_records(r, recs.data());
    return pcs_orient_records(p, bits.data(), recs.data(), (int64_t)recs.size(), stage, out);
}

pcs_status pcs_orient_skeleton(int32_t p, const uint8_t* adj_in, const int32_t* sep_level, const int64_t* sep_offset,
                               const int32_t* members, int32_t stage, const int32_t* directed_in,
                               int64_t n_directed_in, pcs_mixed_graph** out) {
    if (!out || p < 0 || (p > 0 && !adj_in)) return orient_fail(PCS_EINVAL, "orient: bad arguments");
    if ((stage & 1) && p > 1 && (!sep_level || !sep_offset))
        return orient_fail(PCS_EINVAL, "orient: sepsets required for find_v_structures");
    const int W = (p + 31) / 32;
    std::vector<uint32_t> adj((size_t)p * W, 0u), has((size_t)p * W, 0u);
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j)
            if (i != j && adj_in[(size_t)i * p + j]) adj[(size_t)i * W + (j >> 5)] |= 1u << (j & 31);
    std::vector<long long> key, off;
    std::vector<int32_t> len, mem;
    if (stage & 1) {
        size_t slot = 0;
        for (int i = 0; i < p; ++i)
            for (int j = i + 1; j < p; ++j, ++slot) {
                const int ell = sep_level[slot];
                if (ell < 0) continue;
                has[(size_t)i * W + (j >> 5)] |= 1u << (j & 31);
                has[(size_t)j * W + (i >> 5)] |= 1u << (i & 31);
                if (ell == 0) continue;
                key.push_back((long long)i * p + j);
                off.push_back((long long)mem.size());
                len.push_back(ell);
                for (int q = 0; q < ell; ++q) mem.push_back(members[sep_offset[slot] + q]);
            }
    }
    return orient_common(p, adj, key, off, len, mem, &has, stage, directed_in, n_directed_in, out);
}

int64_t pcs_mixed_directed_count(const pcs_mixed_graph* g) { return g ? (int64_t)g->dir.size() / 2 : 0; }
int64_t pcs_mixed_undirected_count(const pcs_mixed_graph* g) { return g ? (int64_t)g->und.size() / 2 : 0; }
void pcs_mixed_directed(const pcs_mixed_graph* g, int32_t* pairs) {
    if (g && !g->dir.empty()) std::memcpy(pairs, g->dir.data(), sizeof(int32_t) * g->dir.size());
}
void pcs_mixed_undirected(const pcs_mixed_graph* g, int32_t* pairs) {
    if (g && !g->und.empty()) std::memcpy(pairs, g->und.data(), sizeof(int32_t) * g->und.size());
}
void pcs_mixed_free(pcs_mixed_graph* g) { delete g; }

}  // extern "C"
