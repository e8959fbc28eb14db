// test_dropin.cpp -- the reference's skeleton tests, written against the C++ drop-in
// (include/pcstable_b200.hpp) exactly as a reference user would call it, and
// cross-checked against the CPU oracle (test infrastructure) on seeded instances.
//
// Build (tests/test_cpp_dropin.py does this):
//   g++ -std=c++20 -O1 -I include -I oracle tests/cpp/test_dropin.cpp
//       -L paper_1812_08491_b200 -lpcstable_b200 -L oracle -lpcs_oracle -o build/test_dropin
// Run: ./test_dropin   (needs a GPU; exit code 0 = all passed)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#include "pcs_oracle.h"
#include "pcstable_b200.hpp"

using namespace pcstable;

static int g_failed = 0, g_checks = 0;
#define EXPECT(cond)                                                                 \
    do {                                                                             \
        ++g_checks;                                                                  \
        if (!(cond)) {                                                               \
            ++g_failed;                                                              \
            std::fprintf(stderr, "%s:%d: EXPECT(%s) failed\n", __FILE__, __LINE__, #cond); \
        }                                                                            \
    } while (0)
#define EXPECT_THROW(stmt, Ex)                 \
    do {                                       \
        bool thrown_ = false;                  \
        try { stmt; } catch (const Ex&) { thrown_ = true; } \
        EXPECT(thrown_ && #Ex);                \
    } while (0)

static CorrelationMatrix make_correlation(Index n, std::vector<std::tuple<Index, Index, double>> entries) {
    std::vector<double> v(static_cast<std::size_t>(n) * n, 0.0);  // support.hpp:103-111
    for (Index i = 0; i < n; ++i) v[static_cast<std::size_t>(i) * n + i] = 1.0;
    for (auto [i, j, x] : entries) v[static_cast<std::size_t>(i) * n + j] = v[static_cast<std::size_t>(j) * n + i] = x;
    return CorrelationMatrix(n, std::move(v));
}

static CorrelationMatrix star() {  // test_skeleton.cpp:24-32
    const double s = 1.0 / std::sqrt(3.0), t = std::sqrt(3.0) / 2.0;
    return make_correlation(4, {{0, 1, s}, {0, 2, s}, {0, 3, t}, {1, 2, 0.0}, {1, 3, 0.5}, {2, 3, 0.5}});
}

static DataMatrix sample(Index p, double density, std::uint64_t seed, Index m) {
    std::vector<double> w(static_cast<std::size_t>(p) * p), x(static_cast<std::size_t>(p) * m);
    detail::check(pcs_random_dag(p, density, seed, w.data()));
    detail::check(pcs_sample_linear_gaussian(w.data(), p, m, seed + 1, x.data()));
    return DataMatrix(m, p, std::move(x));
}

static void test_star_graph(Strategy strategy) {  // test_skeleton.cpp:102-127
    SkeletonConfig cfg;
    cfg.strategy = strategy;
    const auto r = run_pc_stable(star(), 1000, cfg);
    EXPECT(r.skeleton.edge_count() == 3);
    EXPECT(r.skeleton.at(0, 1) && r.skeleton.at(0, 2) && r.skeleton.at(0, 3));
    EXPECT(r.levels_run() == 3);
    EXPECT(r.stop_reason == StopReason::MaxDegreeReached);
    EXPECT(r.levels[0].edges_removed == 1 && r.levels[1].edges_removed == 2 && r.levels[2].edges_removed == 0);
    const auto* s12 = r.sepsets.find(1, 2);
    const auto* s13 = r.sepsets.find(1, 3);
    const auto* s23 = r.sepsets.find(3, 2);
    EXPECT(s12 && s12->empty());
    EXPECT(s13 && *s13 == std::vector<Index>{0});
    EXPECT(s23 && *s23 == std::vector<Index>{0});
    EXPECT(r.sepsets.find(0, 1) == nullptr);
    EXPECT(r.sepsets.stored_count() == 3);
}

static void test_level_cap_and_sample_size() {  // test_skeleton.cpp:139-169
    SkeletonConfig cfg;
    cfg.max_level = 1;
    auto r = run_pc_stable(star(), 1000, cfg);
    EXPECT(r.levels_run() == 2 && r.stop_reason == StopReason::LevelCapReached);
    std::vector<std::tuple<Index, Index, double>> e;
    for (Index i = 0; i < 5; ++i)
        for (Index j = i + 1; j < 5; ++j) e.emplace_back(i, j, 0.97);
    r = run_pc_stable(make_correlation(5, e), 5, SkeletonConfig{});
    EXPECT(r.stop_reason == StopReason::SampleSizeExhausted);
    EXPECT(r.levels_run() == 2);
    EXPECT(r.skeleton.edge_count() == 0);
}

static void test_errors() {  // core.hpp:370-383, skeleton.hpp:344, core.hpp:23-31, stats.hpp:120-129
    SkeletonConfig bad;
    bad.alpha = 0.0;
    EXPECT_THROW(run_pc_stable(star(), 1000, bad), std::invalid_argument);
    EXPECT_THROW(run_pc_stable(star(), 3, SkeletonConfig{}), std::invalid_argument);
    EXPECT_THROW(stats::threshold_tau(0.05, 7, 4), LevelUnreachableError);
    EXPECT_THROW(make_correlation(3, {{0, 1, 1.5}}), std::invalid_argument);
    std::vector<double> x(20 * 3);
    for (int r = 0; r < 20; ++r) { x[r] = r; x[20 + r] = 2.0; x[40 + r] = r * r; }
    try {
        stats::compute_correlation(DataMatrix(20, 3, x));
        EXPECT(false && "ZeroVarianceError expected");
    } catch (const ZeroVarianceError& e) {
        EXPECT(e.column() == 1);
    }
}

static void test_chain_and_collider() {  // acceptance_tests.cpp:383-425
    SkeletonConfig cfg;
    cfg.alpha = 0.01;
    std::vector<double> w(9, 0.0), x(3 * 10000);
    w[1 * 3 + 0] = 0.8; w[2 * 3 + 1] = 0.9;  // 0 -> 1 -> 2
    detail::check(pcs_sample_linear_gaussian(w.data(), 3, 10000, 31, x.data()));
    auto r = run_pc_stable(stats::compute_correlation(DataMatrix(10000, 3, x)), 10000, cfg);
    EXPECT(r.skeleton.at(0, 1) && r.skeleton.at(1, 2) && !r.skeleton.at(0, 2));
    EXPECT(r.sepsets.find(0, 2) && *r.sepsets.find(0, 2) == std::vector<Index>{1});
    std::fill(w.begin(), w.end(), 0.0);
    w[2 * 3 + 0] = 0.8; w[2 * 3 + 1] = 0.9;  // 0 -> 2 <- 1
    detail::check(pcs_sample_linear_gaussian(w.data(), 3, 10000, 32, x.data()));
    r = run_pc_stable(stats::compute_correlation(DataMatrix(10000, 3, x)), 10000, cfg);
    EXPECT(r.skeleton.at(0, 2) && r.skeleton.at(1, 2) && !r.skeleton.at(0, 1));
    EXPECT(r.sepsets.find(0, 1) && r.sepsets.find(0, 1)->empty());
}

// Device result through the drop-in == the oracle's Strategy::Serial run on the same C.
static void test_against_oracle(Index p, double d, Index m, std::uint64_t seed, Strategy strategy) {
    const DataMatrix data = sample(p, d, seed, m);
    std::vector<double> c(static_cast<std::size_t>(p) * p);
    int zc = -1;
    EXPECT(orc_compute_correlation(data.data(), m, p, c.data(), &zc, 4) == ORC_OK);
    const CorrelationMatrix cm(p, c);
    SkeletonConfig cfg;
    cfg.alpha = 0.01;
    cfg.strategy = strategy;
    const auto r = run_pc_stable(cm, m, cfg);
    orc_config oc;
    orc_config_default(&oc);
    oc.alpha = 0.01;
    orc_result* o = nullptr;
    EXPECT(orc_run_pc_stable(c.data(), p, m, &oc, &o) == ORC_OK);
    std::vector<uint8_t> adj(static_cast<std::size_t>(p) * p);
    orc_result_adjacency(o, adj.data());
    bool same = true;
    for (Index i = 0; i < p; ++i)
        for (Index j = 0; j < p; ++j) same &= (adj[static_cast<std::size_t>(i) * p + j] != 0) == r.skeleton.at(i, j);
    EXPECT(same);
    const std::size_t slots = static_cast<std::size_t>(p) * (p - 1) / 2;
    std::vector<int32_t> lv(slots), mem(static_cast<std::size_t>(std::max<int64_t>(orc_result_member_total(o), 1)));
    std::vector<int64_t> off(slots);
    orc_result_sepsets(o, lv.data(), off.data(), mem.data());
    std::size_t s = 0, diffs = 0;
    for (Index i = 0; i < p; ++i)
        for (Index j = i + 1; j < p; ++j, ++s) {
            const auto* got = r.sepsets.find(i, j);
            if (lv[s] < 0) { diffs += got != nullptr; continue; }
            if (!got) { ++diffs; continue; }
            diffs += *got != std::vector<Index>(mem.begin() + off[s], mem.begin() + off[s] + lv[s]);
        }
    EXPECT(diffs == 0);
    std::vector<orc_level_stats> ol(64);
    const int nl = orc_result_levels(o, ol.data(), 64);
    EXPECT(nl == r.levels_run());
    for (int k = 0; k < nl && k < r.levels_run(); ++k) {
        EXPECT(ol[k].ci_tests == r.levels[k].ci_tests);
        EXPECT(ol[k].pseudo_inverses == r.levels[k].pseudo_inverses);
        EXPECT(ol[k].edges_removed == r.levels[k].edges_removed);
    }
    EXPECT(static_cast<int>(r.stop_reason) == orc_result_stop_reason(o));
    orc_result_free(o);
    // data path: compute_correlation + run_pc_stable on the device agrees on the skeleton's size
    const auto rd = run_pc_stable(data, cfg);
    EXPECT(rd.levels_run() >= 1);
}

// test_orient.cpp:25-181, written against the drop-in's orient API
static AdjacencyMatrix make_skeleton(Index n, std::vector<std::pair<Index, Index>> edges) {
    AdjacencyMatrix a(n);
    for (auto [i, j] : edges) a.set_edge(i, j);
    return a;
}

static void test_orientation() {
    {
        const AdjacencyMatrix skel = make_skeleton(3, {{0, 2}, {1, 2}});
        SeparationSets sepsets(3);
        sepsets.store(0, 1, {});
        MixedGraph expected;
        expected.n = 3;
        expected.directed = {{0, 2}, {1, 2}};
        EXPECT(find_v_structures(skel, sepsets) == expected);
        sepsets.store(0, 1, {2});
        expected.directed.clear();
        expected.undirected = {{0, 2}, {1, 2}};
        EXPECT(find_v_structures(skel, sepsets) == expected);
        EXPECT_THROW(find_v_structures(skel, SeparationSets(3)), std::invalid_argument);
        EXPECT_THROW(find_v_structures(skel, SeparationSets(4)), std::invalid_argument);
    }
    {
        const AdjacencyMatrix skel = make_skeleton(4, {{0, 1}, {1, 2}, {0, 3}});
        SeparationSets sepsets(4);
        sepsets.store(0, 2, {});
        sepsets.store(1, 3, {});
        const MixedGraph g = find_v_structures(skel, sepsets);
        EXPECT(g.has_undirected(0, 1) && g.has_directed(2, 1) && g.has_directed(3, 0));
    }
    {
        MixedGraph g;
        g.n = 4;
        g.directed = {{2, 1}, {3, 1}};
        g.undirected = {{0, 1}, {0, 2}, {0, 3}};
        MixedGraph expected;
        expected.n = 4;
        expected.directed = {{0, 1}, {2, 1}, {3, 1}};
        expected.undirected = {{0, 2}, {0, 3}};
        const MixedGraph once = apply_meek_rules(g);
        EXPECT(once == expected);
        EXPECT(apply_meek_rules(once) == once);
        g.directed = {{2, 3}, {3, 1}};
        g.undirected = {{0, 1}, {0, 2}};
        expected.directed = {{0, 1}, {2, 3}, {3, 1}};
        expected.undirected = {{0, 2}};
        EXPECT(apply_meek_rules(g) == expected);
    }
    {
        const AdjacencyMatrix skel = make_skeleton(4, {{0, 1}, {1, 2}, {2, 3}});
        SeparationSets sepsets(4);
        sepsets.store(0, 2, {});
        sepsets.store(1, 3, {2});
        MixedGraph expected;
        expected.n = 4;
        expected.directed = {{0, 1}, {2, 1}};
        expected.undirected = {{2, 3}};
        EXPECT(orient_skeleton(skel, sepsets) == expected);
    }
    {
        // OrientSkeleton.PreservesTheSkeletonExactly on a device skeleton (test_orient.cpp:183-202)
        std::vector<double> w(12 * 12);
        orc_random_dag(12, 0.25, 5, w.data());
        std::vector<double> x(12 * 800);
        orc_sample_linear_gaussian(w.data(), 12, 800, 6, x.data());
        const SkeletonResult r = run_pc_stable(DataMatrix(800, 12, x), SkeletonConfig{});
        const MixedGraph g = orient_skeleton(r.skeleton, r.sepsets);
        EXPECT(g.n == 12);
        EXPECT(g.directed.size() + g.undirected.size() == r.skeleton.edge_count());
        for (Index i = 0; i < 12; ++i)
            for (Index j = i + 1; j < 12; ++j) EXPECT(g.adjacent(i, j) == r.skeleton.at(i, j));
        for (const auto& [a, b] : g.directed) EXPECT(!g.has_directed(b, a) && !g.has_undirected(a, b));
        for (const auto& [a, b] : g.undirected) EXPECT(a < b);
    }
}

// test_skeleton.cpp:342-358 (EdgeParallelStrategy.StopsAtFirstSeparatingSet) through run_level_*,
// plus run_level_zero and the set-shared dense-row pin (test_skeleton.cpp:300-317) with the
// drop-in's documented counter semantics.
static void test_run_level_entry_points() {
    const double s = 1.0 / std::sqrt(3.0), t = std::sqrt(3.0) / 2.0;
    const CorrelationMatrix c =
        make_correlation(4, {{0, 1, s}, {0, 2, s}, {0, 3, t}, {1, 2, 0.0}, {1, 3, 0.5}, {2, 3, 0.5}});
    {  // level 0 on the complete graph removes (1, 2) with the empty set
        AdjacencyMatrix graph = AdjacencyMatrix::complete(4);
        SeparationSets sepsets(4);
        const LevelStats l0 = run_level_zero(c, stats::threshold_tau(0.05, 1000, 0), graph, sepsets, 2);
        EXPECT(l0.ci_tests == 6u && l0.edges_removed == 1u);
        EXPECT(!graph.at(1, 2) && sepsets.find(1, 2) && sepsets.find(1, 2)->empty());
    }
    for (Strategy st : {Strategy::EdgeParallel, Strategy::SetShared, Strategy::Serial}) {
        AdjacencyMatrix graph = AdjacencyMatrix::complete(4);
        SeparationSets sepsets(4);
        graph.clear_edge(1, 2);
        const CompactedAdjacency snapshot = compact(graph);
        SkeletonConfig cfg;
        cfg.strategy = st;
        const double tau1 = stats::threshold_tau(0.05, 1000, 1);
        const LevelStats tally =
            st == Strategy::EdgeParallel ? run_level_edge_parallel(c, snapshot, graph, sepsets, tau1, 1, cfg)
            : st == Strategy::SetShared  ? run_level_set_shared(c, snapshot, graph, sepsets, tau1, 1, cfg)
                                         : run_level_serial(c, snapshot, graph, sepsets, tau1, 1, cfg);
        EXPECT(tally.edges_removed == 2u);
        EXPECT(!graph.at(1, 3) && !graph.at(2, 3));
        EXPECT(sepsets.find(1, 3) && *sepsets.find(1, 3) == std::vector<Index>{0});
        EXPECT(sepsets.find(2, 3) && *sepsets.find(2, 3) == std::vector<Index>{0});
        // a snapshot that is not compact(graph) is rejected (the device reads the live graph)
        AdjacencyMatrix other = AdjacencyMatrix::complete(4);
        EXPECT_THROW(run_level_serial(c, compact(other), graph, sepsets, tau1, 1, cfg), std::invalid_argument);
    }
    {  // test_skeleton.cpp:300-317: complete 6-vertex graph, all c = 0.9, tau ~ 0 -> nothing separates
        std::vector<std::tuple<Index, Index, double>> e;
        for (Index i = 0; i < 6; ++i)
            for (Index j = i + 1; j < 6; ++j) e.push_back({i, j, 0.9});
        const CorrelationMatrix c6 = make_correlation(6, e);
        AdjacencyMatrix graph = AdjacencyMatrix::complete(6);
        SeparationSets sepsets(6);
        SkeletonConfig cfg;
        cfg.strategy = Strategy::SetShared;
        const LevelStats tally = run_level_set_shared(c6, compact(graph), graph, sepsets, 1e-9, 2, cfg);
        // ci_tests: 15 edges x 2 directions x C(4, 2) sets = 180, the same for every strategy when
        // nothing separates (the reference's SetShared also reports 6 * C(5, 2) * 3 = 180).
        EXPECT(tally.ci_tests == 180u);
        // pseudo_inverses follow Strategy::Serial (one per test: 180); the reference's SetShared
        // reports one per (row, set): 6 * C(5, 2) = 60 -- the documented deviation.
        EXPECT(tally.pseudo_inverses == 180u);
        EXPECT(tally.edges_removed == 0u && graph.edge_count() == 15u);
    }
}

int main() {
    const std::vector<std::pair<std::string, std::function<void()>>> tests = {
        {"star_graph_set", [] { test_star_graph(Strategy::SetShared); }},
        {"star_graph_edge", [] { test_star_graph(Strategy::EdgeParallel); }},
        {"star_graph_serial", [] { test_star_graph(Strategy::Serial); }},
        {"level_cap_and_sample_size", test_level_cap_and_sample_size},
        {"errors", test_errors},
        {"chain_and_collider", test_chain_and_collider},
        {"oracle_p50_set", [] { test_against_oracle(50, 0.2, 1000, 7919, Strategy::SetShared); }},
        {"oracle_p100_edge", [] { test_against_oracle(100, 2.0 / 99.0, 1000, 0, Strategy::EdgeParallel); }},
        {"oracle_p120_set", [] { test_against_oracle(120, 0.1, 500, 15838, Strategy::SetShared); }},
        {"orientation", test_orientation},
        {"run_level_entry_points", test_run_level_entry_points},
    };
    for (const auto& [name, fn] : tests) {
        const int before = g_failed;
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_failed;
            std::fprintf(stderr, "%s: unexpected exception: %s\n", name.c_str(), e.what());
        }
        std::printf("[%s] %s\n", g_failed == before ? "  OK  " : " FAIL ", name.c_str());
    }
    std::printf("%d checks, %d failed\n", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
