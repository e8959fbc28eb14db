/*
 * pcstable_b200.hpp -- C++ drop-in for the reference's skeleton API, backed by
 * libpcstable_b200.so (sm_100a) through the C ABI of pcstable_b200.h.
 *
 * A caller of the reference library (proj/include/pcstable) swaps
 *     #include "pcstable/skeleton.hpp"      (and stats.hpp / core.hpp)
 * for
 *     #include "pcstable_b200.hpp"
 * and links -lpcstable_b200.  The names, argument meaning and exceptions below
 * are the reference's:
 *
 *   pcstable::Index, ZeroVarianceError, DegenerateConditioningError,
 *   LevelUnreachableError                                    core.hpp:20-44
 *   pcstable::DataMatrix                                     core.hpp:48-67
 *   pcstable::CorrelationMatrix                              core.hpp:71-103
 *   pcstable::AdjacencyMatrix                                core.hpp:109-194
 *   pcstable::CompactedAdjacency, compact                    core.hpp:200-239
 *   pcstable::SeparationSets                                 core.hpp:267-339
 *   pcstable::Strategy, SkeletonConfig, LevelStats           core.hpp:341-393
 *   pcstable::StopReason, SkeletonResult                     skeleton.hpp:22-40
 *   pcstable::stats::threshold_tau                           stats.hpp:120-129
 *   pcstable::stats::compute_correlation                     stats.hpp:132-156
 *   pcstable::run_pc_stable                                  skeleton.hpp:341-391
 *
 * Every strategy runs on the device and yields Strategy::Serial's skeleton,
 * sepsets and counters (the reference's only deterministic sepset rule);
 * Strategy::EdgeParallel selects the cuPC-E kernels, the others cuPC-S.  The
 * tile-shape knobs and worker_count / schedule_seed are accepted and validated
 * like the reference's but never change a result (proj/README.md:80-82).
 * There is no CPU fallback: without a device the calls throw.
 *
 * Eigen is optional: when <Eigen/Dense> is available the Eigen-typed
 * constructors of the reference are provided as well.
 */
#ifndef PCSTABLE_B200_HPP
#define PCSTABLE_B200_HPP

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <optional>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pcstable_b200.h"

#if defined(__has_include)
#if __has_include(<Eigen/Dense>)
#include <Eigen/Dense>
#define PCSTABLE_B200_HAVE_EIGEN 1
#endif
#endif

namespace pcstable {

using Index = std::int32_t;

class ZeroVarianceError : public std::runtime_error {
public:
    ZeroVarianceError(Index column, std::string what) : std::runtime_error(std::move(what)), column_(column) {}
    Index column() const { return column_; }

private:
    Index column_;
};

class DegenerateConditioningError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

class LevelUnreachableError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

/// Device failure without a reference counterpart (no GPU, CUDA error, level beyond the device path).
class DeviceError : public std::runtime_error {
public:
    DeviceError(int code, std::string what) : std::runtime_error(std::move(what)), code_(code) {}
    int code() const { return code_; }

private:
    int code_;
};

namespace detail {

/// pcs_status -> the reference's exception classes (SURVEY.md §8(b) "Error conventions").
inline void check(pcs_status st, Index column = -1) {
    if (st == PCS_OK) return;
    const std::string msg = pcs_last_error();
    switch (st) {
        case PCS_EINVAL:
        case PCS_ENAN: throw std::invalid_argument(msg);
        case PCS_EZEROVAR: throw ZeroVarianceError(column, msg);
        case PCS_EOVERFLOW: throw std::overflow_error(msg);
        case PCS_ELEVEL: throw LevelUnreachableError(msg);
        default: throw DeviceError(static_cast<int>(st), msg);
    }
}

struct ResultDeleter {
    void operator()(pcs_result* r) const { pcs_result_free(r); }
};
using ResultPtr = std::unique_ptr<pcs_result, ResultDeleter>;

}  // namespace detail

/// m samples x n variables, column-major like Eigen::MatrixXd (value(r, j) = data[j * m + r]).
class DataMatrix {
public:
    DataMatrix(Index samples, Index variables, std::vector<double> column_major)
        : m_(samples), n_(variables), values_(std::move(column_major)) {
        if (m_ < 4) throw std::invalid_argument("DataMatrix: need at least 4 samples, got " + std::to_string(m_));
        if (n_ < 2) throw std::invalid_argument("DataMatrix: need at least 2 variables, got " + std::to_string(n_));
        if (values_.size() != static_cast<std::size_t>(m_) * n_)
            throw std::invalid_argument("DataMatrix: buffer size must be samples * variables");
        for (double v : values_)
            if (!std::isfinite(v)) throw std::invalid_argument("DataMatrix: values must be finite");
    }
#ifdef PCSTABLE_B200_HAVE_EIGEN
    explicit DataMatrix(const Eigen::MatrixXd& values)
        : DataMatrix(static_cast<Index>(values.rows()), static_cast<Index>(values.cols()),
                     std::vector<double>(values.data(), values.data() + values.size())) {}
#endif
    Index sample_count() const { return m_; }
    Index variable_count() const { return n_; }
    double operator()(Index r, Index j) const { return values_[static_cast<std::size_t>(j) * m_ + r]; }
    const double* data() const { return values_.data(); }

private:
    Index m_, n_;
    std::vector<double> values_;
};

/// Pearson correlation matrix; construction validates, symmetrises and clamps exactly like
/// core.hpp:73-95 (the device repeats the same normalisation on upload).
class CorrelationMatrix {
public:
    CorrelationMatrix(Index n, std::vector<double> values) : n_(n), values_(std::move(values)) {
        constexpr double kTol = 1e-12;
        if (n_ < 2 || values_.size() != static_cast<std::size_t>(n_) * n_)
            throw std::invalid_argument("CorrelationMatrix: need a square matrix, n >= 2");
        for (Index i = 0; i < n_; ++i) {
            if (std::abs(at(i, i) - 1.0) > kTol) throw std::invalid_argument("CorrelationMatrix: diagonal must be 1");
            at(i, i) = 1.0;
            for (Index j = i + 1; j < n_; ++j) {
                const double a = at(i, j), b = at(j, i);
                if (!std::isfinite(a) || !std::isfinite(b) || std::abs(a - b) > kTol)
                    throw std::invalid_argument("CorrelationMatrix: matrix must be symmetric");
                double v = 0.5 * (a + b);
                if (std::abs(v) > 1.0 + kTol)
                    throw std::invalid_argument("CorrelationMatrix: entries must lie in [-1, 1]");
                v = std::clamp(v, -1.0, 1.0);
                at(i, j) = v;
                at(j, i) = v;
            }
        }
    }
#ifdef PCSTABLE_B200_HAVE_EIGEN
    explicit CorrelationMatrix(const Eigen::MatrixXd& values)
        : CorrelationMatrix(static_cast<Index>(values.rows()),
                            std::vector<double>(values.data(), values.data() + values.size())) {
        if (values.rows() != values.cols()) throw std::invalid_argument("CorrelationMatrix: need a square matrix, n >= 2");
    }
#endif
    Index size() const { return n_; }
    double operator()(Index i, Index j) const { return values_[static_cast<std::size_t>(i) * n_ + j]; }
    const double* data() const { return values_.data(); }

private:
    double& at(Index i, Index j) { return values_[static_cast<std::size_t>(i) * n_ + j]; }
    Index n_;
    std::vector<double> values_;
};

/// Undirected graph as a dense cell matrix (core.hpp:109-194).  The device returns the final
/// skeleton; clear_edge keeps the reference's claim-once semantics for callers that edit it.
class AdjacencyMatrix {
public:
    explicit AdjacencyMatrix(Index n) : n_(n), cells_(static_cast<std::size_t>(n) * n, 0) {
        if (n < 2) throw std::invalid_argument("AdjacencyMatrix: need n >= 2");
    }
    static AdjacencyMatrix complete(Index n) {
        AdjacencyMatrix a(n);
        for (Index i = 0; i < n; ++i)
            for (Index j = i + 1; j < n; ++j) a.set_edge(i, j);
        return a;
    }
    Index size() const { return n_; }
    bool at(Index i, Index j) const { return cells_[static_cast<std::size_t>(i) * n_ + j] != 0; }
    void set_edge(Index i, Index j) {
        check_pair(i, j);
        cells_[static_cast<std::size_t>(i) * n_ + j] = 1;
        cells_[static_cast<std::size_t>(j) * n_ + i] = 1;
    }
    bool clear_edge(Index i, Index j) {
        check_pair(i, j);
        const bool was = at(i, j);
        cells_[static_cast<std::size_t>(i) * n_ + j] = 0;
        cells_[static_cast<std::size_t>(j) * n_ + i] = 0;
        return was;
    }
    std::size_t edge_count() const {
        std::size_t c = 0;
        for (Index i = 0; i < n_; ++i)
            for (Index j = i + 1; j < n_; ++j) c += at(i, j);
        return c;
    }
    friend bool operator==(const AdjacencyMatrix& a, const AdjacencyMatrix& b) {
        return a.n_ == b.n_ && a.cells_ == b.cells_;
    }
    uint8_t* raw() { return cells_.data(); }

private:
    void check_pair(Index i, Index j) const {
        if (i == j || i < 0 || j < 0 || i >= n_ || j >= n_)
            throw std::invalid_argument("AdjacencyMatrix: invalid vertex pair");
    }
    Index n_;
    std::vector<uint8_t> cells_;
};

/// CSR snapshot (core.hpp:200-225) and its builder (core.hpp:227-239).
class CompactedAdjacency {
public:
    CompactedAdjacency(std::vector<Index> offsets, std::vector<Index> indices)
        : offsets_(std::move(offsets)), indices_(std::move(indices)), max_width_(0) {
        for (std::size_t i = 0; i + 1 < offsets_.size(); ++i)
            max_width_ = std::max(max_width_, offsets_[i + 1] - offsets_[i]);
    }
    Index size() const { return static_cast<Index>(offsets_.size()) - 1; }
    const Index* row(Index i) const { return indices_.data() + offsets_[i]; }
    Index count(Index i) const { return offsets_[i + 1] - offsets_[i]; }
    Index max_width() const { return max_width_; }

private:
    std::vector<Index> offsets_, indices_;
    Index max_width_;
};

inline CompactedAdjacency compact(const AdjacencyMatrix& a) {
    const Index n = a.size();
    std::vector<Index> off(static_cast<std::size_t>(n) + 1, 0), idx;
    for (Index i = 0; i < n; ++i) {
        off[i] = static_cast<Index>(idx.size());
        for (Index j = 0; j < n; ++j)
            if (a.at(i, j)) idx.push_back(j);
    }
    off[n] = static_cast<Index>(idx.size());
    return CompactedAdjacency(std::move(off), std::move(idx));
}

/// One slot per unordered pair, triangular index of core.hpp:329-335.
class SeparationSets {
public:
    explicit SeparationSets(Index n) : n_(n), slots_(n >= 2 ? static_cast<std::size_t>(n) * (n - 1) / 2 : 0) {
        if (n < 2) throw std::invalid_argument("SeparationSets: need n >= 2");
    }
    Index size() const { return n_; }
    void store(Index i, Index j, const std::vector<Index>& set) { slots_[slot(i, j)] = set; }
    /// Null when no set has been recorded for the pair.
    const std::vector<Index>* find(Index i, Index j) const {
        const auto& s = slots_[slot(i, j)];
        return s ? &*s : nullptr;
    }
    std::size_t stored_count() const {
        std::size_t c = 0;
        for (const auto& s : slots_) c += s.has_value();
        return c;
    }
    template <typename Fn>
    void for_each(Fn&& fn) const {
        for (Index i = 0; i < n_; ++i)
            for (Index j = i + 1; j < n_; ++j)
                if (const auto* s = find(i, j)) fn(i, j, *s);
    }

private:
    std::size_t slot(Index i, Index j) const {
        if (i == j || i < 0 || j < 0 || i >= n_ || j >= n_)
            throw std::invalid_argument("SeparationSets: invalid vertex pair");
        if (i > j) std::swap(i, j);
        return static_cast<std::size_t>(i) * (2 * static_cast<std::size_t>(n_) - i - 1) / 2 + (j - i - 1);
    }
    Index n_;
    std::vector<std::optional<std::vector<Index>>> slots_;
};

enum class Strategy { Serial, EdgeParallel, SetShared };

inline const char* to_string(Strategy s) {
    switch (s) {
        case Strategy::Serial: return "serial";
        case Strategy::EdgeParallel: return "edge";
        case Strategy::SetShared: return "set";
    }
    return "?";
}

struct SkeletonConfig {
    double alpha = 0.05;
    std::optional<int> max_level;
    Strategy strategy = Strategy::Serial;
    int edges_per_unit = 2;
    int workers_per_edge = 32;
    int set_groups = 2;
    int unit_width = 64;
    int worker_count = 1;
    std::optional<std::uint64_t> schedule_seed;
    int device = 0;  // CUDA device ordinal (B200 addition)

    void validate() const {  // core.hpp:370-383
        if (!(alpha > 0.0 && alpha < 1.0)) throw std::invalid_argument("SkeletonConfig: alpha must lie in (0, 1)");
        if (max_level && *max_level < 0) throw std::invalid_argument("SkeletonConfig: max_level must be >= 0");
        if (edges_per_unit < 1) throw std::invalid_argument("SkeletonConfig: edges_per_unit must be >= 1");
        if (workers_per_edge < 1) throw std::invalid_argument("SkeletonConfig: workers_per_edge must be >= 1");
        if (set_groups < 1) throw std::invalid_argument("SkeletonConfig: set_groups must be >= 1");
        if (unit_width < 1) throw std::invalid_argument("SkeletonConfig: unit_width must be >= 1");
        if (worker_count < 1) throw std::invalid_argument("SkeletonConfig: worker_count must be >= 1");
    }
};

struct LevelStats {
    int level = 0;
    std::uint64_t ci_tests = 0;         // == Strategy::Serial's count
    std::uint64_t pseudo_inverses = 0;  // == Strategy::Serial's count
    std::uint64_t edges_removed = 0;
    std::chrono::nanoseconds elapsed{0};
    // device additions
    std::uint64_t device_ci_tests = 0;
    std::uint64_t device_pseudo_inverses = 0;
    double kernel_ms = 0.0;
    std::uint64_t device_exact_tests = 0;
    std::uint64_t device_near_threshold = 0;  // tests inside the +-1e-9 threshold band (exact comparison)
};

enum class StopReason { MaxDegreeReached, LevelCapReached, SampleSizeExhausted };

inline const char* to_string(StopReason r) {
    switch (r) {
        case StopReason::MaxDegreeReached: return "max-degree";
        case StopReason::LevelCapReached: return "level-cap";
        case StopReason::SampleSizeExhausted: return "sample-size";
    }
    return "?";
}

struct SkeletonResult {
    AdjacencyMatrix skeleton;
    SeparationSets sepsets;
    std::vector<LevelStats> levels;
    StopReason stop_reason;
    double device_seconds = 0.0;  // CUDA-event time of the device pipeline

    int levels_run() const { return static_cast<int>(levels.size()); }
};

namespace stats {

inline double threshold_tau(double alpha, Index m, int ell) {
    double tau = 0.0;
    detail::check(pcs_threshold_tau(alpha, m, ell, &tau));
    return tau;
}

inline CorrelationMatrix compute_correlation(const DataMatrix& data) {
    const Index p = data.variable_count();
    std::vector<double> c(static_cast<std::size_t>(p) * p);
    int32_t col = -1;
    const pcs_status st = pcs_correlation(data.data(), data.sample_count(), p, c.data(), &col);
    detail::check(st, col);
    return CorrelationMatrix(p, std::move(c));
}

}  // namespace stats

namespace detail {

inline pcs_config to_abi(const SkeletonConfig& cfg) {
    pcs_config c;
    pcs_config_default(&c);
    c.alpha = cfg.alpha;
    c.max_level = cfg.max_level ? *cfg.max_level : -1;
    c.variant = cfg.strategy == Strategy::EdgeParallel ? PCS_VARIANT_EDGE : PCS_VARIANT_SET;
    c.edges_per_unit = cfg.edges_per_unit;
    c.workers_per_edge = cfg.workers_per_edge;
    c.set_groups = cfg.set_groups;
    c.unit_width = cfg.unit_width;
    c.device = cfg.device;
    return c;
}

inline SkeletonResult collect(pcs_result* raw) {
    ResultPtr r(raw);
    const Index p = pcs_result_p(r.get());
    AdjacencyMatrix adj(p);
    pcs_result_adjacency(r.get(), adj.raw());
    SeparationSets sep(p);
    const std::size_t slots = static_cast<std::size_t>(p) * (p - 1) / 2;
    std::vector<int32_t> level(slots);
    std::vector<int64_t> offset(slots);
    std::vector<int32_t> members(static_cast<std::size_t>(std::max<int64_t>(pcs_result_member_total(r.get()), 1)));
    pcs_result_sepsets(r.get(), level.data(), offset.data(), members.data());
    std::size_t s = 0;
    for (Index i = 0; i < p; ++i)
        for (Index j = i + 1; j < p; ++j, ++s)
            if (level[s] >= 0)
                sep.store(i, j, std::vector<Index>(members.begin() + offset[s], members.begin() + offset[s] + level[s]));
    const int32_t nl = pcs_result_levels(r.get(), nullptr, 0);
    std::vector<pcs_level_stats> raw_levels(static_cast<std::size_t>(nl));
    pcs_result_levels(r.get(), raw_levels.data(), nl);
    std::vector<LevelStats> levels;
    for (const auto& L : raw_levels) {
        LevelStats x;
        x.level = L.level;
        x.ci_tests = L.ci_tests;
        x.pseudo_inverses = L.pseudo_inverses;
        x.edges_removed = L.edges_removed;
        x.elapsed = std::chrono::nanoseconds(static_cast<std::int64_t>(L.elapsed_s * 1e9));
        x.device_ci_tests = L.device_ci_tests;
        x.device_pseudo_inverses = L.device_pseudo_inverses;
        x.kernel_ms = L.kernel_ms;
        x.device_exact_tests = L.device_exact_tests;
        x.device_near_threshold = L.device_near_threshold;
        levels.push_back(x);
    }
    StopReason reason = StopReason::MaxDegreeReached;
    switch (pcs_result_stop_reason(r.get())) {
        case PCS_STOP_LEVEL_CAP: reason = StopReason::LevelCapReached; break;
        case PCS_STOP_SAMPLE_SIZE: reason = StopReason::SampleSizeExhausted; break;
        default: break;
    }
    return SkeletonResult{std::move(adj), std::move(sep), std::move(levels), reason,
                          pcs_result_device_seconds(r.get())};
}

}  // namespace detail

/// run_pc_stable (skeleton.hpp:341-391) on the device.
inline SkeletonResult run_pc_stable(const CorrelationMatrix& c, Index sample_count, const SkeletonConfig& cfg) {
    cfg.validate();
    if (sample_count < 4) throw std::invalid_argument("run_pc_stable: need at least 4 samples");
    const pcs_config abi = detail::to_abi(cfg);
    pcs_result* r = nullptr;
    detail::check(pcs_run_pc_stable(c.data(), c.size(), sample_count, &abi, &r));
    return detail::collect(r);
}

namespace detail {

// one level on the device from the caller's live graph (pcs_run_level); the graph doubles as the
// level-start snapshot, so a separate snapshot must equal compact(graph)
inline LevelStats run_level_device(const CorrelationMatrix& c, AdjacencyMatrix& graph, SeparationSets& sepsets,
                                   double tau, int ell, SkeletonConfig cfg, Strategy strategy) {
    const Index n = c.size();
    if (graph.size() != n || sepsets.size() != n) throw std::invalid_argument("run_level: size mismatch");
    cfg.strategy = strategy;
    cfg.validate();
    const pcs_config abi = to_abi(cfg);
    const std::vector<uint8_t> before(graph.raw(), graph.raw() + static_cast<std::size_t>(n) * n);
    pcs_result* raw = nullptr;
    check(pcs_run_level(c.data(), n, ell, tau, &abi, graph.raw(), &raw));
    ResultPtr r(raw);
    const std::size_t slots = static_cast<std::size_t>(n) * (n - 1) / 2;
    std::vector<int32_t> level(slots);
    std::vector<int64_t> offset(slots);
    std::vector<int32_t> members(static_cast<std::size_t>(std::max<int64_t>(pcs_result_member_total(r.get()), 1)));
    pcs_result_sepsets(r.get(), level.data(), offset.data(), members.data());
    std::size_t s = 0;
    for (Index i = 0; i < n; ++i)
        for (Index j = i + 1; j < n; ++j, ++s)
            if (before[static_cast<std::size_t>(i) * n + j] && !graph.at(i, j))  // removed by this level
                sepsets.store(i, j, level[s] == ell ? std::vector<Index>(members.begin() + offset[s],
                                                                         members.begin() + offset[s] + ell)
                                                    : std::vector<Index>{});
    LevelStats out;
    out.level = ell;
    pcs_level_stats L{};
    if (pcs_result_levels(r.get(), &L, 1) == 1) {
        out.ci_tests = L.ci_tests;
        out.pseudo_inverses = L.pseudo_inverses;
        out.edges_removed = L.edges_removed;
        out.elapsed = std::chrono::nanoseconds(static_cast<std::int64_t>(L.elapsed_s * 1e9));
        out.device_ci_tests = L.device_ci_tests;
        out.device_pseudo_inverses = L.device_pseudo_inverses;
        out.kernel_ms = L.kernel_ms;
        out.device_exact_tests = L.device_exact_tests;
        out.device_near_threshold = L.device_near_threshold;
    }
    return out;
}

inline void check_snapshot(const CompactedAdjacency& snapshot, const AdjacencyMatrix& graph) {
    const Index n = graph.size();
    bool same = snapshot.size() == n;
    for (Index i = 0; same && i < n; ++i) {
        Index k = 0;
        for (Index j = 0; j < n && same; ++j)
            if (graph.at(i, j)) same = k < snapshot.count(i) && snapshot.row(i)[k++] == j;
        same = same && k == snapshot.count(i);
    }
    if (!same) throw std::invalid_argument("run_level: the device takes the snapshot from the live graph; "
                                           "snapshot must equal compact(graph)");
}

}  // namespace detail

/// run_level_zero (skeleton.hpp:262-288): one unconditional test per unordered pair; `workers` is
/// accepted for signature parity (the device schedule has no worker count).
inline LevelStats run_level_zero(const CorrelationMatrix& c, double tau0, AdjacencyMatrix& graph,
                                 SeparationSets& sepsets, int workers = 1) {
    if (sepsets.size() != graph.size()) throw std::invalid_argument("run_level_zero: size mismatch");
    (void)workers;
    return detail::run_level_device(c, graph, sepsets, tau0, 0, SkeletonConfig{}, Strategy::Serial);
}

/// run_level_serial (skeleton.hpp:292-307): Strategy::Serial's level (cuPC-S kernels, serial-rule result).
inline LevelStats run_level_serial(const CorrelationMatrix& c, const CompactedAdjacency& snapshot,
                                   AdjacencyMatrix& graph, SeparationSets& sepsets, double tau, int ell,
                                   const SkeletonConfig& cfg) {
    if (ell < 1) throw std::invalid_argument("run_level_serial: need ell >= 1");
    detail::check_snapshot(snapshot, graph);
    return detail::run_level_device(c, graph, sepsets, tau, ell, cfg, Strategy::Serial);
}

/// run_level_edge_parallel (skeleton.hpp:311-320): the cuPC-E kernels.
inline LevelStats run_level_edge_parallel(const CorrelationMatrix& c, const CompactedAdjacency& snapshot,
                                          AdjacencyMatrix& graph, SeparationSets& sepsets, double tau, int ell,
                                          const SkeletonConfig& cfg) {
    if (ell < 1) throw std::invalid_argument("run_level_edge_parallel: need ell >= 1");
    detail::check_snapshot(snapshot, graph);
    return detail::run_level_device(c, graph, sepsets, tau, ell, cfg, Strategy::EdgeParallel);
}

/// run_level_set_shared (skeleton.hpp:325-333): the cuPC-S kernels.
inline LevelStats run_level_set_shared(const CorrelationMatrix& c, const CompactedAdjacency& snapshot,
                                       AdjacencyMatrix& graph, SeparationSets& sepsets, double tau, int ell,
                                       const SkeletonConfig& cfg) {
    if (ell < 1) throw std::invalid_argument("run_level_set_shared: need ell >= 1");
    detail::check_snapshot(snapshot, graph);
    return detail::run_level_device(c, graph, sepsets, tau, ell, cfg, Strategy::SetShared);
}

/// compute_correlation + run_pc_stable in one device pipeline (the pair bench.hpp:107-113 times).
inline SkeletonResult run_pc_stable(const DataMatrix& data, const SkeletonConfig& cfg) {
    cfg.validate();
    const pcs_config abi = detail::to_abi(cfg);
    pcs_result* r = nullptr;
    int32_t col = -1;
    detail::check(pcs_run_pc_stable_data(data.data(), data.sample_count(), data.variable_count(), &abi, &r, &col),
                  col);
    return detail::collect(r);
}

/// Partially directed graph produced by orientation (orient.hpp:15-32).
struct MixedGraph {
    Index n = 0;
    std::set<std::pair<Index, Index>> directed;
    std::set<std::pair<Index, Index>> undirected;

    bool has_directed(Index from, Index to) const { return directed.count({from, to}) > 0; }
    bool has_undirected(Index a, Index b) const {
        if (a > b) std::swap(a, b);
        return undirected.count({a, b}) > 0;
    }
    bool adjacent(Index a, Index b) const { return has_undirected(a, b) || has_directed(a, b) || has_directed(b, a); }
    friend bool operator==(const MixedGraph& x, const MixedGraph& y) {
        return x.n == y.n && x.directed == y.directed && x.undirected == y.undirected;
    }
};

namespace detail {

inline MixedGraph orient_call(const AdjacencyMatrix& skeleton, const SeparationSets* sepsets, int stage,
                              const std::vector<int32_t>& directed_in) {
    const Index n = skeleton.size();
    if (sepsets && sepsets->size() != n)
        throw std::invalid_argument("find_v_structures: skeleton and sepsets sizes differ");
    const std::size_t slots = static_cast<std::size_t>(n) * (n - 1) / 2;
    std::vector<int32_t> level(std::max<std::size_t>(slots, 1), -1), members;
    std::vector<int64_t> offset(std::max<std::size_t>(slots, 1), 0);
    std::vector<uint8_t> cells(static_cast<std::size_t>(n) * n);
    for (Index i = 0; i < n; ++i)
        for (Index j = 0; j < n; ++j) cells[static_cast<std::size_t>(i) * n + j] = i != j && skeleton.at(i, j);
    if (sepsets) {
        std::size_t s = 0;
        for (Index i = 0; i < n; ++i)
            for (Index j = i + 1; j < n; ++j, ++s)
                if (const auto* set = sepsets->find(i, j)) {
                    level[s] = static_cast<int32_t>(set->size());
                    offset[s] = static_cast<int64_t>(members.size());
                    members.insert(members.end(), set->begin(), set->end());
                }
    }
    if (members.empty()) members.push_back(0);
    pcs_mixed_graph* g = nullptr;
    check(pcs_orient_skeleton(n, cells.data(), level.data(), offset.data(), members.data(), stage,
                              directed_in.empty() ? nullptr : directed_in.data(),
                              static_cast<int64_t>(directed_in.size() / 2), &g));
    MixedGraph out;
    out.n = n;
    std::vector<int32_t> d(2 * static_cast<std::size_t>(pcs_mixed_directed_count(g)) + 2),
        u(2 * static_cast<std::size_t>(pcs_mixed_undirected_count(g)) + 2);
    pcs_mixed_directed(g, d.data());
    pcs_mixed_undirected(g, u.data());
    for (int64_t k = 0; k < pcs_mixed_directed_count(g); ++k) out.directed.insert({d[2 * k], d[2 * k + 1]});
    for (int64_t k = 0; k < pcs_mixed_undirected_count(g); ++k) out.undirected.insert({u[2 * k], u[2 * k + 1]});
    pcs_mixed_free(g);
    return out;
}

}  // namespace detail

/// find_v_structures (orient.hpp:40-89): unshielded-triple votes on the device.
inline MixedGraph find_v_structures(const AdjacencyMatrix& skeleton, const SeparationSets& sepsets) {
    return detail::orient_call(skeleton, &sepsets, 1, {});
}

/// apply_meek_rules (orient.hpp:147-167): the reference's visiting order, on the host.
inline MixedGraph apply_meek_rules(MixedGraph g) {
    if (g.n < 2) return g;
    AdjacencyMatrix skel(g.n);
    std::vector<int32_t> din;
    for (const auto& [a, b] : g.directed) {
        skel.set_edge(a, b);
        din.push_back(a);
        din.push_back(b);
    }
    for (const auto& [a, b] : g.undirected) skel.set_edge(a, b);
    return detail::orient_call(skel, nullptr, 2, din);
}

/// orient_skeleton (orient.hpp:170-173).
inline MixedGraph orient_skeleton(const AdjacencyMatrix& skeleton, const SeparationSets& sepsets) {
    return detail::orient_call(skeleton, &sepsets, 3, {});
}

}  // namespace pcstable

#endif  // PCSTABLE_B200_HPP
