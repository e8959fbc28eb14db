// pcstable_b200 -- the reference CLI (proj/tools/pcstable_main.cpp) on the B200 path
// (SURVEY.md §8(f) rows 3 and 4): the same subcommands, flags, file formats
// (io.hpp:121-242), report schema (pcstable_main.cpp:147-173), bench CSV
// (bench.hpp:142-175) and exit codes (pcstable_main.cpp:23-26), with every
// skeleton / correlation / orientation computed by libpcstable_b200.so through the
// C++ drop-in header.  Strategies serial|edge|set all run on the device (edge selects
// the cuPC-E kernels, the others cuPC-S) and return the serial strategy's result.
//
//   pcstable_b200 gen      --n N --d D --m M [--seed S] --out data.csv
//   pcstable_b200 skeleton --data data.csv [--alpha A] [--strategy serial|edge|set] [--beta B]
//                          [--gamma G] [--theta T] [--delta D] [--workers W] [--max-level L]
//                          --out prefix        (writes prefix.edges / .sepsets / .report.json)
//   pcstable_b200 orient   --skeleton prefix.edges --sepsets prefix.sepsets --out cpdag.txt
//   pcstable_b200 bench    --spec "n,d,m[;n,d,m...]" [--strategies serial,edge,set]
//                          [--repeats R] [--seed S] [--alpha A] [--workers W] [--max-level L]
//                          --out bench.csv
#include <algorithm>
#include <bit>
#include <charconv>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "pcstable_b200.hpp"

namespace {

using namespace pcstable;

constexpr int kExitOk = 0, kExitUsage = 1, kExitData = 2, kExitNumerical = 3;

struct ParseError : std::runtime_error {  // io.hpp:23-33
    using std::runtime_error::runtime_error;
};
struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------ io.hpp restated
std::string format_double(double v) {  // shortest round trip (io.hpp:37-41)
    char buf[32];
    const auto res = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, res.ptr);
}
bool parse_double(std::string_view t, double& out) {
    const auto res = std::from_chars(t.data(), t.data() + t.size(), out);
    return res.ec == std::errc() && res.ptr == t.data() + t.size();
}
bool parse_index(std::string_view t, Index& out) {
    const auto res = std::from_chars(t.data(), t.data() + t.size(), out);
    return res.ec == std::errc() && res.ptr == t.data() + t.size() && out >= 0;
}
std::string_view trim(std::string_view s) {
    while (!s.empty() && (s.front() == ' ' || s.front() == '\t' || s.front() == '\r')) s.remove_prefix(1);
    while (!s.empty() && (s.back() == ' ' || s.back() == '\t' || s.back() == '\r')) s.remove_suffix(1);
    return s;
}
std::vector<std::string_view> split(std::string_view line, char sep) {
    std::vector<std::string_view> out;
    std::size_t start = 0;
    for (std::size_t i = 0; i <= line.size(); ++i)
        if (i == line.size() || line[i] == sep) {
            out.push_back(trim(line.substr(start, i - start)));
            start = i + 1;
        }
    return out;
}
std::vector<std::string_view> split_ws(std::string_view line) {
    std::vector<std::string_view> out;
    std::size_t i = 0;
    while (i < line.size()) {
        while (i < line.size() && (line[i] == ' ' || line[i] == '\t' || line[i] == '\r')) ++i;
        const std::size_t s = i;
        while (i < line.size() && line[i] != ' ' && line[i] != '\t' && line[i] != '\r') ++i;
        if (i > s) out.push_back(line.substr(s, i - s));
    }
    return out;
}
std::string read_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw ParseError("cannot open file: " + path);
    std::ostringstream b;
    b << in.rdbuf();
    return std::move(b).str();
}
std::ofstream open_for_write(const std::string& path) {
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw ParseError("cannot open file for writing: " + path);
    return out;
}
template <typename Fn>
void for_each_line(std::string_view text, Fn&& fn) {
    std::size_t no = 0, start = 0;
    for (std::size_t i = 0; i <= text.size(); ++i)
        if (i == text.size() || text[i] == '\n') {
            ++no;
            const std::string_view line = trim(text.substr(start, i - start));
            if (!line.empty()) fn(no, line);
            start = i + 1;
        }
}

// data matrix: m x p column-major values (DataMatrix layout)
struct Data {
    Index m = 0, p = 0;
    std::vector<double> x;  // x[c * m + r]
};

void write_data_csv(const std::string& path, const Data& d) {  // io.hpp:121-135
    std::ofstream out = open_for_write(path);
    std::string line;
    for (Index r = 0; r < d.m; ++r) {
        line.clear();
        for (Index c = 0; c < d.p; ++c) {
            if (c > 0) line.push_back(',');
            line += format_double(d.x[static_cast<std::size_t>(c) * d.m + r]);
        }
        line.push_back('\n');
        out << line;
    }
    if (!out) throw ParseError("failed writing: " + path);
}

Data read_data_csv(const std::string& path) {  // io.hpp:140-182
    const std::string text = read_file(path);
    std::vector<std::vector<double>> rows;
    std::size_t cols = 0;
    bool first = true;
    for_each_line(text, [&](std::size_t no, std::string_view line) {
        const auto cells = split(line, ',');
        std::vector<double> row(cells.size());
        for (std::size_t c = 0; c < cells.size(); ++c)
            if (!parse_double(cells[c], row[c])) {
                if (first) {
                    first = false;
                    return;  // header line
                }
                throw ParseError(path + ": cannot parse '" + std::string(cells[c]) + "' as a number at row " +
                                 std::to_string(no) + ", column " + std::to_string(c + 1));
            }
        first = false;
        if (cols == 0) cols = row.size();
        else if (row.size() != cols)
            throw ParseError(path + ": row " + std::to_string(no) + " has " + std::to_string(row.size()) +
                             " columns, expected " + std::to_string(cols));
        rows.push_back(std::move(row));
    });
    if (rows.empty()) throw ParseError(path + ": no data rows");
    Data d;
    d.m = static_cast<Index>(rows.size());
    d.p = static_cast<Index>(cols);
    if (d.m < 1 || d.p < 1) throw ParseError(path + ": DataMatrix: empty");
    d.x.resize(static_cast<std::size_t>(d.m) * d.p);
    for (Index r = 0; r < d.m; ++r)
        for (Index c = 0; c < d.p; ++c) d.x[static_cast<std::size_t>(c) * d.m + r] = rows[r][c];
    return d;
}

std::uint64_t fingerprint(const Data& d) {  // io.hpp:187-200 (row-major, bytes LSB first)
    std::uint64_t h = 14695981039346656037ULL;
    for (Index r = 0; r < d.m; ++r)
        for (Index c = 0; c < d.p; ++c) {
            const std::uint64_t bits = std::bit_cast<std::uint64_t>(d.x[static_cast<std::size_t>(c) * d.m + r]);
            for (int b = 0; b < 8; ++b) {
                h ^= (bits >> (8 * b)) & 0xffULL;
                h *= 1099511628211ULL;
            }
        }
    return h;
}

void write_edge_list(const std::string& path, const AdjacencyMatrix& g) {  // io.hpp:204-211
    std::ofstream out = open_for_write(path);
    std::string buf;
    const Index n = g.size();
    for (Index i = 0; i < n; ++i)
        for (Index j = i + 1; j < n; ++j)
            if (g.at(i, j)) buf += std::to_string(i) + ' ' + std::to_string(j) + '\n';
    out << buf;
    if (!out) throw ParseError("failed writing: " + path);
}

void write_sepsets(const std::string& path, const SeparationSets& s) {  // io.hpp:232-242
    std::ofstream out = open_for_write(path);
    std::string buf;
    s.for_each([&](Index i, Index j, const std::vector<Index>& set) {
        buf += std::to_string(i) + ' ' + std::to_string(j) + " :";
        std::vector<Index> sorted(set);
        std::sort(sorted.begin(), sorted.end());
        for (Index v : sorted) buf += ' ' + std::to_string(v);
        buf += '\n';
    });
    out << buf;
    if (!out) throw ParseError("failed writing: " + path);
}

void write_mixed_graph(const std::string& path, const MixedGraph& g) {  // io.hpp:215-220
    std::ofstream out = open_for_write(path);
    for (const auto& [a, b] : g.directed) out << a << " > " << b << '\n';
    for (const auto& [a, b] : g.undirected) out << a << ' ' << b << '\n';
    if (!out) throw ParseError("failed writing: " + path);
}

struct EdgeListData {
    std::vector<std::pair<Index, Index>> undirected, directed;
    Index max_vertex = -1;
};

EdgeListData read_edge_list(const std::string& path) {  // io.hpp:251-283
    const std::string text = read_file(path);
    EdgeListData out;
    for_each_line(text, [&](std::size_t no, std::string_view line) {
        const auto tok = split_ws(line);
        const auto bad = [&](const std::string& why) {
            return ParseError(path + ": " + why + " at line " + std::to_string(no));
        };
        Index a = 0, b = 0;
        bool dir = false;
        if (tok.size() == 2) {
            if (!parse_index(tok[0], a) || !parse_index(tok[1], b)) throw bad("expected two vertex ids");
        } else if (tok.size() == 3 && tok[1] == ">") {
            if (!parse_index(tok[0], a) || !parse_index(tok[2], b)) throw bad("expected 'a > b'");
            dir = true;
        } else {
            throw bad("expected 'a b' or 'a > b'");
        }
        if (a == b) throw bad("self edge");
        out.max_vertex = std::max({out.max_vertex, a, b});
        if (dir) out.directed.push_back({a, b});
        else out.undirected.push_back({std::min(a, b), std::max(a, b)});
    });
    return out;
}

struct SepsetRecord {
    Index i = 0, j = 0;
    std::vector<Index> set;
};

std::vector<SepsetRecord> read_sepsets(const std::string& path) {  // io.hpp:292-314
    const std::string text = read_file(path);
    std::vector<SepsetRecord> out;
    for_each_line(text, [&](std::size_t no, std::string_view line) {
        const auto tok = split_ws(line);
        const auto bad = [&](const std::string& why) {
            return ParseError(path + ": " + why + " at line " + std::to_string(no));
        };
        if (tok.size() < 3 || tok[2] != ":") throw bad("expected 'i j : members...'");
        SepsetRecord r;
        if (!parse_index(tok[0], r.i) || !parse_index(tok[1], r.j)) throw bad("expected two vertex ids before ':'");
        if (r.i == r.j) throw bad("self pair");
        for (std::size_t t = 3; t < tok.size(); ++t) {
            Index v = 0;
            if (!parse_index(tok[t], v)) throw bad("bad set member");
            r.set.push_back(v);
        }
        out.push_back(std::move(r));
    });
    return out;
}

// ------------------------------------------------------------------ minimal JSON (report)
struct Json {  // ordered object / array / scalar, dumped like nlohmann::json::dump(2)
    enum Kind { Null, Num, Str, Obj, Arr } kind = Null;
    std::string scalar;
    std::vector<std::pair<std::string, Json>> obj;
    std::vector<Json> arr;
    static Json num(std::uint64_t v) { Json j; j.kind = Num; j.scalar = std::to_string(v); return j; }
    static Json inum(std::int64_t v) { Json j; j.kind = Num; j.scalar = std::to_string(v); return j; }
    static Json dbl(double v) {
        Json j;
        j.kind = Num;
        j.scalar = format_double(v);
        if (j.scalar.find_first_of(".eE") == std::string::npos && j.scalar.find("inf") == std::string::npos)
            j.scalar += ".0";
        return j;
    }
    static Json str(const std::string& s) { Json j; j.kind = Str; j.scalar = s; return j; }
    static Json object() { Json j; j.kind = Obj; return j; }
    static Json array() { Json j; j.kind = Arr; return j; }
    Json& set(const std::string& k, Json v) { obj.emplace_back(k, std::move(v)); return *this; }
    void dump(std::ostream& o, int ind = 0) const {
        const std::string pad(ind + 2, ' '), end(ind, ' ');
        switch (kind) {
            case Null: o << "null"; break;
            case Num: o << scalar; break;
            case Str: o << '"' << scalar << '"'; break;  // paths / enum names: no escapes needed
            case Obj:
                if (obj.empty()) { o << "{}"; break; }
                o << "{\n";
                for (std::size_t k = 0; k < obj.size(); ++k) {
                    o << pad << '"' << obj[k].first << "\": ";
                    obj[k].second.dump(o, ind + 2);
                    o << (k + 1 < obj.size() ? ",\n" : "\n");
                }
                o << end << '}';
                break;
            case Arr:
                if (arr.empty()) { o << "[]"; break; }
                o << "[\n";
                for (std::size_t k = 0; k < arr.size(); ++k) {
                    o << pad;
                    arr[k].dump(o, ind + 2);
                    o << (k + 1 < arr.size() ? ",\n" : "\n");
                }
                o << end << ']';
                break;
        }
    }
};

// ------------------------------------------------------------------ shared helpers
int default_workers() {  // pcstable_main.cpp:30-41
    if (const char* env = std::getenv("PCSTABLE_WORKERS")) {
        try {
            const int v = std::stoi(env);
            if (v >= 1) return v;
        } catch (const std::exception&) {
        }
        std::cerr << "warning: ignoring invalid PCSTABLE_WORKERS='" << env << "'\n";
    }
    const unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : static_cast<int>(hw);
}

Strategy parse_strategy(const std::string& name) {
    if (name == "serial") return Strategy::Serial;
    if (name == "edge") return Strategy::EdgeParallel;
    if (name == "set") return Strategy::SetShared;
    throw UsageError("unknown strategy '" + name + "'");
}

std::string hex_fingerprint(std::uint64_t v) {
    std::ostringstream o;
    o << std::hex << std::setw(16) << std::setfill('0') << v;
    return o.str();
}
std::int64_t to_ms(std::chrono::nanoseconds ns) {
    return std::chrono::duration_cast<std::chrono::milliseconds>(ns).count();
}

// "--flag value" options of one subcommand
struct Args {
    std::map<std::string, std::string> kv;
    std::string need(const std::string& k) const {
        auto it = kv.find(k);
        if (it == kv.end()) throw UsageError("--" + k + " is required");
        return it->second;
    }
    bool has(const std::string& k) const { return kv.count(k) > 0; }
    template <typename T>
    T num(const std::string& k, T dflt, double lo, double hi) const {
        auto it = kv.find(k);
        if (it == kv.end()) return dflt;
        double v = 0;
        if (!parse_double(it->second, v) || !(v >= lo && v <= hi))
            throw UsageError("--" + k + ": value " + it->second + " not in [" + format_double(lo) + ", " +
                             format_double(hi) + "]");
        return static_cast<T>(v);
    }
};

Args parse_args(int argc, char** argv, int first, const std::vector<std::string>& allowed) {
    Args a;
    for (int k = first; k < argc; ++k) {
        std::string t = argv[k];
        if (t.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + t + "'");
        t = t.substr(2);
        std::string v;
        const auto eq = t.find('=');
        if (eq != std::string::npos) {
            v = t.substr(eq + 1);
            t = t.substr(0, eq);
        } else {
            if (k + 1 >= argc) throw UsageError("--" + t + " needs a value");
            v = argv[++k];
        }
        if (std::find(allowed.begin(), allowed.end(), t) == allowed.end())
            throw UsageError("unknown option --" + t);
        a.kv[t] = v;
    }
    return a;
}

Data generate(Index n, double density, Index m, std::uint64_t seed, std::vector<std::pair<Index, Index>>* truth) {
    std::vector<double> w(static_cast<std::size_t>(n) * n);
    detail::check(pcs_random_dag(n, density, seed, w.data()));  // datagen.hpp:42-56
    Data d;
    d.m = m;
    d.p = n;
    d.x.resize(static_cast<std::size_t>(m) * n);
    detail::check(pcs_sample_linear_gaussian(w.data(), n, m, seed + 1, d.x.data()));  // datagen.hpp:62-82
    if (truth)
        for (Index i = 0; i < n; ++i)  // WeightedDag::edges() (datagen.hpp:26-32): ascending effect, then cause
            for (Index j = 0; j < i; ++j)
                if (w[static_cast<std::size_t>(i) * n + j] != 0.0) truth->push_back({j, i});
    return d;
}

// ------------------------------------------------------------------ subcommands
int run_gen(const Args& a) {  // pcstable_main.cpp:78-87
    const Index n = a.num<Index>("n", 0, 2, 1 << 20);
    const double dens = a.num<double>("d", 0.0, 1e-9, 1.0 - 1e-9);
    const Index m = a.num<Index>("m", 0, 4, 1 << 30);
    if (!a.has("n") || !a.has("d") || !a.has("m")) throw UsageError("--n, --d and --m are required");
    const std::uint64_t seed = a.num<std::uint64_t>("seed", 0, 0, 1.8e19);
    const std::string out = a.need("out");
    std::vector<std::pair<Index, Index>> truth;
    const Data d = generate(n, dens, m, seed, &truth);
    write_data_csv(out, d);
    std::ofstream t = open_for_write(out + ".truth");
    for (const auto& [f, to] : truth) t << f << " > " << to << '\n';
    std::cout << "wrote " << out << " (" << m << " samples x " << n << " variables) and " << out << ".truth ("
              << truth.size() << " edges)\n";
    return kExitOk;
}

Json levels_json(const std::vector<LevelStats>& levels) {
    Json arr = Json::array();
    for (const auto& l : levels)
        arr.arr.push_back(Json::object()
                              .set("level", Json::inum(l.level))
                              .set("ci_tests", Json::num(l.ci_tests))
                              .set("pseudo_inverses", Json::num(l.pseudo_inverses))
                              .set("edges_removed", Json::num(l.edges_removed))
                              .set("elapsed_ms", Json::inum(to_ms(l.elapsed))));
    return arr;
}

SkeletonConfig config_from(const Args& a, int workers) {
    SkeletonConfig cfg;
    cfg.alpha = a.num<double>("alpha", 0.05, 1e-12, 1.0 - 1e-12);
    cfg.strategy = parse_strategy(a.has("strategy") ? a.kv.at("strategy") : "serial");
    cfg.edges_per_unit = a.num<int>("beta", 2, 1, 1e9);
    cfg.workers_per_edge = a.num<int>("gamma", 32, 1, 1e9);
    cfg.unit_width = a.num<int>("theta", 64, 1, 1e9);
    cfg.set_groups = a.num<int>("delta", 2, 1, 1e9);
    cfg.worker_count = a.num<int>("workers", workers, 1, 1e9);
    if (a.has("max-level")) cfg.max_level = a.num<int>("max-level", 0, 0, 1e9);
    cfg.validate();
    return cfg;
}

int run_skeleton(const Args& a) {  // pcstable_main.cpp:114-182
    const SkeletonConfig cfg = config_from(a, default_workers());
    const std::string data_path = a.need("data"), out = a.need("out");
    const auto t0 = std::chrono::steady_clock::now();
    const Data d = read_data_csv(data_path);
    const std::uint64_t checksum = fingerprint(d);
    const CorrelationMatrix corr = stats::compute_correlation(DataMatrix(d.m, d.p, d.x));
    const SkeletonResult r = run_pc_stable(corr, d.m, cfg);
    const auto t1 = std::chrono::steady_clock::now();
    write_edge_list(out + ".edges", r.skeleton);
    write_sepsets(out + ".sepsets", r.sepsets);
    std::uint64_t tests = 0, pinvs = 0, removed = 0;
    std::chrono::nanoseconds el{0};
    for (const auto& l : r.levels) {
        tests += l.ci_tests;
        pinvs += l.pseudo_inverses;
        removed += l.edges_removed;
        el += std::chrono::duration_cast<std::chrono::nanoseconds>(l.elapsed);
    }
    Json rep = Json::object();
    rep.set("command", Json::str("skeleton"));
    rep.set("input", Json::object()
                         .set("path", Json::str(data_path))
                         .set("n", Json::inum(d.p))
                         .set("m", Json::inum(d.m))
                         .set("fingerprint", Json::str(hex_fingerprint(checksum))));
    rep.set("config", Json::object()
                          .set("alpha", Json::dbl(cfg.alpha))
                          .set("strategy", Json::str(to_string(cfg.strategy)))
                          .set("beta", Json::inum(cfg.edges_per_unit))
                          .set("gamma", Json::inum(cfg.workers_per_edge))
                          .set("theta", Json::inum(cfg.unit_width))
                          .set("delta", Json::inum(cfg.set_groups))
                          .set("workers", Json::inum(cfg.worker_count))
                          .set("max_level", cfg.max_level ? Json::inum(*cfg.max_level) : Json()));
    rep.set("levels", levels_json(r.levels));
    rep.set("totals", Json::object()
                          .set("ci_tests", Json::num(tests))
                          .set("pseudo_inverses", Json::num(pinvs))
                          .set("edges_removed", Json::num(removed))
                          .set("elapsed_ms", Json::inum(to_ms(el))));
    rep.set("result", Json::object()
                          .set("edges", Json::num(r.skeleton.edge_count()))
                          .set("levels_run", Json::num(r.levels_run()))
                          .set("stop_reason", Json::str(to_string(r.stop_reason))));
    rep.set("wall_ms", Json::inum(to_ms(t1 - t0)));
    std::ofstream ro = open_for_write(out + ".report.json");
    rep.dump(ro);
    ro << '\n';
    if (!ro) throw ParseError("failed writing: " + out + ".report.json");
    std::cout << "skeleton: " << r.skeleton.edge_count() << " edges after " << r.levels_run()
              << " levels (stop: " << to_string(r.stop_reason) << ", " << tests << " tests)\n";
    return kExitOk;
}

int run_orient(const Args& a) {  // pcstable_main.cpp:190-222
    const std::string skel_path = a.need("skeleton"), sep_path = a.need("sepsets"), out = a.need("out");
    const EdgeListData edges = read_edge_list(skel_path);
    if (!edges.directed.empty()) throw ParseError(skel_path + ": skeleton edges must be undirected");
    const std::vector<SepsetRecord> recs = read_sepsets(sep_path);
    Index n = edges.max_vertex + 1;
    for (const auto& r : recs) {
        n = std::max({n, r.i + 1, r.j + 1});
        for (Index s : r.set) n = std::max(n, s + 1);
    }
    if (n < 2) throw ParseError("orient: inputs name fewer than two vertices");
    AdjacencyMatrix skeleton(n);
    for (const auto& [x, y] : edges.undirected) skeleton.set_edge(x, y);
    SeparationSets sepsets(n);
    for (const auto& r : recs) {
        if (skeleton.at(r.i, r.j))
            throw ParseError("orient: pair (" + std::to_string(r.i) + ", " + std::to_string(r.j) +
                             ") has a separating set but is still an edge");
        for (Index s : r.set)
            if (s == r.i || s == r.j)
                throw ParseError("orient: separating set of (" + std::to_string(r.i) + ", " + std::to_string(r.j) +
                                 ") contains an endpoint");
        sepsets.store(r.i, r.j, r.set);
    }
    const MixedGraph g = orient_skeleton(skeleton, sepsets);
    write_mixed_graph(out, g);
    std::cout << "cpdag: " << g.directed.size() << " directed, " << g.undirected.size() << " undirected\n";
    return kExitOk;
}

int run_bench(const Args& a) {  // pcstable_main.cpp:235-250 + bench.hpp:59-175
    struct Case {
        Index n;
        double d;
        Index m;
    };
    std::vector<Case> cases;
    const std::string spec = a.need("spec");
    for (std::string_view triple : split(spec, ';')) {
        if (triple.empty()) continue;
        const auto parts = split(triple, ',');
        double nv = 0, dv = 0, mv = 0;
        if (parts.size() != 3 || !parse_double(parts[0], nv) || !parse_double(parts[1], dv) ||
            !parse_double(parts[2], mv))
            throw std::invalid_argument("bench spec: expected 'n,d,m[;n,d,m...]', got '" + spec + "'");
        Case c{static_cast<Index>(nv), dv, static_cast<Index>(mv)};
        if (c.n < 2 || c.m < 4 || !(c.d > 0.0 && c.d < 1.0))
            throw std::invalid_argument("bench spec: need n >= 2, m >= 4, d in (0, 1)");
        cases.push_back(c);
    }
    if (cases.empty()) throw std::invalid_argument("bench spec: no cases given");
    std::vector<Strategy> strategies;
    for (std::string_view s : split(a.has("strategies") ? a.kv.at("strategies") : "serial,edge,set", ','))
        if (!s.empty()) strategies.push_back(parse_strategy(std::string(s)));
    if (strategies.empty()) throw std::invalid_argument("run_bench: need at least one strategy");
    const int repeats = a.num<int>("repeats", 1, 1, 1e9);
    const std::uint64_t base_seed = a.num<std::uint64_t>("seed", 0, 0, 1.8e19);
    SkeletonConfig base;
    base.alpha = a.num<double>("alpha", 0.05, 1e-12, 1.0 - 1e-12);
    base.worker_count = a.num<int>("workers", default_workers(), 1, 1e9);
    if (a.has("max-level")) base.max_level = a.num<int>("max-level", 0, 0, 1e9);
    base.validate();
    const std::string out = a.need("out");
    std::ofstream o = open_for_write(out);
    o << "n,d,m,seed,strategy,workers,repeat,levels_run,stop_reason,final_edges,"
         "correlation_ms,skeleton_ms,total_ms,ci_tests,pseudo_inverses,edges_removed,"
         "level_ci_tests,level_pseudo_inverses,level_edges_removed,level_ms\n";
    std::size_t rows = 0;
    for (std::size_t ci = 0; ci < cases.size(); ++ci) {
        const Case& c = cases[ci];
        const std::uint64_t case_seed = base_seed + 7919 * ci;  // bench.hpp:94-96
        const Data d = generate(c.n, c.d, c.m, case_seed, nullptr);
        for (Strategy st : strategies) {
            SkeletonConfig cfg = base;
            cfg.strategy = st;
            for (int rep = 0; rep < repeats; ++rep) {
                const auto t0 = std::chrono::steady_clock::now();
                const CorrelationMatrix corr = stats::compute_correlation(DataMatrix(d.m, d.p, d.x));
                const auto t1 = std::chrono::steady_clock::now();
                const SkeletonResult r = run_pc_stable(corr, c.m, cfg);
                const auto t2 = std::chrono::steady_clock::now();
                std::uint64_t tests = 0, pinvs = 0, removed = 0;
                std::string lt, lp, lr, lm;
                for (std::size_t k = 0; k < r.levels.size(); ++k) {
                    const auto& l = r.levels[k];
                    tests += l.ci_tests;
                    pinvs += l.pseudo_inverses;
                    removed += l.edges_removed;
                    const char* sep = k ? ";" : "";
                    lt += sep + std::to_string(l.ci_tests);
                    lp += sep + std::to_string(l.pseudo_inverses);
                    lr += sep + std::to_string(l.edges_removed);
                    lm += sep + std::to_string(to_ms(std::chrono::duration_cast<std::chrono::nanoseconds>(l.elapsed)));
                }
                o << c.n << ',' << format_double(c.d) << ',' << c.m << ',' << case_seed << ',' << to_string(st)
                  << ',' << (st == Strategy::Serial ? 1 : cfg.worker_count) << ',' << rep << ',' << r.levels.size()
                  << ',' << to_string(r.stop_reason) << ',' << r.skeleton.edge_count() << ',' << to_ms(t1 - t0)
                  << ',' << to_ms(t2 - t1) << ',' << to_ms(t2 - t0) << ',' << tests << ',' << pinvs << ','
                  << removed << ',' << lt << ',' << lp << ',' << lr << ',' << lm << '\n';
                ++rows;
            }
        }
    }
    if (!o) throw ParseError("failed writing: " + out);
    std::cout << "bench: " << rows << " rows -> " << out << '\n';
    return kExitOk;
}

void usage() {
    std::cerr << "usage: pcstable_b200 {gen|skeleton|orient|bench} [--option value ...]\n"
                 "  gen      --n --d --m [--seed] --out\n"
                 "  skeleton --data [--alpha] [--strategy serial|edge|set] [--beta] [--gamma] [--theta] [--delta]\n"
                 "           [--workers] [--max-level] --out\n"
                 "  orient   --skeleton --sepsets --out\n"
                 "  bench    --spec n,d,m[;...] [--strategies] [--repeats] [--seed] [--alpha] [--workers]\n"
                 "           [--max-level] --out\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return kExitUsage;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "-h" || cmd == "--help") {
            usage();
            return kExitOk;
        }
        if (cmd == "gen") return run_gen(parse_args(argc, argv, 2, {"n", "d", "m", "seed", "out"}));
        if (cmd == "skeleton")
            return run_skeleton(parse_args(argc, argv, 2, {"data", "alpha", "strategy", "beta", "gamma", "theta",
                                                           "delta", "workers", "max-level", "out"}));
        if (cmd == "orient") return run_orient(parse_args(argc, argv, 2, {"skeleton", "sepsets", "out"}));
        if (cmd == "bench")
            return run_bench(parse_args(argc, argv, 2, {"spec", "strategies", "repeats", "seed", "out", "alpha",
                                                        "workers", "max-level"}));
        usage();
        return kExitUsage;
    } catch (const UsageError& e) {  // CLI11 parse errors (pcstable_main.cpp:326-331)
        std::cerr << "error: " << e.what() << '\n';
        return kExitUsage;
    } catch (const ParseError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitData;
    } catch (const ZeroVarianceError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitNumerical;
    } catch (const LevelUnreachableError& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitNumerical;
    } catch (const std::overflow_error& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitNumerical;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitData;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return kExitNumerical;
    }
}
