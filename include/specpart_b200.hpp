// specpart_b200.hpp — header-only C++ shim: the reference's public C++ API
// (include/specpart/*.hpp) on top of the B200 C-ABI (include/specpart_b200.h).
//
// A caller of the reference switches by including this header instead of
// specpart/{pipeline,graph,sparse,laplacian,eigensolver,preconditioners,
// partitioner,errors}.hpp and linking libspecpart_b200.so: the types keep the
// reference's names and the members its callers use, the free functions keep
// their signatures, and C status codes are rethrown as the reference's
// exception types (errors.hpp:10-54), so the CLI's exit-code mapping
// (tools/specpart.cpp:335-350) and its run_partition body (:63-184) compile and
// behave unchanged. Every computation runs on the device through the C-ABI;
// only file I/O (Matrix Market, partition files) and the report's JSON text are
// host code, as in the reference.
//
// RunReport::to_json() needs nlohmann/json (the reference's serializer) on the
// include path, as the reference itself does.
#pragma once

#include "specpart_b200.h"

#include <algorithm>
#include <cctype>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <istream>
#include <memory>
#include <optional>
#include <ostream>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#if __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
#define SPECPART_B200_HAS_JSON 1
#elif __has_include(<json.hpp>)
#include <json.hpp>
#define SPECPART_B200_HAS_JSON 1
#endif

namespace specpart {

// ---- errors.hpp:10-54 --------------------------------------------------------------------------
class ParseError : public std::runtime_error {
public:
    ParseError(const std::string& msg, std::size_t line)
        : std::runtime_error("line " + std::to_string(line) + ": " + msg), line_(line) {}
    std::size_t line() const noexcept { return line_; }

private:
    std::size_t line_;
};
class BreakdownError : public std::runtime_error {
public:
    BreakdownError(int iteration, bool retried)
        : std::runtime_error("eigensolver breakdown at iteration " + std::to_string(iteration) +
                             (retried ? " (after retry without search directions)" : "")),
          iteration_(iteration), retried_(retried) {}
    int iteration() const noexcept { return iteration_; }
    bool retried() const noexcept { return retried_; }

private:
    int iteration_;
    bool retried_;
};
class InfeasibleError : public std::runtime_error {
public:
    explicit InfeasibleError(const std::string& m) : std::runtime_error(m) {}
};
class DegenerateDegreeError : public std::runtime_error {
public:
    explicit DegenerateDegreeError(const std::string& m) : std::runtime_error(m) {}
};
class DimensionError : public std::logic_error {
public:
    explicit DimensionError(const std::string& m) : std::logic_error(m) {}
};

// ---- sparse.hpp:12-33, dense.hpp:10-39 ---------------------------------------------------------
struct Triplet {
    std::int32_t row;
    std::int32_t col;
    double value;
};

struct SparseMatrix {
    std::int64_t nrows = 0, ncols = 0;
    std::vector<std::int64_t> row_offsets;
    std::vector<std::int32_t> col_indices;
    std::vector<double> values;  // empty = pattern only (unit values)
    std::int64_t nnz() const { return row_offsets.empty() ? 0 : row_offsets.back(); }
    bool has_values() const { return !values.empty(); }
    double value_at(std::int64_t k) const { return has_values() ? values[k] : 1.0; }
};

struct Dense {
    std::int64_t rows = 0, cols = 0;
    std::vector<double> data;  // column-major
    Dense() = default;
    Dense(std::int64_t r, std::int64_t c) : rows(r), cols(c), data(static_cast<std::size_t>(r * c), 0.0) {}
    double& operator()(std::int64_t i, std::int64_t j) { return data[static_cast<std::size_t>(j * rows + i)]; }
    double operator()(std::int64_t i, std::int64_t j) const { return data[static_cast<std::size_t>(j * rows + i)]; }
    double* col(std::int64_t j) { return data.data() + j * rows; }
    const double* col(std::int64_t j) const { return data.data() + j * rows; }
    static Dense identity(std::int64_t n) {
        Dense I(n, n);
        for (std::int64_t i = 0; i < n; ++i) I(i, i) = 1.0;
        return I;
    }
    Dense columns(std::int64_t first, std::int64_t count) const {
        Dense out(rows, count);
        std::copy(col(first), col(first) + rows * count, out.data.begin());
        return out;
    }
};

// ---- graph.hpp:17-49 ---------------------------------------------------------------------------
struct Graph {
    SparseMatrix adjacency;
    std::vector<double> vertex_weights;
    std::int64_t n() const { return adjacency.nrows; }
    std::int64_t edge_count() const { return adjacency.nnz() / 2; }
    std::int64_t degree(std::int64_t v) const { return adjacency.row_offsets[v + 1] - adjacency.row_offsets[v]; }
};

enum class Regularity { Regular, Irregular };

struct GraphKind {
    Regularity kind = Regularity::Regular;
    std::int64_t max_degree = 0;
    double avg_degree = 0.0;
    double ratio = 0.0;
};

struct Partition {
    std::vector<std::int32_t> assignment;
    std::int32_t num_parts = 0;
    std::vector<double> part_weights;
    double cutsize = 0.0;
    double imbalance = 0.0;
};

// ---- laplacian.hpp:14-50 -----------------------------------------------------------------------
enum class ProblemKind { Combinatorial, Generalized, Normalized };

// The explicit operator, assembled on the device (bit-exact, laplacian.cpp:53-144) and
// copied back. `graph` keeps the source graph for the device-side solver entry points.
struct LinearOperator {
    SparseMatrix matrix;
    double spectral_bound = 0.0;
    bool is_diagonal = false;
    std::vector<double> diag;
    std::shared_ptr<const Graph> graph;
    int kind = SP_LAP_COMBINATORIAL;
    std::int64_t n() const { return matrix.nrows; }
};

struct EigenProblem {
    ProblemKind kind = ProblemKind::Combinatorial;
    LinearOperator A;
    std::optional<LinearOperator> B;
};

// ---- eigensolver.hpp:12-35 ---------------------------------------------------------------------
struct SolverConfig {
    int nev = 1;
    double tol = 1e-4;
    int max_iters = 1000;
    std::uint64_t seed = 0;
    bool locking = true;
    bool record_trace = false;
};

struct TraceRecord {
    int iter = 0;
    double min_residual = 0.0;
    double max_residual = 0.0;
    std::vector<double> theta;
};

struct EigenResult {
    std::vector<double> theta;
    Dense X;
    int iterations = 0;
    std::vector<double> residual_norms;
    std::vector<std::uint8_t> converged;
    int breakdown_retries = 0;
    std::vector<TraceRecord> trace;
    bool all_converged() const {
        return !converged.empty() && std::all_of(converged.begin(), converged.end(), [](std::uint8_t c) { return c != 0; });
    }
};

// ---- preconditioners.hpp:12-91 -----------------------------------------------------------------
enum class PrecondKind { Jacobi, Polynomial, Amg };
enum class PolyVariant { GmresRoots, Chebyshev };
enum class AggregationMode { Smoothed, Plain };
enum class CoarseSolverKind { Direct, Chebyshev };

struct PolyConfig {
    int degree = 25;
    std::uint64_t seed = 0;
    PolyVariant variant = PolyVariant::GmresRoots;
};

struct AmgConfig {
    AggregationMode smoothing = AggregationMode::Smoothed;
    double drop_tol = 0.0;
    int max_levels = 20;
    int cheby_degree = 3;
    int power_iters_setup = 10;
    double eig_ratio = 7.0;
    std::int64_t coarse_size_threshold = 500;
    CoarseSolverKind coarse_solver = CoarseSolverKind::Direct;
    int coarse_power_iters = 100;
    std::uint64_t seed = 0;
    static AmgConfig regular_defaults() { return AmgConfig{}; }
    static AmgConfig irregular_defaults() {
        AmgConfig c;
        c.smoothing = AggregationMode::Plain;
        c.drop_tol = 0.4;
        c.max_levels = 5;
        c.coarse_solver = CoarseSolverKind::Chebyshev;
        return c;
    }
};

// The device builds the preconditioner inside the solver call; the object records
// which one and its configuration (operators are immutable, so this is the same
// preconditioner the reference would build on the same operator).
class Preconditioner {
public:
    virtual ~Preconditioner() = default;
    virtual PrecondKind kind() const = 0;
    std::uint64_t seed = 0;
    int degree = 0;
};
class PolynomialPreconditioner : public Preconditioner {
public:
    PrecondKind kind() const override { return PrecondKind::Polynomial; }
    int requested_degree() const { return degree; }
};
class AmgPreconditioner : public Preconditioner {
public:
    PrecondKind kind() const override { return PrecondKind::Amg; }
};
namespace b200 {
class JacobiPreconditioner final : public Preconditioner {
public:
    PrecondKind kind() const override { return PrecondKind::Jacobi; }
};
} // namespace b200

// ---- partitioner.hpp:13-42 ---------------------------------------------------------------------
struct Embedding {
    Dense coords;  // n x (d-1)
    int d = 0;
};

// ---- pipeline.hpp:16-110 -----------------------------------------------------------------------
enum class ProblemChoice { Auto, Combinatorial, Generalized, Normalized };
enum class PrecondChoice { Auto, Jacobi, Polynomial, Amg, None };
enum class InitChoice { Auto, Random, PiecewiseConstant };

struct RunConfig {
    std::int64_t num_parts = 2;
    ProblemChoice problem = ProblemChoice::Auto;
    PrecondChoice precond = PrecondChoice::Auto;
    std::optional<double> tol;
    int max_iters = 1000;
    std::uint64_t seed = 42;
    double epsilon = 0.01;
    bool doubled_cut = false;
    InitChoice init = InitChoice::Auto;
    bool record_trace = false;
};

struct ResolvedConfig {
    ProblemKind problem = ProblemKind::Combinatorial;
    PrecondChoice precond = PrecondChoice::Jacobi;
    double tol = 1e-2;
    InitChoice init = InitChoice::Random;
    int eigenvectors = 0;
};

struct StageTimes {
    double laplacian_s = 0.0, eigensolve_s = 0.0, partition_s = 0.0, total_s = 0.0;
};

struct AmgLevelStats {
    std::int64_t n = 0;
    std::int64_t nnz = 0;
};

inline const char* problem_name(ProblemKind k) {
    switch (k) {
    case ProblemKind::Combinatorial: return "combinatorial";
    case ProblemKind::Generalized: return "generalized";
    case ProblemKind::Normalized: return "normalized";
    }
    return "?";
}
inline const char* problem_choice_name(ProblemChoice c) {
    switch (c) {
    case ProblemChoice::Auto: return "auto";
    case ProblemChoice::Combinatorial: return "combinatorial";
    case ProblemChoice::Generalized: return "generalized";
    case ProblemChoice::Normalized: return "normalized";
    }
    return "?";
}
inline const char* precond_choice_name(PrecondChoice c) {
    switch (c) {
    case PrecondChoice::Auto: return "auto";
    case PrecondChoice::Jacobi: return "jacobi";
    case PrecondChoice::Polynomial: return "polynomial";
    case PrecondChoice::Amg: return "amg";
    case PrecondChoice::None: return "none";
    }
    return "?";
}
inline const char* init_choice_name(InitChoice c) {
    switch (c) {
    case InitChoice::Auto: return "auto";
    case InitChoice::Random: return "random";
    case InitChoice::PiecewiseConstant: return "piecewise";
    }
    return "?";
}
inline const char* precond_name(PrecondKind k) {
    switch (k) {
    case PrecondKind::Jacobi: return "jacobi";
    case PrecondKind::Polynomial: return "polynomial";
    case PrecondKind::Amg: return "amg";
    }
    return "?";
}

struct RunReport {
    std::int64_t n = 0, edges = 0;
    GraphKind graph_kind;
    std::int64_t dropped_vertices = 0;
    std::int64_t num_parts = 0;
    ResolvedConfig resolved;
    std::uint64_t seed = 0;
    int max_iters = 0;
    double epsilon = 0.0;
    bool doubled_cut = false;
    int iterations = 0;
    std::vector<double> theta, residual_norms;
    std::vector<std::uint8_t> converged;
    std::vector<TraceRecord> trace;
    std::vector<AmgLevelStats> amg_levels;
    StageTimes times;
    double cutsize = 0.0, imbalance = 0.0;
    std::vector<double> part_weights;
    std::vector<std::string> warnings;
    sp_report raw{};  // the C report (device-side accounting included)

#ifdef SPECPART_B200_HAS_JSON
    // pipeline.cpp:169-215 (docs/report_schema.md), same library, so same text
    std::string to_json() const {
        nlohmann::json j;
        j["graph"] = {{"n", n},
                      {"edges", edges},
                      {"max_degree", graph_kind.max_degree},
                      {"avg_degree", graph_kind.avg_degree},
                      {"degree_ratio", graph_kind.ratio},
                      {"kind", graph_kind.kind == Regularity::Regular ? "regular" : "irregular"},
                      {"dropped_vertices", dropped_vertices}};
        j["config"] = {{"parts", num_parts},
                       {"problem", problem_name(resolved.problem)},
                       {"preconditioner", precond_choice_name(resolved.precond)},
                       {"tolerance", resolved.tol},
                       {"initial_vectors", init_choice_name(resolved.init)},
                       {"eigenvectors", resolved.eigenvectors},
                       {"seed", seed},
                       {"max_iters", max_iters},
                       {"epsilon", epsilon},
                       {"doubled_cut", doubled_cut}};
        j["solver"] = {{"iterations", iterations},
                       {"theta", theta},
                       {"residual_norms", residual_norms},
                       {"converged", std::vector<bool>(converged.begin(), converged.end())}};
        if (!amg_levels.empty()) {
            nlohmann::json lv = nlohmann::json::array();
            for (const AmgLevelStats& l : amg_levels) lv.push_back({{"n", l.n}, {"nnz", l.nnz}});
            j["solver"]["amg_levels"] = lv;
        }
        if (!trace.empty()) {
            nlohmann::json tr = nlohmann::json::array();
            for (const TraceRecord& t : trace)
                tr.push_back({{"iter", t.iter},
                              {"min_residual", t.min_residual},
                              {"max_residual", t.max_residual},
                              {"theta", t.theta}});
            j["solver"]["trace"] = tr;
        }
        j["times"] = {{"laplacian_s", times.laplacian_s},
                      {"eigensolve_s", times.eigensolve_s},
                      {"partition_s", times.partition_s},
                      {"total_s", times.total_s}};
        j["partition"] = {{"cutsize", cutsize}, {"imbalance", imbalance}, {"part_weights", part_weights}};
        j["warnings"] = warnings;
        return j.dump(2);
    }
#endif
};

struct RunResult {
    Partition partition;
    RunReport report;
};

// ---- the device context and status mapping -------------------------------------------------------
namespace b200 {

// One context per thread/GPU, created lazily on device `SPECPART_B200_DEVICE` (default 0).
inline sp_context* context() {
    thread_local struct Holder {
        sp_context* c = nullptr;
        ~Holder() { sp_context_destroy(c); }
    } h;
    if (!h.c) {
        int dev = 0;
        if (const char* e = std::getenv("SPECPART_B200_DEVICE")) dev = std::atoi(e);
        if (sp_context_create(dev, &h.c) != SP_OK) throw std::runtime_error("specpart_b200: no CUDA device");
    }
    return h.c;
}

inline void rethrow(sp_status st, sp_context* c) {
    if (st == SP_OK) return;
    const std::string msg = sp_last_error(c) ? sp_last_error(c) : "";
    switch (st) {
    case SP_PARSE: throw ParseError(msg, 0);
    case SP_BREAKDOWN: {
        // "eigensolver breakdown at iteration N[ (after retry ...)]"
        const std::size_t p = msg.find("iteration ");
        const int it = p == std::string::npos ? 0 : std::atoi(msg.c_str() + p + 10);
        throw BreakdownError(it, msg.find("after retry") != std::string::npos);
    }
    case SP_INFEASIBLE: throw InfeasibleError(msg);
    case SP_DEGENERATE: throw DegenerateDegreeError(msg);
    case SP_DIMENSION: throw DimensionError(msg);
    case SP_INVALID: throw std::invalid_argument(msg);
    default: throw std::runtime_error(msg);
    }
}

inline sp_graph c_graph(const Graph& g) {
    return sp_graph{g.n(), g.adjacency.row_offsets.data(), g.adjacency.col_indices.data(),
                    g.adjacency.values.empty() ? nullptr : g.adjacency.values.data(),
                    g.vertex_weights.empty() ? nullptr : g.vertex_weights.data()};
}

inline std::string lower(std::string s) {
    for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    return s;
}
inline bool blank_or_comment(const std::string& line) {
    for (char ch : line) {
        if (ch == '%') return true;
        if (!std::isspace(static_cast<unsigned char>(ch))) return false;
    }
    return true;
}

inline GraphKind kind_of(const sp_graph_info& info) {
    GraphKind k;
    k.kind = info.regular ? Regularity::Regular : Regularity::Irregular;
    k.max_degree = info.max_degree;
    k.avg_degree = info.avg_degree;
    k.ratio = info.degree_ratio;
    return k;
}

inline Graph download(sp_context* c, sp_device_graph* dg, std::vector<std::int64_t>* old_ids) {
    sp_graph_info info{};
    rethrow(sp_device_graph_info(c, dg, &info), c);
    Graph g;
    g.adjacency.nrows = g.adjacency.ncols = info.n;
    g.adjacency.row_offsets.resize(static_cast<std::size_t>(info.n + 1));
    g.adjacency.col_indices.resize(static_cast<std::size_t>(info.nnz));
    if (old_ids) old_ids->resize(static_cast<std::size_t>(info.n));
    rethrow(sp_device_graph_download(c, dg, g.adjacency.row_offsets.data(), g.adjacency.col_indices.data(),
                                     old_ids ? old_ids->data() : nullptr), c);
    g.adjacency.values.assign(static_cast<std::size_t>(info.nnz), 1.0);  // unit edge costs, as graph.cpp:61
    g.vertex_weights.assign(static_cast<std::size_t>(info.n), 1.0);
    return g;
}

struct DeviceGraphHolder {
    sp_device_graph* p = nullptr;
    ~DeviceGraphHolder() { sp_graph_free(p); }
};

inline int32_t precond_code(const Preconditioner* M) {
    if (!M) return SP_PRECOND_NONE;
    switch (M->kind()) {
    case PrecondKind::Jacobi: return SP_PRECOND_JACOBI;
    case PrecondKind::Polynomial: return SP_PRECOND_POLYNOMIAL;
    case PrecondKind::Amg: return SP_PRECOND_AMG;
    }
    return SP_PRECOND_NONE;
}

} // namespace b200

// ---- sparse.cpp:106-176: Matrix Market (host file I/O) ----------------------------------------
inline SparseMatrix parse_matrix_market(std::istream& in) {
    using b200::lower;
    std::string line;
    std::size_t lineno = 0;
    if (!std::getline(in, line)) throw ParseError("empty input", 1);
    ++lineno;
    std::istringstream banner(line);
    std::string tag, object, format, field, symmetry;
    banner >> tag >> object >> format >> field >> symmetry;
    if (lower(tag) != "%%matrixmarket" || lower(object) != "matrix")
        throw ParseError("malformed MatrixMarket banner", lineno);
    format = lower(format);
    field = lower(field);
    symmetry = lower(symmetry);
    if (format != "coordinate") throw ParseError("unsupported format '" + format + "' (coordinate only)", lineno);
    const bool pattern = field == "pattern";
    if (!pattern && field != "real" && field != "integer") throw ParseError("unsupported field '" + field + "'", lineno);
    const bool symmetric = symmetry == "symmetric";
    if (!symmetric && symmetry != "general") throw ParseError("unsupported symmetry '" + symmetry + "'", lineno);
    std::int64_t nrows = 0, ncols = 0, declared = 0;
    for (;;) {
        if (!std::getline(in, line)) throw ParseError("missing size line", lineno + 1);
        ++lineno;
        if (b200::blank_or_comment(line)) continue;
        std::istringstream sz(line);
        if (!(sz >> nrows >> ncols >> declared) || nrows < 0 || ncols < 0 || declared < 0)
            throw ParseError("malformed size line", lineno);
        std::string extra;
        if (sz >> extra) throw ParseError("trailing tokens on size line", lineno);
        break;
    }
    std::vector<Triplet> ent;
    ent.reserve(static_cast<std::size_t>(symmetric ? 2 * declared : declared));
    std::int64_t seen = 0;
    while (seen < declared) {
        if (!std::getline(in, line))
            throw ParseError("entry list truncated: expected " + std::to_string(declared) + " entries, got " +
                                 std::to_string(seen),
                             lineno + 1);
        ++lineno;
        if (b200::blank_or_comment(line)) continue;
        std::istringstream es(line);
        std::int64_t r = 0, c = 0;
        double v = 1.0;
        if (!(es >> r >> c)) throw ParseError("malformed entry", lineno);
        if (!pattern && !(es >> v)) throw ParseError("missing value", lineno);
        std::string extra;
        if (es >> extra) throw ParseError("trailing tokens on entry", lineno);
        if (r < 1 || r > nrows || c < 1 || c > ncols)
            throw ParseError("index out of range: (" + std::to_string(r) + ", " + std::to_string(c) + ")", lineno);
        ent.push_back({static_cast<std::int32_t>(r - 1), static_cast<std::int32_t>(c - 1), v});
        if (symmetric && r != c) ent.push_back({static_cast<std::int32_t>(c - 1), static_cast<std::int32_t>(r - 1), v});
        ++seen;
    }
    // canonical CSR (from_triplets, sparse.cpp:36-65): rows sorted, duplicates summed
    std::stable_sort(ent.begin(), ent.end(),
                     [](const Triplet& a, const Triplet& b) { return a.row != b.row ? a.row < b.row : a.col < b.col; });
    SparseMatrix m;
    m.nrows = nrows;
    m.ncols = ncols;
    m.row_offsets.assign(static_cast<std::size_t>(nrows + 1), 0);
    for (std::size_t k = 0; k < ent.size();) {
        std::size_t k2 = k + 1;
        double v = ent[k].value;
        while (k2 < ent.size() && ent[k2].row == ent[k].row && ent[k2].col == ent[k].col) v += ent[k2++].value;
        m.col_indices.push_back(ent[k].col);
        if (!pattern) m.values.push_back(v);
        ++m.row_offsets[static_cast<std::size_t>(ent[k].row) + 1];
        k = k2;
    }
    for (std::int64_t i = 0; i < nrows; ++i) m.row_offsets[i + 1] += m.row_offsets[i];
    return m;
}

inline SparseMatrix parse_matrix_market_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw ParseError("cannot open '" + path + "'", 0);
    return parse_matrix_market(in);
}

// ---- graph.hpp:53-83 ---------------------------------------------------------------------------
// symmetrize (graph.cpp:44-64), on the device
inline Graph symmetrize(const SparseMatrix& A) {
    if (A.nrows != A.ncols) throw std::invalid_argument("symmetrize: matrix not square");
    sp_context* c = b200::context();
    b200::DeviceGraphHolder h;
    b200::rethrow(sp_ingest(c, A.nrows, A.row_offsets.data(), A.col_indices.data(), 0, &h.p), c);
    return b200::download(c, h.p, nullptr);
}

// largest_connected_component (graph.cpp:118-171), on the device
inline std::pair<Graph, std::vector<std::int64_t>> largest_connected_component(const Graph& g) {
    sp_context* c = b200::context();
    b200::DeviceGraphHolder h;
    b200::rethrow(sp_ingest(c, g.n(), g.adjacency.row_offsets.data(), g.adjacency.col_indices.data(), 1, &h.p), c);
    std::vector<std::int64_t> old;
    Graph sub = b200::download(c, h.p, &old);
    return {std::move(sub), std::move(old)};
}

// classify (graph.cpp:173-182)
inline GraphKind classify(const Graph& g) {
    sp_context* c = b200::context();
    sp_graph cg{g.n(), g.adjacency.row_offsets.data(), g.adjacency.col_indices.data(), nullptr, nullptr};
    sp_graph_info info{};
    b200::rethrow(sp_classify(c, &cg, &info), c);
    return b200::kind_of(info);
}

// cutsize (graph.cpp:184-196)
inline double cutsize(const Graph& g, std::span<const std::int32_t> assignment, bool doubled = false) {
    if (static_cast<std::int64_t>(assignment.size()) != g.n())
        throw std::invalid_argument("cutsize: assignment length mismatch");
    sp_context* c = b200::context();
    const sp_graph cg = b200::c_graph(g);
    double cut = 0.0;
    b200::rethrow(sp_cutsize(c, &cg, assignment.data(), doubled ? 1 : 0, &cut), c);
    return cut;
}

// imbalance (graph.cpp:198-207): a K-element reduction on the host
inline double imbalance(std::span<const double> part_weights) {
    if (part_weights.empty()) throw std::invalid_argument("imbalance: no parts");
    double total = 0.0, maxw = 0.0;
    for (double w : part_weights) {
        total += w;
        maxw = std::max(maxw, w);
    }
    if (total <= 0.0) throw std::invalid_argument("imbalance: total weight not positive");
    return maxw / (total / static_cast<double>(part_weights.size()));
}

// make_partition (graph.cpp:209-230)
inline Partition make_partition(const Graph& g, std::vector<std::int32_t> assignment, std::int32_t num_parts,
                                bool doubled_cut = false) {
    if (static_cast<std::int64_t>(assignment.size()) != g.n())
        throw std::invalid_argument("make_partition: assignment length mismatch");
    sp_context* c = b200::context();
    const sp_graph cg = b200::c_graph(g);
    Partition p;
    p.num_parts = num_parts;
    p.part_weights.resize(static_cast<std::size_t>(num_parts > 0 ? num_parts : 1));
    b200::rethrow(sp_cut_imbalance(c, &cg, assignment.data(), num_parts, doubled_cut ? 1 : 0, &p.cutsize,
                                   &p.imbalance, p.part_weights.data()),
                  c);
    p.assignment = std::move(assignment);
    return p;
}

// write_partition / read_partition (graph.cpp:232-254): file formats, host
inline void write_partition(std::ostream& out, std::span<const std::int32_t> assignment,
                            std::span<const std::int64_t> original_ids) {
    for (std::size_t v = 0; v < assignment.size(); ++v)
        out << (original_ids.empty() ? static_cast<std::int64_t>(v) : original_ids[v]) << ' ' << assignment[v] << '\n';
}

inline std::vector<std::pair<std::int64_t, std::int32_t>> read_partition(std::istream& in) {
    std::vector<std::pair<std::int64_t, std::int32_t>> rows;
    std::string line;
    std::size_t lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (line.empty()) continue;
        std::istringstream ls(line);
        std::int64_t id;
        std::int32_t part;
        if (!(ls >> id >> part)) throw ParseError("malformed partition line", lineno);
        rows.emplace_back(id, part);
    }
    return rows;
}

// ---- laplacian.hpp:24-50: operators assembled on the device ----------------------------------------
namespace b200 {
inline LinearOperator build_kind(const Graph& g, int kind) {
    sp_context* c = context();
    const sp_graph cg = c_graph(g);
    LinearOperator op;
    const std::int64_t n = g.n();
    const std::int64_t nnz = kind == SP_LAP_DEGREE ? n : g.adjacency.nnz() + n;
    op.matrix.nrows = op.matrix.ncols = n;
    op.matrix.row_offsets.resize(static_cast<std::size_t>(n + 1));
    op.matrix.col_indices.resize(static_cast<std::size_t>(std::max<std::int64_t>(nnz, 1)));
    op.matrix.values.resize(static_cast<std::size_t>(std::max<std::int64_t>(nnz, 1)));
    op.diag.resize(static_cast<std::size_t>(n));
    std::int32_t isdiag = 0;
    rethrow(sp_build_laplacian(c, kind, &cg, op.matrix.row_offsets.data(), op.matrix.col_indices.data(),
                               op.matrix.values.data(), op.diag.data(), &op.spectral_bound, &isdiag),
            c);
    op.matrix.col_indices.resize(static_cast<std::size_t>(nnz));
    op.matrix.values.resize(static_cast<std::size_t>(nnz));
    op.is_diagonal = isdiag != 0;
    op.graph = std::make_shared<const Graph>(g);
    op.kind = kind;
    return op;
}
} // namespace b200

inline LinearOperator build_combinatorial(const Graph& g) { return b200::build_kind(g, SP_LAP_COMBINATORIAL); }
inline LinearOperator build_normalized(const Graph& g) { return b200::build_kind(g, SP_LAP_NORMALIZED); }
inline LinearOperator build_degree(const Graph& g) { return b200::build_kind(g, SP_LAP_DEGREE); }

// build_problem (laplacian.cpp:161-180)
inline EigenProblem build_problem(const Graph& g, ProblemKind kind) {
    EigenProblem p;
    p.kind = kind;
    p.A = kind == ProblemKind::Normalized ? build_normalized(g) : build_combinatorial(g);
    if (kind == ProblemKind::Generalized) p.B = build_degree(g);
    return p;
}

// apply_block (laplacian.cpp:146-159): Y = op V on the device (spmv_block order, bit-exact)
inline void apply_block(const LinearOperator& op, const Dense& V, Dense& Y) {
    if (V.rows != op.n()) throw DimensionError("apply_block: shape mismatch");
    sp_context* c = b200::context();
    Y = Dense(V.rows, V.cols);
    if (V.cols == 0) return;
    b200::rethrow(sp_spmm_csr(c, op.n(), op.n(), op.matrix.row_offsets.data(), op.matrix.col_indices.data(),
                              op.matrix.values.data(), V.data.data(), static_cast<std::int32_t>(V.cols), Y.data.data()),
                  c);
}
inline Dense apply_block(const LinearOperator& op, const Dense& V) {
    Dense Y;
    apply_block(op, V, Y);
    return Y;
}

// ---- kernels.hpp:20-28: the block products LOBPCG is built from, on the device -------------------
namespace kernels {
inline Dense gram(const Dense& U, const Dense& V) {  // U^T V
    if (U.rows != V.rows) throw DimensionError("gram: row mismatch");
    sp_context* c = b200::context();
    Dense G(U.cols, V.cols);
    if (U.cols == 0 || V.cols == 0) return G;
    b200::rethrow(sp_gram(c, U.rows, U.data.data(), static_cast<std::int32_t>(U.cols), V.data.data(),
                          static_cast<std::int32_t>(V.cols), nullptr, G.data.data()),
                  c);
    return G;
}
inline void mult(const Dense& X, const Dense& C, Dense& Y) {  // Y = X C
    if (X.cols != C.rows) throw DimensionError("mult: inner dimension mismatch");
    sp_context* c = b200::context();
    Y = Dense(X.rows, C.cols);
    if (X.rows == 0 || C.cols == 0) return;
    b200::rethrow(sp_block_combine(c, X.rows, X.data.data(), static_cast<std::int32_t>(X.cols), C.data.data(),
                                   static_cast<std::int32_t>(C.cols), 0, Y.data.data()),
                  c);
}
inline void mult_sub(Dense& Y, const Dense& X, const Dense& C) {  // Y -= X C
    if (X.cols != C.rows || Y.rows != X.rows || Y.cols != C.cols) throw DimensionError("mult_sub: shape mismatch");
    sp_context* c = b200::context();
    if (X.rows == 0 || C.cols == 0) return;
    b200::rethrow(sp_block_combine(c, X.rows, X.data.data(), static_cast<std::int32_t>(X.cols), C.data.data(),
                                   static_cast<std::int32_t>(C.cols), 1, Y.data.data()),
                  c);
}
} // namespace kernels

// ---- preconditioner builders (preconditioners.hpp:30-91) -----------------------------------------
inline std::unique_ptr<Preconditioner> jacobi_build(const LinearOperator&) {
    return std::make_unique<b200::JacobiPreconditioner>();
}
inline std::unique_ptr<PolynomialPreconditioner> polynomial_build(const LinearOperator&, const PolyConfig& cfg) {
    if (cfg.degree < 1) throw InfeasibleError("polynomial_build: degree < 1");
    if (cfg.variant != PolyVariant::GmresRoots)
        throw std::invalid_argument("polynomial_build: only the GMRES-roots variant runs on the device");
    auto p = std::make_unique<PolynomialPreconditioner>();
    p->seed = cfg.seed;
    p->degree = cfg.degree;
    return p;
}
inline std::unique_ptr<AmgPreconditioner> amg_build(const LinearOperator& A, const AmgConfig& cfg) {
    if (cfg.max_levels < 1) throw InfeasibleError("amg_build: max_levels < 1");
    if (cfg.drop_tol < 0.0 || cfg.drop_tol >= 1.0) throw InfeasibleError("amg_build: drop_tol outside [0,1)");
    if (cfg.cheby_degree < 1) throw InfeasibleError("amg_build: cheby_degree < 1");
    // the device builds the preset of A's graph kind (pipeline.cpp:107-112)
    if (A.graph) {
        const bool regular = classify(*A.graph).kind == Regularity::Regular;
        const AmgConfig want = regular ? AmgConfig::regular_defaults() : AmgConfig::irregular_defaults();
        if (cfg.smoothing != want.smoothing || cfg.drop_tol != want.drop_tol || cfg.max_levels != want.max_levels ||
            cfg.coarse_solver != want.coarse_solver)
            throw std::invalid_argument("amg_build: the device runs the regular/irregular presets of AmgConfig");
    }
    auto p = std::make_unique<AmgPreconditioner>();
    p->seed = cfg.seed;
    return p;
}

// ---- eigensolver.hpp:37-65 ---------------------------------------------------------------------
inline Dense initial_guess_random(std::int64_t n, int d, std::uint64_t seed) {
    Dense X(n, d);
    b200::rethrow(sp_initial_guess(b200::context(), SP_INIT_RANDOM, n, d, seed, X.data.data()), b200::context());
    return X;
}
inline Dense initial_guess_piecewise(std::int64_t n, int d) {
    Dense X(n, d);
    b200::rethrow(sp_initial_guess(b200::context(), SP_INIT_PIECEWISE, n, d, 0, X.data.data()), b200::context());
    return X;
}

// lobpcg (eigensolver.cpp:177-337) on the problem's graph, preconditioner built on problem.A
inline EigenResult lobpcg(const EigenProblem& problem, const Preconditioner* M, const Dense& X0,
                          const SolverConfig& cfg) {
    if (!problem.A.graph) throw std::invalid_argument("lobpcg: problem was not built by build_problem");
    if (X0.cols != cfg.nev) throw DimensionError("lobpcg: X0 must have nev columns");
    if (X0.rows != problem.A.n()) throw DimensionError("lobpcg: X0 rows != n");
    sp_context* c = b200::context();
    const sp_graph cg = b200::c_graph(*problem.A.graph);
    const std::int32_t prob = problem.kind == ProblemKind::Combinatorial ? SP_PROBLEM_COMBINATORIAL
                              : problem.kind == ProblemKind::Generalized ? SP_PROBLEM_GENERALIZED
                                                                         : SP_PROBLEM_NORMALIZED;
    EigenResult r;
    r.theta.resize(static_cast<std::size_t>(cfg.nev));
    r.residual_norms.resize(static_cast<std::size_t>(cfg.nev));
    r.converged.resize(static_cast<std::size_t>(cfg.nev));
    r.X = Dense(X0.rows, cfg.nev);
    std::int32_t it = 0, rt = 0;
    b200::rethrow(sp_lobpcg(c, &cg, prob, b200::precond_code(M), M ? M->seed : 0, M ? M->degree : 0, X0.data.data(),
                            cfg.nev, cfg.tol, cfg.max_iters, cfg.locking ? 1 : 0, r.theta.data(), r.X.data.data(),
                            r.residual_norms.data(), r.converged.data(), &it, &rt),
                  c);
    r.iterations = it;
    r.breakdown_retries = rt;
    return r;
}

// ---- partitioner.hpp:13-42 ---------------------------------------------------------------------
inline int eigenvector_count(std::int64_t num_parts) {
    if (num_parts < 2) throw InfeasibleError("eigenvector_count: K must be >= 2");
    int d = 0;
    for (std::uint64_t k = static_cast<std::uint64_t>(num_parts); k; k >>= 1) ++d;  // bit_width
    return d;
}

inline Embedding embed(const Dense& eigenvectors) {
    if (eigenvectors.cols < 2) throw DimensionError("embed: need at least two eigenvectors");
    Embedding e;
    e.d = static_cast<int>(eigenvectors.cols);
    e.coords = eigenvectors.columns(1, eigenvectors.cols - 1);
    return e;
}

inline Partition mj_partition(const Embedding& emb, std::span<const double> weights, std::int64_t num_parts) {
    sp_context* c = b200::context();
    const std::int64_t n = emb.coords.rows;
    Partition p;
    p.num_parts = static_cast<std::int32_t>(num_parts);
    p.assignment.resize(static_cast<std::size_t>(n));
    p.part_weights.resize(static_cast<std::size_t>(num_parts > 0 ? num_parts : 1));
    b200::rethrow(sp_mj_partition(c, n, static_cast<std::int32_t>(emb.coords.cols), emb.coords.data.data(),
                                  weights.empty() ? nullptr : weights.data(), num_parts, p.assignment.data(),
                                  p.part_weights.data(), &p.imbalance),
                  c);
    return p;
}

// ---- pipeline.cpp:20-45: the Auto decision table (host logic) -----------------------------------
inline std::pair<ProblemKind, double> select_defaults(const GraphKind& kind, PrecondChoice precond) {
    const bool regular = kind.kind == Regularity::Regular;
    switch (precond) {
    case PrecondChoice::Jacobi:
    case PrecondChoice::None:
        return regular ? std::pair{ProblemKind::Combinatorial, 1e-3} : std::pair{ProblemKind::Generalized, 1e-2};
    case PrecondChoice::Polynomial:
        return regular ? std::pair{ProblemKind::Combinatorial, 1e-3} : std::pair{ProblemKind::Normalized, 1e-2};
    case PrecondChoice::Amg:
        return regular ? std::pair{ProblemKind::Combinatorial, 1e-2} : std::pair{ProblemKind::Generalized, 1e-2};
    case PrecondChoice::Auto: break;
    }
    throw std::invalid_argument("select_defaults: preconditioner must be resolved");
}
inline PrecondChoice select_precond_auto(const GraphKind& kind) {
    return kind.kind == Regularity::Regular ? PrecondChoice::Amg : PrecondChoice::Polynomial;
}
inline InitChoice select_initial_vectors(const GraphKind& kind) {
    return kind.kind == Regularity::Regular ? InitChoice::Random : InitChoice::PiecewiseConstant;
}

// ---- pipeline.hpp:106: partition_graph on the device ------------------------------------------------
inline RunResult partition_graph(const Graph& g, const RunConfig& cfg) {
    sp_context* c = b200::context();
    const sp_graph cg = b200::c_graph(g);
    sp_config cc{};
    cc.num_parts = cfg.num_parts;
    cc.problem = static_cast<int32_t>(cfg.problem);
    cc.precond = static_cast<int32_t>(cfg.precond);
    cc.tol = cfg.tol ? *cfg.tol : -1.0;
    cc.max_iters = cfg.max_iters;
    cc.init = static_cast<int32_t>(cfg.init);
    cc.seed = cfg.seed;
    cc.epsilon = cfg.epsilon;
    cc.doubled_cut = cfg.doubled_cut;
    cc.record_trace = cfg.record_trace;
    RunResult out;
    out.partition.assignment.resize(static_cast<std::size_t>(g.n()));
    out.partition.part_weights.resize(static_cast<std::size_t>(cfg.num_parts > 0 ? cfg.num_parts : 1));
    sp_report& r = out.report.raw;
    r.part_weights = out.partition.part_weights.data();
    std::vector<sp_trace_record> tr;
    if (cfg.record_trace) {
        tr.resize(static_cast<std::size_t>(cfg.max_iters > 0 ? cfg.max_iters : 0) + 1);
        r.trace = tr.data();
        r.trace_capacity = static_cast<int32_t>(tr.size());
    }
    b200::rethrow(sp_partition(c, &cg, &cc, out.partition.assignment.data(), &r, nullptr), c);
    out.partition.num_parts = static_cast<std::int32_t>(cfg.num_parts);
    out.partition.cutsize = r.cutsize;
    out.partition.imbalance = r.imbalance;
    RunReport& R = out.report;
    R.n = r.n;
    R.edges = r.edges;
    R.graph_kind.kind = r.graph_regular ? Regularity::Regular : Regularity::Irregular;
    R.graph_kind.max_degree = r.max_degree;
    R.graph_kind.avg_degree = r.avg_degree;
    R.graph_kind.ratio = r.degree_ratio;
    R.num_parts = r.num_parts;
    R.resolved.problem = r.problem == SP_PROBLEM_GENERALIZED  ? ProblemKind::Generalized
                         : r.problem == SP_PROBLEM_NORMALIZED ? ProblemKind::Normalized
                                                              : ProblemKind::Combinatorial;
    R.resolved.precond = static_cast<PrecondChoice>(r.precond);
    R.resolved.tol = r.tol;
    R.resolved.init = static_cast<InitChoice>(r.init);
    R.resolved.eigenvectors = r.eigenvectors;
    R.seed = r.seed;
    R.max_iters = r.max_iters;
    R.epsilon = r.epsilon;
    R.doubled_cut = r.doubled_cut != 0;
    R.iterations = r.iterations;
    R.theta.assign(r.theta, r.theta + r.eigenvectors);
    R.residual_norms.assign(r.residual_norms, r.residual_norms + r.eigenvectors);
    R.converged.assign(r.converged, r.converged + r.eigenvectors);
    for (int32_t k = 0; k < r.trace_len; ++k)
        R.trace.push_back({tr[k].iter, tr[k].min_residual, tr[k].max_residual,
                           std::vector<double>(tr[k].theta, tr[k].theta + tr[k].ntheta)});
    for (int32_t l = 0; l < r.amg_levels; ++l) R.amg_levels.push_back({r.amg_n[l], r.amg_nnz[l]});
    R.times = {r.laplacian_s, r.eigensolve_s, r.partition_s, r.total_s};
    R.cutsize = r.cutsize;
    R.imbalance = r.imbalance;
    R.part_weights = out.partition.part_weights;
    // warnings in the reference's order (pipeline.cpp:116-117, 140-148, 161-163)
    if (r.warnings & SP_WARN_AMG_STAGNATED) R.warnings.emplace_back("amg coarsening stagnated; hierarchy stopped early");
    if (r.warnings & SP_WARN_BREAKDOWN_RECOVERED)
        R.warnings.emplace_back("eigensolver recovered from a basis breakdown by clearing the search directions");
    if (r.warnings & SP_WARN_UNCONVERGED)
        R.warnings.emplace_back("eigensolver reached max_iters with unconverged columns; "
                                "partitioning on partially converged eigenvectors");
    if (r.warnings & SP_WARN_IMBALANCE)
        R.warnings.emplace_back("imbalance " + std::to_string(r.imbalance) + " exceeds 1+epsilon = " +
                                std::to_string(1.0 + cfg.epsilon));
    r.part_weights = nullptr;
    r.trace = nullptr;
    return out;
}

} // namespace specpart
