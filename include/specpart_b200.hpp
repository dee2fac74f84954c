// specpart_b200.hpp — header-only C++ shim: `specpart::partition_graph` on top of
// the B200 C-ABI (include/specpart_b200.h).
//
// A caller of the reference (`#include "specpart/pipeline.hpp"`) switches by
// including this header instead and linking libspecpart_b200.so. The types keep
// the reference's names and members used by its callers (graph.hpp:17-49,
// sparse.hpp:18-33, pipeline.hpp:16-110) and the C status codes are rethrown as
// the reference's exception types (errors.hpp:10-54), so the CLI's exit-code
// mapping (tools/specpart.cpp:335-350) keeps working unchanged.
#pragma once

#include "specpart_b200.h"

#include <cstdint>
#include <cstdlib>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace specpart {

class ParseError : public std::runtime_error {
public:
    explicit ParseError(const std::string& m) : std::runtime_error(m) {}
};
class BreakdownError : public std::runtime_error {
public:
    explicit BreakdownError(const std::string& m)
        : std::runtime_error(m), retried_(m.find("after retry") != std::string::npos) {}
    bool retried() const noexcept { return retried_; }

private:
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

struct SparseMatrix {
    std::int64_t nrows = 0, ncols = 0;
    std::vector<std::int64_t> row_offsets;
    std::vector<std::int32_t> col_indices;
    std::vector<double> values;  // empty = unit
    std::int64_t nnz() const { return row_offsets.empty() ? 0 : row_offsets.back(); }
};

struct Graph {
    SparseMatrix adjacency;
    std::vector<double> vertex_weights;
    std::int64_t n() const { return adjacency.nrows; }
    std::int64_t edge_count() const { return adjacency.nnz() / 2; }
};

enum class Regularity { Regular, Irregular };

// graph.hpp:35-41
struct GraphKind {
    Regularity kind = Regularity::Regular;
    std::int64_t max_degree = 0;
    double avg_degree = 0.0;
    double ratio = 0.0;
};

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

struct Partition {
    std::vector<std::int32_t> assignment;
    std::int32_t num_parts = 0;
    std::vector<double> part_weights;
    double cutsize = 0.0;
    double imbalance = 0.0;
};

struct StageTimes {
    double laplacian_s = 0.0, eigensolve_s = 0.0, partition_s = 0.0, total_s = 0.0;
};

struct RunReport {
    std::int64_t n = 0, edges = 0, num_parts = 0;
    int iterations = 0;
    std::vector<double> theta, residual_norms;
    std::vector<std::uint8_t> converged;
    StageTimes times;
    double cutsize = 0.0, imbalance = 0.0;
    std::vector<double> part_weights;
    std::vector<std::string> warnings;
    sp_report raw{};  // every resolved field of the C report
};

struct RunResult {
    Partition partition;
    RunReport report;
};

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
    const std::string msg = sp_last_error(c);
    switch (st) {
    case SP_OK: return;
    case SP_PARSE: throw ParseError(msg);
    case SP_BREAKDOWN: throw BreakdownError(msg);
    case SP_INFEASIBLE: throw InfeasibleError(msg);
    case SP_DEGENERATE: throw DegenerateDegreeError(msg);
    case SP_DIMENSION: throw DimensionError(msg);
    case SP_INVALID: throw std::invalid_argument(msg);
    default: throw std::runtime_error(msg);
    }
}

} // namespace b200

// pipeline.hpp:106
inline RunResult partition_graph(const Graph& g, const RunConfig& cfg) {
    sp_context* c = b200::context();
    sp_graph cg{g.n(), g.adjacency.row_offsets.data(), g.adjacency.col_indices.data(),
                g.adjacency.values.empty() ? nullptr : g.adjacency.values.data(),
                g.vertex_weights.empty() ? nullptr : g.vertex_weights.data()};
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
    out.partition.assignment.resize(static_cast<size_t>(g.n()));
    out.partition.part_weights.resize(static_cast<size_t>(cfg.num_parts > 0 ? cfg.num_parts : 1));
    sp_report& r = out.report.raw;
    r.part_weights = out.partition.part_weights.data();
    b200::rethrow(sp_partition(c, &cg, &cc, out.partition.assignment.data(), &r, nullptr), c);
    out.partition.num_parts = static_cast<std::int32_t>(cfg.num_parts);
    out.partition.cutsize = r.cutsize;
    out.partition.imbalance = r.imbalance;
    RunReport& R = out.report;
    R.n = r.n;
    R.edges = r.edges;
    R.num_parts = r.num_parts;
    R.iterations = r.iterations;
    R.theta.assign(r.theta, r.theta + r.eigenvectors);
    R.residual_norms.assign(r.residual_norms, r.residual_norms + r.eigenvectors);
    R.converged.assign(r.converged, r.converged + r.eigenvectors);
    R.times = {r.laplacian_s, r.eigensolve_s, r.partition_s, r.total_s};
    R.cutsize = r.cutsize;
    R.imbalance = r.imbalance;
    R.part_weights = out.partition.part_weights;
    if (r.warnings & SP_WARN_BREAKDOWN_RECOVERED)
        R.warnings.emplace_back("eigensolver recovered from a basis breakdown by clearing the search directions");
    if (r.warnings & SP_WARN_UNCONVERGED)
        R.warnings.emplace_back("eigensolver reached max_iters with unconverged columns; "
                                "partitioning on partially converged eigenvectors");
    if (r.warnings & SP_WARN_IMBALANCE)
        R.warnings.emplace_back("imbalance " + std::to_string(r.imbalance) + " exceeds 1+epsilon = " +
                                std::to_string(1.0 + cfg.epsilon));
    return out;
}

namespace b200 {
inline Graph download(sp_context* c, sp_device_graph* dg, std::vector<std::int64_t>* old_ids) {
    sp_graph_info info{};
    rethrow(sp_device_graph_info(c, dg, &info), c);
    Graph g;
    g.adjacency.nrows = g.adjacency.ncols = info.n;
    g.adjacency.row_offsets.resize(static_cast<size_t>(info.n + 1));
    g.adjacency.col_indices.resize(static_cast<size_t>(info.nnz));
    if (old_ids) old_ids->resize(static_cast<size_t>(info.n));
    rethrow(sp_device_graph_download(c, dg, g.adjacency.row_offsets.data(), g.adjacency.col_indices.data(),
                                     old_ids ? old_ids->data() : nullptr), c);
    g.adjacency.values.assign(static_cast<size_t>(info.nnz), 1.0);  // unit edge costs, as graph.cpp:61
    g.vertex_weights.assign(static_cast<size_t>(info.n), 1.0);
    return g;
}

struct DeviceGraphHolder {
    sp_device_graph* p = nullptr;
    ~DeviceGraphHolder() { sp_graph_free(p); }
};
} // namespace b200

// graph.hpp:53 (graph.cpp:44-64), on the device
inline Graph symmetrize(const SparseMatrix& A) {
    if (A.nrows != A.ncols) throw std::invalid_argument("symmetrize: matrix not square");
    sp_context* c = b200::context();
    b200::DeviceGraphHolder h;
    b200::rethrow(sp_ingest(c, A.nrows, A.row_offsets.data(), A.col_indices.data(), 0, &h.p), c);
    return b200::download(c, h.p, nullptr);
}

// graph.hpp:62 (graph.cpp:118-171), on the device
inline std::pair<Graph, std::vector<std::int64_t>> largest_connected_component(const Graph& g) {
    sp_context* c = b200::context();
    b200::DeviceGraphHolder h;
    b200::rethrow(sp_ingest(c, g.n(), g.adjacency.row_offsets.data(), g.adjacency.col_indices.data(), 1, &h.p), c);
    std::vector<std::int64_t> old;
    Graph sub = b200::download(c, h.p, &old);
    return {std::move(sub), std::move(old)};
}

// graph.hpp:65 (graph.cpp:173-182)
inline GraphKind classify(const Graph& g) {
    sp_context* c = b200::context();
    sp_graph cg{g.n(), g.adjacency.row_offsets.data(), g.adjacency.col_indices.data(), nullptr, nullptr};
    sp_graph_info info{};
    b200::rethrow(sp_classify(c, &cg, &info), c);
    GraphKind k;
    k.kind = info.regular ? Regularity::Regular : Regularity::Irregular;
    k.max_degree = info.max_degree;
    k.avg_degree = info.avg_degree;
    k.ratio = info.degree_ratio;
    return k;
}

} // namespace specpart
