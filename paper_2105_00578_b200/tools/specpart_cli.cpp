// specpart_b200 — the reference's command-line front end (tools/specpart.cpp) on the B200 C-ABI.
//
// Same options, subcommands `gen` and `sweep`, output formats and exit codes as tools/specpart.cpp:
//   * Matrix Market parsing (sparse.cpp:105-171) on the host — file I/O, no device work;
//   * symmetrize + largest_connected_component (graph.cpp:44-171) on the device (sp_ingest);
//   * partition_graph (pipeline.cpp:47-167) on the device graph (sp_partition_resident), or the
//     --init-file warm start (tools/specpart.cpp:94-157, x0 passed to the same call);
//   * write_partition "origId partId" lines (graph.cpp:232-238) and the JSON run report
//     (pipeline.cpp:169-215, docs/report_schema.md: nlohmann::json::dump(2) layout, keys sorted).
// Exit codes (tools/specpart.cpp:19-22, 335-350): 0 ok, 1 other error, 2 parse error, 3 solver
// breakdown, 4 infeasible configuration / degenerate degree. Option errors use CLI11's codes.
#include "specpart_b200.h"

#include <json.hpp>  // nlohmann/json (header-only; the reference's report serializer)

#include <algorithm>
#include <cctype>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

namespace {

constexpr int kExitParse = 2, kExitBreakdown = 3, kExitInfeasible = 4;
// CLI11 exit codes for option errors (CLI11 ExitCodes)
constexpr int kCliConversion = 101, kCliValidation = 105, kCliRequired = 106, kCliExtras = 109;

struct Fail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const std::string& m) { throw Fail{code, m}; }

// ---- Matrix Market (sparse.cpp:79-171) --------------------------------------------------------
std::string lower(std::string s) {
    for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

bool blank_or_comment(const std::string& line) {
    for (char c : line) {
        if (c == '%') return true;
        if (!std::isspace(static_cast<unsigned char>(c))) return false;
    }
    return true;
}

// ParseError::what() (errors.hpp:10-19)
std::string perr(const std::string& m, std::size_t line) {
    return "line " + std::to_string(line) + ": " + m;
}

// Pattern CSR of the parsed matrix, rows bucketed in file order (duplicates kept: sp_ingest's
// sort + unique is from_triplets(sum_duplicates=false), and symmetrize ignores values).
struct Pattern {
    int64_t nrows = 0, ncols = 0;
    std::vector<int64_t> offsets;
    std::vector<int32_t> cols;
};

Pattern parse_matrix_market(std::istream& in) {
    std::string line;
    std::size_t lineno = 0;
    if (!std::getline(in, line)) fail(kExitParse, perr("empty input", 1));
    ++lineno;
    std::istringstream banner(line);
    std::string tag, object, format, field, symmetry;
    banner >> tag >> object >> format >> field >> symmetry;
    if (lower(tag) != "%%matrixmarket" || lower(object) != "matrix")
        fail(kExitParse, perr("malformed MatrixMarket banner", lineno));
    format = lower(format);
    field = lower(field);
    symmetry = lower(symmetry);
    if (format != "coordinate")
        fail(kExitParse, perr("unsupported format '" + format + "' (coordinate only)", lineno));
    const bool pattern = field == "pattern";
    if (!pattern && field != "real" && field != "integer")
        fail(kExitParse, perr("unsupported field '" + field + "'", lineno));
    const bool symmetric = symmetry == "symmetric";
    if (!symmetric && symmetry != "general")
        fail(kExitParse, perr("unsupported symmetry '" + symmetry + "'", lineno));

    int64_t nrows = 0, ncols = 0, declared = 0;
    for (;;) {
        if (!std::getline(in, line)) fail(kExitParse, perr("missing size line", lineno + 1));
        ++lineno;
        if (blank_or_comment(line)) continue;
        std::istringstream sz(line);
        if (!(sz >> nrows >> ncols >> declared) || nrows < 0 || ncols < 0 || declared < 0)
            fail(kExitParse, perr("malformed size line", lineno));
        std::string extra;
        if (sz >> extra) fail(kExitParse, perr("trailing tokens on size line", lineno));
        break;
    }
    std::vector<int32_t> rr, cc;
    rr.reserve(static_cast<size_t>(symmetric ? 2 * declared : declared));
    cc.reserve(rr.capacity());
    int64_t seen = 0;
    while (seen < declared) {
        if (!std::getline(in, line))
            fail(kExitParse, perr("entry list truncated: expected " + std::to_string(declared) +
                                      " entries, got " + std::to_string(seen),
                                  lineno + 1));
        ++lineno;
        if (blank_or_comment(line)) continue;
        std::istringstream es(line);
        int64_t r = 0, c = 0;
        double v = 1.0;
        if (!(es >> r >> c)) fail(kExitParse, perr("malformed entry", lineno));
        if (!pattern && !(es >> v)) fail(kExitParse, perr("missing value", lineno));
        std::string extra;
        if (es >> extra) fail(kExitParse, perr("trailing tokens on entry", lineno));
        if (r < 1 || r > nrows || c < 1 || c > ncols)
            fail(kExitParse, perr("index out of range: (" + std::to_string(r) + ", " + std::to_string(c) + ")",
                                  lineno));
        rr.push_back(static_cast<int32_t>(r - 1));
        cc.push_back(static_cast<int32_t>(c - 1));
        if (symmetric && r != c) {
            rr.push_back(static_cast<int32_t>(c - 1));
            cc.push_back(static_cast<int32_t>(r - 1));
        }
        ++seen;
    }
    Pattern p;
    p.nrows = nrows;
    p.ncols = ncols;
    p.offsets.assign(static_cast<size_t>(nrows + 1), 0);
    for (int32_t r : rr) ++p.offsets[static_cast<size_t>(r) + 1];
    for (int64_t i = 0; i < nrows; ++i) p.offsets[i + 1] += p.offsets[i];
    std::vector<int64_t> pos(p.offsets.begin(), p.offsets.end() - 1);
    p.cols.resize(rr.size());
    for (size_t k = 0; k < rr.size(); ++k) p.cols[static_cast<size_t>(pos[rr[k]]++)] = cc[k];
    return p;
}

std::vector<double> vec(const double* v, int n) { return std::vector<double>(v, v + n); }

const char* problem_name(int p) {
    switch (p) {
    case SP_PROBLEM_COMBINATORIAL: return "combinatorial";
    case SP_PROBLEM_GENERALIZED: return "generalized";
    case SP_PROBLEM_NORMALIZED: return "normalized";
    default: return "auto";
    }
}
const char* precond_name(int p) {
    switch (p) {
    case SP_PRECOND_JACOBI: return "jacobi";
    case SP_PRECOND_POLYNOMIAL: return "polynomial";
    case SP_PRECOND_AMG: return "amg";
    case SP_PRECOND_NONE: return "none";
    default: return "auto";
    }
}
const char* init_name(int p) {
    switch (p) {
    case SP_INIT_RANDOM: return "random";
    case SP_INIT_PIECEWISE: return "piecewise";
    default: return "auto";
    }
}

// RunReport::to_json (pipeline.cpp:169-215), serialized with the same header-only library the
// reference uses (nlohmann::json, sorted keys, dump(2)), so reports compare byte-for-byte.
std::string report_json(const sp_report& r, const std::vector<double>& part_weights, int64_t dropped,
                        const std::vector<std::string>& warnings, bool with_trace) {
    using nlohmann::json;
    json j;
    j["graph"] = {{"n", r.n},
                  {"edges", r.edges},
                  {"max_degree", r.max_degree},
                  {"avg_degree", r.avg_degree},
                  {"degree_ratio", r.degree_ratio},
                  {"kind", r.graph_regular ? "regular" : "irregular"},
                  {"dropped_vertices", dropped}};
    j["config"] = {{"parts", r.num_parts},
                   {"problem", problem_name(r.problem)},
                   {"preconditioner", precond_name(r.precond)},
                   {"tolerance", r.tol},
                   {"initial_vectors", init_name(r.init)},
                   {"eigenvectors", r.eigenvectors},
                   {"seed", r.seed},
                   {"max_iters", r.max_iters},
                   {"epsilon", r.epsilon},
                   {"doubled_cut", r.doubled_cut != 0}};
    std::vector<bool> conv;
    for (int k = 0; k < r.eigenvectors; ++k) conv.push_back(r.converged[k] != 0);
    j["solver"] = {{"iterations", r.iterations},
                   {"theta", vec(r.theta, r.eigenvectors)},
                   {"residual_norms", vec(r.residual_norms, r.eigenvectors)},
                   {"converged", conv}};
    if (r.amg_levels > 0) {
        json lv = json::array();
        for (int l = 0; l < r.amg_levels; ++l) lv.push_back({{"n", r.amg_n[l]}, {"nnz", r.amg_nnz[l]}});
        j["solver"]["amg_levels"] = lv;
    }
    if (with_trace && r.trace_len > 0) {
        json tr = json::array();
        for (int t = 0; t < r.trace_len; ++t) {
            const sp_trace_record& rec = r.trace[t];
            tr.push_back({{"iter", rec.iter},
                          {"min_residual", rec.min_residual},
                          {"max_residual", rec.max_residual},
                          {"theta", vec(rec.theta, rec.ntheta)}});
        }
        j["solver"]["trace"] = tr;
    }
    j["times"] = {{"laplacian_s", r.laplacian_s},
                  {"eigensolve_s", r.eigensolve_s},
                  {"partition_s", r.partition_s},
                  {"total_s", r.total_s}};
    j["partition"] = {{"cutsize", r.cutsize}, {"imbalance", r.imbalance}, {"part_weights", part_weights}};
    j["warnings"] = warnings;
    return j.dump(2);
}

// ---- status → the reference's exception classes (tools/specpart.cpp:335-350) ----------------
void check(sp_status st, sp_context* ctx) {
    if (st == SP_OK) return;
    const std::string m = sp_last_error(ctx) ? sp_last_error(ctx) : "";
    switch (st) {
    case SP_PARSE: fail(kExitParse, "parse error: " + m);
    case SP_BREAKDOWN: fail(kExitBreakdown, "solver breakdown: " + m);
    case SP_INFEASIBLE:
    case SP_DEGENERATE: fail(kExitInfeasible, "infeasible: " + m);
    default: fail(1, "error: " + m);
    }
}

// ---- generators (generators.cpp:126-175) ----------------------------------------------------
// Deterministic meshes only; nbrs(i) lists every neighbour of vertex i in ascending id order, the
// row of graph_from_edges' CSR.
struct MeshGen {
    std::string kind;
    int64_t a = 0, b = 0, c = 0;
    int stencil = 27;
    std::vector<std::vector<int64_t>> adj;  // seeded random graphs: explicit sorted rows
    int64_t n() const {
        return kind == "grid2d" ? a * b : kind == "stencil3d" ? a * b * c : a;
    }
    void nbrs(int64_t i, std::vector<int64_t>& nb) const {
        if (!adj.empty()) {
            nb.insert(nb.end(), adj[static_cast<size_t>(i)].begin(), adj[static_cast<size_t>(i)].end());
        } else if (kind == "grid2d") {
            const int64_t x = i % a, y = i / a;
            if (y > 0) nb.push_back(i - a);
            if (x > 0) nb.push_back(i - 1);
            if (x + 1 < a) nb.push_back(i + 1);
            if (y + 1 < b) nb.push_back(i + a);
        } else if (kind == "stencil3d") {
            const int64_t x = i % a, y = (i / a) % b, z = i / (a * b);
            for (int64_t dz = -1; dz <= 1; ++dz)
                for (int64_t dy = -1; dy <= 1; ++dy)
                    for (int64_t dx = -1; dx <= 1; ++dx) {
                        if (dx == 0 && dy == 0 && dz == 0) continue;
                        if (stencil == 7 && std::abs(dx) + std::abs(dy) + std::abs(dz) != 1) continue;
                        const int64_t X = x + dx, Y = y + dy, Z = z + dz;
                        if (X < 0 || X >= a || Y < 0 || Y >= b || Z < 0 || Z >= c) continue;
                        nb.push_back((Z * b + Y) * a + X);  // (dz, dy, dx) order is id order
                    }
        } else if (kind == "ring") {
            const int64_t p = (i + a - 1) % a, q = (i + 1) % a;
            nb.push_back(std::min(p, q));
            nb.push_back(std::max(p, q));
        } else {  // path
            if (i > 0) nb.push_back(i - 1);
            if (i + 1 < a) nb.push_back(i + 1);
        }
    }
};

// graph_from_edges (graph.cpp:66-81): both directions, self-loops dropped, rows sorted and unique
std::vector<std::vector<int64_t>> rows_from_edges(int64_t n, const std::vector<std::pair<int32_t, int32_t>>& edges) {
    std::vector<std::vector<int64_t>> adj(static_cast<size_t>(n));
    for (const auto& [u, v] : edges)
        if (u != v) {
            adj[static_cast<size_t>(u)].push_back(v);
            adj[static_cast<size_t>(v)].push_back(u);
        }
    for (auto& r : adj) {
        std::sort(r.begin(), r.end());
        r.erase(std::unique(r.begin(), r.end()), r.end());
    }
    return adj;
}

bool connected(const std::vector<std::vector<int64_t>>& adj) {
    std::vector<char> seen(adj.size(), 0);
    std::vector<int64_t> todo{0};
    seen[0] = 1;
    size_t count = 1;
    while (!todo.empty()) {
        const int64_t v = todo.back();
        todo.pop_back();
        for (int64_t u : adj[static_cast<size_t>(v)])
            if (!seen[static_cast<size_t>(u)]) {
                seen[static_cast<size_t>(u)] = 1;
                ++count;
                todo.push_back(u);
            }
    }
    return count == adj.size();
}

// random_regular_graph (generators.cpp:201-234): configuration model on a std::mt19937_64
// stream; a pairing with a self-loop or a repeated edge is redrawn (200 draws per stream),
// a disconnected one too; the stream is reseeded (seed + attempt * golden ratio) after 200.
std::vector<std::vector<int64_t>> random_regular_rows(int64_t n, int64_t deg, uint64_t seed) {
    if (n < 2 || deg < 1 || deg >= n) fail(kExitInfeasible, "infeasible: randomregular: need 1 <= deg < n >= 2");
    if ((n * deg) % 2 != 0) fail(kExitInfeasible, "infeasible: randomregular: n*deg must be even");
    std::vector<int32_t> stubs(static_cast<size_t>(n * deg));
    std::vector<std::pair<int32_t, int32_t>> pairs;
    for (uint64_t attempt = 0;; ++attempt) {
        std::mt19937_64 rng(seed + attempt * 0x9e3779b97f4a7c15ULL);
        for (int draw = 0; draw < 200; ++draw) {
            for (size_t k = 0; k < stubs.size(); ++k) stubs[k] = static_cast<int32_t>(k / static_cast<size_t>(deg));
            std::shuffle(stubs.begin(), stubs.end(), rng);
            pairs.clear();
            bool loop = false;
            for (size_t k = 0; k + 1 < stubs.size(); k += 2) {
                if (stubs[k] == stubs[k + 1]) {
                    loop = true;
                    break;
                }
                pairs.emplace_back(std::min(stubs[k], stubs[k + 1]), std::max(stubs[k], stubs[k + 1]));
            }
            if (loop) continue;
            std::sort(pairs.begin(), pairs.end());
            if (std::adjacent_find(pairs.begin(), pairs.end()) != pairs.end()) continue;
            auto adj = rows_from_edges(n, pairs);
            if (connected(adj)) return adj;
        }
    }
}

// scale_free_graph (generators.cpp:238-266): a star on attach+1 vertices, then each new vertex
// takes `attach` distinct targets drawn uniformly from the endpoint list (degree-proportional).
std::vector<std::vector<int64_t>> scale_free_rows(int64_t n, int64_t attach, uint64_t seed) {
    if (attach < 1 || n <= attach) fail(kExitInfeasible, "infeasible: scalefree: need n > attach >= 1");
    std::mt19937_64 rng(seed);
    std::vector<std::pair<int32_t, int32_t>> edges;
    std::vector<int32_t> ends;
    for (int64_t v = 1; v <= attach; ++v) {
        edges.emplace_back(0, static_cast<int32_t>(v));
        ends.push_back(0);
        ends.push_back(static_cast<int32_t>(v));
    }
    std::vector<int32_t> chosen;
    for (int64_t v = attach + 1; v < n; ++v) {
        chosen.clear();
        while (static_cast<int64_t>(chosen.size()) < attach) {
            const int32_t t = ends[rng() % ends.size()];
            if (std::find(chosen.begin(), chosen.end(), t) == chosen.end()) chosen.push_back(t);
        }
        for (int32_t t : chosen) {
            edges.emplace_back(t, static_cast<int32_t>(v));
            ends.push_back(t);
            ends.push_back(static_cast<int32_t>(v));
        }
    }
    return rows_from_edges(n, edges);
}

// generate() argument checks (generators.cpp:126-175)
MeshGen make_gen(const std::string& kind, const std::vector<int64_t>& dims, int stencil, uint64_t seed = 0) {
    auto dim = [&](size_t i) -> int64_t {
        if (i >= dims.size()) fail(kExitInfeasible, "infeasible: gen: missing dimension for " + kind);
        return dims[i];
    };
    MeshGen g;
    g.kind = kind;
    g.stencil = stencil;
    if (kind == "grid2d") {
        g.a = dim(0), g.b = dim(1);
        if (g.a < 1 || g.b < 1) fail(kExitInfeasible, "infeasible: grid2d: dimensions must be positive");
    } else if (kind == "stencil3d") {
        g.a = dim(0), g.b = dim(1), g.c = dim(2);
        if (g.a < 1 || g.b < 1 || g.c < 1) fail(kExitInfeasible, "infeasible: stencil3d: dimensions must be positive");
        if (stencil != 7 && stencil != 27) fail(kExitInfeasible, "infeasible: stencil3d: stencil must be 7 or 27");
    } else if (kind == "ring") {
        g.a = dim(0);
        if (g.a < 3) fail(kExitInfeasible, "infeasible: ring: need n >= 3");
    } else if (kind == "path") {
        g.a = dim(0);
        if (g.a < 1) fail(kExitInfeasible, "infeasible: path: need n >= 1");
    } else if (kind == "randomregular") {
        g.a = dim(0);
        g.adj = random_regular_rows(g.a, dim(1), seed);
    } else if (kind == "scalefree") {
        g.a = dim(0);
        g.adj = scale_free_rows(g.a, dim(1), seed);
    } else {
        fail(kExitInfeasible, "infeasible: gen: unknown kind '" + kind + "'");
    }
    return g;
}

// write_matrix_market_pattern_symmetric (sparse.cpp:179-191): the lower triangle, row order
int run_gen(const MeshGen& g, std::ostream& out) {
    const int64_t n = g.n();
    std::vector<int64_t> nb;
    int64_t lower = 0;
    for (int64_t i = 0; i < n; ++i) {
        nb.clear();
        g.nbrs(i, nb);
        for (int64_t j : nb) lower += j < i;
    }
    std::string buf = "%%MatrixMarket matrix coordinate pattern symmetric\n" + std::to_string(n) + ' ' +
                      std::to_string(n) + ' ' + std::to_string(lower) + '\n';
    char line[48];
    for (int64_t i = 0; i < n; ++i) {
        nb.clear();
        g.nbrs(i, nb);
        for (int64_t j : nb)
            if (j < i) buf.append(line, static_cast<size_t>(std::snprintf(line, sizeof line, "%lld %lld\n",
                                                                           static_cast<long long>(i + 1),
                                                                           static_cast<long long>(j + 1))));
    }
    out << buf;
    return 0;
}

// ---- sweep (tools/specpart.cpp:265-327, run_sweep + SweepTable::to_tsv, generators.cpp:283-315)
// GeneratorSpec::parse (generators.cpp:64-105) of "kind:a,b[,c][,p7|p27]"
MeshGen parse_spec(const std::string& text) {
    const size_t colon = text.find(':');
    const std::string head = text.substr(0, colon);
    std::vector<std::string> args;
    if (colon != std::string::npos) {
        std::istringstream rest(text.substr(colon + 1));
        std::string tok;
        while (std::getline(rest, tok, ',')) args.push_back(tok);
    }
    std::vector<int64_t> dims;
    int stencil = 27;
    uint64_t seed = 0;
    const size_t need = head == "stencil3d" ? 3 : (head == "ring" || head == "path") ? 1 : 2;
    for (size_t i = 0; i < args.size(); ++i) {
        if (i < need) dims.push_back(std::stoll(args[i]));
        else if (args[i] == "p7") stencil = 7;
        else if (args[i] == "p27") stencil = 27;
        else if (!args[i].empty() && args[i][0] == 's') seed = std::stoull(args[i].substr(1));
    }
    if (dims.size() < need) fail(1, "error: generator spec '" + text + "': missing argument");
    return make_gen(head, dims, stencil, seed);
}

struct SweepArgs {
    std::vector<std::string> graphs, preconds, problems;
    std::vector<double> tols;
    int64_t parts = 8;
    uint64_t seed = 42;
    int max_iters = 1000;
};

int run_sweep(const SweepArgs& s) {
    auto precond_of = [](const std::string& v) {
        if (v == "jacobi") return SP_PRECOND_JACOBI;
        if (v == "polynomial") return SP_PRECOND_POLYNOMIAL;
        if (v == "amg") return SP_PRECOND_AMG;
        if (v == "none") return SP_PRECOND_NONE;
        fail(kExitInfeasible, "infeasible: sweep: unknown preconditioner '" + v + "'");
    };
    auto problem_of = [](const std::string& v) {
        if (v == "combinatorial") return SP_PROBLEM_COMBINATORIAL;
        if (v == "generalized") return SP_PROBLEM_GENERALIZED;
        if (v == "normalized") return SP_PROBLEM_NORMALIZED;
        fail(kExitInfeasible, "infeasible: sweep: unknown problem '" + v + "'");
    };
    struct Csr {
        std::string name;
        std::vector<int64_t> off;
        std::vector<int32_t> col;
    };
    std::vector<Csr> graphs;
    for (const std::string& spec : s.graphs) {
        const MeshGen g = parse_spec(spec);
        Csr c;
        c.name = spec;
        c.off.push_back(0);
        std::vector<int64_t> nb;
        for (int64_t i = 0; i < g.n(); ++i) {
            nb.clear();
            g.nbrs(i, nb);
            for (int64_t j : nb) c.col.push_back(static_cast<int32_t>(j));
            c.off.push_back(static_cast<int64_t>(c.col.size()));
        }
        graphs.push_back(std::move(c));
    }
    struct Cfg {
        std::string label;
        sp_config c;
    };
    std::vector<Cfg> cfgs;
    const std::vector<std::string> preconds = s.preconds.empty() ? std::vector<std::string>{"jacobi"} : s.preconds;
    const std::vector<std::string> problems = s.problems.empty() ? std::vector<std::string>{"auto"} : s.problems;
    const std::vector<double> tols = s.tols.empty() ? std::vector<double>{0.0} : s.tols;
    for (const std::string& pc : preconds)
        for (const std::string& pr : problems)
            for (double t : tols) {
                sp_config c{};
                c.num_parts = s.parts;
                c.seed = s.seed;
                c.max_iters = s.max_iters;
                c.epsilon = 0.01;
                c.precond = precond_of(pc);
                c.problem = pr != "auto" ? problem_of(pr) : SP_PROBLEM_AUTO;
                c.init = SP_INIT_AUTO;
                c.tol = t > 0.0 ? t : -1.0;
                cfgs.push_back({pc + "/" + pr + "/tol=" + (t > 0.0 ? std::to_string(t) : "auto"), c});
            }
    sp_context* ctx = nullptr;
    if (sp_context_create(0, &ctx) != SP_OK) fail(1, "error: cannot create the CUDA context");
    std::ostringstream os;
    os << "graph\tconfig\titerations\tcut\timbalance\tseconds\terror\n";
    for (const Csr& g : graphs) {
        const int64_t n = static_cast<int64_t>(g.off.size()) - 1;
        const sp_graph sg{n, g.off.data(), g.col.data(), nullptr, nullptr};
        std::vector<int32_t> asg(static_cast<size_t>(n));
        for (const Cfg& c : cfgs) {
            std::vector<double> pw(static_cast<size_t>(std::max<int64_t>(c.c.num_parts, 1)));
            sp_report rep{};
            rep.part_weights = pw.data();
            const sp_status st = sp_partition(ctx, &sg, &c.c, asg.data(), &rep, nullptr);
            int iters = 0;
            double cut = 0.0, imb = 0.0, secs = 0.0;
            std::string err;
            if (st == SP_OK) iters = rep.iterations, cut = rep.cutsize, imb = rep.imbalance, secs = rep.total_s;
            else err = sp_last_error(ctx) ? sp_last_error(ctx) : "error";
            os << g.name << '\t' << c.label << '\t' << iters << '\t' << cut << '\t' << imb << '\t' << secs << '\t'
               << err << '\n';
        }
    }
    sp_context_destroy(ctx);
    std::cout << os.str();
    return 0;
}

// ---- partition (tools/specpart.cpp:62-196) ---------------------------------------------------
struct Args {
    std::string input, problem = "auto", precond = "auto", init = "auto", output, report, init_file;
    int64_t parts = 0;
    double tolerance = -1.0;
    int max_iters = 1000;
    uint64_t seed = 42;
    double epsilon = 0.01;
    bool doubled_cut = false, trace = false;
};

std::vector<double> load_dense_block_colmajor(const std::string& path, int64_t* rows, int64_t* cols) {
    std::ifstream in(path);
    if (!in) fail(kExitParse, "parse error: " + perr("cannot open '" + path + "'", 0));
    if (!(in >> *rows >> *cols) || *rows < 1 || *cols < 1)
        fail(kExitParse, "parse error: " + perr("malformed block header in '" + path + "'", 1));
    std::vector<double> X(static_cast<size_t>(*rows * *cols));
    for (int64_t i = 0; i < *rows; ++i)
        for (int64_t j = 0; j < *cols; ++j)
            if (!(in >> X[static_cast<size_t>(j * *rows + i)]))
                fail(kExitParse, "parse error: " + perr("truncated block data in '" + path + "'", 0));
    return X;
}

int eigenvector_count(int64_t K) {  // partitioner.cpp:13-17: bit_width(K)
    int b = 0;
    for (uint64_t k = static_cast<uint64_t>(K); k; k >>= 1) ++b;
    return b;
}

int run_partition(const Args& a) {
    Pattern raw;
    {
        std::ifstream in(a.input);
        if (!in) fail(kExitParse, "parse error: " + perr("cannot open '" + a.input + "'", 0));
        try {
            raw = parse_matrix_market(in);
        } catch (const Fail& f) {
            fail(f.code, "parse error: " + f.msg);
        }
    }
    if (raw.nrows != raw.ncols) fail(1, "error: symmetrize: matrix not square");

    sp_context* ctx = nullptr;
    if (sp_context_create(0, &ctx) != SP_OK) fail(1, "error: cannot create the CUDA context");
    struct Guard {
        sp_context* c;
        sp_device_graph* g = nullptr;
        ~Guard() {
            if (g) sp_graph_free(g);
            sp_context_destroy(c);
        }
    } guard{ctx};

    check(sp_ingest(ctx, raw.nrows, raw.offsets.data(), raw.cols.data(), 1, &guard.g), ctx);
    sp_graph_info info{};
    check(sp_device_graph_info(ctx, guard.g, &info), ctx);
    const int64_t dropped = info.n_symmetrized - info.n;
    std::vector<int64_t> old_ids(static_cast<size_t>(std::max<int64_t>(info.n, 1)));
    check(sp_device_graph_download(ctx, guard.g, nullptr, nullptr, old_ids.data()), ctx);

    sp_config cfg{};
    cfg.num_parts = a.parts;
    cfg.problem = a.problem == "combinatorial" ? SP_PROBLEM_COMBINATORIAL
                  : a.problem == "generalized" ? SP_PROBLEM_GENERALIZED
                  : a.problem == "normalized"  ? SP_PROBLEM_NORMALIZED
                                               : SP_PROBLEM_AUTO;
    cfg.precond = a.precond == "jacobi"       ? SP_PRECOND_JACOBI
                  : a.precond == "polynomial" ? SP_PRECOND_POLYNOMIAL
                  : a.precond == "amg"        ? SP_PRECOND_AMG
                  : a.precond == "none"       ? SP_PRECOND_NONE
                                              : SP_PRECOND_AUTO;
    cfg.init = a.init == "random" ? SP_INIT_RANDOM : a.init == "piecewise" ? SP_INIT_PIECEWISE : SP_INIT_AUTO;
    cfg.tol = a.tolerance > 0.0 ? a.tolerance : -1.0;
    cfg.max_iters = a.max_iters;
    cfg.seed = a.seed;
    cfg.epsilon = a.epsilon;
    cfg.doubled_cut = a.doubled_cut;
    cfg.record_trace = a.trace;

    std::vector<double> x0;
    if (!a.init_file.empty()) {
        int64_t rows = 0, cols = 0;
        x0 = load_dense_block_colmajor(a.init_file, &rows, &cols);
        if (rows != info.n)
            fail(kExitInfeasible, "infeasible: initial block has " + std::to_string(rows) +
                                      " rows but the graph has " + std::to_string(info.n) + " vertices");
        if (cols != eigenvector_count(a.parts))
            fail(kExitInfeasible, "infeasible: initial block must have d=" +
                                      std::to_string(eigenvector_count(a.parts)) + " columns");
    }

    std::vector<int32_t> assignment(static_cast<size_t>(info.n));
    std::vector<double> part_weights(static_cast<size_t>(std::max<int64_t>(a.parts, 1)));
    std::vector<sp_trace_record> trace(a.trace ? static_cast<size_t>(a.max_iters) + 2 : 0);
    sp_report rep{};
    rep.part_weights = part_weights.data();
    rep.trace = trace.empty() ? nullptr : trace.data();
    rep.trace_capacity = static_cast<int32_t>(trace.size());
    check(sp_partition_resident(ctx, guard.g, &cfg, assignment.data(), &rep, x0.empty() ? nullptr : x0.data()),
          ctx);

    // pipeline.cpp:140-163 warnings; the --init-file path reports only its own (specpart.cpp:156)
    std::vector<std::string> warnings;
    if (!a.init_file.empty()) {
        rep.init = SP_INIT_RANDOM;
        warnings.push_back("initial vectors loaded from " + a.init_file);
    } else {
        if (rep.warnings & SP_WARN_AMG_STAGNATED) warnings.emplace_back("amg coarsening stagnated; hierarchy stopped early");
        if (rep.warnings & SP_WARN_BREAKDOWN_RECOVERED)
            warnings.emplace_back("eigensolver recovered from a basis breakdown by clearing the search directions");
        if (rep.warnings & SP_WARN_UNCONVERGED)
            warnings.emplace_back("eigensolver reached max_iters with unconverged columns; "
                                  "partitioning on partially converged eigenvectors");
        if (rep.warnings & SP_WARN_IMBALANCE)
            warnings.emplace_back("imbalance " + std::to_string(rep.imbalance) + " exceeds 1+epsilon = " +
                                  std::to_string(1.0 + a.epsilon));
    }
    if (dropped > 0)
        warnings.push_back("input graph was disconnected; kept the largest component (" + std::to_string(info.n) +
                           " of " + std::to_string(info.n_symmetrized) + " vertices)");

    // write_partition (graph.cpp:232-238): "origId partId" per vertex
    {
        std::string buf;
        buf.reserve(assignment.size() * 16);
        char line[48];
        for (size_t v = 0; v < assignment.size(); ++v) {
            const int len = std::snprintf(line, sizeof line, "%lld %d\n", static_cast<long long>(old_ids[v]),
                                          assignment[v]);
            buf.append(line, static_cast<size_t>(len));
        }
        if (!a.output.empty()) {
            std::ofstream out(a.output, std::ios::binary);
            out << buf;
        } else {
            std::cout << buf;
        }
    }
    if (!a.report.empty()) {
        std::ofstream out(a.report);
        out << report_json(rep, part_weights, dropped, warnings, a.trace) << '\n';
    }
    std::ostringstream imb;
    imb << rep.imbalance;  // default ostream formatting, as specpart.cpp:189-191
    std::cerr << "n=" << rep.n << " K=" << rep.num_parts << " cutsize=" << rep.cutsize << " imbalance=" << imb.str()
              << " iters=" << rep.iterations << '\n';
    for (const std::string& w : warnings) std::cerr << "warning: " << w << '\n';
    return 0;
}

// ---- option parsing (the CLI11 surface of tools/specpart.cpp:200-235) ------------------------
bool take(int argc, char** argv, int& i, const char* name, std::string& val) {
    const size_t L = std::strlen(name);
    if (std::strncmp(argv[i], name, L) != 0) return false;
    if (argv[i][L] == '=') {
        val = argv[i] + L + 1;
        return true;
    }
    if (argv[i][L] != '\0') return false;
    if (i + 1 >= argc) fail(kCliConversion, std::string(name) + " requires an argument");
    val = argv[++i];
    return true;
}

template <class T>
T num(const std::string& s, const char* name) {
    T v{};
    auto r = std::from_chars(s.data(), s.data() + s.size(), v);
    if (r.ec != std::errc() || r.ptr != s.data() + s.size())
        fail(kCliConversion, std::string("Could not convert: ") + name + " = " + s);
    return v;
}

void member(const std::string& v, const char* name, std::initializer_list<const char*> allowed) {
    for (const char* a : allowed)
        if (v == a) return;
    fail(kCliValidation, std::string(name) + ": " + v + " not in allowed set");
}

void usage() {
    std::cout << "spectral graph partitioner (B200)\n"
                 "Usage: specpart_b200 [OPTIONS] [SUBCOMMAND]\n"
                 "  --input FILE        Matrix Market graph file\n"
                 "  --parts K           number of parts K\n"
                 "  --problem P         auto|combinatorial|generalized|normalized\n"
                 "  --precond P         auto|jacobi|polynomial|amg|none\n"
                 "  --init I            auto|random|piecewise\n"
                 "  --tolerance T       eigensolver residual tolerance\n"
                 "  --max-iters N       eigensolver iteration cap\n"
                 "  --seed S            random seed\n"
                 "  --epsilon E         allowed imbalance ratio (default 0.01)\n"
                 "  --threads N         accepted for compatibility (the solve runs on the GPU)\n"
                 "  --doubled-cut       report cut edges counted twice\n"
                 "  --trace             record per-iteration solver trace in the report\n"
                 "  --output FILE       partition file (default stdout)\n"
                 "  --report FILE       write a JSON run report\n"
                 "  --init-file FILE    dense initial block: 'rows cols' header, row-major values\n"
                 "Subcommands:\n"
                 "  gen KIND DIMS... [--stencil 7|27] [--seed S] [--out FILE]\n"
                 "        grid2d W H | stencil3d X Y Z | ring N | path N | randomregular N DEG | scalefree N ATTACH\n"
                 "  sweep --gen SPEC... [--parts K] [--tolerances T...] [--preconds P...] [--problems P...]\n"
                 "        [--seed S] [--max-iters N]   TSV table (graph, config, iterations, cut, imbalance, s)\n";
}

int main_impl(int argc, char** argv) {
    Args a;
    int i = 1;
    if (argc > 1 && std::strcmp(argv[1], "gen") == 0) {
        std::string kind, out, v;
        std::vector<int64_t> dims;
        int stencil = 27;
        uint64_t gseed = 0;
        for (i = 2; i < argc; ++i) {
            if (take(argc, argv, i, "--stencil", v)) stencil = num<int>(v, "--stencil");
            else if (take(argc, argv, i, "--seed", v)) gseed = num<uint64_t>(v, "--seed");
            else if (take(argc, argv, i, "--out", out)) {
            } else if (argv[i][0] == '-' && argv[i][1] == '-') fail(kCliExtras, std::string("The following argument was not expected: ") + argv[i]);
            else if (kind.empty()) kind = argv[i];
            else dims.push_back(num<int64_t>(argv[i], "dims"));
        }
        if (kind.empty() || dims.empty()) fail(kCliRequired, "gen: kind and dims are required");
        const MeshGen g = make_gen(kind, dims, stencil, gseed);
        if (!out.empty()) {
            std::ofstream f(out);
            return run_gen(g, f);
        }
        return run_gen(g, std::cout);
    }
    if (argc > 1 && std::strcmp(argv[1], "sweep") == 0) {
        SweepArgs s;
        std::string v;
        // CLI11 vector options: values follow the flag until the next option
        auto many = [&](int& k, std::vector<std::string>& dst) {
            while (k + 1 < argc && std::strncmp(argv[k + 1], "--", 2) != 0) dst.push_back(argv[++k]);
        };
        for (i = 2; i < argc; ++i) {
            std::vector<std::string> tmp;
            if (!std::strcmp(argv[i], "--gen")) many(i, s.graphs);
            else if (!std::strcmp(argv[i], "--preconds")) many(i, s.preconds);
            else if (!std::strcmp(argv[i], "--problems")) many(i, s.problems);
            else if (!std::strcmp(argv[i], "--tolerances")) {
                many(i, tmp);
                for (const std::string& t : tmp) s.tols.push_back(num<double>(t, "--tolerances"));
            } else if (take(argc, argv, i, "--parts", v)) s.parts = num<int64_t>(v, "--parts");
            else if (take(argc, argv, i, "--seed", v)) s.seed = num<uint64_t>(v, "--seed");
            else if (take(argc, argv, i, "--max-iters", v)) s.max_iters = num<int>(v, "--max-iters");
            else fail(kCliExtras, std::string("The following argument was not expected: ") + argv[i]);
        }
        if (s.graphs.empty()) fail(kCliRequired, "--gen is required");
        return run_sweep(s);
    }
    for (; i < argc; ++i) {
        std::string v;
        if (!std::strcmp(argv[i], "--help") || !std::strcmp(argv[i], "-h")) {
            usage();
            return 0;
        }
        if (!std::strcmp(argv[i], "--doubled-cut")) a.doubled_cut = true;
        else if (!std::strcmp(argv[i], "--trace")) a.trace = true;
        else if (take(argc, argv, i, "--input", a.input)) {
        } else if (take(argc, argv, i, "--parts", v)) a.parts = num<int64_t>(v, "--parts");
        else if (take(argc, argv, i, "--problem", a.problem))
            member(a.problem, "--problem", {"auto", "combinatorial", "generalized", "normalized"});
        else if (take(argc, argv, i, "--precond", a.precond))
            member(a.precond, "--precond", {"auto", "jacobi", "polynomial", "amg", "none"});
        else if (take(argc, argv, i, "--init", a.init)) member(a.init, "--init", {"auto", "random", "piecewise"});
        else if (take(argc, argv, i, "--tolerance", v)) a.tolerance = num<double>(v, "--tolerance");
        else if (take(argc, argv, i, "--max-iters", v)) a.max_iters = num<int>(v, "--max-iters");
        else if (take(argc, argv, i, "--seed", v)) a.seed = num<uint64_t>(v, "--seed");
        else if (take(argc, argv, i, "--epsilon", v)) a.epsilon = num<double>(v, "--epsilon");
        else if (take(argc, argv, i, "--threads", v)) (void)num<int>(v, "--threads");
        else if (take(argc, argv, i, "--output", a.output)) {
        } else if (take(argc, argv, i, "--report", a.report)) {
        } else if (take(argc, argv, i, "--init-file", a.init_file)) {
        } else fail(kCliExtras, std::string("The following argument was not expected: ") + argv[i]);
    }
    if (a.input.empty() || a.parts < 2) {
        std::cerr << "error: --input and --parts >= 2 are required (see --help)\n";
        return kExitInfeasible;
    }
    return run_partition(a);
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return main_impl(argc, argv);
    } catch (const Fail& f) {
        std::cerr << f.msg << '\n';
        return f.code;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}
