// A reference caller compiled against the shim (include/specpart_b200.hpp) instead of
// specpart/*.hpp: the call sequence of tools/specpart.cpp's run_partition (:63-184) —
// Matrix Market parse, symmetrize, largest component, partition_graph, and the
// --init-file path that resolves the Auto table and runs build_problem ->
// {jacobi,polynomial,amg}_build -> lobpcg -> embed -> mj_partition -> make_partition
// by hand — plus write/read_partition, cutsize/imbalance, to_json and the exception
// types the CLI maps to exit codes. Usage: caller_test <graph.mtx>
#include "specpart_b200.hpp"

#include <cstdio>
#include <sstream>
#include <string>
#include <vector>

using namespace specpart;

static int fails = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            ++fails;                                                          \
            std::printf("FAILED line %d: %s\n", __LINE__, #c);                 \
        }                                                                     \
    } while (0)

// the init-file branch: every stage by hand on an explicit X0
static RunResult by_hand(const Graph& g, const RunConfig& cfg, const Dense& X0) {
    GraphKind kind = classify(g);
    PrecondChoice pc = cfg.precond == PrecondChoice::Auto ? select_precond_auto(kind) : cfg.precond;
    auto [prob, tol_auto] = select_defaults(kind, pc);
    const double tol = cfg.tol.value_or(tol_auto);
    const int d = eigenvector_count(cfg.num_parts);
    EigenProblem problem = build_problem(g, prob);
    std::unique_ptr<Preconditioner> M;
    if (pc == PrecondChoice::Jacobi) M = jacobi_build(problem.A);
    else if (pc == PrecondChoice::Polynomial) {
        PolyConfig poly;
        poly.seed = cfg.seed ^ 0x706f6c79ULL;
        M = polynomial_build(problem.A, poly);
    } else if (pc == PrecondChoice::Amg) {
        AmgConfig ac = kind.kind == Regularity::Regular ? AmgConfig::regular_defaults() : AmgConfig::irregular_defaults();
        ac.seed = cfg.seed ^ 0x616d67ULL;
        M = amg_build(problem.A, ac);
    }
    SolverConfig sc;
    sc.nev = d;
    sc.tol = tol;
    sc.max_iters = cfg.max_iters;
    sc.seed = cfg.seed;
    EigenResult eig = lobpcg(problem, M.get(), X0, sc);
    Embedding emb = embed(eig.X);
    Partition part = mj_partition(emb, g.vertex_weights, cfg.num_parts);
    RunResult result;
    result.partition = make_partition(g, std::move(part.assignment), static_cast<std::int32_t>(cfg.num_parts),
                                      cfg.doubled_cut);
    result.report.n = g.n();
    result.report.graph_kind = kind;
    result.report.resolved = {prob, pc, tol, InitChoice::Random, d};
    result.report.iterations = eig.iterations;
    result.report.theta = eig.theta;
    result.report.cutsize = result.partition.cutsize;
    return result;
}

int main(int argc, char** argv) {
    if (argc < 2) {
        std::printf("usage: caller_test <graph.mtx>\n");
        return 2;
    }
    SparseMatrix raw = parse_matrix_market_file(argv[1]);
    Graph whole = symmetrize(raw);
    auto [g, original_ids] = largest_connected_component(whole);
    CHECK(g.n() > 0 && g.n() <= whole.n());

    for (PrecondChoice pc : {PrecondChoice::Jacobi, PrecondChoice::Polynomial, PrecondChoice::Amg}) {
        RunConfig cfg;
        cfg.num_parts = 4;
        cfg.precond = pc;
        cfg.seed = 11;
        cfg.record_trace = true;
        RunResult r = partition_graph(g, cfg);
        CHECK(r.report.resolved.precond == pc);
        CHECK(r.report.resolved.eigenvectors == 3);
        CHECK(static_cast<int>(r.report.trace.size()) == r.report.iterations + 1);
        CHECK(r.partition.cutsize == cutsize(g, r.partition.assignment));
        CHECK(r.partition.imbalance == imbalance(r.partition.part_weights));
        CHECK((pc == PrecondChoice::Amg) == !r.report.amg_levels.empty());
        // the same run through the individual stages on the same initial block
        Dense X0 = initial_guess_random(g.n(), 3, cfg.seed);
        RunResult h = by_hand(g, cfg, X0);
        CHECK(h.report.iterations == r.report.iterations);
        CHECK(h.partition.assignment == r.partition.assignment);
        CHECK(h.partition.cutsize == r.partition.cutsize);
        // write_partition / read_partition round trip with the original ids
        std::stringstream ss;
        write_partition(ss, r.partition.assignment, original_ids);
        auto rows = read_partition(ss);
        CHECK(static_cast<std::int64_t>(rows.size()) == g.n());
        CHECK(rows.front().first == original_ids.front() && rows.front().second == r.partition.assignment.front());
        r.report.dropped_vertices = whole.n() - g.n();
        const std::string js = r.report.to_json();
        CHECK(js.find("\"dropped_vertices\"") != std::string::npos && js.find("\"iterations\"") != std::string::npos);
        CHECK((js.find("\"amg_levels\"") != std::string::npos) == (pc == PrecondChoice::Amg));
        std::printf("%s: cut %.0f, imbalance %.6f, %d iterations\n", precond_choice_name(pc), r.report.cutsize,
                    r.report.imbalance, r.report.iterations);
    }
    // the CLI's exit-code classes (tools/specpart.cpp:335-350)
    try {
        RunConfig bad;
        bad.num_parts = g.n() + 1;
        partition_graph(g, bad);
        CHECK(false);
    } catch (const InfeasibleError&) {
    }
    try {
        std::istringstream in("%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1.0\n");
        parse_matrix_market(in);
        CHECK(false);
    } catch (const ParseError& e) {
        CHECK(e.line() == 4);
    }
    try {
        Dense X0(g.n(), 3);  // rank-0 block: breakdown after the retry (acceptance c9)
        RunConfig cfg;
        cfg.num_parts = 4;
        cfg.precond = PrecondChoice::Jacobi;
        by_hand(g, cfg, X0);
        CHECK(false);
    } catch (const BreakdownError& e) {
        CHECK(e.retried());
    }
    std::printf("caller_test: %d failures\n", fails);
    return fails ? 1 : 0;
}
