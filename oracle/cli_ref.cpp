// oracle/cli_ref.cpp — TEST INFRASTRUCTURE ONLY. The reference CLI's partition and gen paths
// (tools/specpart.cpp:62-196, 237-263) without CLI11 (absent here), linked against the
// unmodified reference objects in oracle/_ref. Used by tests/golden/make_cli_golden.py to record
// the partition files, reports and .mtx outputs the B200 CLI must reproduce.
//   cli_ref gen KIND STENCIL DIMS... [SEED]       -> .mtx on stdout (SEED: randomregular/scalefree)
//   cli_ref part MTX K PROBLEM PRECOND SEED OUT REPORT
//   cli_ref sweep K SEED SPEC,SPEC PRECOND,PRECOND PROBLEM,PROBLEM   (tools/specpart.cpp:265-327)
#include "specpart/generators.hpp"
#include "specpart/graph.hpp"
#include "specpart/pipeline.hpp"
#include "specpart/sparse.hpp"

#include <cstdlib>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

using namespace specpart;

int main(int argc, char** argv) {
    if (argc < 2) return 1;
    const std::string mode = argv[1];
    if (mode == "gen") {
        const std::string kind = argv[2];
        const int stencil = std::atoi(argv[3]);
        std::vector<std::int64_t> d;
        for (int i = 4; i < argc; ++i) d.push_back(std::atoll(argv[i]));
        GeneratorSpec spec;
        if (kind == "grid2d") spec = GeneratorSpec::grid2d(d[0], d[1]);
        else if (kind == "stencil3d") spec = GeneratorSpec::stencil3d(d[0], d[1], d[2], stencil);
        else if (kind == "ring") spec.kind = GeneratorSpec::Kind::Ring, spec.a = d[0];
        else if (kind == "path") spec.kind = GeneratorSpec::Kind::Path, spec.a = d[0];
        else if (kind == "randomregular") spec = GeneratorSpec::random_regular(d[0], d[1], static_cast<std::uint64_t>(d[2]));
        else if (kind == "scalefree") spec = GeneratorSpec::scale_free(d[0], d[1], static_cast<std::uint64_t>(d[2]));
        else return 1;
        write_matrix_market_pattern_symmetric(std::cout, generate(spec).adjacency);
        return 0;
    }
    if (mode == "sweep") {
        auto split = [](const std::string& t) {
            std::vector<std::string> v;
            std::size_t p = 0;
            while (p <= t.size()) {
                const std::size_t q = t.find(';', p);
                v.push_back(t.substr(p, q == std::string::npos ? std::string::npos : q - p));
                if (q == std::string::npos) break;
                p = q + 1;
            }
            return v;
        };
        std::vector<Graph> storage;
        std::vector<std::pair<std::string, const Graph*>> graphs;
        const auto specs = split(argv[4]);
        storage.reserve(specs.size());
        for (const std::string& t : specs) {
            storage.push_back(generate(GeneratorSpec::parse(t)));
            graphs.emplace_back(t, &storage.back());
        }
        std::vector<std::pair<std::string, RunConfig>> configs;
        for (const std::string& pc : split(argv[5]))
            for (const std::string& pr : split(argv[6])) {
                RunConfig c;
                c.num_parts = std::atoll(argv[2]);
                c.seed = std::strtoull(argv[3], nullptr, 10);
                c.precond = pc == "polynomial" ? PrecondChoice::Polynomial
                            : pc == "none"     ? PrecondChoice::None
                                               : PrecondChoice::Jacobi;
                if (pr == "combinatorial") c.problem = ProblemChoice::Combinatorial;
                else if (pr == "generalized") c.problem = ProblemChoice::Generalized;
                else if (pr == "normalized") c.problem = ProblemChoice::Normalized;
                configs.emplace_back(pc + "/" + pr + "/tol=auto", c);
            }
        std::cout << run_sweep(graphs, configs).to_tsv();
        return 0;
    }
    const std::string problem = argv[4], precond = argv[5];
    RunConfig cfg;
    cfg.num_parts = std::atoll(argv[3]);
    cfg.seed = std::strtoull(argv[6], nullptr, 10);
    if (problem == "combinatorial") cfg.problem = ProblemChoice::Combinatorial;
    else if (problem == "generalized") cfg.problem = ProblemChoice::Generalized;
    else if (problem == "normalized") cfg.problem = ProblemChoice::Normalized;
    if (precond == "jacobi") cfg.precond = PrecondChoice::Jacobi;
    else if (precond == "polynomial") cfg.precond = PrecondChoice::Polynomial;
    else if (precond == "none") cfg.precond = PrecondChoice::None;
    else if (precond == "amg") cfg.precond = PrecondChoice::Amg;
    SparseMatrix raw = parse_matrix_market_file(argv[2]);
    Graph whole = symmetrize(raw);
    auto [g, original_ids] = largest_connected_component(whole);
    const std::int64_t dropped = whole.n() - g.n();
    RunResult result = partition_graph(g, cfg);
    result.report.dropped_vertices = dropped;
    if (dropped > 0)
        result.report.warnings.push_back("input graph was disconnected; kept the largest component (" +
                                         std::to_string(g.n()) + " of " + std::to_string(whole.n()) +
                                         " vertices)");
    std::ofstream out(argv[7]);
    write_partition(out, result.partition.assignment, original_ids);
    std::ofstream rep(argv[8]);
    rep << result.report.to_json() << '\n';
    return 0;
}
