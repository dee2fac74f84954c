// A reference-style caller compiled against the header-only shim (include/specpart_b200.hpp)
// instead of specpart/pipeline.hpp: pipeline_test.cpp:66-110 KATs, unchanged call syntax.
#include "specpart_b200.hpp"

#include <cstdio>
#include <utility>
#include <vector>

using namespace specpart;

static Graph ring(int n) {
    Graph g;
    g.adjacency.nrows = g.adjacency.ncols = n;
    g.adjacency.row_offsets.push_back(0);
    for (int i = 0; i < n; ++i) {
        int a = (i + n - 1) % n, b = (i + 1) % n;
        if (a > b) std::swap(a, b);
        g.adjacency.col_indices.push_back(a);
        g.adjacency.col_indices.push_back(b);
        g.adjacency.values.push_back(1.0);
        g.adjacency.values.push_back(1.0);
        g.adjacency.row_offsets.push_back(g.adjacency.col_indices.size());
    }
    g.vertex_weights.assign(n, 1.0);
    return g;
}

int main() {
    int fails = 0;
    RunConfig cfg;
    cfg.num_parts = 2;
    cfg.tol = 1e-6;
    cfg.seed = 5;
    cfg.precond = PrecondChoice::Jacobi;
    RunResult r = partition_graph(ring(8), cfg);
    int boundaries = 0;
    for (int i = 0; i < 8; ++i) boundaries += r.partition.assignment[i] != r.partition.assignment[(i + 1) % 8];
    if (r.report.cutsize != 2.0 || boundaries != 2) ++fails;
    if (r.partition.part_weights[0] != 4.0 || r.partition.part_weights[1] != 4.0) ++fails;
    try {
        RunConfig bad = cfg;
        bad.num_parts = 9;
        partition_graph(ring(8), bad);
        ++fails;
    } catch (const InfeasibleError&) {
    }
    std::printf("shim_test: cut %.0f, %d boundaries, %d failures\n", r.report.cutsize, boundaries, fails);
    return fails ? 1 : 0;
}
