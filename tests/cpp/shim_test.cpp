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
    // CLI ingestion (tools/specpart.cpp:89-90): a directed 3-cycle with a self-loop and a
    // directed path 3 -> 5 -> 4; two components of 3 vertices, the tie goes to {0, 1, 2}
    SparseMatrix raw;
    raw.nrows = raw.ncols = 6;
    raw.row_offsets = {0, 2, 3, 4, 5, 5, 6};
    raw.col_indices = {1, 0, 2, 0, 5, 4};
    Graph whole = symmetrize(raw);
    auto [lcc, old] = largest_connected_component(whole);
    if (whole.adjacency.nnz() != 10 || lcc.n() != 3 || lcc.adjacency.nnz() != 6 || old != std::vector<std::int64_t>{0, 1, 2})
        ++fails;
    if (classify(lcc).kind != Regularity::Regular || classify(lcc).max_degree != 2) ++fails;
    // kernels.hpp: gram / mult / mult_sub on small exact integers (every product exact in fp64)
    Dense X(5, 2), C(2, 3);
    for (int i = 0; i < 5; ++i) { X(i, 0) = i + 1; X(i, 1) = 2 - i; }
    for (int j = 0; j < 3; ++j) { C(0, j) = j - 1; C(1, j) = 2 * j + 1; }
    Dense Y;
    kernels::mult(X, C, Y);
    Dense Z = Y;
    kernels::mult_sub(Z, X, C);
    Dense G = kernels::gram(X, Y);
    for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 3; ++j) {
            if (Y(i, j) != X(i, 0) * C(0, j) + X(i, 1) * C(1, j)) ++fails;
            if (Z(i, j) != 0.0) ++fails;
        }
    for (int a = 0; a < 2; ++a)
        for (int j = 0; j < 3; ++j) {
            double s = 0;
            for (int i = 0; i < 5; ++i) s += X(i, a) * Y(i, j);
            if (G(a, j) != s) ++fails;
        }
    std::printf("shim_test: cut %.0f, %d boundaries, %d failures\n", r.report.cutsize, boundaries, fails);
    return fails ? 1 : 0;
}
