// graph_dev.cuh — device-resident graph (a row block of it on multi-GPU) and
// the Laplacian operators built from it.
#pragma once

#include "ops.cuh"

#include <cstring>
#include <vector>

namespace spb {

// Graph (graph.hpp:17-32) on the device. On one GPU the block is the whole
// graph (row0 = 0, n_local = n_global). Offsets are rebased to the block;
// column ids stay global.
struct DevGraph {
    int64_t n_global = 0;
    int64_t nnz_global = 0;
    int64_t row0 = 0;
    int64_t n_local = 0;
    int64_t nnz_local = 0;
    DBuf<int64_t> offs;   // n_local + 1, offs[0] = 0
    DBuf<int32_t> cols;   // nnz_local
    DBuf<double> vals;    // nnz_local, empty = unit costs
    DBuf<double> vw;      // n_local vertex weights, empty = unit
    DBuf<double> vw_all;  // n_global vertex weights as given (empty = unit)
    DBuf<double> deg;     // n_local weighted degrees (Graph::weighted_degree)
    DBuf<double> deg_all; // n_global degrees (multi-GPU); empty on one GPU
    bool unit_values = true;
    bool unit_weights = true;
    bool positive_weights = true;
    bool prepared = false;
    bool positive_degrees_local = true;
    bool positive_degrees = true;   // all vertices (the generalized problem needs B = D > 0)
    int64_t max_degree_local = 0;
    int64_t max_degree_global = 0;

    const double* deg_global() const { return deg_all.p ? deg_all.p : deg.p; }
};

struct DevLaplacian {
    int kind = 0;  // 0 combinatorial, 1 normalized, 2 degree
    DevOp op;
    DBuf<double> diag;
    DBuf<double> isd;     // normalized: n_global entries
    DBuf<int64_t> offs_L; // explicit form
    DBuf<int32_t> cols_L;
    DBuf<double> vals_L;
    DBuf<int32_t> long_rows;
    RowBins bins;  // irregular graphs in the solver (spmm_vec.cu)
    DBuf<int32_t> cols_halo;  // multi-GPU: op columns in local halo numbering
    DBuf<double> isd_halo;    // multi-GPU normalized: isd of own + halo rows
    DBuf<int32_t> dpos;       // multi-GPU: per-row diagonal storage slot
};

// Weighted degrees, unit-cost detection and max degree of the local block.
void graph_degrees(DevGraph& g, cudaStream_t s);
// Builds L_C (kind 0), L_N (kind 1) or D (kind 2). With materialize the explicit
// CSR of L is formed (bit-exact, laplacian.cpp:53-144); otherwise unit-cost
// graphs use the pattern operators (same results, 4 B/nnz).
void build_laplacian(int kind, const DevGraph& g, bool materialize, DevLaplacian& L, cudaStream_t s);
void collect_long_rows(const DevGraph& g, DevLaplacian& L, int64_t threshold, cudaStream_t s);
void inverse_diagonal(const DevLaplacian& L, DBuf<double>& inv, cudaStream_t s);

// Degree-descending vertex order of a one-GPU graph (relabel.cu): new vertex r is old
// vertex perm[r] (ties by ascending id); out holds the relabelled CSR.
struct Relabel {
    DBuf<int32_t> perm, inv;  // new -> old, old -> new
    bool on = false;
};
void relabel_by_degree(const DevGraph& g, DevGraph& out, Relabel& rl, cudaStream_t s);
// dst_new(r, :) = src_old(perm[r], :)  /  dst_old(perm[r], :) = src_new(r, :)
void permute_rows_in(const Relabel& rl, int64_t n, int m, const View& src_old, const View& dst_new, cudaStream_t s);
void permute_rows_out(const Relabel& rl, int64_t n, int m, const View& src_new, const View& dst_old, cudaStream_t s);

} // namespace spb
