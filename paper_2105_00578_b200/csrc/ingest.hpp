// ingest.hpp — symmetrize + largest_connected_component on the device (ingest.cu).
#pragma once

#include "common.cuh"

namespace spb {

struct IngestResult {
    int64_t n_sym = 0, nnz_sym = 0;  // symmetrized pattern (before the component cut)
    int64_t n = 0, nnz = 0;          // result graph
    int32_t components_root = 0;     // minimum vertex id of the kept component
    DBuf<int64_t> offs;              // n + 1
    DBuf<int32_t> cols;              // nnz, strictly increasing per row
    DBuf<int64_t> old_ids;           // n: original vertex id of every kept vertex
};

// symmetrize (graph.cpp:44-64) of the square pattern (n, d_offs, d_cols) and, with
// lcc, largest_connected_component (graph.cpp:118-171). Device inputs and outputs.
void ingest_graph(int64_t n, const int64_t* d_offs, const int32_t* d_cols, int64_t nnz_in, bool lcc,
                  IngestResult& out, cudaStream_t s);

} // namespace spb
