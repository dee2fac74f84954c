// relabel.cu — degree-descending vertex order for irregular (power-law) graphs.
//
// The binned SpMM on a power-law graph (spmm_vec.cu) gathers one X row per stored
// entry; with the R-MAT generator's random vertex labels those rows are scattered
// over the whole block, so every gather is a DRAM access (the block of a BASELINE
// R-MAT config is 134-400 MB, larger than the 126 MB L2). Most entries point at the
// few high-degree vertices, so numbering the vertices by descending degree packs
// the rows the gathers hit into the first few megabytes of every block, where they
// stay L2-resident. The solver runs in the new numbering; the initial block is
// generated in the reference's numbering and permuted in, and the eigenvectors are
// permuted back before the multi-jagged stage (which breaks coordinate ties by the
// original vertex id, partitioner.cpp:96-98) and the metrics. The LOBPCG result is
// the same up to rounding (the binned SpMM was already not in storage order).
#include "graph_dev.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

namespace spb {

namespace {

__global__ void deg_key_kernel(int64_t n, const int64_t* offs, uint32_t* key, int32_t* id) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        key[i] = static_cast<uint32_t>(offs[i + 1] - offs[i]);
        id[i] = static_cast<int32_t>(i);
    }
}

__global__ void inverse_kernel(int64_t n, const int32_t* perm, int32_t* inv, const int64_t* offs_old,
                               int64_t* len_new) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t o = perm[r];
        inv[o] = static_cast<int32_t>(r);
        len_new[r] = offs_old[o + 1] - offs_old[o];
    }
}

// new row r = old row perm[r], columns mapped old -> new (warp per row)
__global__ void relabel_rows_kernel(int64_t n, const int32_t* perm, const int32_t* inv, const int64_t* offs_old,
                                    const int32_t* cols_old, const double* vals_old, const int64_t* offs_new,
                                    int32_t* cols_new, double* vals_new) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t r = w0; r < n; r += nw) {
        const int64_t o = perm[r];
        const int64_t k0 = offs_old[o], len = offs_old[o + 1] - k0, d0 = offs_new[r];
        for (int64_t k = lane; k < len; k += 32) {
            cols_new[d0 + k] = inv[cols_old[k0 + k]];
            if (vals_old) vals_new[d0 + k] = vals_old[k0 + k];
        }
    }
}

template <bool OUT>
__global__ void permute_rows_kernel(int64_t n, int m, const int32_t* perm, View src, View dst) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * m;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = t / m;
        const int c = static_cast<int>(t - r * m);
        if (OUT) dst.at(perm[r], c) = src.at(r, c);  // new -> old
        else dst.at(r, c) = src.at(perm[r], c);      // old -> new
    }
}

template <class F> void cub_do(F&& f, DBuf<char>& temp) {
    size_t need = 0;
    SPB_CUDA(f(static_cast<void*>(nullptr), need));
    if (need > temp.n) temp.alloc(need);
    SPB_CUDA(f(static_cast<void*>(temp.p), need));
    launch_counter() += 4;
}

} // namespace

void relabel_by_degree(const DevGraph& g, DevGraph& out, Relabel& rl, cudaStream_t s) {
    const int64_t n = g.n_local, nnz = g.nnz_local;
    if (g.row0 != 0 || n != g.n_global) throw SpError(1, "relabel_by_degree: one-GPU graphs only");
    DBuf<uint32_t> k0(n), k1(n);
    DBuf<int32_t> v0(n);
    DBuf<char> temp;
    rl.perm.alloc(n);
    rl.inv.alloc(n);
    deg_key_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, g.offs.p, k0.p, v0.p);
    SPB_LAUNCH_CHECK();
    // descending degree, ties by ascending id (the radix sort is stable)
    const int bits = 32;
    cub_do([&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairsDescending(t, b, k0.p, k1.p, v0.p, rl.perm.p, n, 0, bits, s);
    }, temp);
    DBuf<int64_t> len(n + 1);
    SPB_CUDA(cudaMemsetAsync(len.p + n, 0, sizeof(int64_t), s));
    inverse_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, rl.perm.p, rl.inv.p, g.offs.p, len.p);
    SPB_LAUNCH_CHECK();
    out.offs.alloc(n + 1);
    cub_do([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, len.p, out.offs.p, n + 1, s); },
           temp);
    out.cols.alloc(std::max<int64_t>(nnz, 1));
    if (g.vals.p) out.vals.alloc(std::max<int64_t>(nnz, 1));
    else out.vals.release();
    relabel_rows_kernel<<<grid_for(n * 32, 256, 8), 256, 0, s>>>(n, rl.perm.p, rl.inv.p, g.offs.p, g.cols.p,
                                                                 g.vals.p, out.offs.p, out.cols.p, out.vals.p);
    SPB_LAUNCH_CHECK();
    out.n_global = out.n_local = n;
    out.nnz_global = out.nnz_local = nnz;
    out.row0 = 0;
    out.vw.release();
    out.vw_all.release();
    out.prepared = false;
    rl.on = true;
}

void permute_rows_in(const Relabel& rl, int64_t n, int m, const View& src_old, const View& dst_new, cudaStream_t s) {
    if (n <= 0 || m <= 0) return;
    permute_rows_kernel<false><<<grid_for(n * m, 256, 8), 256, 0, s>>>(n, m, rl.perm.p, src_old, dst_new);
    SPB_LAUNCH_CHECK();
}

void permute_rows_out(const Relabel& rl, int64_t n, int m, const View& src_new, const View& dst_old, cudaStream_t s) {
    if (n <= 0 || m <= 0) return;
    permute_rows_kernel<true><<<grid_for(n * m, 256, 8), 256, 0, s>>>(n, m, rl.perm.p, src_new, dst_old);
    SPB_LAUNCH_CHECK();
}

} // namespace spb
