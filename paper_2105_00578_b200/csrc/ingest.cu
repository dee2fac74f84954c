// ingest.cu — graph ingestion on the device: what the
// reference's CLI runs on the host before partition_graph
// (tools/specpart.cpp:89-90, 104):
//   symmetrize                  graph.cpp:44-64   pattern of A + A^T, diagonal
//                                                 dropped, rows sorted, unit costs
//   largest_connected_component graph.cpp:118-171 union-find with component-minimum
//                                                 roots; ties -> smallest id; kept
//                                                 vertices keep their relative order
//   classify                    graph.cpp:173-182 (abi.cu, on the result)
//
// All integer work, HBM-bound, bit-exact by construction:
//   1. every stored entry (i, j), i != j, emits the two packed keys
//      (i << sh | j) and (j << sh | i) (sh = bit width of n-1); a diagonal entry
//      emits two copies of the sentinel key (all ones in 2·sh bits, never a valid
//      off-diagonal pair). Sorting the keys on 2·sh bits and dropping duplicates
//      is exactly from_triplets(sum_duplicates=false) (sparse.cpp:36-63): rows
//      ascending, columns strictly ascending within a row.
//   2. row offsets come from the row boundaries of the unique key array.
//   3. connected components: lock-free union-find over the upper triangle
//      (hook the larger root under the smaller with atomicCAS, path halving),
//      then full compression. Every parent pointer points to a smaller id of the
//      same component, so each component's root is its minimum vertex — the
//      reference's DisjointSets roots (graph.cpp:100-111), independent of the
//      order the hooks land in.
//   4. component sizes (atomics on integers), best root = max size, smallest
//      root among ties (graph.cpp:134-141) via one 64-bit atomicMax.
//   5. relabel: new id = exclusive scan of the keep flags (ascending old id, as
//      graph.cpp:143-150), offsets = scan of kept degrees, columns remapped per
//      entry (monotone map: rows stay sorted).
#include "context.hpp"
#include "ingest.hpp"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <bit>

namespace spb {

namespace {

__global__ void emit_pairs_kernel(int64_t n, const int64_t* __restrict__ offs, const int32_t* __restrict__ cols,
                                  int sh, uint64_t sentinel, uint64_t* __restrict__ keys, int* __restrict__ bad) {
    // one warp per row, lanes over the row's entries (raw inputs may have hub rows)
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        const int64_t k0 = offs[i], k1 = offs[i + 1];
        for (int64_t k = k0 + lane; k < k1; k += 32) {
            const int32_t j = cols[k];
            uint64_t a = sentinel, b = sentinel;
            if (j < 0 || j >= n) {
                atomicOr(bad, 1);
            } else if (j != i) {
                a = (static_cast<uint64_t>(i) << sh) | static_cast<uint64_t>(j);
                b = (static_cast<uint64_t>(j) << sh) | static_cast<uint64_t>(i);
            }
            keys[2 * k] = a;
            keys[2 * k + 1] = b;
        }
    }
}

// offs[r] = first k with row(key[k]) >= r, for r in [0, n]; cols[k] = col(key[k])
__global__ void csr_from_keys_kernel(int64_t nnz, int64_t n, const uint64_t* __restrict__ keys, int sh,
                                     int64_t* __restrict__ offs, int32_t* __restrict__ cols) {
    const uint64_t mask = (uint64_t(1) << sh) - 1;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k <= nnz;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = k < nnz ? static_cast<int64_t>(keys[k] >> sh) : n;
        const int64_t prev = k > 0 ? static_cast<int64_t>(keys[k - 1] >> sh) : -1;
        for (int64_t rr = prev + 1; rr <= r; ++rr) offs[rr] = k;
        if (k < nnz) cols[k] = static_cast<int32_t>(keys[k] & mask);
    }
}

__global__ void iota_i32_kernel(int64_t n, int32_t* p) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = static_cast<int32_t>(i);
}

// root of v with path halving; parent[x] <= x always holds
__device__ __forceinline__ int32_t find_root(volatile int32_t* parent, int32_t v) {
    int32_t cur = parent[v];
    if (cur == v) return v;
    int32_t prev = v, next;
    while (cur > (next = parent[cur])) {
        parent[prev] = next;
        prev = cur;
        cur = next;
    }
    return cur;
}

__global__ void hook_kernel(int64_t nnz, const uint64_t* __restrict__ keys, int sh, int32_t* parent) {
    const uint64_t mask = (uint64_t(1) << sh) - 1;
    volatile int32_t* vp = parent;
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t key = keys[k];
        const int32_t u = static_cast<int32_t>(key >> sh), v = static_cast<int32_t>(key & mask);
        if (v >= u) continue;  // each undirected edge once (the pattern is symmetric)
        int32_t ru = find_root(vp, u), rv = find_root(vp, v);
        while (ru != rv) {
            const int32_t hi = ru > rv ? ru : rv, lo = ru > rv ? rv : ru;
            const int32_t old = atomicCAS(parent + hi, hi, lo);
            if (old == hi) break;
            ru = find_root(vp, old);
            rv = find_root(vp, lo);
        }
    }
}

// full compression + component sizes
__global__ void compress_count_kernel(int64_t n, int32_t* parent, int32_t* size) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int32_t r = parent[i];
        while (parent[r] != r) r = parent[r];
        parent[i] = r;
        atomicAdd(size + r, 1);
    }
}

// best = max over roots of (size << 32 | ~root): largest component, smallest root among ties
__global__ void best_root_kernel(int64_t n, const int32_t* __restrict__ size, unsigned long long* best) {
    unsigned long long mine = 0;
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t s = size[r];
        if (s > 0) {
            const unsigned long long v = (static_cast<unsigned long long>(s) << 32) |
                                         (0xFFFFFFFFull - static_cast<unsigned long long>(r));
            mine = v > mine ? v : mine;
        }
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, mine, o);
        mine = x > mine ? x : mine;
    }
    if ((threadIdx.x & 31) == 0 && mine) atomicMax(best, mine);
}

__global__ void keep_flags_kernel(int64_t n, const int32_t* __restrict__ parent, int32_t best,
                                  const int64_t* __restrict__ offs, int32_t* __restrict__ keep,
                                  int64_t* __restrict__ kdeg) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const bool k = parent[i] == best;
        keep[i] = k ? 1 : 0;
        kdeg[i] = k ? offs[i + 1] - offs[i] : 0;
    }
}

// scatter: old_ids[new_id[i]] = i and the kept rows' offsets (kdeg scanned)
__global__ void relabel_rows_kernel(int64_t n, const int32_t* __restrict__ keep, const int32_t* __restrict__ new_id,
                                    const int64_t* __restrict__ koff, int64_t* __restrict__ old_ids,
                                    int64_t* __restrict__ offs_new, int64_t nnz_new, int64_t n_new) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (keep[i]) {
            old_ids[new_id[i]] = i;
            offs_new[new_id[i]] = koff[i];
        }
        if (i == 0) offs_new[n_new] = nnz_new;
    }
}

__global__ void remap_cols_kernel(int64_t nnz, const uint64_t* __restrict__ keys, int sh,
                                  const int64_t* __restrict__ offs, const int32_t* __restrict__ cols,
                                  const int32_t* __restrict__ keep, const int32_t* __restrict__ new_id,
                                  const int64_t* __restrict__ koff, int32_t* __restrict__ cols_new) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t u = static_cast<int64_t>(keys[k] >> sh);
        if (!keep[u]) continue;
        cols_new[koff[u] + (k - offs[u])] = new_id[cols[k]];
    }
}

__global__ void iota_i64_kernel(int64_t n, int64_t* p) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[i] = i;
}

template <class F> void cub_call(F&& f, DBuf<char>& temp, cudaStream_t) {
    size_t need = 0;
    SPB_CUDA(f(static_cast<void*>(nullptr), need));
    if (need > temp.n) temp.alloc(need);
    SPB_CUDA(f(static_cast<void*>(temp.p), need));
}

} // namespace

void ingest_graph(int64_t n, const int64_t* d_offs, const int32_t* d_cols, int64_t nnz_in, bool lcc,
                  IngestResult& out, cudaStream_t s) {
    if (n <= 0) throw_invalid(lcc ? "largest_connected_component: empty graph" : "symmetrize: empty matrix");
    if (n > 0x7FFFFFFF) throw_invalid("symmetrize: more than 2^31-1 vertices");
    const int sh = std::max(1, static_cast<int>(std::bit_width(static_cast<uint64_t>(n - 1))));
    const int end_bit = 2 * sh;
    const uint64_t sentinel = (end_bit >= 64) ? ~uint64_t(0) : ((uint64_t(1) << end_bit) - 1);
    const int64_t nk = 2 * nnz_in;
    DBuf<char> temp;

    // 1. emit + sort + unique
    DBuf<uint64_t> ka(std::max<int64_t>(nk, 1)), kb(std::max<int64_t>(nk, 1));
    DBuf<int> bad(1);
    DBuf<int64_t> nsel(1);
    SPB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    int64_t nuniq = 0;
    uint64_t last = 0;
    if (nk > 0) {
        emit_pairs_kernel<<<grid_for(n * 32, 256, 8), 256, 0, s>>>(n, d_offs, d_cols, sh, sentinel, ka.p, bad.p);
        SPB_LAUNCH_CHECK();
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, ka.p, kb.p, nk, 0, end_bit, s);
        }, temp, s);
        launch_counter() += (end_bit + 7) / 8 + 1;
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceSelect::Unique(t, b, kb.p, ka.p, nsel.p, nk, s);
        }, temp, s);
        launch_counter() += 2;
        SPB_CUDA(cudaMemcpyAsync(&nuniq, nsel.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    }
    int hbad = 0;
    SPB_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    if (hbad) throw_invalid("symmetrize: column index out of range");
    if (nuniq > 0) {
        SPB_CUDA(cudaMemcpyAsync(&last, ka.p + nuniq - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
    }
    kb.release();
    const int64_t nnz = nuniq - ((nuniq > 0 && last == sentinel) ? 1 : 0);

    // 2. CSR of the symmetrized pattern
    DBuf<int64_t> offs(n + 1);
    DBuf<int32_t> cols(std::max<int64_t>(nnz, 1));
    csr_from_keys_kernel<<<grid_for(nnz + 1, 256, 8), 256, 0, s>>>(nnz, n, ka.p, sh, offs.p, cols.p);
    SPB_LAUNCH_CHECK();

    out.n_sym = n;
    out.nnz_sym = nnz;
    if (!lcc) {
        out.n = n;
        out.nnz = nnz;
        out.offs = std::move(offs);
        out.cols = std::move(cols);
        out.old_ids.alloc(n);
        iota_i64_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, out.old_ids.p);
        SPB_LAUNCH_CHECK();
        return;
    }

    // 3-4. components, sizes, best root
    DBuf<int32_t> parent(n), size(n);
    DBuf<unsigned long long> best(1);
    iota_i32_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, parent.p);
    SPB_LAUNCH_CHECK();
    SPB_CUDA(cudaMemsetAsync(size.p, 0, sizeof(int32_t) * n, s));
    SPB_CUDA(cudaMemsetAsync(best.p, 0, sizeof(unsigned long long), s));
    if (nnz > 0) {
        hook_kernel<<<grid_for(nnz, 256, 8), 256, 0, s>>>(nnz, ka.p, sh, parent.p);
        SPB_LAUNCH_CHECK();
    }
    compress_count_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, parent.p, size.p);
    SPB_LAUNCH_CHECK();
    best_root_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, size.p, best.p);
    SPB_LAUNCH_CHECK();
    unsigned long long hb = 0;
    SPB_CUDA(cudaMemcpyAsync(&hb, best.p, sizeof(hb), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    const int64_t n_new = static_cast<int64_t>(hb >> 32);
    const int32_t root = static_cast<int32_t>(0xFFFFFFFFull - (hb & 0xFFFFFFFFull));
    out.components_root = root;

    if (n_new == n) {  // connected: the symmetrized graph itself
        out.n = n;
        out.nnz = nnz;
        out.offs = std::move(offs);
        out.cols = std::move(cols);
        out.old_ids.alloc(n);
        iota_i64_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, out.old_ids.p);
        SPB_LAUNCH_CHECK();
        return;
    }

    // 5. relabel
    DBuf<int32_t> keep(n), new_id(n);
    DBuf<int64_t> kdeg(n), koff(n + 1);
    keep_flags_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, parent.p, root, offs.p, keep.p, kdeg.p);
    SPB_LAUNCH_CHECK();
    size.release();
    cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, keep.p, new_id.p, n, s); },
             temp, s);
    cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, kdeg.p, koff.p, n, s); },
             temp, s);
    launch_counter() += 4;
    int64_t tail[2] = {0, 0};  // koff[n-1], kdeg[n-1]
    SPB_CUDA(cudaMemcpyAsync(&tail[0], koff.p + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaMemcpyAsync(&tail[1], kdeg.p + n - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    const int64_t nnz_new = tail[0] + tail[1];

    out.n = n_new;
    out.nnz = nnz_new;
    out.offs.alloc(n_new + 1);
    out.cols.alloc(std::max<int64_t>(nnz_new, 1));
    out.old_ids.alloc(n_new);
    relabel_rows_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, keep.p, new_id.p, koff.p, out.old_ids.p,
                                                            out.offs.p, nnz_new, n_new);
    SPB_LAUNCH_CHECK();
    if (nnz > 0) {
        remap_cols_kernel<<<grid_for(nnz, 256, 8), 256, 0, s>>>(nnz, ka.p, sh, offs.p, cols.p, keep.p, new_id.p,
                                                                koff.p, out.cols.p);
        SPB_LAUNCH_CHECK();
    }
}

} // namespace spb
