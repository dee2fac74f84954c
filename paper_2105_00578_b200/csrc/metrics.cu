// metrics.cu — make_partition / cutsize / imbalance (src/graph.cpp:184-230) on the device.
//
// Exactness: part weights are sums over the part's vertices in ascending vertex
// order (the reference's loop order) — for unit or integer weights they are
// exact integer counts; otherwise a stable sort by part followed by one
// sequential sum per part reproduces the reference's order on one GPU. The cut
// counts each undirected edge once (j > i) with integer-exact accumulation for
// unit costs. imbalance() is evaluated on the host on the K part weights with
// the reference's formula and order.
#include "metrics.hpp"

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>

namespace spb {

namespace {

constexpr int kT = 256;

__global__ void validate_kernel(int64_t n, const int32_t* a, int64_t K, int* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (a[i] < 0 || a[i] >= K) atomicOr(bad, 1);
}

// per-CTA shared histogram (K <= 4096) then one global atomic per bin (exact)
__global__ void count_kernel(int64_t n, const int32_t* a, int64_t K, unsigned long long* cnt) {
    extern __shared__ unsigned int hist[];
    const bool local = K <= 4096;
    if (local) {
        for (int64_t k = threadIdx.x; k < K; k += blockDim.x) hist[k] = 0;
        __syncthreads();
    }
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (local) atomicAdd(hist + a[i], 1u);
        else atomicAdd(cnt + a[i], 1ull);
    }
    if (local) {
        __syncthreads();
        for (int64_t k = threadIdx.x; k < K; k += blockDim.x)
            if (hist[k]) atomicAdd(cnt + k, static_cast<unsigned long long>(hist[k]));
    }
}

__global__ void iota32_kernel(int64_t n, int32_t* v) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        v[i] = static_cast<int32_t>(i);
}

// one thread per part: sequential sum of its (vertex-ordered) weights
__global__ void part_sum_kernel(int64_t n, const int32_t* sorted_parts, const int32_t* sorted_vtx,
                                const double* w, int64_t K, double* out) {
    const int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (k >= K) return;
    // lower bound of part k in the sorted part array
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (sorted_parts[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    double s = 0.0;
    for (int64_t p = lo; p < n && sorted_parts[p] == k; ++p) s += w[sorted_vtx[p]];
    out[k] = s;
}

__global__ void cut_kernel(int64_t n, int64_t row0, const int64_t* offs, const int32_t* cols,
                           const double* vals, const int32_t* a_global, double* partial) {
    // warp per row, lanes over the row's entries (balanced on power-law rows;
    // unit costs make the sum an exact integer in any order)
    double s = 0.0;
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = warp0; i < n; i += nwarps) {
        const int64_t gi = row0 + i;
        const int32_t pi = a_global[gi];
        for (int64_t k = offs[i] + lane; k < offs[i + 1]; k += 32) {
            const int32_t j = cols[k];
            if (j > gi && a_global[j] != pi) s += vals ? vals[k] : 1.0;
        }
    }
    __shared__ double red[kT];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = kT / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void sum_kernel(const double* partial, int rows, double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double s = 0.0;
    for (int r = 0; r < rows; ++r) s += partial[r];
    out[0] = s;
}

} // namespace

PartitionMetrics make_partition_dev(sp_context* ctx, const DevGraph& g, const int32_t* a_global,
                                    int64_t K, bool doubled) {
    cudaStream_t s = ctx->stream;
    Comm& cm = ctx->comm;
    const int64_t n = g.n_local;
    const int32_t* a_local = a_global + g.row0;
    PartitionMetrics out;
    // validate ids (graph.cpp:215-218)
    DBuf<int> bad(1);
    SPB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    if (n > 0) {
        validate_kernel<<<grid_for(n, kT, 8), kT, 0, s>>>(n, a_local, K, bad.p);
        SPB_LAUNCH_CHECK();
    }
    int hbad = 0;
    SPB_CUDA(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    if (cm.active()) {
        DBuf<int64_t> t(1);
        int64_t v = hbad;
        SPB_CUDA(cudaMemcpyAsync(t.p, &v, sizeof(v), cudaMemcpyHostToDevice, s));
        cm.sum_i64(t.p, 1, s);
        SPB_CUDA(cudaMemcpyAsync(&v, t.p, sizeof(v), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        hbad = v != 0;
    }
    if (hbad) throw_invalid("make_partition: part id out of range");

    // part weights
    out.part_weights.assign(K, 0.0);
    if (g.unit_weights) {
        DBuf<unsigned long long> cnt(K);
        SPB_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * K, s));
        if (n > 0) {
            count_kernel<<<grid_for(n, kT, 2), kT, K <= 4096 ? sizeof(unsigned int) * K : 0, s>>>(n, a_local, K, cnt.p);
            SPB_LAUNCH_CHECK();
        }
        cm.sum_i64(reinterpret_cast<int64_t*>(cnt.p), static_cast<int>(K), s);
        std::vector<unsigned long long> h(K);
        SPB_CUDA(cudaMemcpyAsync(h.data(), cnt.p, sizeof(unsigned long long) * K, cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        for (int64_t k = 0; k < K; ++k) out.part_weights[k] = static_cast<double>(h[k]);
    } else {
        DBuf<int32_t> vin(std::max<int64_t>(n, 1)), vout(std::max<int64_t>(n, 1)), kout(std::max<int64_t>(n, 1));
        DBuf<double> pw(K);
        SPB_CUDA(cudaMemsetAsync(pw.p, 0, sizeof(double) * K, s));
        if (n > 0) {
            iota32_kernel<<<grid_for(n, kT, 8), kT, 0, s>>>(n, vin.p);
            size_t need = 0;
            SPB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need, a_local, kout.p, vin.p, vout.p, n, 0, 32, s));
            DBuf<char> tmp(need);
            SPB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, need, a_local, kout.p, vin.p, vout.p, n, 0, 32, s));
            launch_counter() += 6;
            part_sum_kernel<<<ceil_div(K, 128), 128, 0, s>>>(n, kout.p, vout.p, g.vw.p, K, pw.p);
            SPB_LAUNCH_CHECK();
        }
        cm.sum_small(pw.p, static_cast<int>(K), s);
        SPB_CUDA(cudaMemcpyAsync(out.part_weights.data(), pw.p, sizeof(double) * K, cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
    }
    for (double w : out.part_weights)
        if (w <= 0.0) throw_invalid("make_partition: empty part");

    out.cut = cutsize_dev(ctx, g, a_global, doubled);
    out.imbalance = imbalance_of(out.part_weights);
    return out;
}

// cutsize (graph.cpp:184-196): no validation of the ids, as in the reference
double cutsize_dev(sp_context* ctx, const DevGraph& g, const int32_t* a_global, bool doubled) {
    cudaStream_t s = ctx->stream;
    const int64_t n = g.n_local;
    const int grid = grid_for(std::max<int64_t>(n, 1), kT, 4);
    DBuf<double> part(grid), tot(1);
    cut_kernel<<<grid, kT, 0, s>>>(n, g.row0, g.offs.p, g.cols.p, g.unit_values ? nullptr : g.vals.p,
                                   a_global, part.p);
    SPB_LAUNCH_CHECK();
    sum_kernel<<<1, 32, 0, s>>>(part.p, grid, tot.p);
    SPB_LAUNCH_CHECK();
    ctx->comm.sum_small(tot.p, 1, s);
    double cut = 0.0;
    SPB_CUDA(cudaMemcpyAsync(&cut, tot.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    return doubled ? 2.0 * cut : cut;
}

// imbalance (graph.cpp:198-207)
double imbalance_of(const std::vector<double>& w) {
    if (w.empty()) throw_invalid("imbalance: no parts");
    double total = 0.0, maxw = 0.0;
    for (double x : w) {
        total += x;
        maxw = std::max(maxw, x);
    }
    if (total <= 0.0) throw_invalid("imbalance: total weight not positive");
    return maxw / (total / static_cast<double>(w.size()));
}

} // namespace spb
