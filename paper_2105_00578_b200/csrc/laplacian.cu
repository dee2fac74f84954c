// laplacian.cu — bit-exact Laplacian assembly on the device.
//
// Restates, as data-parallel kernels, build_combinatorial (src/laplacian.cpp:53-83),
// build_normalized (:85-127), build_degree (:129-144), make_operator /
// gershgorin_bound / extract_diag (:14-51) and Graph::weighted_degree
// (src/graph.cpp:15-20). Bit-exactness rules (SURVEY §7 hard part 5): per-row
// sums are sequential in storage order (one thread per row), products use
// __dmul_rn (no FMA), 1/sqrt uses IEEE __dsqrt_rn/__ddiv_rn, and the diagonal
// is inserted before the first column > i. The L structure is a pure function of
// A's: offsets_L[i] = offsets_A[i] + i.
#include "graph_dev.cuh"

#include <algorithm>

namespace spb {

namespace {

__global__ void degree_kernel(int64_t n, const int64_t* offs, const double* vals, double* deg,
                              int* nonunit) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k0 = offs[i], k1 = offs[i + 1];
        if (!vals) {
            deg[i] = static_cast<double>(k1 - k0);  // sum of 1.0s is exact
            if (k1 == k0) atomicOr(nonunit, 2);
            continue;
        }
        double s = 0.0;
        bool unit = true;
        for (int64_t k = k0; k < k1; ++k) {
            const double v = vals[k];
            s = __dadd_rn(s, v);
            unit &= (v == 1.0);
        }
        deg[i] = s;
        if (!unit) atomicOr(nonunit, 1);
        if (!(s > 0.0)) atomicOr(nonunit, 2);
    }
}

__global__ void max_degree_kernel(int64_t n, const int64_t* offs, unsigned long long* out) {
    unsigned long long best = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        best = max(best, static_cast<unsigned long long>(offs[i + 1] - offs[i]));
    for (int off = 16; off > 0; off >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, off));
    if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

__global__ void isd_kernel(int64_t n, const double* deg, double* isd, unsigned long long* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double d = deg[i];
        if (d <= 0.0) {
            atomicMin(bad, static_cast<unsigned long long>(i));
            isd[i] = 0.0;
        } else {
            isd[i] = __ddiv_rn(1.0, __dsqrt_rn(d));
        }
    }
}

// Explicit L_C / L_N rows. kind 0: combinatorial, 1: normalized.
__global__ void assemble_kernel(int kind, int64_t n, int64_t row0, const int64_t* offs,
                                const int32_t* cols, const double* vals, const double* deg,
                                const double* isd, int64_t* offs_L, int32_t* cols_L, double* vals_L) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k0 = offs[i], k1 = offs[i + 1];
        const int64_t gi = row0 + i;
        int64_t o = k0 + i;
        offs_L[i] = o;
        if (i == n - 1) offs_L[n] = k1 + n;
        const double dval = kind == 0 ? deg[i] : 1.0;
        const double isdi = kind == 1 ? isd[gi] : 0.0;
        bool placed = false;
        for (int64_t k = k0; k < k1; ++k) {
            const int32_t j = cols[k];
            if (!placed && j > gi) {
                cols_L[o] = static_cast<int32_t>(gi);
                vals_L[o] = dval;
                ++o;
                placed = true;
            }
            const double a = vals ? vals[k] : 1.0;
            cols_L[o] = j;
            vals_L[o] = kind == 0 ? -a : __dmul_rn(__dmul_rn(-a, isdi), isd[j]);
            ++o;
        }
        if (!placed) {
            cols_L[o] = static_cast<int32_t>(gi);
            vals_L[o] = dval;
        }
    }
}

// Gershgorin bound of an explicit CSR (laplacian.cpp:14-28) and its diagonal
// (:30-36): sequential per row, max over rows (exact, order-free).
__global__ void bound_diag_kernel(int64_t n, int64_t row0, const int64_t* offs,
                                  const int32_t* cols, const double* vals, double* diag,
                                  unsigned long long* bound_bits) {
    double best = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double dsum = 0.0, off = 0.0, dlast = 0.0;
        for (int64_t k = offs[i]; k < offs[i + 1]; ++k) {
            const double v = vals ? vals[k] : 1.0;
            if (cols[k] == row0 + i) {
                dsum = __dadd_rn(dsum, v);
                dlast = v;
            } else {
                off = __dadd_rn(off, fabs(v));
            }
        }
        diag[i] = dlast;
        best = fmax(best, __dadd_rn(dsum, off));
    }
    // non-negative doubles order like their bit patterns
    unsigned long long b = __double_as_longlong(best);
    for (int off = 16; off > 0; off >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, off));
    if ((threadIdx.x & 31) == 0) atomicMax(bound_bits, b);
}

// Gershgorin bound of the unit-cost L_N from the pattern (no materialization):
// row i = 1 + sum_k |(-1*isd_i)*isd_j| in storage order; the diagonal term is
// added first because gershgorin_bound keeps separate diag/off accumulators.
// Warp per row: the 32 lanes compute 32 consecutive terms in parallel (coalesced
// column loads, independent isd gathers), then every lane folds them into the
// row sum in storage order via shuffles, so power-law hub rows cost one
// shuffle+add per entry instead of one dependent memory latency.
__global__ void normal_bound_kernel(int64_t n, int64_t row0, const int64_t* offs,
                                    const int32_t* cols, const double* isd,
                                    unsigned long long* bound_bits) {
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    double best = 0.0;
    for (int64_t i = warp0; i < n; i += nwarps) {
        const double nisdi = -isd[row0 + i];
        const int64_t k0 = offs[i], k1 = offs[i + 1];
        double off = 0.0;
        // the next 32 terms are loaded while the current ones are folded in; full
        // groups issue their 32 shuffles back to back so only the adds form the chain
        double term = (k0 + lane < k1) ? fabs(__dmul_rn(nisdi, isd[cols[k0 + lane]])) : 0.0;
        for (int64_t kb = k0; kb < k1; kb += 32) {
            const int cnt = static_cast<int>(min(static_cast<int64_t>(32), k1 - kb));
            const int64_t kn = kb + 32 + lane;
            const double next = kn < k1 ? fabs(__dmul_rn(nisdi, isd[cols[kn]])) : 0.0;
            if (cnt == 32) {
                double t[32];
#pragma unroll
                for (int q = 0; q < 32; ++q) t[q] = __shfl_sync(0xffffffffu, term, q);
#pragma unroll
                for (int q = 0; q < 32; ++q) off = __dadd_rn(off, t[q]);
            } else {
                for (int q = 0; q < cnt; ++q) off = __dadd_rn(off, __shfl_sync(0xffffffffu, term, q));
            }
            term = next;
        }
        best = fmax(best, __dadd_rn(1.0, off));
    }
    unsigned long long b = __double_as_longlong(best);
    for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    if (lane == 0) atomicMax(bound_bits, b);
}

__global__ void max_value_kernel(int64_t n, const double* v, unsigned long long* bits) {
    double best = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        best = fmax(best, v[i]);
    unsigned long long b = __double_as_longlong(best);
    for (int off = 16; off > 0; off >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, off));
    if ((threadIdx.x & 31) == 0) atomicMax(bits, b);
}

__global__ void fill_const_kernel(int64_t n, double* out, double v) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = v;
}

// Jacobi inverse diagonal (preconditioners.cpp:44-49)
__global__ void inv_diag_kernel(int64_t n, const double* d, double* inv) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        inv[i] = fabs(d[i]) < 1e-300 ? 1.0 : __ddiv_rn(1.0, d[i]);
}

__global__ void collect_long_rows_kernel(int64_t n, const int64_t* offs, int64_t thr, int32_t* out,
                                         unsigned long long* count) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (offs[i + 1] - offs[i] > thr) out[atomicAdd(count, 1ull)] = static_cast<int32_t>(i);
}

int g1(int64_t n) { return grid_for(n, 256, 8); }

} // namespace

void graph_degrees(DevGraph& g, cudaStream_t s) {
    g.deg.alloc(std::max<int64_t>(g.n_local, 1));
    DBuf<int> flag(1);
    SPB_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), s));
    degree_kernel<<<g1(g.n_local), 256, 0, s>>>(g.n_local, g.offs.p, g.vals.p, g.deg.p, flag.p);
    SPB_LAUNCH_CHECK();
    DBuf<unsigned long long> md(1);
    SPB_CUDA(cudaMemsetAsync(md.p, 0, sizeof(unsigned long long), s));
    max_degree_kernel<<<g1(g.n_local), 256, 0, s>>>(g.n_local, g.offs.p, md.p);
    SPB_LAUNCH_CHECK();
    int nonunit = 0;
    unsigned long long maxdeg = 0;
    SPB_CUDA(cudaMemcpyAsync(&nonunit, flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaMemcpyAsync(&maxdeg, md.p, sizeof(maxdeg), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    g.unit_values = (g.vals.p == nullptr) || (nonunit & 1) == 0;
    g.positive_degrees_local = (nonunit & 2) == 0;
    g.max_degree_local = static_cast<int64_t>(maxdeg);
}

void collect_long_rows(const DevGraph& g, DevLaplacian& L, int64_t threshold, cudaStream_t s) {
    L.long_rows.alloc(std::max<int64_t>(g.n_local, 1));
    DBuf<unsigned long long> cnt(1);
    SPB_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), s));
    collect_long_rows_kernel<<<g1(g.n_local), 256, 0, s>>>(g.n_local, g.offs.p, threshold,
                                                           L.long_rows.p, cnt.p);
    SPB_LAUNCH_CHECK();
    unsigned long long c = 0;
    SPB_CUDA(cudaMemcpyAsync(&c, cnt.p, sizeof(c), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    if (c > 1) {
        // atomics leave the list in arbitrary order: sort it so the partial-sum
        // layout (and hence every reduction) is identical run to run
        std::vector<int32_t> h(c);
        SPB_CUDA(cudaMemcpyAsync(h.data(), L.long_rows.p, sizeof(int32_t) * c, cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        std::sort(h.begin(), h.end());
        SPB_CUDA(cudaMemcpyAsync(L.long_rows.p, h.data(), sizeof(int32_t) * c, cudaMemcpyHostToDevice, s));
    }
    L.op.long_rows = L.long_rows.p;
    L.op.n_long = static_cast<int64_t>(c);
    L.op.long_threshold = threshold;
}

void build_laplacian(int kind, const DevGraph& g, bool materialize, DevLaplacian& L, cudaStream_t s) {
    const int64_t n = g.n_local;
    L.kind = kind;
    L.op = DevOp{};
    L.op.n = n;
    L.op.row0 = g.row0;
    L.op.x_rows = g.n_global;
    L.op.long_threshold = int64_t(1) << 40;
    L.diag.alloc(std::max<int64_t>(n, 1));
    DBuf<unsigned long long> bb(1);
    SPB_CUDA(cudaMemsetAsync(bb.p, 0, sizeof(unsigned long long), s));

    if (kind == 2) {  // build_degree: diagonal operator of weighted degrees
        SPB_CUDA(cudaMemcpyAsync(L.diag.p, g.deg.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        L.op.mode = OP_DIAGONAL;
        L.op.diag = L.diag.p;
        L.op.is_diagonal = true;
        L.op.nnz = n;
        L.op.max_row = 1;
        if (materialize) {
            // the diagonal CSR: offsets i, cols i, vals deg (laplacian.cpp:134-143)
            L.offs_L.alloc(n + 1);
            L.cols_L.alloc(std::max<int64_t>(n, 1));
            L.vals_L.alloc(std::max<int64_t>(n, 1));
            std::vector<int64_t> ho(n + 1);
            std::vector<int32_t> hc(std::max<int64_t>(n, 1));
            for (int64_t i = 0; i <= n; ++i) ho[i] = i;
            for (int64_t i = 0; i < n; ++i) hc[i] = static_cast<int32_t>(g.row0 + i);
            SPB_CUDA(cudaMemcpyAsync(L.offs_L.p, ho.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
            SPB_CUDA(cudaMemcpyAsync(L.cols_L.p, hc.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s));
            SPB_CUDA(cudaMemcpyAsync(L.vals_L.p, g.deg.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
        }
        // Gershgorin of a diagonal operator: max_i (d_i + 0); degrees are >= 0
        max_value_kernel<<<g1(n), 256, 0, s>>>(n, g.deg.p, bb.p);
        SPB_LAUNCH_CHECK();
        unsigned long long bits = 0;
        SPB_CUDA(cudaMemcpyAsync(&bits, bb.p, sizeof(bits), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        std::memcpy(&L.op.bound, &bits, sizeof(bits));
        return;
    }

    if (kind == 1) {
        L.isd.alloc(std::max<int64_t>(g.n_global, 1));
        DBuf<unsigned long long> bad(1);
        const unsigned long long none = ~0ull;
        SPB_CUDA(cudaMemcpyAsync(bad.p, &none, sizeof(none), cudaMemcpyHostToDevice, s));
        // isd over GLOBAL vertices (the kernel gathers isd_j for halo columns)
        isd_kernel<<<g1(g.n_global), 256, 0, s>>>(g.n_global, g.deg_global(), L.isd.p, bad.p);
        SPB_LAUNCH_CHECK();
        unsigned long long first_bad = 0;
        SPB_CUDA(cudaMemcpyAsync(&first_bad, bad.p, sizeof(first_bad), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        if (first_bad != none)
            throw_degenerate("normalized Laplacian requires degree >= 1 at vertex " +
                             std::to_string(first_bad));
    }

    const bool pattern_ok = g.unit_values && !materialize;
    if (materialize || !g.unit_values) {
        const int64_t nnzL = g.nnz_local + n;
        L.offs_L.alloc(n + 1);
        L.cols_L.alloc(std::max<int64_t>(nnzL, 1));
        L.vals_L.alloc(std::max<int64_t>(nnzL, 1));
        if (n > 0) {
            assemble_kernel<<<g1(n), 256, 0, s>>>(kind, n, g.row0, g.offs.p, g.cols.p, g.vals.p,
                                                  g.deg.p, kind == 1 ? L.isd.p : nullptr,
                                                  L.offs_L.p, L.cols_L.p, L.vals_L.p);
            SPB_LAUNCH_CHECK();
        }
        // offsets of a row block are relative to the block
        bound_diag_kernel<<<g1(n), 256, 0, s>>>(n, g.row0, L.offs_L.p, L.cols_L.p, L.vals_L.p,
                                                L.diag.p, bb.p);
        SPB_LAUNCH_CHECK();
        L.op.mode = OP_EXPLICIT;
        L.op.offs = L.offs_L.p;
        L.op.cols = L.cols_L.p;
        L.op.vals = L.vals_L.p;
        L.op.nnz = nnzL;
        L.op.max_row = static_cast<int>(std::min<int64_t>(g.max_degree_local + 1, 1 << 30));
    }
    if (pattern_ok) {
        L.op.offs = g.offs.p;
        L.op.cols = g.cols.p;
        L.op.nnz = g.nnz_local;
        L.op.max_row = static_cast<int>(std::min<int64_t>(g.max_degree_local, 1 << 30));
        if (kind == 0) {
            L.op.mode = OP_LAPLACE_UNIT;
            SPB_CUDA(cudaMemcpyAsync(L.diag.p, g.deg.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
            // Gershgorin row bound deg + sum|-1| = 2*deg exactly (integers)
            L.op.bound = 2.0 * static_cast<double>(g.max_degree_global);
        } else {
            L.op.mode = OP_NORMAL_UNIT;
            fill_const_kernel<<<g1(n), 256, 0, s>>>(n, L.diag.p, 1.0);
            SPB_LAUNCH_CHECK();
            normal_bound_kernel<<<g1(n), 256, 0, s>>>(n, g.row0, g.offs.p, g.cols.p, L.isd.p, bb.p);
            SPB_LAUNCH_CHECK();
        }
    }
    L.op.diag = L.diag.p;
    L.op.isd = L.isd.p;
    if (!(pattern_ok && kind == 0)) {
        unsigned long long bits = 0;
        SPB_CUDA(cudaMemcpyAsync(&bits, bb.p, sizeof(bits), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        std::memcpy(&L.op.bound, &bits, sizeof(bits));
    }
    if (kind == 1) L.op.bound = std::min(L.op.bound, 2.0);  // laplacian.cpp:124-125
    L.op.is_diagonal = (g.nnz_global == 0);  // nnz == nrows with only diagonal entries
}

void inverse_diagonal(const DevLaplacian& L, DBuf<double>& inv, cudaStream_t s) {
    inv.alloc(std::max<int64_t>(L.op.n, 1));
    inv_diag_kernel<<<g1(L.op.n), 256, 0, s>>>(L.op.n, L.diag.p, inv.p);
    SPB_LAUNCH_CHECK();
}

} // namespace spb
