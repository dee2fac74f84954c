// amg.cu — aggregation AMG preconditioner (preconditioners.cpp:384-728) on the device.
//
// Setup, level by level (AmgPreconditionerImpl::build, :567-650):
//   strength graph        device (count + fill kernels, |a_ij| >= tol sqrt|a_ii a_jj|)
//   greedy aggregation    host: the reference's pass order (roots in ascending id, then
//                         leftovers, then singletons) is inherently sequential — the result
//                         depends on the visiting order — so it runs as one O(nnz) host pass
//                         over the downloaded strength pattern; everything else is on the GPU
//   tentative P           device (1/sqrt(|aggregate|))
//   lambda_max(D^-1 A)    device power iteration from the reference's seeded mt19937_64 vector
//   smoothed P, P^T,      device expand-sort-reduce: products keyed (row, col) in 64 bits,
//   A P, P^T (A P)        CUB radix sort (stable) + reduce-by-key, row-batched to bound memory
//   coarse direct solve   host Cholesky of the <= coarse_size_threshold dense matrix with the
//                         reference's shift escalation (:619-633); its inverse is applied on
//                         the device
// Apply (vcycle, :667-706): Chebyshev pre-smoothing from zero, residual, restriction,
// recursion, prolongation, residual, Chebyshev post-smoothing — every product a device SpMM
// (level 0 through the solver's own fine-grid kernels), every update a fused vector kernel.
// Numerically equivalent to the reference, not bit-identical (its spgemm and std::sort-based
// triplet merge fix a different summation order).
#include "amg.hpp"

#include "dense_host.hpp"

#include <cub/cub.cuh>
#include <cuda/std/functional>

#include <algorithm>
#include <bit>
#include <cmath>

namespace spb {

AmgCfg AmgCfg::regular_defaults() {
    AmgCfg c;  // preconditioners.cpp:24-31
    c.smoothed = true;
    c.drop_tol = 0.0;
    c.max_levels = 20;
    c.coarse_direct = true;
    return c;
}

AmgCfg AmgCfg::irregular_defaults() {
    AmgCfg c;  // preconditioners.cpp:33-40
    c.smoothed = false;
    c.drop_tol = 0.4;
    c.max_levels = 5;
    c.coarse_direct = false;
    return c;
}

DevOp CsrDev::op() const {
    DevOp o;
    o.mode = OP_EXPLICIT;
    o.n = nrows;
    o.nnz = nnz;
    o.offs = offs.p;
    o.cols = cols.p;
    o.vals = vals.p;
    o.long_threshold = int64_t(1) << 40;
    o.max_row = max_row;
    o.x_rows = ncols;
    return o;
}

std::vector<int32_t> greedy_aggregate(int64_t n, const std::vector<int64_t>& offs, const std::vector<int32_t>& cols,
                                      int64_t& num_aggregates) {
    std::vector<int32_t> agg(static_cast<size_t>(n), -1);
    int32_t next = 0;
    // pass 1: a vertex none of whose strong neighbours is aggregated roots a new
    // aggregate and absorbs them
    for (int64_t i = 0; i < n; ++i) {
        if (agg[i] != -1) continue;
        bool free_nbhd = true;
        for (int64_t k = offs[i]; k < offs[i + 1]; ++k)
            if (agg[cols[k]] != -1) {
                free_nbhd = false;
                break;
            }
        if (!free_nbhd) continue;
        agg[i] = next;
        for (int64_t k = offs[i]; k < offs[i + 1]; ++k) agg[cols[k]] = next;
        ++next;
    }
    // pass 2: leftovers join the aggregate of their first aggregated strong neighbour
    for (int64_t i = 0; i < n; ++i) {
        if (agg[i] != -1) continue;
        for (int64_t k = offs[i]; k < offs[i + 1]; ++k)
            if (agg[cols[k]] != -1) {
                agg[i] = agg[cols[k]];
                break;
            }
    }
    // pass 3: isolated leftovers become singletons
    for (int64_t i = 0; i < n; ++i)
        if (agg[i] == -1) agg[i] = next++;
    num_aggregates = next;
    return agg;
}

namespace {

constexpr int kT = 256;
int g1(int64_t n) { return grid_for(n, kT, 8); }

template <class F> void cub_run(F&& f, DBuf<char>& temp) {
    size_t need = 0;
    SPB_CUDA(f(static_cast<void*>(nullptr), need));
    if (need > temp.n) temp.alloc(need);
    SPB_CUDA(f(static_cast<void*>(temp.p), need));
    launch_counter() += 4;
}

// inverse_diagonal (preconditioners.cpp:44-49) + extract_diag (laplacian.cpp:30-36)
__global__ void diag_kernel(int64_t n, const int64_t* offs, const int32_t* cols, const double* vals, double* d,
                            double* inv) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double v = 0.0;
        for (int64_t k = offs[i]; k < offs[i + 1]; ++k)
            if (cols[k] == i) v = vals[k];
        d[i] = v;
        inv[i] = fabs(v) < 1e-300 ? 1.0 : 1.0 / v;
    }
}

// strength_graph (preconditioners.cpp:389-407)
__device__ __forceinline__ bool strong(int64_t i, int32_t j, double a, const double* d, double tol) {
    return j != i && fabs(a) >= tol * sqrt(fabs(d[i] * d[j]));
}
__global__ void strength_count_kernel(int64_t n, const int64_t* offs, const int32_t* cols, const double* vals,
                                      const double* d, double tol, int64_t* cnt) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t c = 0;
        for (int64_t k = offs[i]; k < offs[i + 1]; ++k) c += strong(i, cols[k], vals[k], d, tol) ? 1 : 0;
        cnt[i] = c;
    }
}
__global__ void strength_fill_kernel(int64_t n, const int64_t* offs, const int32_t* cols, const double* vals,
                                     const double* d, double tol, const int64_t* soffs, int32_t* scols) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int64_t o = soffs[i];
        for (int64_t k = offs[i]; k < offs[i + 1]; ++k)
            if (strong(i, cols[k], vals[k], d, tol)) scols[o++] = cols[k];
    }
}

// tentative_prolongator (preconditioners.cpp:452-470)
__global__ void agg_count_kernel(int64_t n, const int32_t* agg, int* cnt) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        atomicAdd(cnt + agg[i], 1);
}
__global__ void ptent_kernel(int64_t n, const int32_t* agg, const int* cnt, int64_t* poffs, int32_t* pcols,
                             double* pvals) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        poffs[i] = i;
        if (i < n) {
            pcols[i] = agg[i];
            pvals[i] = 1.0 / sqrt(static_cast<double>(cnt[agg[i]]));
        }
    }
}

// P = P_tent - omega D^{-1} A P_tent (:590-610): row i emits (agg[i], p_i) then, per
// stored a_ij, (agg[j], -omega inv_i a_ij p_j); warp per row
__global__ void smooth_expand_kernel(int64_t n, const int64_t* offs, const int32_t* cols, const double* vals,
                                     const double* inv, const int32_t* agg, const double* pt, double omega,
                                     int64_t nc, uint64_t* keys, double* out) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = w0; i < n; i += nw) {
        const int64_t base = offs[i] + i;
        const double sc = -omega * inv[i];
        if (lane == 0) {
            keys[base] = static_cast<uint64_t>(i) * nc + agg[i];
            out[base] = pt[i];
        }
        for (int64_t k = offs[i] + lane; k < offs[i + 1]; k += 32) {
            const int32_t j = cols[k];
            keys[base + 1 + (k - offs[i])] = static_cast<uint64_t>(i) * nc + agg[j];
            out[base + 1 + (k - offs[i])] = sc * (vals[k] * pt[j]);
        }
    }
}

// plain_galerkin (:478-520): every a_ij lands in (agg[i], agg[j])
__global__ void plain_expand_kernel(int64_t n, const int64_t* offs, const int32_t* cols, const double* vals,
                                    const int32_t* agg, int64_t nc, uint64_t* keys, double* out) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = w0; i < n; i += nw)
        for (int64_t k = offs[i] + lane; k < offs[i + 1]; k += 32) {
            keys[k] = static_cast<uint64_t>(agg[i]) * nc + agg[cols[k]];
            out[k] = vals[k];
        }
}
__global__ void plain_scale_kernel(int64_t nnz, const uint64_t* keys, int64_t nc, const int* cnt, double* vals) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nnz;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t I = static_cast<int64_t>(keys[e] / nc), J = static_cast<int64_t>(keys[e] % nc);
        vals[e] = vals[e] / sqrt(static_cast<double>(cnt[I])) / sqrt(static_cast<double>(cnt[J]));
    }
}

// transpose (sparse.cpp:67-87): key (col, row) per entry
__global__ void transpose_expand_kernel(int64_t n, const int64_t* offs, const int32_t* cols, const double* vals,
                                        int64_t nrows_out_stride, uint64_t* keys, double* out) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = w0; i < n; i += nw)
        for (int64_t k = offs[i] + lane; k < offs[i + 1]; k += 32) {
            keys[k] = static_cast<uint64_t>(cols[k]) * nrows_out_stride + i;
            out[k] = vals[k];
        }
}

// row-wise SpGEMM C = A B, expand step for rows [r0, r1): entry e of row i emits
// a_e * B(j, :) at pre[e] - p0 onward, keys (i - r0, col)
__global__ void entry_count_kernel(int64_t nnz, const int32_t* acols, const int64_t* boffs, int64_t* cnt) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e <= nnz;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        cnt[e] = e < nnz ? boffs[acols[e] + 1] - boffs[acols[e]] : 0;
}
__global__ void row_pre_kernel(int64_t n, const int64_t* aoffs, const int64_t* pre, int64_t* rpre) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i <= n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        rpre[i] = pre[aoffs[i]];
}
__global__ void spgemm_expand_kernel(int64_t r0, int64_t r1, const int64_t* aoffs, const int32_t* acols,
                                     const double* avals, const int64_t* boffs, const int32_t* bcols,
                                     const double* bvals, const int64_t* pre, int64_t p0, int64_t ncols,
                                     uint64_t* keys, double* out) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
    for (int64_t i = r0 + w0; i < r1; i += nw)
        for (int64_t e = aoffs[i] + lane; e < aoffs[i + 1]; e += 32) {
            const int32_t j = acols[e];
            const double a = avals[e];
            int64_t o = pre[e] - p0;
            const uint64_t rk = static_cast<uint64_t>(i - r0) * ncols;
            for (int64_t t = boffs[j]; t < boffs[j + 1]; ++t, ++o) {
                keys[o] = rk + bcols[t];
                out[o] = a * bvals[t];
            }
        }
}

// sorted unique keys (row * ncols + col) -> CSR columns / offsets of rows [0, nrows)
__global__ void keys_cols_kernel(int64_t nu, const uint64_t* keys, int64_t ncols, int32_t* cols) {
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < nu;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x)
        cols[e] = static_cast<int32_t>(keys[e] % ncols);
}
__global__ void keys_offs_kernel(int64_t nrows, int64_t nu, const uint64_t* keys, int64_t ncols, int64_t base,
                                 int64_t* offs) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r <= nrows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t k = static_cast<uint64_t>(r) * ncols;
        int64_t lo = 0, hi = nu;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < k) lo = mid + 1;
            else hi = mid;
        }
        offs[r] = base + lo;
    }
}
__global__ void max_row_kernel(int64_t n, const int64_t* offs, int* mx) {
    int m = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t len = offs[i + 1] - offs[i];
        m = max(m, static_cast<int>(len < (1 << 30) ? len : (1 << 30)));
    }
    atomicMax(mx, m);
}

// ---- V-cycle vector kernels (column-major or row-major views, rows x k) ----
// chebyshev_solve (:115-156): dir = inv_d rhs / theta, Z = dir
__global__ void cheb_init_kernel(int64_t n, int k, const double* inv, View rhs, View dir, View z, double theta) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = t % n;
        const int c = static_cast<int>(t / n);
        const double d = inv[i] * rhs.at(i, c) / theta;
        dir.at(i, c) = d;
        z.at(i, c) = d;
    }
}
// dir = c1 dir + c2 inv_d (rhs - AZ); Z += dir
__global__ void cheb_step_kernel(int64_t n, int k, const double* inv, View rhs, View az, View dir, View z, double c1,
                                 double c2) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = t % n;
        const int c = static_cast<int>(t / n);
        const double r = rhs.at(i, c) - az.at(i, c);
        const double d = c1 * dir.at(i, c) + c2 * inv[i] * r;
        dir.at(i, c) = d;
        z.at(i, c) += d;
    }
}
__global__ void sub_kernel(int64_t n, int k, View a, View b, View out) {  // out = a - b
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = t % n;
        const int c = static_cast<int>(t / n);
        out.at(i, c) = a.at(i, c) - b.at(i, c);
    }
}
__global__ void add_kernel(int64_t n, int k, View z, View d) {  // z += d
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n * k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = t % n;
        const int c = static_cast<int>(t / n);
        z.at(i, c) += d.at(i, c);
    }
}
// y(i, :) (+)= sum_e v_e x(col_e, :) for a rectangular CSR (P, P^T); thread per (row, column)
template <bool ADD>
__global__ void rect_spmm_kernel(int64_t nrows, int k, const int64_t* offs, const int32_t* cols, const double* vals,
                                 View x, View y) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nrows * k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = t % nrows;
        const int c = static_cast<int>(t / nrows);
        double acc = 0.0;
        for (int64_t e = offs[i]; e < offs[i + 1]; ++e) acc += vals[e] * x.at(cols[e], c);
        if (ADD) y.at(i, c) += acc;
        else y.at(i, c) = acc;
    }
}
// coarse direct solve: Z = Ainv rhs (dense nc x nc, column-major)
__global__ void dense_apply_kernel(int64_t nc, int k, const double* ainv, View rhs, View z) {
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nc * k;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = t % nc;
        const int c = static_cast<int>(t / nc);
        double acc = 0.0;
        for (int64_t j = 0; j < nc; ++j) acc += ainv[j * nc + i] * rhs.at(j, c);
        z.at(i, c) = acc;
    }
}
// power iteration helpers: w *= inv_d with per-CTA sums of squares (fixed order)
__global__ void scale_sq_kernel(int64_t n, View w, const double* inv, double* part) {
    __shared__ double red[kT];
    double s = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = w.at(i, 0) * inv[i];
        w.at(i, 0) = v;
        s += v * v;
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int h = kT / 2; h > 0; h >>= 1) {
        if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void div_kernel(int64_t n, View in, View out, double d) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out.at(i, 0) = in.at(i, 0) / d;
}

// expand-sort-reduce into a CSR (nrows x ncols); keys are row * ncols + col (rows
// relative to the batch), summed in expansion order (stable radix sort)
struct Esc {
    DBuf<char> temp;
    DBuf<uint64_t> k0, k1;
    DBuf<double> v0, v1;
    DBuf<int64_t> nrun;
    void reserve(int64_t cnt) {
        k0.alloc(std::max<int64_t>(cnt, 1));
        k1.alloc(std::max<int64_t>(cnt, 1));
        v0.alloc(std::max<int64_t>(cnt, 1));
        v1.alloc(std::max<int64_t>(cnt, 1));
        nrun.alloc(1);
    }
    // sorts k0/v0[0, cnt) and reduces runs into k0/v0; returns the run count
    int64_t sort_reduce(int64_t cnt, uint64_t max_key, cudaStream_t s) {
        if (cnt == 0) return 0;
        const int end_bit = std::max(1, static_cast<int>(std::bit_width(max_key)));
        cub_run([&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(t, b, k0.p, k1.p, v0.p, v1.p, cnt, 0, end_bit, s);
        }, temp);
        cub_run([&](void* t, size_t& b) {
            return cub::DeviceReduce::ReduceByKey(t, b, k1.p, k0.p, v1.p, v0.p, nrun.p, ::cuda::std::plus<double>(),
                                                  cnt, s);
        }, temp);
        int64_t nu = 0;
        SPB_CUDA(cudaMemcpyAsync(&nu, nrun.p, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        return nu;
    }
};

// batch results appended into one CSR
struct CsrBuilder {
    std::vector<DBuf<int32_t>> cols;
    std::vector<DBuf<double>> vals;
    std::vector<int64_t> cnt;
    DBuf<int64_t> offs;
    int64_t nnz = 0;
    void finish(CsrDev& out, int64_t nrows, int64_t ncols, cudaStream_t s) {
        out.nrows = nrows;
        out.ncols = ncols;
        out.nnz = nnz;
        out.offs = std::move(offs);
        out.cols.alloc(std::max<int64_t>(nnz, 1));
        out.vals.alloc(std::max<int64_t>(nnz, 1));
        int64_t o = 0;
        for (size_t b = 0; b < cols.size(); ++b) {
            if (cnt[b]) {
                SPB_CUDA(cudaMemcpyAsync(out.cols.p + o, cols[b].p, sizeof(int32_t) * cnt[b], cudaMemcpyDeviceToDevice, s));
                SPB_CUDA(cudaMemcpyAsync(out.vals.p + o, vals[b].p, sizeof(double) * cnt[b], cudaMemcpyDeviceToDevice, s));
            }
            o += cnt[b];
        }
        DBuf<int> mx(1);
        SPB_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(int), s));
        max_row_kernel<<<g1(nrows), kT, 0, s>>>(nrows, out.offs.p, mx.p);
        SPB_LAUNCH_CHECK();
        SPB_CUDA(cudaMemcpyAsync(&out.max_row, mx.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        cols.clear();
        vals.clear();
    }
};

// the sorted unique keys of rows [r0, r0 + rows) -> CSR pieces
void append_rows(Esc& e, int64_t nu, int64_t r0, int64_t rows, int64_t ncols, CsrBuilder& cb, cudaStream_t s) {
    keys_offs_kernel<<<g1(rows + 1), kT, 0, s>>>(rows, nu, e.k0.p, ncols, cb.nnz, cb.offs.p + r0);
    SPB_LAUNCH_CHECK();
    DBuf<int32_t> c(std::max<int64_t>(nu, 1));
    DBuf<double> v(std::max<int64_t>(nu, 1));
    if (nu) {
        keys_cols_kernel<<<g1(nu), kT, 0, s>>>(nu, e.k0.p, ncols, c.p);
        SPB_LAUNCH_CHECK();
        SPB_CUDA(cudaMemcpyAsync(v.p, e.v0.p, sizeof(double) * nu, cudaMemcpyDeviceToDevice, s));
    }
    cb.cols.push_back(std::move(c));
    cb.vals.push_back(std::move(v));
    cb.cnt.push_back(nu);
    cb.nnz += nu;
}

constexpr int64_t kBatchProducts = int64_t(1) << 27;  // 2 GB of (key, value) pairs per batch

// C = A B (row-wise expand-sort-reduce, rows batched by product count)
void spgemm(const CsrDev& A, const CsrDev& B, CsrDev& C, cudaStream_t s) {
    const int64_t m = A.nrows, nnz = A.nnz;
    DBuf<int64_t> pre(nnz + 1), rpre(m + 1);
    DBuf<char> temp;
    entry_count_kernel<<<g1(nnz + 1), kT, 0, s>>>(nnz, A.cols.p, B.offs.p, pre.p);
    SPB_LAUNCH_CHECK();
    cub_run([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, pre.p, pre.p, nnz + 1, s); }, temp);
    row_pre_kernel<<<g1(m + 1), kT, 0, s>>>(m, A.offs.p, pre.p, rpre.p);
    SPB_LAUNCH_CHECK();
    std::vector<int64_t> hr(static_cast<size_t>(m + 1));
    SPB_CUDA(cudaMemcpyAsync(hr.data(), rpre.p, sizeof(int64_t) * (m + 1), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    CsrBuilder cb;
    cb.offs.alloc(m + 1);
    Esc e;
    int64_t r0 = 0;
    while (r0 < m) {
        int64_t r1 = r0 + 1;
        // grow the batch while it stays under the product budget (a single row may exceed it)
        {
            int64_t lo = r0 + 1, hi = m;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (hr[mid] - hr[r0] <= kBatchProducts) lo = mid;
                else hi = mid - 1;
            }
            r1 = lo;
        }
        const int64_t cnt = hr[r1] - hr[r0];
        e.reserve(cnt);
        if (cnt) {
            spgemm_expand_kernel<<<grid_for((r1 - r0) * 32, kT, 8), kT, 0, s>>>(
                r0, r1, A.offs.p, A.cols.p, A.vals.p, B.offs.p, B.cols.p, B.vals.p, pre.p, hr[r0], B.ncols, e.k0.p, e.v0.p);
            SPB_LAUNCH_CHECK();
        }
        const int64_t nu = e.sort_reduce(cnt, static_cast<uint64_t>(r1 - r0) * B.ncols, s);
        append_rows(e, nu, r0, r1 - r0, B.ncols, cb, s);
        r0 = r1;
    }
    cb.finish(C, m, B.ncols, s);
}

void transpose(const CsrDev& A, CsrDev& T, cudaStream_t s) {
    Esc e;
    e.reserve(A.nnz);
    if (A.nnz) {
        transpose_expand_kernel<<<grid_for(A.nrows * 32, kT, 8), kT, 0, s>>>(A.nrows, A.offs.p, A.cols.p, A.vals.p,
                                                                              A.nrows, e.k0.p, e.v0.p);
        SPB_LAUNCH_CHECK();
    }
    // keys are unique: the reduce keeps every entry
    const int64_t nu = e.sort_reduce(A.nnz, static_cast<uint64_t>(A.ncols) * A.nrows, s);
    CsrBuilder cb;
    cb.offs.alloc(A.ncols + 1);
    append_rows(e, nu, 0, A.ncols, A.nrows, cb, s);
    cb.finish(T, A.ncols, A.nrows, s);
}

} // namespace

// ---------------------------------------------------------------------------

Amg::Amg(sp_context* ctx, CsrDev&& A0, DBuf<double>&& diag0, const AmgCfg& cfg, SpmmFn fine_spmm,
         std::function<double*(int, DBuf<double>&)> fine_alloc, std::function<View(double*, int)> fine_view,
         int max_cols)
    : ctx_(ctx), s_(ctx->stream), cfg_(cfg), fine_spmm_(std::move(fine_spmm)), fine_view_(std::move(fine_view)),
      max_cols_(max_cols) {
    if (cfg.max_levels < 1) throw_infeasible("amg_build: max_levels < 1");
    if (cfg.drop_tol < 0.0 || cfg.drop_tol >= 1.0) throw_infeasible("amg_build: drop_tol outside [0,1)");
    if (cfg.cheby_degree < 1) throw_infeasible("amg_build: cheby_degree < 1");
    lv_.emplace_back();
    lv_[0].A = std::move(A0);
    lv_[0].diag = std::move(diag0);
    fz_ = fine_alloc(max_cols_, f_z_);
    fdir_ = fine_alloc(max_cols_, f_dir_);
    ft_ = fine_alloc(max_cols_, f_t_);
    fres_ = fine_alloc(max_cols_, f_res_);
    fpost_ = fine_alloc(max_cols_, f_post_);
    red_.alloc(4096);
    build();
}

void Amg::spmm(int l, const View& X, int m, const View& Y) {
    if (l == 0) {
        fine_spmm_(X, m, Y);
        return;
    }
    EpiArgs ea;
    ea.mode = EPI_STORE;
    ea.Y = Y;
    spmm_launch(lv_[l].A.op(), X, m, ea, s_);
}

// estimate_lambda_max (preconditioners.cpp:91-112): power iteration on D^{-1} A
double Amg::power_lambda(int l, int iters, uint64_t seed) {
    AmgLevelDev& L = lv_[l];
    const int64_t n = L.A.nrows;
    if (n == 1) return 1.0;
    const View v = l == 0 ? fv(fz_, 1) : colmajor(L.z.p, L.ld, 1);
    const View w = l == 0 ? fv(ft_, 1) : colmajor(L.t.p, L.ld, 1);
    mt_uniform_block(seed, n, 1, 0, n, v, s_);
    double lambda = 1.0;
    const int grid = std::min(g1(n), 2048);
    for (int it = 0; it < iters; ++it) {
        spmm(l, v, 1, w);
        scale_sq_kernel<<<grid, kT, 0, s_>>>(n, w, L.inv_diag.p, red_.p);
        SPB_LAUNCH_CHECK();
        std::vector<double> part(grid);
        SPB_CUDA(cudaMemcpyAsync(part.data(), red_.p, sizeof(double) * grid, cudaMemcpyDeviceToHost, s_));
        SPB_CUDA(cudaStreamSynchronize(s_));
        double ss = 0.0;
        for (double x : part) ss += x;
        const double nrm = std::sqrt(ss);
        if (nrm == 0.0) return 1.0;
        lambda = nrm;
        div_kernel<<<g1(n), kT, 0, s_>>>(n, w, v, nrm);
        SPB_LAUNCH_CHECK();
    }
    return lambda;
}

void Amg::build() {
    auto finish_level = [&](AmgLevelDev& L) {
        const int64_t n = L.A.nrows;
        if (!L.diag.p || L.diag.n < static_cast<size_t>(n)) L.diag.alloc(std::max<int64_t>(n, 1));
        L.inv_diag.alloc(std::max<int64_t>(n, 1));
        diag_kernel<<<g1(n), kT, 0, s_>>>(n, L.A.offs.p, L.A.cols.p, L.A.vals.p, L.diag.p, L.inv_diag.p);
        SPB_LAUNCH_CHECK();
        if (&L != &lv_[0]) {
            L.ld = std::max<int64_t>(n, 1);
            const size_t e = static_cast<size_t>(L.ld) * max_cols_;
            L.z.alloc(e);
            L.dir.alloc(e);
            L.t.alloc(e);
            L.res.alloc(e);
            L.post.alloc(e);
        }
        L.crhs.release();
    };
    finish_level(lv_[0]);
    DBuf<char> temp;
    while (static_cast<int>(lv_.size()) < cfg_.max_levels && lv_.back().A.nrows > cfg_.coarse_size_threshold) {
        AmgLevelDev& F = lv_.back();
        const int64_t n = F.A.nrows;
        // strength graph -> host greedy aggregation
        DBuf<int64_t> soffs(n + 1);
        strength_count_kernel<<<g1(n), kT, 0, s_>>>(n, F.A.offs.p, F.A.cols.p, F.A.vals.p, F.diag.p, cfg_.drop_tol,
                                                    soffs.p);
        SPB_LAUNCH_CHECK();
        SPB_CUDA(cudaMemsetAsync(soffs.p + n, 0, sizeof(int64_t), s_));
        cub_run([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, soffs.p, soffs.p, n + 1, s_); },
                temp);
        int64_t snnz = 0;
        SPB_CUDA(cudaMemcpyAsync(&snnz, soffs.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s_));
        SPB_CUDA(cudaStreamSynchronize(s_));
        DBuf<int32_t> scols(std::max<int64_t>(snnz, 1));
        strength_fill_kernel<<<g1(n), kT, 0, s_>>>(n, F.A.offs.p, F.A.cols.p, F.A.vals.p, F.diag.p, cfg_.drop_tol,
                                                   soffs.p, scols.p);
        SPB_LAUNCH_CHECK();
        std::vector<int64_t> ho(static_cast<size_t>(n + 1));
        std::vector<int32_t> hc(static_cast<size_t>(std::max<int64_t>(snnz, 1)));
        SPB_CUDA(cudaMemcpyAsync(ho.data(), soffs.p, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost, s_));
        if (snnz) SPB_CUDA(cudaMemcpyAsync(hc.data(), scols.p, sizeof(int32_t) * snnz, cudaMemcpyDeviceToHost, s_));
        SPB_CUDA(cudaStreamSynchronize(s_));
        int64_t nagg = 0;
        const std::vector<int32_t> hagg = greedy_aggregate(n, ho, hc, nagg);
        if (nagg >= n) {
            stagnated_ = true;
            break;
        }
        DBuf<int32_t> agg(n);
        SPB_CUDA(cudaMemcpyAsync(agg.p, hagg.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, s_));
        DBuf<int> cnt(nagg);
        SPB_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int) * nagg, s_));
        agg_count_kernel<<<g1(n), kT, 0, s_>>>(n, agg.p, cnt.p);
        SPB_LAUNCH_CHECK();
        CsrDev Pt0;  // tentative prolongator
        Pt0.nrows = n;
        Pt0.ncols = nagg;
        Pt0.nnz = n;
        Pt0.max_row = 1;
        Pt0.offs.alloc(n + 1);
        Pt0.cols.alloc(n);
        Pt0.vals.alloc(n);
        ptent_kernel<<<g1(n + 1), kT, 0, s_>>>(n, agg.p, cnt.p, Pt0.offs.p, Pt0.cols.p, Pt0.vals.p);
        SPB_LAUNCH_CHECK();
        AmgLevelDev C;
        if (!cfg_.smoothed) {
            // plain aggregation: P = P_tent, coarse = plain_galerkin (:478-520)
            Esc e;
            e.reserve(F.A.nnz);
            plain_expand_kernel<<<grid_for(n * 32, kT, 8), kT, 0, s_>>>(n, F.A.offs.p, F.A.cols.p, F.A.vals.p, agg.p,
                                                                        nagg, e.k0.p, e.v0.p);
            SPB_LAUNCH_CHECK();
            const int64_t nu = e.sort_reduce(F.A.nnz, static_cast<uint64_t>(nagg) * nagg, s_);
            plain_scale_kernel<<<g1(std::max<int64_t>(nu, 1)), kT, 0, s_>>>(nu, e.k0.p, nagg, cnt.p, e.v0.p);
            SPB_LAUNCH_CHECK();
            CsrBuilder cb;
            cb.offs.alloc(nagg + 1);
            append_rows(e, nu, 0, nagg, nagg, cb, s_);
            cb.finish(C.A, nagg, nagg, s_);
            F.P = std::move(Pt0);
        } else {
            // P = (I - omega D^{-1} A) P_tent (:585-612), coarse = P^T (A P)
            const double lambda = power_lambda(static_cast<int>(lv_.size()) - 1, cfg_.power_iters_setup,
                                               cfg_.seed ^ (0xabcdefULL + lv_.size()));
            const double omega = 4.0 / (3.0 * std::max(lambda, 1e-30));
            Esc e;
            const int64_t cntp = F.A.nnz + n;
            e.reserve(cntp);
            smooth_expand_kernel<<<grid_for(n * 32, kT, 8), kT, 0, s_>>>(n, F.A.offs.p, F.A.cols.p, F.A.vals.p,
                                                                         F.inv_diag.p, agg.p, Pt0.vals.p, omega,
                                                                         nagg, e.k0.p, e.v0.p);
            SPB_LAUNCH_CHECK();
            const int64_t nu = e.sort_reduce(cntp, static_cast<uint64_t>(n) * nagg, s_);
            CsrBuilder cb;
            cb.offs.alloc(n + 1);
            append_rows(e, nu, 0, n, nagg, cb, s_);
            cb.finish(F.P, n, nagg, s_);
        }
        transpose(F.P, F.Pt, s_);
        if (cfg_.smoothed) {
            CsrDev AP;
            spgemm(F.A, F.P, AP, s_);
            spgemm(F.Pt, AP, C.A, s_);
        }
        lv_.push_back(std::move(C));
        finish_level(lv_.back());
    }
    // smoother data for every level but the coarsest (:622-630)
    const int L = static_cast<int>(lv_.size());
    for (int l = 0; l + 1 < L; ++l) {
        AmgLevelDev& V = lv_[l];
        V.lambda_max = power_lambda(l, cfg_.power_iters_setup, cfg_.seed ^ (0x517cc1ULL + static_cast<uint64_t>(l)));
        V.low = V.lambda_max / cfg_.eig_ratio;
        V.high = 1.1 * V.lambda_max;
        V.degree = cfg_.cheby_degree;
    }
    // coarse solver (:633-660)
    AmgLevelDev& Lc = lv_.back();
    direct_ = cfg_.coarse_direct;
    if (direct_) {
        const int64_t nc = Lc.A.nrows;
        nc_ = nc;
        std::vector<int64_t> o(static_cast<size_t>(nc + 1));
        std::vector<int32_t> c(static_cast<size_t>(std::max<int64_t>(Lc.A.nnz, 1)));
        std::vector<double> v(static_cast<size_t>(std::max<int64_t>(Lc.A.nnz, 1))), d(static_cast<size_t>(nc));
        SPB_CUDA(cudaMemcpyAsync(o.data(), Lc.A.offs.p, sizeof(int64_t) * (nc + 1), cudaMemcpyDeviceToHost, s_));
        if (Lc.A.nnz) {
            SPB_CUDA(cudaMemcpyAsync(c.data(), Lc.A.cols.p, sizeof(int32_t) * Lc.A.nnz, cudaMemcpyDeviceToHost, s_));
            SPB_CUDA(cudaMemcpyAsync(v.data(), Lc.A.vals.p, sizeof(double) * Lc.A.nnz, cudaMemcpyDeviceToHost, s_));
        }
        SPB_CUDA(cudaMemcpyAsync(d.data(), Lc.diag.p, sizeof(double) * nc, cudaMemcpyDeviceToHost, s_));
        SPB_CUDA(cudaStreamSynchronize(s_));
        if (nc > 8192) throw SpError(1, "amg: coarse level too large for the direct solver");
        double trace = 0.0;
        for (double x : d) trace += x;
        const double shift = 1e-8 * (trace > 0.0 ? trace / static_cast<double>(nc) : 1.0);
        Mat base(nc, nc);
        for (int64_t i = 0; i < nc; ++i)
            for (int64_t k = o[i]; k < o[i + 1]; ++k) base(static_cast<int>(i), c[k]) = v[k];
        Mat Lf;
        double sh = shift;
        for (;;) {
            Lf = base;
            for (int64_t i = 0; i < nc; ++i) Lf(static_cast<int>(i), static_cast<int>(i)) += sh;
            if (cholesky_lower(Lf)) break;
            sh *= 100.0;  // singular beyond the kernel shift; escalate
        }
        // inverse = L^{-T} L^{-1}, column by column
        std::vector<double> inv(static_cast<size_t>(nc) * nc);
        std::vector<double> e(static_cast<size_t>(nc));
        for (int64_t j = 0; j < nc; ++j) {
            std::fill(e.begin(), e.end(), 0.0);
            e[j] = 1.0;
            solve_lower(Lf, e.data());
            solve_lower_transposed(Lf, e.data());
            std::copy(e.begin(), e.end(), inv.begin() + j * nc);
        }
        coarse_inv_.alloc(inv.size());
        SPB_CUDA(cudaMemcpyAsync(coarse_inv_.p, inv.data(), sizeof(double) * inv.size(), cudaMemcpyHostToDevice, s_));
        SPB_CUDA(cudaStreamSynchronize(s_));
    } else {
        Lc.lambda_max = power_lambda(L - 1, cfg_.coarse_power_iters, cfg_.seed ^ (0x9e3779ULL + static_cast<uint64_t>(L)));
        Lc.low = Lc.lambda_max / cfg_.eig_ratio;
        Lc.high = 1.1 * Lc.lambda_max;
        Lc.degree = cfg_.cheby_degree;
    }
}

// chebyshev_solve (preconditioners.cpp:115-156), Z from zero
void Amg::chebyshev(int l, const View& rhs, int k, const View& Z) {
    AmgLevelDev& L = lv_[l];
    const int64_t n = L.A.nrows;
    const double theta = 0.5 * (L.high + L.low), delta = 0.5 * (L.high - L.low);
    const double sigma1 = theta / delta;
    const View dir = l == 0 ? fv(fdir_, k) : colmajor(L.dir.p, L.ld, k);
    const View T = l == 0 ? fv(ft_, k) : colmajor(L.t.p, L.ld, k);
    cheb_init_kernel<<<g1(n * k), kT, 0, s_>>>(n, k, L.inv_diag.p, rhs, dir, Z, theta);
    SPB_LAUNCH_CHECK();
    double rho_prev = 1.0 / sigma1;
    for (int it = 1; it < L.degree; ++it) {
        spmm(l, Z, k, T);
        const double rho = 1.0 / (2.0 * sigma1 - rho_prev);
        const double c1 = rho * rho_prev, c2 = 2.0 * rho / delta;
        cheb_step_kernel<<<g1(n * k), kT, 0, s_>>>(n, k, L.inv_diag.p, rhs, T, dir, Z, c1, c2);
        SPB_LAUNCH_CHECK();
        rho_prev = rho;
    }
}

void Amg::coarse_solve(const View& rhs, int k, const View& Z) {
    AmgLevelDev& L = lv_.back();
    if (!direct_) {
        chebyshev(static_cast<int>(lv_.size()) - 1, rhs, k, Z);
        return;
    }
    dense_apply_kernel<<<g1(nc_ * k), kT, 0, s_>>>(nc_, k, coarse_inv_.p, rhs, Z);
    SPB_LAUNCH_CHECK();
    (void)L;
}

// vcycle (preconditioners.cpp:679-706)
void Amg::vcycle(int l, const View& rhs, int k, const View& Z) {
    if (l + 1 == static_cast<int>(lv_.size())) {
        coarse_solve(rhs, k, Z);
        return;
    }
    AmgLevelDev& L = lv_[l];
    AmgLevelDev& C = lv_[l + 1];
    const int64_t n = L.A.nrows, nc = C.A.nrows;
    const View T = l == 0 ? fv(ft_, k) : colmajor(L.t.p, L.ld, k);
    const View res = l == 0 ? fv(fres_, k) : colmajor(L.res.p, L.ld, k);
    const View post = l == 0 ? fv(fpost_, k) : colmajor(L.post.p, L.ld, k);
    if (!C.crhs.p) C.crhs.alloc(static_cast<size_t>(C.ld) * max_cols_);
    const View crhs = colmajor(C.crhs.p, C.ld, k);
    const View cz = colmajor(C.z.p, C.ld, k);
    chebyshev(l, rhs, k, Z);  // pre-smoothing from zero
    spmm(l, Z, k, T);
    sub_kernel<<<g1(n * k), kT, 0, s_>>>(n, k, rhs, T, res);
    SPB_LAUNCH_CHECK();
    rect_spmm_kernel<false><<<g1(nc * k), kT, 0, s_>>>(nc, k, L.Pt.offs.p, L.Pt.cols.p, L.Pt.vals.p, res, crhs);
    SPB_LAUNCH_CHECK();
    vcycle(l + 1, crhs, k, cz);
    rect_spmm_kernel<true><<<g1(n * k), kT, 0, s_>>>(n, k, L.P.offs.p, L.P.cols.p, L.P.vals.p, cz, Z);
    SPB_LAUNCH_CHECK();
    spmm(l, Z, k, T);  // post-smoothing: one more Chebyshev solve on the updated residual
    sub_kernel<<<g1(n * k), kT, 0, s_>>>(n, k, rhs, T, res);
    SPB_LAUNCH_CHECK();
    chebyshev(l, res, k, post);
    add_kernel<<<g1(n * k), kT, 0, s_>>>(n, k, Z, post);
    SPB_LAUNCH_CHECK();
}

void Amg::apply(const View& R, int k, const View& H) {
    if (k <= 0) return;
    if (k > max_cols_) throw_dimension("amg apply: shape mismatch");
    const int64_t n = lv_[0].A.nrows;
    vcycle(0, R.sub(0, k), k, fv(fz_, k));
    copy_view(n, fv(fz_, k), H.sub(0, k), s_);
}

} // namespace spb
