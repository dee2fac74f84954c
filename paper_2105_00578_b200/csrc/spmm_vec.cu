// spmm_vec.cu — SpMM for irregular (power-law) graphs in the solver: rows binned
// by length, S lanes per row (S = 4, 8, 16, 32 by bin), the S lanes stride over
// the row's entries and each lane gathers whole X rows (all m columns,
// contiguous in the row-major block), so one warp instruction serves 32 entries
// instead of one. The S partial sums are combined by a fixed butterfly, so the
// result is deterministic (run to run and rank count for a fixed partition),
// but — unlike the order-exact group kernel used by the kernel-level sp_spmm —
// not in the reference's per-row storage order. Rows with more than the
// long-row threshold keep one CTA each (spmm_long_kernel).
#include "spmm_epilogue.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <vector>

namespace spb {

namespace {

constexpr int kVThreads = 256;
#ifndef SPB_VEC_U
#define SPB_VEC_U 4
#endif

// Binned rows (all four bins by default), lanes over columns: R rows per warp,
// L = 32 / R lanes per row, G = pow2(m) lanes per entry (lane = column),
// E = L / G entries per instruction, U instructions in flight; the E slot sums
// combine by a fixed butterfly (deterministic). Coalesced whole-row gathers: 1-2
// L1 wavefronts per entry instead of one per column and entry.
template <int G, int R, int MODE, int EPI>
__global__ void __launch_bounds__(kVThreads) spmm_rowcols_kernel(const DevOp op, const View X, const EpiArgs ea,
                                                                 const int m, const int32_t* rows,
                                                                 const int64_t nrows, const int partial_base) {
    constexpr int L = 32 / R;
    static_assert(L >= G, "a row group must hold one entry's columns");
    constexpr int E = L / G;
    constexpr int U = SPB_VEC_U;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / L, gl = lane % L;
    const int sub = gl / G, c = gl % G;
    const bool act = c < m;
    // warp-uniform row loop (the butterfly below is a full-warp shuffle)
    const int64_t w0 = (blockIdx.x * static_cast<int64_t>(kVThreads) + threadIdx.x) >> 5;
    const int64_t nw = static_cast<int64_t>(gridDim.x) * (kVThreads / 32);
    double sq = 0.0;
    for (int64_t rb = w0 * R; rb < nrows; rb += nw * R) {
        const int64_t r = rb + grp;
        const bool valid = r < nrows;
        const int64_t row = valid ? rows[r] : 0;
        const int64_t grow = op.row0 + row;
        const int64_t k0 = valid ? op.offs[row] : 0, k1 = valid ? op.offs[row + 1] : 0;
        double nisdi = 0.0;
        if (MODE == OP_NORMAL_UNIT && valid) nisdi = -op.isd[grow];
        double acc = 0.0;
        int64_t k = k0 + sub;
        for (; k + (U - 1) * E < k1; k += U * E) {
            int32_t j[U];
            double w[U], x[U];
#pragma unroll
            for (int u = 0; u < U; ++u) j[u] = op.cols[k + u * E];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (MODE == OP_EXPLICIT) w[u] = op.vals[k + u * E];
                else if (MODE == OP_NORMAL_UNIT) w[u] = nisdi * op.isd[j[u]];
                else w[u] = -1.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) x[u] = act ? __ldg(X.ptr + static_cast<int64_t>(j[u]) * X.rs + c) : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u) acc = fma(w[u], x[u], acc);
        }
        for (; k < k1; k += E) {
            const int64_t j = op.cols[k];
            double w;
            if (MODE == OP_EXPLICIT) w = op.vals[k];
            else if (MODE == OP_NORMAL_UNIT) w = nisdi * op.isd[j];
            else w = -1.0;
            const double x = act ? __ldg(X.ptr + j * X.rs + c) : 0.0;
            acc = fma(w, x, acc);
        }
#pragma unroll
        for (int off = L / 2; off >= G; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        if (valid && sub == 0 && act) {
            const double xi = X.at(grow, c);
            double v = acc;
            if (MODE == OP_LAPLACE_UNIT) v = __dadd_rn(v, __dmul_rn(op.diag[row], xi));
            if (MODE == OP_NORMAL_UNIT) v = __dadd_rn(v, xi);
            epilogue<EPI>(ea, row, c, v, xi, sq);
        }
    }
    if (EPI == EPI_RESIDUAL) {
        __shared__ double s_sq[kVThreads / 32][32];
        s_sq[warp][lane] = sq;  // zero on lanes that never ran an epilogue
        __syncthreads();
        if (threadIdx.x < m) {
            double t = 0.0;
            for (int w = 0; w < kVThreads / 32; ++w)
                for (int g = 0; g < R; ++g) t += s_sq[w][g * L + threadIdx.x];
            ea.partial[static_cast<int64_t>(partial_base + blockIdx.x) * m + threadIdx.x] = t;
        }
    }
}

// Long rows (bin 4) in chunks of kChunk entries, one CTA per chunk, lanes over columns:
// G = pow2(m) lanes per entry (lane = column), E = 32 / G entries per warp instruction,
// U instructions in flight per warp; one warp instruction gathers E whole X rows coalesced
// (an m*8-byte row is 1-2 L1 wavefronts). Deterministic: entry k of the chunk goes to
// slot (k - kb) mod (NW*E), the slots combine in slot order into one partial per chunk;
// long_finish_kernel then adds each row's chunk partials in order, the diagonal term and
// the epilogue (one warp per row, lane = column).
constexpr int64_t kChunk = 4096;

template <int G, int MODE>
__global__ void __launch_bounds__(kVThreads) long_chunk_cols_kernel(const DevOp op, const View X, const int m,
                                                                    const int32_t* chunk_row,
                                                                    const int64_t* chunk_k0, double* chunk_part) {
    constexpr int E = 32 / G;
    constexpr int NW = kVThreads / 32;
    constexpr int STRIDE = NW * E;
    constexpr int U = SPB_VEC_U;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane / G, c = lane % G;
    const int slot = warp * E + sub;
    const int64_t row = chunk_row[blockIdx.x];
    const int64_t grow = op.row0 + row;
    const int64_t kb = chunk_k0[blockIdx.x];
    const int64_t ke = min(kb + kChunk, op.offs[row + 1]);
    const bool act = c < m;
    double nisdi = 0.0;
    if (MODE == OP_NORMAL_UNIT) nisdi = -op.isd[grow];
    double acc = 0.0;
    int64_t k = kb + slot;
    for (; k + (U - 1) * STRIDE < ke; k += U * STRIDE) {
        int32_t j[U];
        double w[U], x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) j[u] = op.cols[k + u * STRIDE];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (MODE == OP_EXPLICIT) w[u] = op.vals[k + u * STRIDE];
            else if (MODE == OP_NORMAL_UNIT) w[u] = nisdi * op.isd[j[u]];
            else w[u] = -1.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = act ? __ldg(X.ptr + static_cast<int64_t>(j[u]) * X.rs + c) : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) acc = fma(w[u], x[u], acc);
    }
    for (; k < ke; k += STRIDE) {
        const int64_t j = op.cols[k];
        double w;
        if (MODE == OP_EXPLICIT) w = op.vals[k];
        else if (MODE == OP_NORMAL_UNIT) w = nisdi * op.isd[j];
        else w = -1.0;
        const double x = act ? __ldg(X.ptr + j * X.rs + c) : 0.0;
        acc = fma(w, x, acc);
    }
    __shared__ double red[STRIDE][G];
    red[slot][c] = acc;
    __syncthreads();
    if (threadIdx.x < m) {
        double v = 0.0;
        for (int t = 0; t < STRIDE; ++t) v += red[t][threadIdx.x];
        chunk_part[static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x] = v;
    }
}

template <int MODE, int EPI>
__global__ void __launch_bounds__(kVThreads) long_finish_kernel(const DevOp op, const View X, const EpiArgs ea,
                                                                const int m, const int64_t* row_chunk0,
                                                                const double* chunk_part, const int partial_base) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * (kVThreads / 32) + warp;
    __shared__ double s_sq[kVThreads / 32][32];
    double sq = 0.0;
    if (i < op.n_long && lane < m) {
        const int64_t row = op.long_rows[i];
        const int64_t grow = op.row0 + row;
        double v = 0.0;
        for (int64_t ch = row_chunk0[i]; ch < row_chunk0[i + 1]; ++ch) v += chunk_part[ch * 32 + lane];
        const double xi = X.at(grow, lane);
        if (MODE == OP_LAPLACE_UNIT) v = __dadd_rn(v, __dmul_rn(op.diag[row], xi));
        if (MODE == OP_NORMAL_UNIT) v = __dadd_rn(v, xi);
        epilogue<EPI>(ea, row, lane, v, xi, sq);
    }
    if (EPI == EPI_RESIDUAL) {
        s_sq[warp][lane] = sq;
        __syncthreads();
        if (threadIdx.x < m) {
            double s = 0.0;
            for (int w = 0; w < kVThreads / 32; ++w) s += s_sq[w][threadIdx.x];
            ea.partial[static_cast<int64_t>(partial_base + blockIdx.x) * m + threadIdx.x] = s;
        }
    }
}

__global__ void chunk_count_kernel(int64_t nl, const int32_t* long_rows, const int64_t* offs, int64_t* cnt) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nl;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = long_rows[i];
        cnt[i] = (offs[r + 1] - offs[r] + kChunk - 1) / kChunk;
    }
}

__global__ void chunk_fill_kernel(int64_t nl, const int32_t* long_rows, const int64_t* offs, const int64_t* start,
                                  int32_t* chunk_row, int64_t* chunk_k0) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nl;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = long_rows[i];
        int64_t c = start[i];
        for (int64_t k = offs[r]; k < offs[r + 1]; k += kChunk, ++c) {
            chunk_row[c] = static_cast<int32_t>(r);
            chunk_k0[c] = k;
        }
    }
}

__global__ void bin_keys_kernel(int64_t n, const int64_t* offs, int64_t long_thr, uint8_t* key, int32_t* ids,
                                unsigned long long* counts) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t len = offs[i + 1] - offs[i];
        const uint8_t b = len > long_thr ? 4 : (len <= 16 ? 0 : (len <= 64 ? 1 : (len <= 256 ? 2 : 3)));
        key[i] = b;
        ids[i] = static_cast<int32_t>(i);
        atomicAdd(&counts[b], 1ull);
    }
}

template <int S, int MODE, int EPI>
int launch_bin(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s, const int32_t* rows,
               int64_t nrows, int partial_base) {
    // rows of the S = 4 / 8 bins: several rows per warp (L = 8 or 16 lanes per row) when m fits
    constexpr int RS = S == 4 ? 4 : (S == 8 ? 2 : 1);
    int grid;
    if (m <= 8) {
        grid = grid_for(nrows, (kVThreads / 32) * RS, 8);
        spmm_rowcols_kernel<8, RS, MODE, EPI><<<grid, kVThreads, 0, s>>>(op, X, ea, m, rows, nrows, partial_base);
    } else if (m <= 16) {
        constexpr int R16 = RS > 2 ? 2 : RS;
        grid = grid_for(nrows, (kVThreads / 32) * R16, 8);
        spmm_rowcols_kernel<16, R16, MODE, EPI><<<grid, kVThreads, 0, s>>>(op, X, ea, m, rows, nrows, partial_base);
    } else {
        grid = grid_for(nrows, kVThreads / 32, 8);
        spmm_rowcols_kernel<32, 1, MODE, EPI><<<grid, kVThreads, 0, s>>>(op, X, ea, m, rows, nrows, partial_base);
    }
    SPB_LAUNCH_CHECK();
    return grid;
}

template <int MODE, int EPI>
int launch_mode(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s) {
    int rows_out = 0;
    constexpr int kS[4] = {4, 8, 16, 32};
    for (int b = 0; b < 4; ++b) {
        const int64_t nb = op.bin_off[b + 1] - op.bin_off[b];
        if (nb <= 0) continue;
        const int32_t* r = op.bin_rows + op.bin_off[b];
        switch (kS[b]) {
        case 4: rows_out += launch_bin<4, MODE, EPI>(op, X, m, ea, s, r, nb, rows_out); break;
        case 8: rows_out += launch_bin<8, MODE, EPI>(op, X, m, ea, s, r, nb, rows_out); break;
        case 16: rows_out += launch_bin<16, MODE, EPI>(op, X, m, ea, s, r, nb, rows_out); break;
        default: rows_out += launch_bin<32, MODE, EPI>(op, X, m, ea, s, r, nb, rows_out); break;
        }
    }
    return rows_out;
}

template <int MODE, int EPI>
int launch_long(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s, int partial_base) {
    if (op.n_long <= 0) return 0;
    const int nch = static_cast<int>(op.long_nchunks);
    if (m <= 8) long_chunk_cols_kernel<8, MODE><<<nch, kVThreads, 0, s>>>(op, X, m, op.long_chunk_row, op.long_chunk_k0, op.long_part);
    else if (m <= 16) long_chunk_cols_kernel<16, MODE><<<nch, kVThreads, 0, s>>>(op, X, m, op.long_chunk_row, op.long_chunk_k0, op.long_part);
    else long_chunk_cols_kernel<32, MODE><<<nch, kVThreads, 0, s>>>(op, X, m, op.long_chunk_row, op.long_chunk_k0, op.long_part);
    SPB_LAUNCH_CHECK();
    const int grid = ceil_div(op.n_long, kVThreads / 32);
    long_finish_kernel<MODE, EPI><<<grid, kVThreads, 0, s>>>(op, X, ea, m, op.long_row_chunk0, op.long_part, partial_base);
    SPB_LAUNCH_CHECK();
    return grid;
}

} // namespace

bool spmm_vec_ok(const DevOp& op, const View& X, int m, const EpiArgs& ea) {
    return op.bin_rows && op.mode != OP_DIAGONAL && X.cs == 1 && m <= 32 && !(ea.mode == EPI_RESIDUAL && m > 16) &&
           (ea.mode != EPI_POLY || (ea.Y.cs == 1 && ea.H.cs == 1));
}

int spmm_vec_launch(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s) {
    auto go = [&](auto mode_tag) -> int {
        constexpr int MODE = decltype(mode_tag)::value;
        int rows = 0;
        switch (ea.mode) {
        case EPI_STORE:
            rows = launch_mode<MODE, EPI_STORE>(op, X, m, ea, s);
            return rows + launch_long<MODE, EPI_STORE>(op, X, m, ea, s, rows);
        case EPI_RESIDUAL:
            rows = launch_mode<MODE, EPI_RESIDUAL>(op, X, m, ea, s);
            return rows + launch_long<MODE, EPI_RESIDUAL>(op, X, m, ea, s, rows);
        default:
            rows = launch_mode<MODE, EPI_POLY>(op, X, m, ea, s);
            return rows + launch_long<MODE, EPI_POLY>(op, X, m, ea, s, rows);
        }
    };
    switch (op.mode) {
    case OP_EXPLICIT: return go(std::integral_constant<int, OP_EXPLICIT>{});
    case OP_LAPLACE_UNIT: return go(std::integral_constant<int, OP_LAPLACE_UNIT>{});
    default: return go(std::integral_constant<int, OP_NORMAL_UNIT>{});
    }
}

void build_row_bins(DevOp& op, int64_t long_thr, RowBins& st, cudaStream_t s) {
    const int64_t n = op.n;
    if (n <= 0 || op.mode == OP_DIAGONAL) return;
    DBuf<uint8_t> key(n), key_out(n);
    DBuf<int32_t> ids(n);
    DBuf<unsigned long long> counts(5);
    st.rows.alloc(n);
    SPB_CUDA(cudaMemsetAsync(counts.p, 0, 5 * sizeof(unsigned long long), s));
    bin_keys_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(n, op.offs, long_thr, key.p, ids.p, counts.p);
    SPB_LAUNCH_CHECK();
    // stable: rows keep ascending order inside each bin (deterministic schedules)
    size_t tmp_bytes = 0;
    SPB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key.p, key_out.p, ids.p, st.rows.p, n, 0, 3, s));
    DBuf<unsigned char> tmp(std::max<size_t>(tmp_bytes, 1));
    SPB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, key.p, key_out.p, ids.p, st.rows.p, n, 0, 3, s));
    unsigned long long h[5];
    SPB_CUDA(cudaMemcpyAsync(h, counts.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    op.bin_off[0] = 0;
    for (int b = 0; b < 5; ++b) op.bin_off[b + 1] = op.bin_off[b] + static_cast<int64_t>(h[b]);
    op.bin_rows = st.rows.p;
    // the long rows (bin 4), cut into chunks of kChunk entries (ascending row order)
    op.long_rows = st.rows.p + op.bin_off[4];
    op.n_long = static_cast<int64_t>(h[4]);
    op.long_threshold = long_thr;
    const int64_t nl = op.n_long;
    if (nl > 0) {
        st.row_chunk0.alloc(nl + 1);
        DBuf<int64_t> cnt(nl + 1);
        chunk_count_kernel<<<grid_for(nl, 256, 4), 256, 0, s>>>(nl, op.long_rows, op.offs, cnt.p);
        SPB_LAUNCH_CHECK();
        SPB_CUDA(cudaMemsetAsync(cnt.p + nl, 0, sizeof(int64_t), s));
        size_t tb = 0;
        SPB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, st.row_chunk0.p, nl + 1, s));
        DBuf<unsigned char> t2(std::max<size_t>(tb, 1));
        SPB_CUDA(cub::DeviceScan::ExclusiveSum(t2.p, tb, cnt.p, st.row_chunk0.p, nl + 1, s));
        int64_t nch = 0;
        SPB_CUDA(cudaMemcpyAsync(&nch, st.row_chunk0.p + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        st.chunk_row.alloc(std::max<int64_t>(nch, 1));
        st.chunk_k0.alloc(std::max<int64_t>(nch, 1));
        st.part.alloc(static_cast<size_t>(std::max<int64_t>(nch, 1)) * 32);
        chunk_fill_kernel<<<grid_for(nl, 256, 4), 256, 0, s>>>(nl, op.long_rows, op.offs, st.row_chunk0.p,
                                                                st.chunk_row.p, st.chunk_k0.p);
        SPB_LAUNCH_CHECK();
        op.long_nchunks = nch;
        op.long_row_chunk0 = st.row_chunk0.p;
        op.long_chunk_row = st.chunk_row.p;
        op.long_chunk_k0 = st.chunk_k0.p;
        op.long_part = st.part.p;
    }
}

} // namespace spb
