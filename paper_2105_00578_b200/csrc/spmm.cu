// spmm.cu — CSR SpMM over a row-major block of vectors, with fused epilogues.
//
// Replaces kernels::spmv_block (src/kernels.cpp:36-62), the residual update of
// lobpcg (src/eigensolver.cpp:210-222), kernels::diag_scale (kernels.cpp:187-197)
// and the product-form GMRES-polynomial step (src/preconditioners.cpp:171-193).
//
// Mapping: a group of G lanes (G = next pow2 >= m, <= 32) owns one row; lane c
// owns column c of the block. The row's column indices are fetched G at a time
// with one coalesced load and broadcast by shuffles, so every X gather of the
// group is one contiguous m*8-byte segment of a row-major block. Accumulation is
// sequential over the row in storage order with explicit round-to-nearest
// multiply/add intrinsics (no FMA contraction), which makes the result
// bit-identical to spmv_block. Rows longer than long_threshold are handled by a
// CTA-per-row kernel with a fixed-order tree reduction (deterministic, not
// bit-identical to the sequential sum).
#include "ops.cuh"

namespace spb {

namespace {

constexpr int kThreads = 256;

struct RowAcc {
    // returns acc for (row, column c); xi = X(grow, c)
    template <int MODE, int G>
    static __device__ __forceinline__ double run(const DevOp& op, const View& X, int64_t row,
                                                 int64_t grow, int c, bool act, double xi,
                                                 unsigned gmask, int gl) {
        const int64_t k0 = op.offs[row];
        const int64_t k1 = op.offs[row + 1];
        double acc = 0.0;
        bool placed = false;
        double dval = 0.0, isdi = 0.0;
        if (MODE == OP_LAPLACE_UNIT) dval = op.diag[row];
        if (MODE == OP_NORMAL_UNIT) isdi = op.isd[grow];
        for (int64_t kb = k0; kb < k1; kb += G) {
            const int cnt = static_cast<int>(min(static_cast<int64_t>(G), k1 - kb));
            int jl = 0;
            double vl = 0.0;
            if (gl < cnt) {
                jl = __ldg(op.cols + kb + gl);
                if (MODE == OP_EXPLICIT) vl = __ldg(op.vals + kb + gl);
                if (MODE == OP_NORMAL_UNIT) vl = __dmul_rn(-isdi, __ldg(op.isd + jl));
            }
#pragma unroll 4
            for (int t = 0; t < cnt; ++t) {
                const int j = __shfl_sync(gmask, jl, t, G);
                double v = 0.0;
                if (MODE == OP_EXPLICIT || MODE == OP_NORMAL_UNIT) v = __shfl_sync(gmask, vl, t, G);
                const double xj = act ? X.at(j, c) : 0.0;
                if (MODE == OP_LAPLACE_UNIT) {
                    if (!placed && j > grow) {
                        acc = __dadd_rn(acc, __dmul_rn(dval, xi));
                        placed = true;
                    }
                    acc = __dsub_rn(acc, xj);  // (-1.0) * x_j added: exact negation
                } else if (MODE == OP_NORMAL_UNIT) {
                    if (!placed && j > grow) {
                        acc = __dadd_rn(acc, xi);  // 1.0 * x_i
                        placed = true;
                    }
                    acc = __dadd_rn(acc, __dmul_rn(v, xj));
                } else {
                    acc = __dadd_rn(acc, __dmul_rn(v, xj));
                }
            }
        }
        if (MODE == OP_LAPLACE_UNIT && !placed) acc = __dadd_rn(acc, __dmul_rn(dval, xi));
        if (MODE == OP_NORMAL_UNIT && !placed) acc = __dadd_rn(acc, xi);
        return acc;
    }
};

template <int EPI>
__device__ __forceinline__ void epilogue(const EpiArgs& ea, int64_t row, int c, double acc,
                                         double xi, double& sq) {
    if (EPI == EPI_STORE) {
        ea.Y.at(row, c) = acc;
    } else if (EPI == EPI_RESIDUAL) {
        // R = AX - BX * diag(theta)   (eigensolver.cpp:212-218): bx = d_i*x_i, r = ax - t*bx
        const double bx = ea.bdiag ? __dmul_rn(ea.bdiag[row], xi) : xi;
        const double r = __dsub_rn(acc, __dmul_rn(ea.theta[c], bx));
        ea.Y.at(row, c) = r;
        sq = fma(r, r, sq);
    } else {
        // prod_{i+1} = prod_i - inv_i * (A prod_i); H += inv_{i+1} * prod_{i+1}
        // (preconditioners.cpp:183-190, unrolled one step ahead)
        const double pn = __dsub_rn(xi, __dmul_rn(ea.inv_cur, acc));
        ea.Y.at(row, c) = pn;
        double h = ea.first ? __dmul_rn(ea.inv_cur, xi) : ea.H.at(row, c);
        h = __dadd_rn(h, __dmul_rn(ea.inv_next, pn));
        ea.H.at(row, c) = h;
    }
}

template <int G, int MODE, int EPI>
__global__ void __launch_bounds__(kThreads) spmm_group_kernel(const DevOp op, const View X,
                                                              const EpiArgs ea, const int m) {
    constexpr int GPW = 32 / G;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int gw = lane / G;
    const int warp = threadIdx.x >> 5;
    const int64_t group = (static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + warp) * GPW + gw;
    const int64_t ngroups = static_cast<int64_t>(gridDim.x) * (kThreads / 32) * GPW;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (gw * G));
    double sq = 0.0;

    for (int64_t row = group; row < op.n; row += ngroups) {
        const int64_t grow = op.row0 + row;
        if (MODE == OP_DIAGONAL) {
            for (int c0 = 0; c0 < m; c0 += G) {
                const int c = c0 + gl;
                if (c < m) {
                    const double xi = X.at(grow, c);
                    epilogue<EPI>(ea, row, c, __dmul_rn(op.diag[row], xi), xi, sq);
                }
            }
            continue;
        }
        if (op.offs[row + 1] - op.offs[row] > op.long_threshold) continue;  // long-row bin
        for (int c0 = 0; c0 < m; c0 += G) {
            const int c = c0 + gl;
            const bool act = c < m;
            const double xi = act ? X.at(grow, c) : 0.0;
            const double acc = RowAcc::run<MODE, G>(op, X, row, grow, c, act, xi, gmask, gl);
            if (act) epilogue<EPI>(ea, row, c, acc, xi, sq);
        }
    }

    if (EPI == EPI_RESIDUAL) {
        __shared__ double red[kThreads];
        red[threadIdx.x] = sq;
        __syncthreads();
        if (threadIdx.x < m) {
            double s = 0.0;
            for (int g = 0; g < kThreads / G; ++g) s += red[g * G + threadIdx.x];
            ea.partial[static_cast<int64_t>(blockIdx.x) * m + threadIdx.x] = s;
        }
    }
}


// Warp-tiled kernel for short rows (max_row <= 32: meshes). A warp owns 32
// consecutive rows: it loads their 33 offsets and the contiguous column-index
// segment (<= 32*32 entries) with coalesced loads into shared memory, then its
// 32/G groups walk the rows. The diagonal slot is located before accumulating,
// so the inner loops are branch-free and their gathers independent.
constexpr int kTileRows = 32;
constexpr int kTileCap = 32 * 32;

template <int G, int MODE, int EPI>
__global__ void __launch_bounds__(kThreads) spmm_tile_kernel(const DevOp op, const View X, const EpiArgs ea,
                                                             const int m) {
    constexpr int GPW = 32 / G;
    extern __shared__ int32_t s_cols_all[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    int32_t* sc = s_cols_all + warp * kTileCap;
    double* sv = reinterpret_cast<double*>(s_cols_all + (kThreads / 32) * kTileCap) + warp * kTileCap;
    const int gl = lane & (G - 1);
    const int gw = lane / G;
    double sq = 0.0;
    const int64_t ntiles = (op.n + kTileRows - 1) / kTileRows;
    const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + warp;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
    for (int64_t tile = gwarp; tile < ntiles; tile += nwarps) {
        const int64_t r0 = tile * kTileRows;
        const int nr = static_cast<int>(min(static_cast<int64_t>(kTileRows), op.n - r0));
        const int64_t ko = op.offs[r0 + min(lane, nr)];
        const int64_t kbeg = __shfl_sync(0xffffffffu, ko, 0);
        const int64_t kend = op.offs[r0 + nr];
        const int total = static_cast<int>(kend - kbeg);
        __syncwarp();
        for (int e = lane; e < total; e += 32) {
            sc[e] = __ldg(op.cols + kbeg + e);
            if (MODE == OP_EXPLICIT) sv[e] = __ldg(op.vals + kbeg + e);
        }
        __syncwarp();
        const int rows_per_group = (nr + GPW - 1) / GPW;
        for (int it = 0; it < rows_per_group; ++it) {
            const int rr = it * GPW + gw;
            const int rclamp = min(rr, nr - 1);
            const int64_t o_lo = __shfl_sync(0xffffffffu, ko, rclamp);
            const int64_t o_hi = __shfl_sync(0xffffffffu, ko, min(rclamp + 1, 31));
            const int k0 = static_cast<int>(o_lo - kbeg);
            const int k1 = static_cast<int>((rclamp + 1 >= nr ? kend : o_hi) - kbeg);
            if (rr >= nr) continue;
            const int64_t row = r0 + rr;
            const int64_t grow = op.row0 + row;
            for (int c0 = 0; c0 < m; c0 += G) {
                const int c = c0 + gl;
                if (c >= m) continue;
                const double xi = X.at(grow, c);
                double acc = 0.0;
                if (MODE == OP_EXPLICIT) {
                    for (int k = k0; k < k1; ++k) acc = __dadd_rn(acc, __dmul_rn(sv[k], X.at(sc[k], c)));
                } else {
                    // storage position of the diagonal: before the first column > grow
                    int kd = k0;
                    while (kd < k1 && sc[kd] < grow) ++kd;
                    if (MODE == OP_LAPLACE_UNIT) {
#pragma unroll 4
                        for (int k = k0; k < kd; ++k) acc = __dsub_rn(acc, X.at(sc[k], c));
                        acc = __dadd_rn(acc, __dmul_rn(op.diag[row], xi));
#pragma unroll 4
                        for (int k = kd; k < k1; ++k) acc = __dsub_rn(acc, X.at(sc[k], c));
                    } else {
                        const double nisdi = -op.isd[grow];
#pragma unroll 4
                        for (int k = k0; k < kd; ++k) {
                            const int j = sc[k];
                            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(nisdi, op.isd[j]), X.at(j, c)));
                        }
                        acc = __dadd_rn(acc, xi);
#pragma unroll 4
                        for (int k = kd; k < k1; ++k) {
                            const int j = sc[k];
                            acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(nisdi, op.isd[j]), X.at(j, c)));
                        }
                    }
                }
                epilogue<EPI>(ea, row, c, acc, xi, sq);
            }
        }
    }
    if (EPI == EPI_RESIDUAL) {
        __shared__ double red[kThreads];
        red[threadIdx.x] = sq;
        __syncthreads();
        if (threadIdx.x < m) {
            double s = 0.0;
            for (int g = 0; g < kThreads / G; ++g) s += red[g * G + threadIdx.x];
            ea.partial[static_cast<int64_t>(blockIdx.x) * m + threadIdx.x] = s;
        }
    }
}

// One CTA per long row (power-law hubs). Thread t accumulates entries
// k0+t, k0+t+256, ... for every column; fixed-order warp butterfly + smem tree.
template <int MODE, int EPI>
__global__ void __launch_bounds__(kThreads) spmm_long_kernel(const DevOp op, const View X,
                                                             const EpiArgs ea, const int m,
                                                             const int partial_base) {
    const int64_t row = op.long_rows[blockIdx.x];
    const int64_t grow = op.row0 + row;
    const int64_t k0 = op.offs[row], k1 = op.offs[row + 1];
    __shared__ double red[kThreads / 32][32];
    __shared__ double sqs[32];
    double isdi = 0.0;
    if (MODE == OP_NORMAL_UNIT) isdi = op.isd[grow];
    for (int c0 = 0; c0 < m; c0 += 32) {
        const int mc = min(32, m - c0);
        double acc[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) acc[c] = 0.0;
        for (int64_t k = k0 + threadIdx.x; k < k1; k += kThreads) {
            const int j = op.cols[k];
            double v;
            if (MODE == OP_EXPLICIT) v = op.vals[k];
            else if (MODE == OP_NORMAL_UNIT) v = __dmul_rn(-isdi, op.isd[j]);
            else v = -1.0;
            const double* xr = &X.at(j, c0);
#pragma unroll
            for (int c = 0; c < 32; ++c)
                if (c < mc) acc[c] = __dadd_rn(acc[c], __dmul_rn(v, xr[c * X.cs]));
        }
        // fixed-order reductions
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            double a = acc[c];
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
            acc[c] = a;
        }
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        if (lane == 0)
            for (int c = 0; c < 32; ++c) red[warp][c] = acc[c];
        __syncthreads();
        if (threadIdx.x < mc) {
            const int c = threadIdx.x;
            double s = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) s += red[w][c];
            const double xi = X.at(grow, c0 + c);
            if (MODE == OP_LAPLACE_UNIT) s = __dadd_rn(s, __dmul_rn(op.diag[row], xi));
            if (MODE == OP_NORMAL_UNIT) s = __dadd_rn(s, xi);
            double sq = 0.0;
            epilogue<EPI>(ea, row, c0 + c, s, xi, sq);
            sqs[c] = sq;
        }
        __syncthreads();
        if (EPI == EPI_RESIDUAL && threadIdx.x < mc)
            ea.partial[static_cast<int64_t>(partial_base + blockIdx.x) * m + c0 + threadIdx.x] =
                sqs[threadIdx.x];
        __syncthreads();
    }
}

template <int MODE, int EPI>
int launch_mode_epi(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s) {
    int G = 1;
    while (G < m && G < 32) G <<= 1;
    if (MODE != OP_DIAGONAL && op.max_row <= 32 && op.n_long == 0) {
        const int64_t ntiles = (op.n + kTileRows - 1) / kTileRows;
        const int grid = grid_for(ntiles, kThreads / 32, 8);
        const size_t smem = (kThreads / 32) * kTileCap * (sizeof(int32_t) + (MODE == OP_EXPLICIT ? sizeof(double) : 0));
        auto go = [&](auto kern) {
            static bool attr = false;
            if (!attr) {
                SPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                attr = true;
            }
            kern<<<grid, kThreads, smem, s>>>(op, X, ea, m);
        };
        switch (G) {
        case 1: go(spmm_tile_kernel<1, MODE, EPI>); break;
        case 2: go(spmm_tile_kernel<2, MODE, EPI>); break;
        case 4: go(spmm_tile_kernel<4, MODE, EPI>); break;
        case 8: go(spmm_tile_kernel<8, MODE, EPI>); break;
        case 16: go(spmm_tile_kernel<16, MODE, EPI>); break;
        default: go(spmm_tile_kernel<32, MODE, EPI>); break;
        }
        SPB_LAUNCH_CHECK();
        return grid;
    }
    const int groups_per_block = kThreads / G;
    const int grid = grid_for(op.n, groups_per_block, 8);
    switch (G) {
    case 1: spmm_group_kernel<1, MODE, EPI><<<grid, kThreads, 0, s>>>(op, X, ea, m); break;
    case 2: spmm_group_kernel<2, MODE, EPI><<<grid, kThreads, 0, s>>>(op, X, ea, m); break;
    case 4: spmm_group_kernel<4, MODE, EPI><<<grid, kThreads, 0, s>>>(op, X, ea, m); break;
    case 8: spmm_group_kernel<8, MODE, EPI><<<grid, kThreads, 0, s>>>(op, X, ea, m); break;
    case 16: spmm_group_kernel<16, MODE, EPI><<<grid, kThreads, 0, s>>>(op, X, ea, m); break;
    default: spmm_group_kernel<32, MODE, EPI><<<grid, kThreads, 0, s>>>(op, X, ea, m); break;
    }
    SPB_LAUNCH_CHECK();
    if (MODE != OP_DIAGONAL && op.n_long > 0) {
        spmm_long_kernel<MODE, EPI>
            <<<static_cast<int>(op.n_long), kThreads, 0, s>>>(op, X, ea, m, grid);
        SPB_LAUNCH_CHECK();
    }
    return grid + (MODE != OP_DIAGONAL ? static_cast<int>(op.n_long) : 0);
}

template <int EPI>
int launch_epi(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s) {
    switch (op.mode) {
    case OP_EXPLICIT: return launch_mode_epi<OP_EXPLICIT, EPI>(op, X, m, ea, s);
    case OP_LAPLACE_UNIT: return launch_mode_epi<OP_LAPLACE_UNIT, EPI>(op, X, m, ea, s);
    case OP_NORMAL_UNIT: return launch_mode_epi<OP_NORMAL_UNIT, EPI>(op, X, m, ea, s);
    default: return launch_mode_epi<OP_DIAGONAL, EPI>(op, X, m, ea, s);
    }
}

__global__ void reduce_partials_kernel(const double* partial, int rows, int m, double* out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= m) return;
    double s = 0.0;
    for (int r = 0; r < rows; ++r) s += partial[static_cast<int64_t>(r) * m + c];
    out[c] = s;
}

} // namespace

int spmm_launch(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s) {
    if (m <= 0) return 0;
    if (ea.mode != EPI_STORE && m > 32)
        throw_dimension("spmm: fused epilogues support at most 32 columns");
    switch (ea.mode) {
    case EPI_STORE: return launch_epi<EPI_STORE>(op, X, m, ea, s);
    case EPI_RESIDUAL: return launch_epi<EPI_RESIDUAL>(op, X, m, ea, s);
    default: return launch_epi<EPI_POLY>(op, X, m, ea, s);
    }
}

void reduce_partials(const double* partial, int rows, int m, double* out, cudaStream_t s) {
    reduce_partials_kernel<<<1, 64, 0, s>>>(partial, rows, m, out);
    SPB_LAUNCH_CHECK();
}

} // namespace spb
