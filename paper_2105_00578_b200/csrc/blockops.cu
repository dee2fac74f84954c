// blockops.cu — tall-skinny block kernels on row-major (or column-major) views.
//
// Replaces the tall-skinny kernels of src/kernels.cpp: gram (:79-110), mult
// (:127-142), mult_sub (:144-157), dot/norm2/axpy (:159-185), diag_scale
// (:187-197), scale_columns (:199-207), and the column copies in lobpcg.
//
// One kernel (ts_tile_kernel) streams row tiles of up to three input blocks
// through shared memory, optionally transforms them (V - U*C for block
// Gram-Schmidt, V*C for block combines), writes the result, and accumulates a
// Gram matrix [left]^T diag(b) [right] of the tile in registers (2x2 register
// blocks, row slices). Per-CTA partials are reduced in a fixed order by a second
// kernel, so every Gram is bit-reproducible run to run (the reference's
// chunked-reduction determinism contract, kernels.hpp:10-13).
#include "bulk.cuh"
#include "ops.cuh"

#include <algorithm>
#include <cstdint>
#include <cstdlib>

namespace spb {

namespace {

constexpr int kTsThreads = 256;
constexpr int kTR = 64;  // rows per tile

struct TsDev {
    int64_t n;
    View U0, U1, V, W, W2;
    const double* C;
    int ldc;
    const double* b;
    int transform;
    int gram, left_u, left_self;
    int u0, u1, kv, kw;
    int P, Q;
    int nb, slices;
    double* partial;
    // fused final reduction (small Grams): the last CTA to finish sums every CTA's
    // partial in CTA order into gram_out; counter is zero on entry and on exit
    double* gram_out;
    unsigned* counter;
};

constexpr int kStages = 3;

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Tile rows [r0, r0+rows) of view v -> smem columns [c0, c0+cols) of a row-major
// tile with row stride ldt. Column-major views (rs == 1): warp per column, lane
// per row (coalesced 256 B per warp request). Row-major views: a flat walk over
// the rows x cols elements with an incremental (r, c) cursor (no divisions).
__device__ __forceinline__ void issue_view(double* tile, int ldt, int c0, const View& v, int64_t r0, int rows,
                                           int cols) {
    if (v.rs == 1 && cols > 1) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int c = warp; c < cols; c += kTsThreads / 32) {
            const double* src = v.ptr + static_cast<int64_t>(c) * v.cs + r0;
            double* dst = tile + c0 + c;
            for (int r = lane; r < rows; r += 32) cp_async8(dst + r * ldt, src + r);
        }
        return;
    }
    const int total = rows * cols;
    int r = threadIdx.x / cols, c = threadIdx.x - (threadIdx.x / cols) * cols;
    const int dr = kTsThreads / cols, dc = kTsThreads - dr * cols;
    for (int e = threadIdx.x; e < total; e += kTsThreads) {
        cp_async8(tile + r * ldt + c0 + c, v.ptr + (r0 + r) * v.rs + static_cast<int64_t>(c) * v.cs);
        r += dr;
        c += dc;
        if (c >= cols) {
            c -= cols;
            ++r;
        }
    }
}

__device__ __forceinline__ void store_view(const View& v, const double* tile, int ldt, int c0, int64_t r0,
                                           int rows, int cols) {
    if (v.rs == 1 && cols > 1) {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int c = warp; c < cols; c += kTsThreads / 32) {
            double* dst = v.ptr + static_cast<int64_t>(c) * v.cs + r0;
            const double* src = tile + c0 + c;
            for (int r = lane; r < rows; r += 32) dst[r] = src[r * ldt];
        }
        return;
    }
    const int total = rows * cols;
    int r = threadIdx.x / cols, c = threadIdx.x - (threadIdx.x / cols) * cols;
    const int dr = kTsThreads / cols, dc = kTsThreads - dr * cols;
    for (int e = threadIdx.x; e < total; e += kTsThreads) {
        v.ptr[(r0 + r) * v.rs + static_cast<int64_t>(c) * v.cs] = tile[r * ldt + c0 + c];
        r += dr;
        c += dc;
        if (c >= cols) {
            c -= cols;
            ++r;
        }
    }
}

// One smem row layout per stage: [ U (u) | V (kv) | W (kw) | b ], row stride LDT.
// A Gram operand column is then a fixed column offset inside the row, and the
// per-row inner loops are 4 LDS + 4 DFMA per 2x2 register block.
template <int MAXB>
__global__ void __launch_bounds__(kTsThreads) ts_tile_kernel(const TsDev a) {
    extern __shared__ double smem[];
    constexpr int TR = kTR;
    const int u = a.u0 + a.u1;
    const bool need_u = (a.transform == TS_UPDATE) || (a.gram && a.left_u);
    const int cu = need_u ? u : 0;
    const int cv = cu, cw = cu + a.kv, cb = cw + a.kw;
    const int LDT = (cb + 1) | 1;  // odd row stride: conflict-free column-wise smem access
    const int stage_elems = TR * LDT;
    const int inner = a.transform == TS_UPDATE ? u : a.kv;
    double* Cs = smem + kStages * stage_elems;  // inner x kw, column-major
    if (a.transform != TS_NONE)
        for (int i = threadIdx.x; i < inner * a.kw; i += blockDim.x) {
            const int c = i / inner, q = i - c * inner;
            Cs[i] = a.C[q + static_cast<int64_t>(c) * a.ldc];
        }

    // transform mapping: thread -> (fixed output column, row slice)
    const int kwp = a.kw > 0 ? a.kw : 1;
    const int t_col = threadIdx.x % kwp;
    const int t_r0 = threadIdx.x / kwp;
    const int t_rstep = max(1, kTsThreads / kwp);
    const bool t_on = t_r0 < t_rstep && a.transform != TS_NONE;
    const int a_off = a.transform == TS_UPDATE ? 0 : cv;      // transform operand columns
    const double* Ccol = Cs + t_col * inner;

    // gram mapping: left col i -> [U | right], right col j -> right block
    const int right_off = (a.transform == TS_NONE) ? cv : cw;
    const int uL = a.left_u ? u : 0;
    double acc[MAXB][4];
    int lc0[MAXB], lc1[MAXB], rc0[MAXB], rc1[MAXB];
    bool on[MAXB];
    const int nbi = (a.P + 1) / 2;
    const int sl = (MAXB == 1) ? threadIdx.x / max(a.nb, 1) : 0;
#pragma unroll
    for (int bb = 0; bb < MAXB; ++bb) {
        acc[bb][0] = acc[bb][1] = acc[bb][2] = acc[bb][3] = 0.0;
        const int blk = (MAXB == 1) ? (threadIdx.x % max(a.nb, 1)) : (threadIdx.x + bb * blockDim.x);
        on[bb] = a.gram && blk < a.nb && sl < a.slices;
        const int i0 = 2 * (blk % nbi), j0 = 2 * (blk / nbi);
        const int i1 = min(i0 + 1, a.P - 1), j1 = min(j0 + 1, a.Q - 1);
        lc0[bb] = i0 < uL ? i0 : right_off + (i0 - uL);
        lc1[bb] = i1 < uL ? i1 : right_off + (i1 - uL);
        rc0[bb] = right_off + j0;
        rc1[bb] = right_off + j1;
    }

    const int64_t ntiles = (a.n + TR - 1) / TR;
    const int64_t nt = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto issue = [&](int64_t i) {
        const int64_t r0 = (blockIdx.x + i * gridDim.x) * TR;
        const int rows = static_cast<int>(min(static_cast<int64_t>(TR), a.n - r0));
        double* T = smem + (i % kStages) * stage_elems;
        if (need_u) {
            if (a.u0) issue_view(T, LDT, 0, a.U0, r0, rows, a.u0);
            if (a.u1) issue_view(T, LDT, a.u0, a.U1, r0, rows, a.u1);
        }
        issue_view(T, LDT, cv, a.V, r0, rows, a.kv);
        if (a.gram && a.b)
            for (int r = threadIdx.x; r < rows; r += blockDim.x) cp_async8(T + r * LDT + cb, a.b + r0 + r);
    };

    for (int st = 0; st < kStages - 1; ++st) {
        if (st < nt) issue(st);
        cp_commit();
    }
    for (int64_t i = 0; i < nt; ++i) {
        if (i + kStages - 1 < nt) issue(i + kStages - 1);
        cp_commit();
        cp_wait<kStages - 1>();
        __syncthreads();
        const int64_t r0 = (blockIdx.x + i * gridDim.x) * TR;
        const int rows = static_cast<int>(min(static_cast<int64_t>(TR), a.n - r0));
        double* T = smem + (i % kStages) * stage_elems;

        if (a.transform != TS_NONE) {
            if (t_on) {
                for (int r = t_r0; r < rows; r += t_rstep) {
                    const double* ar = T + r * LDT + a_off;
                    double sacc = 0.0;
                    for (int q = 0; q < inner; ++q) sacc = fma(ar[q], Ccol[q], sacc);
                    T[r * LDT + cw + t_col] = (a.transform == TS_UPDATE) ? T[r * LDT + cv + t_col] - sacc : sacc;
                }
            }
            __syncthreads();
            const int w1 = min(a.kw, a.W.cols);
            if (w1 > 0) store_view(a.W, T, LDT, cw, r0, rows, w1);
            if (a.kw > w1) store_view(a.W2, T, LDT, cw + w1, r0, rows, a.kw - w1);
        }
        if (a.gram) {
#pragma unroll
            for (int bb = 0; bb < MAXB; ++bb) {
                if (!on[bb]) continue;
                const int step = (MAXB == 1) ? a.slices : 1;
                const int rstart = (MAXB == 1) ? sl : 0;
                const double* row = T + rstart * LDT;
                double a0 = acc[bb][0], a1 = acc[bb][1], a2 = acc[bb][2], a3 = acc[bb][3];
                for (int r = rstart; r < rows; r += step, row += step * LDT) {
                    const double l0 = row[lc0[bb]], l1 = row[lc1[bb]];
                    double q0 = row[rc0[bb]], q1 = row[rc1[bb]];
                    if (a.b) {
                        const double bw = row[cb];
                        q0 *= bw;
                        q1 *= bw;
                    }
                    a0 = fma(l0, q0, a0);
                    a1 = fma(l1, q0, a1);
                    a2 = fma(l0, q1, a2);
                    a3 = fma(l1, q1, a3);
                }
                acc[bb][0] = a0;
                acc[bb][1] = a1;
                acc[bb][2] = a2;
                acc[bb][3] = a3;
            }
        }
        __syncthreads();
    }
    cp_wait<0>();

    if (!a.gram) return;
    double* part = a.partial + static_cast<int64_t>(blockIdx.x) * a.P * a.Q;
    auto put = [&](int blk, const double* v) {
        const int i0 = 2 * (blk % nbi), j0 = 2 * (blk / nbi);
        part[i0 + j0 * a.P] = v[0];
        if (i0 + 1 < a.P) part[i0 + 1 + j0 * a.P] = v[1];
        if (j0 + 1 < a.Q) part[i0 + (j0 + 1) * a.P] = v[2];
        if (i0 + 1 < a.P && j0 + 1 < a.Q) part[i0 + 1 + (j0 + 1) * a.P] = v[3];
    };
    if (MAXB == 1) {
        // reduce row slices in fixed order through shared memory
        __syncthreads();
        double* red = smem;  // blockDim x 4
        for (int k = 0; k < 4; ++k) red[k * blockDim.x + threadIdx.x] = acc[0][k];
        __syncthreads();
        if (threadIdx.x < a.nb) {
            const int blk = threadIdx.x;
            double sred[4] = {0.0, 0.0, 0.0, 0.0};
            for (int s2 = 0; s2 < a.slices; ++s2)
                for (int k = 0; k < 4; ++k) sred[k] += red[k * blockDim.x + s2 * a.nb + blk];
            put(blk, sred);
        }
    } else {
#pragma unroll
        for (int bb = 0; bb < MAXB; ++bb) {
            const int blk = threadIdx.x + bb * blockDim.x;
            if (blk < a.nb) put(blk, acc[bb]);
        }
    }
}

// ---------------------------------------------------------------------------
// FP64 tensor-core variant (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4). Same
// staging and smem row layout as ts_tile_kernel; the block transform is a
// (64 x inner) x (inner x kw) product per tile (warp w owns rows 8w..8w+7) and
// the Gram is L^T diag(b) R with K = tile rows, 8x8 output blocks spread over
// warps by (block, k-step group). Per-warp fragments are combined in a fixed
// order, so results are run-to-run deterministic.
constexpr int kMaxItems = 4;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kTsThreads) ts_mma_kernel(const TsDev a) {
    extern __shared__ double smem[];
    constexpr int TR = kTR;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int u = a.u0 + a.u1;
    const bool need_u = (a.transform == TS_UPDATE) || (a.gram && a.left_u);
    const int cu = need_u ? u : 0;
    const int cv = cu, cw = cu + a.kv, cb = cw + a.kw;
    const int LDT = (cb + 1) | 1;
    const int stage_elems = TR * LDT;
    const int inner = a.transform == TS_UPDATE ? u : a.kv;
    double* Cs = smem + kStages * stage_elems;  // inner x kw, column-major
    if (a.transform != TS_NONE)
        for (int i = threadIdx.x; i < inner * a.kw; i += blockDim.x) {
            const int c = i / inner, q = i - c * inner;
            Cs[i] = a.C[q + static_cast<int64_t>(c) * a.ldc];
        }
    const int a_off = a.transform == TS_UPDATE ? 0 : cv;
    const int right_off = (a.transform == TS_NONE) ? cv : cw;
    const int uL = a.left_u ? u : 0;

    // gram work items: (8x8 block, k-step group)
    const int MB = (a.P + 7) / 8, NB = (a.Q + 7) / 8, nblk = MB * NB;
    const int kgroups = a.gram ? max(1, min(16, 8 / max(nblk, 1))) : 1;
    const int nitems = nblk * kgroups;
    double acc0[kMaxItems], acc1[kMaxItems];
    int lcol[kMaxItems], rcol[kMaxItems], kgi[kMaxItems];
    bool lok[kMaxItems], rok[kMaxItems], ion[kMaxItems];
#pragma unroll
    for (int t = 0; t < kMaxItems; ++t) {
        const int item = warp + t * (kTsThreads / 32);
        ion[t] = a.gram && item < nitems;
        const int blk = item % max(nblk, 1), kg = item / max(nblk, 1);
        const int mb = blk % max(MB, 1), nb = blk / max(MB, 1);
        const int mrow = mb * 8 + gid, ncol = nb * 8 + gid;
        lok[t] = mrow < a.P;
        rok[t] = ncol < a.Q;
        lcol[t] = mrow < uL ? mrow : right_off + (mrow - uL);
        rcol[t] = right_off + ncol;
        kgi[t] = kg;
        acc0[t] = acc1[t] = 0.0;
    }

    const int64_t ntiles = (a.n + TR - 1) / TR;
    const int64_t nt = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    auto issue = [&](int64_t i) {
        const int64_t r0 = (blockIdx.x + i * gridDim.x) * TR;
        const int rows = static_cast<int>(min(static_cast<int64_t>(TR), a.n - r0));
        double* T = smem + (i % kStages) * stage_elems;
        if (need_u) {
            if (a.u0) issue_view(T, LDT, 0, a.U0, r0, rows, a.u0);
            if (a.u1) issue_view(T, LDT, a.u0, a.U1, r0, rows, a.u1);
        }
        issue_view(T, LDT, cv, a.V, r0, rows, a.kv);
        if (a.gram && a.b)
            for (int r = threadIdx.x; r < rows; r += blockDim.x) cp_async8(T + r * LDT + cb, a.b + r0 + r);
        // zero the rows of a short tail tile so the fixed-size MMA steps read zeros
        for (int e = threadIdx.x; e < (TR - rows) * LDT; e += blockDim.x) T[rows * LDT + e] = 0.0;
    };

    for (int st = 0; st < kStages - 1; ++st) {
        if (st < nt) issue(st);
        cp_commit();
    }
    for (int64_t i = 0; i < nt; ++i) {
        if (i + kStages - 1 < nt) issue(i + kStages - 1);
        cp_commit();
        cp_wait<kStages - 1>();
        __syncthreads();
        const int64_t r0 = (blockIdx.x + i * gridDim.x) * TR;
        const int rows = static_cast<int>(min(static_cast<int64_t>(TR), a.n - r0));
        double* T = smem + (i % kStages) * stage_elems;

        if (a.transform != TS_NONE) {
            // rows 8*warp .. 8*warp+7 of W = A_in * C  (UPDATE: W = V - U*C)
            const double* arow = T + (warp * 8 + gid) * LDT + a_off;
            for (int nb = 0; nb * 8 < a.kw; ++nb) {
                double d0 = 0.0, d1 = 0.0;
                const int n = nb * 8 + gid;
                const double* ccol = Cs + min(n, a.kw - 1) * inner;
                for (int k0 = 0; k0 < inner; k0 += 4) {
                    const int k = k0 + tig;
                    const double av = k < inner ? arow[k] : 0.0;
                    const double bv = (k < inner && n < a.kw) ? ccol[k] : 0.0;
                    dmma(d0, d1, av, bv);
                }
                // d0, d1 = W[8*warp + gid][nb*8 + 2*tig + {0,1}]
                const int r = warp * 8 + gid;
                const int c0 = nb * 8 + 2 * tig;
                double* wrow = T + r * LDT;
                if (c0 < a.kw) wrow[cw + c0] = (a.transform == TS_UPDATE) ? wrow[cv + c0] - d0 : d0;
                if (c0 + 1 < a.kw) wrow[cw + c0 + 1] = (a.transform == TS_UPDATE) ? wrow[cv + c0 + 1] - d1 : d1;
            }
            __syncthreads();
            const int w1 = min(a.kw, a.W.cols);
            if (w1 > 0) store_view(a.W, T, LDT, cw, r0, rows, w1);
            if (a.kw > w1) store_view(a.W2, T, LDT, cw + w1, r0, rows, a.kw - w1);
        }
        if (a.gram) {
#pragma unroll
            for (int t = 0; t < kMaxItems; ++t) {
                if (!ion[t]) continue;
                for (int ks = kgi[t]; ks < TR / 4; ks += kgroups) {
                    const double* row = T + (ks * 4 + tig) * LDT;
                    const double av = lok[t] ? row[lcol[t]] : 0.0;
                    double bv = rok[t] ? row[rcol[t]] : 0.0;
                    if (a.b) bv *= row[cb];
                    dmma(acc0[t], acc1[t], av, bv);
                }
            }
        }
        __syncthreads();
    }
    cp_wait<0>();

    if (!a.gram) return;
    // fixed-order reduction: fragments -> smem [item][64] -> sum over k-groups per block
    __syncthreads();
    double* red = smem;  // nitems x 64
#pragma unroll
    for (int t = 0; t < kMaxItems; ++t) {
        if (!ion[t]) continue;
        const int item = warp + t * (kTsThreads / 32);
        red[item * 64 + gid * 8 + 2 * tig] = acc0[t];
        red[item * 64 + gid * 8 + 2 * tig + 1] = acc1[t];
    }
    __syncthreads();
    double* part = a.partial + static_cast<int64_t>(blockIdx.x) * a.P * a.Q;
    for (int e = threadIdx.x; e < a.P * a.Q; e += blockDim.x) {
        const int i = e % a.P, j = e / a.P;
        const int blk = (i / 8) + (j / 8) * MB;
        const int off = (i % 8) * 8 + (j % 8);
        double sum = 0.0;
        for (int kg = 0; kg < kgroups; ++kg) sum += red[(kg * nblk + blk) * 64 + off];
        part[i + j * a.P] = sum;
    }
}

// ---------------------------------------------------------------------------
// Column-major blocks fed by the bulk-copy engine (ts_bulk_kernel). Every
// operand column's tile segment (TR rows, contiguous) is one cp.async.bulk
// issued by a single thread into a ring of smem stages tracked by mbarriers,
// so staging costs a handful of instructions per tile instead of one per
// element. Smem columns have stride SC = TR + 4 doubles: both DMMA fragment
// shapes used here (8 rows x 4 columns for the transform's A, 4 rows x 8
// columns for the Gram) then hit every bank pair exactly twice (two
// wavefronts, conflict-free). The transform (W = V - U C or V C) runs on
// DMMA.8x8x4 per 8-row strip; the Gram splits the tile's k-steps over the
// warps; per-warp fragments are summed in a fixed order (deterministic).
constexpr int kBulkMaxBlk = 9;
constexpr size_t kFusedGramMax = 64;  // P*Q up to which the bulk kernel reduces its own Gram
constexpr int kBulkThreads = kTsThreads + 32;  // 8 consumer warps + 1 producer warp

// Stage layout (columns of SC doubles): U [0, u) | V [cV, cV+kv) | 3 zero | b.
// The zero columns pad the transform's k-steps past V (COMBINE) and stand in
// for Gram fragment rows/columns past P/Q; past U (UPDATE) the k-steps read V
// columns against zero rows of the padded C. Warp w owns the 8-row strips
// w, w+8, ... of every tile for both the transform and the Gram, so W (one
// per-CTA smem buffer) needs only warp-level synchronization and each tile
// costs one block barrier.
struct BulkCfg {
    int TR, SC, nst;
    int nload;        // bulk-loaded columns per stage
    int has_b;
    int ncol;         // columns per stage
    int cV, cb, zc;
};

template <int NBLK>  // Gram 8x8 blocks (MB*NB), compile-time so the k-step loop is straight-line
__global__ void __launch_bounds__(kBulkThreads, 2) ts_bulk_kernel(const TsDev a, const BulkCfg g) {
    constexpr int NCH = NBLK <= 2 ? 4 : (NBLK <= 4 ? 2 : 1);  // independent accumulator chains per block
    extern __shared__ __align__(128) double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int TR = g.TR, SC = g.SC;
    const int u = a.u0 + a.u1;
    const int inner = a.transform == TS_UPDATE ? u : (a.transform == TS_COMBINE_UV ? u + a.kv : a.kv);
    const int KBp = (inner + 3) / 4 * 4, NWp = (a.kw + 7) / 8 * 8;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem);  // full[nst] then empty[nst]
    uint64_t* ebar = bar + g.nst;
    const double** src = reinterpret_cast<const double**>(smem + 8);
    int* scol = reinterpret_cast<int*>(smem + 8 + 64);
    double* st0 = smem + 8 + 64 + 64;
    const size_t stage_elems = static_cast<size_t>(g.ncol) * SC;
    double* Wb = st0 + g.nst * stage_elems;              // kw columns
    double* Cs = Wb + static_cast<size_t>(a.kw) * SC;     // KBp x NWp column-major, zero padded
    if (threadIdx.x == 0) {
        for (int s2 = 0; s2 < g.nst; ++s2) {
            mbar_init(bar + s2, 1);
            mbar_init(ebar + s2, kTsThreads / 32);  // one arrival per consumer warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        int c = 0;
        if ((a.transform == TS_UPDATE) || (a.transform == TS_COMBINE_UV) || (a.gram && a.left_u)) {
            for (int j = 0; j < a.u0; ++j, ++c) { src[c] = a.U0.ptr + static_cast<int64_t>(j) * a.U0.cs; scol[c] = j; }
            for (int j = 0; j < a.u1; ++j, ++c) { src[c] = a.U1.ptr + static_cast<int64_t>(j) * a.U1.cs; scol[c] = a.u0 + j; }
        }
        for (int j = 0; j < a.kv; ++j, ++c) { src[c] = a.V.ptr + static_cast<int64_t>(j) * a.V.cs; scol[c] = g.cV + j; }
        if (g.has_b) { src[c] = a.b; scol[c] = g.cb; }
    }
    if (a.transform != TS_NONE)
        for (int i = threadIdx.x; i < KBp * NWp; i += blockDim.x) {
            const int c = i / KBp, q = i - c * KBp;
            Cs[i] = (q < inner && c < a.kw) ? a.C[q + static_cast<int64_t>(c) * a.ldc] : 0.0;
        }
    for (int s2 = 0; s2 < g.nst; ++s2)
        for (int e = threadIdx.x; e < 3 * TR; e += blockDim.x) {
            const int zz = e / TR, r = e - zz * TR;
            st0[s2 * stage_elems + static_cast<size_t>(g.zc + zz) * SC + r] = 0.0;
        }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();

    const int ntiles = static_cast<int>((a.n + TR - 1) / TR);
    const int nt = ntiles > static_cast<int>(blockIdx.x) ? (ntiles - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1 : 0;
    auto issue = [&](int tile, int s2) {
        const int64_t r0 = static_cast<int64_t>(tile) * TR;
        const int rows = static_cast<int>(min(static_cast<int64_t>(TR), a.n - r0));
        const int brows = rows & ~1;  // bulk sizes are multiples of 16 B
        double* T = st0 + s2 * stage_elems;
        mbar_expect_tx(bar + s2, static_cast<unsigned>(brows) * 8u * g.nload);
        if (brows > 0)
            for (int c = 0; c < g.nload; ++c) bulk_g2s(T + scol[c] * SC, src[c] + r0, brows * 8u, bar + s2);
    };
    const bool right_w = a.transform != TS_NONE;
    const int uL = a.left_u ? u : 0;
    const int MB = a.gram ? (a.P + 7) / 8 : 0, NB = a.gram ? (a.Q + 7) / 8 : 0;
    const int nblk = MB * NB;
    // per block: this lane's fragment column, in the stage (>= 0) or in W (-1 - col).
    // Two accumulator chains per block (DMMA latency ~137 cycles: independent
    // chains keep the tensor pipe busy); summed in a fixed order at the end.
    constexpr int NB1 = NBLK > 0 ? NBLK : 1;
    int lcol[NB1], rcol[NB1];
    double acc0[NB1][NCH], acc1[NB1][NCH];
    {
        int mb = 0, nb = 0;
#pragma unroll
        for (int t = 0; t < NB1; ++t) {
            const int mrow = mb * 8 + gid, ncol = nb * 8 + gid;
            int l = g.zc, r = g.zc;
            if (t < nblk && mrow < a.P) l = mrow < uL ? mrow : (right_w ? -1 - (mrow - uL) : g.cV + mrow - uL);
            if (t < nblk && ncol < a.Q) r = right_w ? -1 - ncol : g.cV + ncol;
            lcol[t] = l;
            rcol[t] = r;
#pragma unroll
            for (int c = 0; c < NCH; ++c) acc0[t][c] = acc1[t][c] = 0.0;
            if (++mb == MB) {
                mb = 0;
                ++nb;
            }
        }
    }
    const int a_col = (a.transform == TS_UPDATE || a.transform == TS_COMBINE_UV) ? 0 : g.cV;
    const int w1 = a.W.cols;
    const int spw = TR / 64;  // strips per warp per tile (warp w: strips w, w+8, ...)

    if (warp == kTsThreads / 32) {
        // producer warp: refill stage s once all consumer warps released it
        if (lane == 0) {
            int s2 = 0;
            unsigned eph = 0;
            for (int i = 0; i < nt; ++i) {
                if (i >= g.nst) mbar_wait(ebar + s2, eph);
                issue(blockIdx.x + i * gridDim.x, s2);
                if (++s2 == g.nst) {
                    s2 = 0;
                    if (i >= g.nst) eph ^= 1u;
                    else if (i + 1 == g.nst) eph = 0;
                }
            }
        }
    }
    else {
    int tile = blockIdx.x, s2 = 0;
    unsigned ph = 0;
    for (int i = 0; i < nt; ++i, tile += gridDim.x) {
        const int64_t r0 = static_cast<int64_t>(tile) * TR;
        const int rows = static_cast<int>(min(static_cast<int64_t>(TR), a.n - r0));
        double* T = st0 + s2 * stage_elems;
        mbar_wait(bar + s2, ph);
        if (rows < TR) {
            // tail tile (the CTA's last): odd last row by hand, zero rows [rows, TR)
            if (rows & 1)
                for (int c = threadIdx.x; c < g.nload; c += kTsThreads) T[scol[c] * SC + rows - 1] = src[c][r0 + rows - 1];
            for (int e = threadIdx.x; e < g.nload * (TR - rows); e += kTsThreads) {
                const int c = e / (TR - rows), r = rows + e - c * (TR - rows);
                T[scol[c] * SC + r] = 0.0;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kTsThreads) : "memory");  // consumers only
        }
        const double* lp[NB1];
        const double* rp[NB1];
#pragma unroll
        for (int t = 0; t < NB1; ++t) {
            lp[t] = (lcol[t] >= 0 ? T + lcol[t] * SC : Wb + (-1 - lcol[t]) * SC) + tig;
            rp[t] = (rcol[t] >= 0 ? T + rcol[t] * SC : Wb + (-1 - rcol[t]) * SC) + tig;
        }
        const double* bcol = T + g.cb * SC + tig;
        // groups of 4 strips: 4 independent DMMA chains in the transform
        for (int j0 = 0; j0 < spw; j0 += 4) {
            if (right_w) {
                for (int nb = 0; nb * 8 < a.kw; ++nb) {
                    double d0[4] = {0.0, 0.0, 0.0, 0.0}, d1[4] = {0.0, 0.0, 0.0, 0.0};
                    const double* ap = T + (a_col + tig) * SC + (warp + 8 * j0) * 8 + gid;
                    const double* cp = Cs + (nb * 8 + gid) * KBp + tig;
                    for (int k0 = 0; k0 < KBp; k0 += 4) {
                        const double cv = *cp;
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            if (j0 + j < spw) dmma(d0[j], d1[j], ap[j * 64], cv);
                        ap += 4 * SC;
                        cp += 4;
                    }
                    const int c0 = nb * 8 + 2 * tig;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (j0 + j >= spw) break;
                        const int rr = (warp + 8 * (j0 + j)) * 8 + gid;
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int cc = c0 + h;
                            if (cc < a.kw) {
                                double w = h ? d1[j] : d0[j];
                                if (a.transform == TS_UPDATE) w = T[(g.cV + cc) * SC + rr] - w;
                                Wb[cc * SC + rr] = w;
                                if (rr < rows) {
                                    double* dst = cc < w1 ? a.W.ptr + static_cast<int64_t>(cc) * a.W.cs
                                                          : a.W2.ptr + static_cast<int64_t>(cc - w1) * a.W2.cs;
                                    dst[r0 + rr] = w;
                                }
                            }
                        }
                    }
                }
                __syncwarp();
            }
            if (NBLK > 0) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (j0 + j >= spw) break;
                    const int sr = (warp + 8 * (j0 + j)) * 8;
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const int k0 = sr + 4 * kk;
                        const int ch = (j * 2 + kk) % NCH;
                        const double bb = g.has_b ? bcol[k0] : 1.0;
#pragma unroll
                        for (int t = 0; t < NBLK; ++t) {
                            double bv = rp[t][k0];
                            if (g.has_b) bv *= bb;
                            dmma(acc0[t][ch], acc1[t][ch], lp[t][k0], bv);
                        }
                    }
                }
            }
            if (right_w) __syncwarp();  // W rows of these strips are rewritten next tile
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(ebar + s2)) : "memory");
        if (++s2 == g.nst) {
            s2 = 0;
            ph ^= 1u;
        }
    }

    }
    if (!a.gram) return;
    double* red = st0;
    __syncthreads();  // all stages consumed (every full barrier waited)
#pragma unroll
    for (int t = 0; t < NB1; ++t) {
        if (warp < kTsThreads / 32 && t < nblk) {
            double s0 = acc0[t][0], s1 = acc1[t][0];
#pragma unroll
            for (int c = 1; c < NCH; ++c) {
                s0 += acc0[t][c];
                s1 += acc1[t][c];
            }
            red[(warp * nblk + t) * 64 + gid * 8 + 2 * tig] = s0;
            red[(warp * nblk + t) * 64 + gid * 8 + 2 * tig + 1] = s1;
        }
    }
    __syncthreads();
    double* part = a.partial + static_cast<int64_t>(blockIdx.x) * a.P * a.Q;
    for (int e = threadIdx.x; e < a.P * a.Q; e += blockDim.x) {
        const int i2 = e % a.P, j = e / a.P;
        const int blk = (i2 / 8) + (j / 8) * MB;
        const int off = (i2 % 8) * 8 + (j % 8);
        double sum = 0.0;
        for (int w = 0; w < kTsThreads / 32; ++w) sum += red[(w * nblk + blk) * 64 + off];
        part[i2 + j * a.P] = sum;
    }
    if (!a.counter) return;
    // last CTA: fixed-order (CTA 0, 1, ...) sum of the partials — the result does not
    // depend on which CTA finishes last (deterministic, same order as reduce_gram_kernel)
    __shared__ unsigned ticket;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) ticket = atomicAdd(a.counter, 1u);
    __syncthreads();
    if (ticket != gridDim.x - 1) return;
    __threadfence();
    const int PQ = a.P * a.Q;
    const int lane2 = threadIdx.x & 31;
    for (int e = warp; e < PQ; e += kBulkThreads / 32) {
        double s = 0.0;
        for (int r = lane2; r < static_cast<int>(gridDim.x); r += 32) s += __ldcg(a.partial + static_cast<int64_t>(r) * PQ + e);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (lane2 == 0) a.gram_out[e] = s;
    }
    if (threadIdx.x == 0) *a.counter = 0u;
}

__global__ void reduce_gram_kernel(const double* partial, int rows, int PQ, double* out) {
    const int e = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (e >= PQ) return;
    double s = 0.0;
    for (int r = lane; r < rows; r += 32) s += partial[static_cast<int64_t>(r) * PQ + e];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) out[e] = s;
}

__global__ void scale_cols_kernel(View v, const double* sc, int64_t n) {
    const int64_t total = n * v.cols;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = idx / v.cols;
        const int c = static_cast<int>(idx - r * v.cols);
        v.at(r, c) *= sc[c];
    }
}

__global__ void diag_apply_kernel(int64_t n, const double* d, View in, View out) {
    const int64_t total = n * in.cols;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = idx / in.cols;
        const int c = static_cast<int>(idx - r * in.cols);
        out.at(r, c) = __dmul_rn(d[r], in.at(r, c));
    }
}

struct ColList {
    int k;
    int idx[kMaxCols];
};

__global__ void gather_cols_kernel(int64_t n, View in, ColList cl, View out) {
    const int64_t total = n * cl.k;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = idx / cl.k;
        const int c = static_cast<int>(idx - r * cl.k);
        out.at(r, c) = in.at(r, cl.idx[c]);
    }
}

__global__ void fill_kernel(int64_t n, View v, double value) {
    const int64_t total = n * v.cols;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = idx / v.cols;
        const int c = static_cast<int>(idx - r * v.cols);
        v.at(r, c) = value;
    }
}

__global__ void scal_kernel(int64_t n, double a, View in, View out) {
    const int64_t total = n * in.cols;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = idx / in.cols;
        const int c = static_cast<int>(idx - r * in.cols);
        out.at(r, c) = __dmul_rn(a, in.at(r, c));
    }
}

int elem_grid(int64_t total) { return grid_for(total, 256, 8); }

__global__ void colsum_kernel(int64_t n, View v, double* partial) {
    // thread-private sums over a grid-stride of rows, then fixed-order CTA tree
    __shared__ double red[256];
    for (int c = 0; c < v.cols; ++c) {
        double s = 0.0;
        for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < n;
             r += static_cast<int64_t>(gridDim.x) * blockDim.x)
            s += v.at(r, c);
        red[threadIdx.x] = s;
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) partial[static_cast<int64_t>(blockIdx.x) * v.cols + c] = red[0];
        __syncthreads();
    }
}

struct Theta {
    double t[kMaxCols];
};
__global__ void residual_ax_kernel(int64_t n, int m, View X, View AX, const double* bdiag, const Theta th, View R,
                                   double* partial) {
    __shared__ double red[256];
    for (int c = 0; c < m; ++c) {
        double s = 0.0;
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const double x = X.at(i, c);
            const double bx = bdiag ? __dmul_rn(bdiag[i], x) : x;
            const double r = __dsub_rn(AX.at(i, c), __dmul_rn(th.t[c], bx));
            R.at(i, c) = r;
            s += r * r;
        }
        red[threadIdx.x] = s;
        __syncthreads();
        for (int w = 128; w > 0; w >>= 1) {
            if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
            __syncthreads();
        }
        if (threadIdx.x == 0) partial[static_cast<int64_t>(blockIdx.x) * m + c] = red[0];
        __syncthreads();
    }
}

} // namespace

int residual_from_ax(int64_t n, const View& X, const View& AX, const double* bdiag, const double* theta_host,
                     int m, const View& R, double* partial, cudaStream_t s) {
    if (m > kMaxCols) throw_dimension("residual_from_ax: too many columns");
    Theta th{};
    for (int c = 0; c < m; ++c) th.t[c] = theta_host[c];
    const int grid = grid_for(std::max<int64_t>(n, 1), 256, 2);
    residual_ax_kernel<<<grid, 256, 0, s>>>(n, m, X, AX, bdiag, th, R, partial);
    SPB_LAUNCH_CHECK();
    return grid;
}

int colsum_partials(int64_t n, const View& v, double* scratch, cudaStream_t s) {
    const int grid = grid_for(n, 256, 2);
    colsum_kernel<<<grid, 256, 0, s>>>(n, v, scratch);
    SPB_LAUNCH_CHECK();
    return grid;
}

int ts_run(const TsSpec& s, double* gram_out, double* scratch, size_t scratch_elems, cudaStream_t st) {
    TsDev a{};
    a.n = s.n;
    a.U0 = s.U0;
    a.U1 = s.U1;
    a.V = s.V;
    a.W = s.W;
    a.W2 = s.W2;
    a.C = s.C;
    a.b = s.b;
    a.transform = s.transform;
    a.u0 = s.U0.ptr ? s.U0.cols : 0;
    a.u1 = s.U1.ptr ? s.U1.cols : 0;
    a.kv = s.V.cols;
    a.kw = 0;
    if (s.transform == TS_UPDATE) a.kw = a.kv;
    if (s.transform == TS_COMBINE || s.transform == TS_COMBINE_UV) a.kw = s.W.cols + (s.W2.ptr ? s.W2.cols : 0);
    a.gram = s.gram ? 1 : 0;
    a.left_u = s.gram_left_u ? 1 : 0;
    a.left_self = s.gram_left_self ? 1 : 0;
    const int rq = s.transform == TS_NONE ? a.kv : a.kw;
    a.Q = rq;
    a.P = (a.left_u ? a.u0 + a.u1 : 0) + (a.left_self ? rq : 0);
    if (s.n <= 0) return a.P;

    int maxb = 1;
    if (a.gram) {
        a.nb = ((a.P + 1) / 2) * ((a.Q + 1) / 2);
        if (a.nb <= kTsThreads) {
            a.slices = kTsThreads / a.nb;
        } else {
            a.slices = 1;
            maxb = (a.nb + kTsThreads - 1) / kTsThreads;
        }
    } else {
        a.nb = 1;
        a.slices = 1;
    }
    const int u = a.u0 + a.u1;
    const int inner = s.transform == TS_UPDATE ? u : (s.transform == TS_COMBINE_UV ? u + a.kv : a.kv);
    a.ldc = s.ldc > 0 ? s.ldc : inner;
    const bool need_u = (s.transform == TS_UPDATE) || (s.transform == TS_COMBINE_UV) || (s.gram && s.gram_left_u);
    const int LDT = ((need_u ? u : 0) + a.kv + a.kw + 1) | 1;
    size_t sm = sizeof(double) * (static_cast<size_t>(kStages) * kTR * LDT +
                                  (s.transform != TS_NONE ? static_cast<size_t>(inner) * a.kw : 0));
    sm = std::max(sm, sizeof(double) * 4 * kTsThreads);
    const int per_sm = static_cast<int>(std::max<size_t>(1, std::min<size_t>(8, (200 * 1024) / sm)));
    const int64_t ntiles = (s.n + kTR - 1) / kTR;
    int grid = grid_for(ntiles, 1, per_sm);
    const size_t PQ = static_cast<size_t>(a.P) * a.Q;
    if (a.gram) {
        // shrink the grid if the partial scratch is too small (keeps determinism: grid is a
        // pure function of (n, P, Q, scratch size))
        while (static_cast<size_t>(grid) * PQ > scratch_elems && grid > 1) grid = (grid + 1) / 2;
        if (static_cast<size_t>(grid) * PQ > scratch_elems)
            throw SpError(1, "ts_run: gram scratch too small");
    }
    a.partial = scratch;
    auto launch = [&](auto kern) {
        if (sm > 48 * 1024) SPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
        kern<<<grid, kTsThreads, sm, st>>>(a);
    };
    const int nblk = ((a.P + 7) / 8) * ((a.Q + 7) / 8);
    // column-major operands: direct-fragment kernel (no staging)
    auto cm = [](const View& v, int cols) { return cols == 0 || v.rs == 1; };
    const bool colmajor_all = cm(s.U0, a.u0) && cm(s.U1, a.u1) && cm(s.V, a.kv) &&
                              (s.transform == TS_NONE || (cm(s.W, s.W.cols) && (!s.W2.ptr || cm(s.W2, s.W2.cols))));
    // bulk-copy kernel for aligned column-major operands (meshes' default)
    auto aligned = [](const View& v, int cols) {
        return cols == 0 || (reinterpret_cast<uintptr_t>(v.ptr) % 16 == 0 && (cols == 1 || v.cs % 2 == 0));
    };
    const int nblk_b = a.gram ? ((a.P + 7) / 8) * ((a.Q + 7) / 8) : 0;
    const int nw1 = s.transform == TS_NONE ? 0 : s.W.cols, nw2 = s.transform == TS_NONE ? 0 : a.kw - nw1;
    if (colmajor_all && aligned(s.U0, a.u0) && aligned(s.U1, a.u1) &&
        aligned(s.V, a.kv) && aligned(s.W, nw1) && aligned(s.W2, nw2) &&
        (!s.b || reinterpret_cast<uintptr_t>(s.b) % 16 == 0) && nblk_b <= kBulkMaxBlk &&
        a.u0 + a.u1 + a.kv + 1 <= 64 && a.kw <= 64) {
        BulkCfg g{};
        g.has_b = (a.gram && s.b) ? 1 : 0;
        const int cu_b = need_u ? u : 0;
        g.nload = cu_b + a.kv + g.has_b;
        g.cV = cu_b;
        g.zc = g.cV + a.kv;
        g.cb = g.zc + 3;
        g.ncol = g.cb + g.has_b;
        size_t smb = 0;
        bool found = false;
        const int KBp = (inner + 3) / 4 * 4, NWp = (a.kw + 7) / 8 * 8;
        // tile rows: ~48 KB of loaded columns per stage, 64..2048 rows
        int TR = 64;
        while (TR < 2048 && static_cast<size_t>(g.nload) * (2 * TR) * 8 <= static_cast<size_t>(48) * 1024) TR *= 2;
        for (; TR >= 64 && !found; TR /= 2) {
            for (int nst : {4, 3, 2}) {
                const int SC = TR + 4;
                const size_t stage = static_cast<size_t>(g.ncol) * SC;
                size_t bytes = sizeof(double) * (8 + 64 + 64 + nst * stage + static_cast<size_t>(a.kw) * SC +
                                                 static_cast<size_t>(KBp) * NWp);
                const size_t red = sizeof(double) * (200 + 64 * static_cast<size_t>(kTsThreads / 32) * std::max(nblk_b, 1));
                bytes = std::max(bytes, red);
                if (bytes <= 112 * 1024) {
                    g.TR = TR;
                    g.SC = SC;
                    g.nst = nst;
                    smb = bytes;
                    found = true;
                    break;
                }
            }
        }
        if (found) {
            const int per_sm = static_cast<int>(std::max<size_t>(1, std::min<size_t>(2, (227 * 1024) / smb)));
            const int64_t nt2 = (s.n + g.TR - 1) / g.TR;
            int gridb = grid_for(nt2, 1, per_sm);
            if (a.gram) {
                // the last scratch element is the fused reduction's counter
                while (static_cast<size_t>(gridb) * PQ + 1 > scratch_elems && gridb > 1) gridb = (gridb + 1) / 2;
            }
            static void (*const kerns[kBulkMaxBlk + 1])(const TsDev, const BulkCfg) = {
                ts_bulk_kernel<0>, ts_bulk_kernel<1>, ts_bulk_kernel<2>, ts_bulk_kernel<3>, ts_bulk_kernel<4>,
                ts_bulk_kernel<5>, ts_bulk_kernel<6>, ts_bulk_kernel<7>, ts_bulk_kernel<8>, ts_bulk_kernel<9>};
            static bool attr_set = false;  // once, at the maximum (no attribute changes between launches)
            if (!attr_set) {
                for (auto k : kerns)
                    SPB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
                attr_set = true;
            }
            // small Grams reduce inside the kernel (the last CTA); larger ones keep the
            // separate wide reduction (one warp per element over every CTA)
            const bool fused = a.gram && PQ <= kFusedGramMax && scratch_elems >= PQ * gridb + 1;
            a.gram_out = fused ? gram_out : nullptr;
            a.counter = fused ? reinterpret_cast<unsigned*>(scratch + scratch_elems - 1) : nullptr;
            kerns[nblk_b]<<<gridb, kBulkThreads, smb, st>>>(a, g);
            SPB_LAUNCH_CHECK();
            if (a.gram && !fused) {
                reduce_gram_kernel<<<ceil_div(static_cast<int64_t>(PQ), 4), 128, 0, st>>>(scratch, gridb,
                                                                                      static_cast<int>(PQ), gram_out);
                SPB_LAUNCH_CHECK();
            }
            return a.P;
        }
    }
    if (s.transform == TS_COMBINE_UV) throw SpError(1, "ts_run: combine over [U | V] needs aligned column-major operands");
    const bool mma_ok = (!a.gram || nblk <= kMaxItems * (kTsThreads / 32));
    if (mma_ok) {
        // reduction scratch: nitems x 64 doubles must fit in the staged smem
        const int kgroups = a.gram ? std::max(1, std::min(16, 8 / std::max(nblk, 1))) : 1;
        const size_t need = sizeof(double) * 64 * static_cast<size_t>(nblk * kgroups);
        size_t sm2 = std::max(sm, need);
        if (sm2 > 48 * 1024)
            SPB_CUDA(cudaFuncSetAttribute(ts_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm2)));
        ts_mma_kernel<<<grid, kTsThreads, sm2, st>>>(a);
    } else if (maxb <= 1) launch(ts_tile_kernel<1>);
    else if (maxb <= 2) launch(ts_tile_kernel<2>);
    else if (maxb <= 4) launch(ts_tile_kernel<4>);
    else if (maxb <= 8) launch(ts_tile_kernel<8>);
    else if (maxb <= 16) launch(ts_tile_kernel<16>);
    else throw_dimension("ts_run: gram too large");
    SPB_LAUNCH_CHECK();
    if (a.gram) {
        reduce_gram_kernel<<<ceil_div(static_cast<int64_t>(PQ), 4), 128, 0, st>>>(
            scratch, grid, static_cast<int>(PQ), gram_out);
        SPB_LAUNCH_CHECK();
    }
    return a.P;
}

void scale_cols(View V, const double* colscale_dev, cudaStream_t s, int64_t n) {
    if (n <= 0 || V.cols <= 0) return;
    scale_cols_kernel<<<elem_grid(n * V.cols), 256, 0, s>>>(V, colscale_dev, n);
    SPB_LAUNCH_CHECK();
}

void diag_apply(int64_t n, const double* d, View in, View out, cudaStream_t s) {
    if (n <= 0 || in.cols <= 0) return;
    diag_apply_kernel<<<elem_grid(n * in.cols), 256, 0, s>>>(n, d, in, out);
    SPB_LAUNCH_CHECK();
}

void jacobi_apply(int64_t n, const double* inv_diag, View in, View out, cudaStream_t s) {
    diag_apply(n, inv_diag, in, out, s);
}

void copy_view(int64_t n, View in, View out, cudaStream_t s) {
    if (n <= 0 || in.cols <= 0) return;
    scal_kernel<<<elem_grid(n * in.cols), 256, 0, s>>>(n, 1.0, in, out);
    SPB_LAUNCH_CHECK();
}

void poly_first_only(int64_t n, double inv0, View R, View H, cudaStream_t s) {
    if (n <= 0 || R.cols <= 0) return;
    scal_kernel<<<elem_grid(n * R.cols), 256, 0, s>>>(n, inv0, R, H);
    SPB_LAUNCH_CHECK();
}

void gather_cols(int64_t n, View in, const int* cols_host, int k, View out, cudaStream_t s) {
    if (n <= 0 || k <= 0) return;
    if (k > kMaxCols) throw_dimension("gather_cols: too many columns");
    ColList cl{};
    cl.k = k;
    for (int i = 0; i < k; ++i) cl.idx[i] = cols_host[i];
    gather_cols_kernel<<<elem_grid(n * k), 256, 0, s>>>(n, in, cl, out);
    SPB_LAUNCH_CHECK();
}

void fill_view(int64_t n, View v, double value, cudaStream_t s) {
    if (n <= 0 || v.cols <= 0) return;
    fill_kernel<<<elem_grid(n * v.cols), 256, 0, s>>>(n, v, value);
    SPB_LAUNCH_CHECK();
}

} // namespace spb
