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
#include "p2p.cuh"
#include "spmm_epilogue.cuh"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace spb {

namespace {

constexpr int kThreads = 256;

// X loads of the SpMM kernels. With the halo exchange fused in (HF), peers write
// the halo rows of X while the kernel runs, so X is not read-only for the
// kernel's lifetime and ld.global.nc is not allowed: use L2-coherent loads.
template <bool HF> __device__ __forceinline__ double ldx(const double* p) {
    if constexpr (HF) return __ldcg(p);
    else return __ldg(p);
}

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
        const int64_t kdiag = op.dpos ? k0 + op.dpos[row] : -1;
        for (int64_t kb = k0; kb < k1; kb += G) {
            const int cnt = static_cast<int>(min(static_cast<int64_t>(G), k1 - kb));
            int jl = 0;
            double vl = 0.0;
            if (gl < cnt) {
                jl = __ldg(op.cols + kb + gl);
                if (MODE == OP_EXPLICIT) vl = __ldg(op.vals + kb + gl);
                if (MODE == OP_NORMAL_UNIT) vl = __dmul_rn(-isdi, __ldg(op.isd + jl));
            }
            // gathers issued U at a time ahead of the ordered accumulation
            constexpr int U = G < 8 ? G : 8;
#pragma unroll
            for (int t0 = 0; t0 < G; t0 += U) {
            if (t0 >= cnt) break;
            int jt[U];
            double xt[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                jt[u] = __shfl_sync(gmask, jl, t0 + u, G);
                xt[u] = (act && t0 + u < cnt) ? X.at(jt[u], c) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = t0 + u;
                if (t >= cnt) break;
                const int j = jt[u];
                double v = 0.0;
                if (MODE == OP_EXPLICIT || MODE == OP_NORMAL_UNIT) v = __shfl_sync(gmask, vl, t, G);
                const double xj = xt[u];
                const bool at_diag = op.dpos ? (kb + t == kdiag) : (j > grow);
                if (MODE == OP_LAPLACE_UNIT) {
                    if (!placed && at_diag) {
                        acc = __dadd_rn(acc, __dmul_rn(dval, xi));
                        placed = true;
                    }
                    acc = __dsub_rn(acc, xj);  // (-1.0) * x_j added: exact negation
                } else if (MODE == OP_NORMAL_UNIT) {
                    if (!placed && at_diag) {
                        acc = __dadd_rn(acc, xi);  // 1.0 * x_i
                        placed = true;
                    }
                    acc = __dadd_rn(acc, __dmul_rn(v, xj));
                } else {
                    acc = __dadd_rn(acc, __dmul_rn(v, xj));
                }
            }
            }
        }
        if (MODE == OP_LAPLACE_UNIT && !placed) acc = __dadd_rn(acc, __dmul_rn(dval, xi));
        if (MODE == OP_NORMAL_UNIT && !placed) acc = __dadd_rn(acc, xi);
        return acc;
    }
};

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
// consecutive rows: it loads their offsets and the contiguous column-index
// segment (<= 32*32 entries) with coalesced loads into shared memory, computes
// each row's length and diagonal slot once (lane = row), then its 32/G groups
// walk (row, column-chunk) items. Each item issues all its gathers before
// accumulating (fully unrolled, predicated, 32-bit index math), and short rows
// are processed two items per group iteration to keep more loads in flight.
// X, Y and H are row-major (cs == 1) with 32-bit row*ld products.
constexpr int kTileRows = 32;
constexpr int kTileCap = 32 * 32;

struct TileArgs {
    const double* X;
    int ldx;
    double* Y;
    int ldy;
    double* H;
    int ldh;
    int m;
};

template <int MAXR, int MODE>
struct ItemLoad {
    double xv[MAXR];
    double vv[MAXR];  // explicit values / normalized coefficients
    double xi, h;
    int len, kd, c;
    int64_t row;
    bool act;
};

template <int G, int MAXR, int MODE, int EPI>
__device__ __forceinline__ void tile_item_load(ItemLoad<MAXR, MODE>& it, const DevOp& op, const TileArgs& ta,
                                               const EpiArgs& ea, const int32_t* sc, const double* sv,
                                               const int* s_start, const int* s_len, const int* s_kd,
                                               int64_t r0, int rr, int ch, int gl, const char* xbase,
                                               uint32_t ld8) {
    it.c = ch * G + gl;
    it.act = it.c < ta.m;
    it.row = r0 + rr;
    const int st = s_start[rr];
    it.len = it.act ? s_len[rr] : 0;
    it.kd = s_kd[rr];
    const char* xc = xbase + 8u * static_cast<uint32_t>(it.c);
    const uint32_t grow = static_cast<uint32_t>(op.row0 + it.row);
    it.xi = it.act ? *reinterpret_cast<const double*>(xc + static_cast<uint64_t>(grow) * ld8) : 0.0;
    it.h = 0.0;
    if (EPI == EPI_POLY && !ea.first && ea.h_terms && it.act) it.h = ta.H[static_cast<int>(it.row) * ta.ldh + it.c];
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
        if (k < it.len) {
            const uint32_t j = static_cast<uint32_t>(sc[st + k]);
            it.xv[k] = __ldg(reinterpret_cast<const double*>(xc + static_cast<uint64_t>(j) * ld8));
            if (MODE == OP_EXPLICIT || MODE == OP_NORMAL_UNIT) it.vv[k] = sv[st + k];
        }
    }
}

template <int MAXR, int MODE, int EPI>
__device__ __forceinline__ void tile_item_finish(const ItemLoad<MAXR, MODE>& it, const DevOp& op,
                                                 const TileArgs& ta, const EpiArgs& ea, const double* s_theta,
                                                 double& sq) {
    if (!it.act) return;
    double acc = 0.0;
    double dterm = 0.0;
    if (MODE == OP_LAPLACE_UNIT) dterm = __dmul_rn(op.diag[it.row], it.xi);
    if (MODE == OP_NORMAL_UNIT) dterm = it.xi;
#pragma unroll
    for (int k = 0; k < MAXR; ++k) {
        if (k < it.len) {
            if (MODE == OP_LAPLACE_UNIT) {
                if (k == it.kd) acc = __dadd_rn(acc, dterm);
                acc = __dsub_rn(acc, it.xv[k]);
            } else if (MODE == OP_NORMAL_UNIT) {
                if (k == it.kd) acc = __dadd_rn(acc, dterm);
                acc = __dadd_rn(acc, __dmul_rn(it.vv[k], it.xv[k]));
            } else {
                acc = __dadd_rn(acc, __dmul_rn(it.vv[k], it.xv[k]));
            }
        }
    }
    if ((MODE == OP_LAPLACE_UNIT || MODE == OP_NORMAL_UNIT) && it.kd >= it.len) acc = __dadd_rn(acc, dterm);
    const int yoff = static_cast<int>(it.row) * ta.ldy + it.c;
    if (EPI == EPI_STORE) {
        ta.Y[yoff] = acc;
    } else if (EPI == EPI_RESIDUAL) {
        const double bx = ea.bdiag ? __dmul_rn(ea.bdiag[it.row], it.xi) : it.xi;
        const double r = __dsub_rn(acc, __dmul_rn(s_theta[it.c], bx));
        ta.Y[yoff] = r;
        sq = fma(r, r, sq);
    } else {
        const double pn = __dsub_rn(it.xi, __dmul_rn(ea.inv_cur, acc));
        ta.Y[yoff] = pn;
        if (ea.h_terms) ta.H[static_cast<int>(it.row) * ta.ldh + it.c] = poly_h(ea, it.h, it.xi, pn);
    }
}

template <int G, int MAXR, int RPI, int MODE, int EPI>
__global__ void __launch_bounds__(kThreads) spmm_tile_kernel(const DevOp op, const TileArgs ta, const EpiArgs ea) {
    constexpr int GPW = 32 / G;
    constexpr bool kVals = (MODE == OP_EXPLICIT || MODE == OP_NORMAL_UNIT);
    extern __shared__ int32_t s_dyn[];
    __shared__ int s_start_all[kThreads / 32][kTileRows + 1];
    __shared__ int s_len_all[kThreads / 32][kTileRows];
    __shared__ int s_kd_all[kThreads / 32][kTileRows];
    __shared__ double s_theta[kMaxCols];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    int32_t* sc = s_dyn + warp * kTileCap;
    double* sv = reinterpret_cast<double*>(s_dyn + (kThreads / 32) * kTileCap) + warp * kTileCap;
    int* s_start = s_start_all[warp];
    int* s_len = s_len_all[warp];
    int* s_kd = s_kd_all[warp];
    if (EPI == EPI_RESIDUAL) {
        for (int c = threadIdx.x; c < ta.m; c += kThreads) s_theta[c] = ea.theta[c];
        __syncthreads();
    }
    const int gl = lane & (G - 1);
    const int gw = lane / G;
    const int nch = (ta.m + G - 1) / G;
    const char* xbase = reinterpret_cast<const char*>(ta.X);
    const uint32_t ld8 = 8u * static_cast<uint32_t>(ta.ldx);
    double sq = 0.0;
    const int64_t ntiles = (op.n + kTileRows - 1) / kTileRows;
    const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + warp;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
    for (int64_t tile = gwarp; tile < ntiles; tile += nwarps) {
        const int64_t r0 = tile * kTileRows;
        const int nr = static_cast<int>(min(static_cast<int64_t>(kTileRows), op.n - r0));
        const int64_t ko = op.offs[r0 + min(lane, nr)];
        const int64_t kbeg = __shfl_sync(0xffffffffu, ko, 0);
        const int64_t kn = __shfl_down_sync(0xffffffffu, ko, 1);
        const int64_t kend = op.offs[r0 + nr];
        const int total = static_cast<int>(kend - kbeg);
        __syncwarp();
        for (int e = lane; e < total; e += 32) {
            const int j = __ldg(op.cols + kbeg + e);
            sc[e] = j;
            if (MODE == OP_EXPLICIT) sv[e] = __ldg(op.vals + kbeg + e);
            if (MODE == OP_NORMAL_UNIT) sv[e] = __ldg(op.isd + j);
        }
        __syncwarp();
        if (lane < nr) {
            const int st = static_cast<int>(ko - kbeg);
            const int len = static_cast<int>((lane + 1 < nr ? kn : kend) - ko);
            const int64_t grow = op.row0 + r0 + lane;
            int kd = 0;
            if (MODE == OP_LAPLACE_UNIT || MODE == OP_NORMAL_UNIT) {
                if (op.dpos) kd = op.dpos[r0 + lane];
                else
                    while (kd < len && sc[st + kd] < grow) ++kd;
                if (MODE == OP_NORMAL_UNIT) {
                    const double nisdi = -op.isd[grow];
                    for (int k = 0; k < len; ++k) sv[st + k] = __dmul_rn(nisdi, sv[st + k]);
                }
            }
            s_start[lane] = st;
            s_len[lane] = len;
            s_kd[lane] = kd;
        }
        __syncwarp();
        const int items = nr * nch;
        for (int it0 = gw; it0 < items; it0 += GPW * RPI) {
            ItemLoad<MAXR, MODE> A;
            const int rA = nch == 1 ? it0 : it0 / nch;
            tile_item_load<G, MAXR, MODE, EPI>(A, op, ta, ea, sc, sv, s_start, s_len, s_kd, r0, rA,
                                               it0 - rA * nch, gl, xbase, ld8);
            if (RPI == 2) {
                const int it1 = it0 + GPW;
                ItemLoad<MAXR, MODE> B;
                const int rB = nch == 1 ? it1 : it1 / nch;
                if (it1 < items)
                    tile_item_load<G, MAXR, MODE, EPI>(B, op, ta, ea, sc, sv, s_start, s_len, s_kd, r0, rB,
                                                       it1 - rB * nch, gl, xbase, ld8);
                tile_item_finish<MAXR, MODE, EPI>(A, op, ta, ea, s_theta, sq);
                if (it1 < items) tile_item_finish<MAXR, MODE, EPI>(B, op, ta, ea, s_theta, sq);
            } else {
                tile_item_finish<MAXR, MODE, EPI>(A, op, ta, ea, s_theta, sq);
            }
        }
        __syncwarp();
    }
    if (EPI == EPI_RESIDUAL) {
        __shared__ double red[kThreads];
        red[threadIdx.x] = sq;
        __syncthreads();
        if (threadIdx.x < ta.m) {
            double s = 0.0;
            for (int g = 0; g < kThreads / G; ++g) s += red[g * G + threadIdx.x];
            ea.partial[static_cast<int64_t>(blockIdx.x) * ta.m + threadIdx.x] = s;
        }
    }
}


// Column-major "row per lane" kernel for short rows (max_row <= 32, meshes).
// X, Y, H column-major: element (r, c) at c*ld + r. A warp owns 32 consecutive
// rows (one per lane). Each lane first turns its row into MAXR slots
// (byte offset, weight) in the exact storage order of the explicit CSR of L —
// off-diagonals (offset j, weight -1 / (-isd_i)*isd_j / a_ij) with the diagonal
// (offset i, weight deg / 1.0) spliced in before the first column > i — then
// every column is a branch-free chain acc += w_k * X[c][o_k]. The products are
// the reference's products (spmv_block: acc += a_ik * x_k), so the result is
// bit-identical; padded slots add +-0, which cannot change an accumulator that
// starts at +0 (round-to-nearest never produces -0 from +0 by addition).
// For mesh orderings the 32 lanes gather 32 consecutive addresses per slot.
template <int MAXR, int MODE, int EPI, int CBT = 2, int MINB = 1, bool HF = false>
__global__ void __launch_bounds__(kThreads, MINB) spmm_col_kernel(const DevOp op, const TileArgs ta, const EpiArgs ea,
                                                                   const HaloFuse hf) {
    constexpr bool kRegs = MAXR <= 8;       // slots in registers, several columns per pass
    constexpr int NS = MAXR + 1;            // + the diagonal slot
    constexpr int NSR = kRegs ? NS : 1;
    __shared__ double s_sq[kThreads / 32][kMaxCols];
    __shared__ double s_theta[kMaxCols];
    extern __shared__ uint32_t s_slot_dyn[];  // !kRegs: [warp][slot][lane] offsets, then weights
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int m = ta.m;
    // multi-GPU: push this rank's boundary rows into the peers' X first (p2p.cuh)
    if (HF && !hf.nopush)
        halo_push_part(hf, m, [&](int64_t r, int c) {
            return const_cast<double*>(ta.X) + static_cast<int64_t>(c) * ta.ldx + r;
        });
    if (EPI == EPI_RESIDUAL) {
        for (int c = threadIdx.x; c < m; c += kThreads) s_theta[c] = ea.theta[c];
        for (int c = lane; c < m; c += 32) s_sq[warp][c] = 0.0;
        __syncthreads();
    }
    uint32_t* so = s_slot_dyn + warp * NS * 32;
    double* sw = reinterpret_cast<double*>(s_slot_dyn + (kThreads / 32) * NS * 32) + warp * NS * 32;
    const int64_t ntiles = (op.n + 31) / 32;
    const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + warp;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
    const uint64_t ldx8 = 8ull * static_cast<uint32_t>(ta.ldx);
    const char* xbase = reinterpret_cast<const char*>(ta.X);
    bool waited = false;
    for (int64_t lt = gwarp; lt < ntiles; lt += nwarps) {
        int64_t tile = lt;
        if (HF) {
            // interior tiles first; the first halo-reading tile waits for the peers
            if (lt >= hf.n_int && !waited) {
                halo_wait_warp(hf);
                waited = true;
            }
            tile = (lt + hf.rot) % ntiles;
        }
        const int64_t row = tile * 32 + lane;
        const bool live = row < op.n;
        const int64_t grow = op.row0 + row;
        const uint32_t grow8 = 8u * static_cast<uint32_t>(live ? grow : op.row0);
        int64_t k0 = 0;
        int len = 0;
        if (live) {
            k0 = op.offs[row];
            len = static_cast<int>(op.offs[row + 1] - k0);
        }
        // ---- slots of this row: independent loads first, then the splice
        uint32_t ro[NSR];
        double rw[NSR];
        {
            double dw = 0.0, nisdi = 0.0;
            if (MODE == OP_LAPLACE_UNIT && live) dw = op.diag[row];
            if (MODE == OP_NORMAL_UNIT && live) {
                dw = 1.0;
                nisdi = -op.isd[grow];
            }
            int jv[MAXR];
            double wv[MAXR];
#pragma unroll
            for (int k = 0; k < MAXR; ++k) jv[k] = (k < len) ? __ldg(op.cols + k0 + k) : 0;
#pragma unroll
            for (int k = 0; k < MAXR; ++k) {
                wv[k] = 0.0;
                if (k < len) {
                    if (MODE == OP_LAPLACE_UNIT) wv[k] = -1.0;
                    else if (MODE == OP_NORMAL_UNIT) wv[k] = __dmul_rn(nisdi, __ldg(op.isd + jv[k]));
                    else wv[k] = __ldg(op.vals + k0 + k);
                }
            }
            int kd = MAXR + 1;  // explicit CSR: the diagonal is a stored entry
            if (MODE != OP_EXPLICIT) {
                kd = 0;
                if (op.dpos) {
                    kd = live ? op.dpos[row] : 0;
                } else {
#pragma unroll
                    for (int k = 0; k < MAXR; ++k) kd += (k < len && jv[k] < grow) ? 1 : 0;
                }
            }
#pragma unroll
            for (int sidx = 0; sidx < NS; ++sidx) {
                // slot sidx holds entry sidx before the diagonal, entry sidx-1 after it
                uint32_t o = grow8;
                double w = 0.0;
                if (sidx < kd) {
                    if (sidx < MAXR && sidx < len) {
                        o = 8u * static_cast<uint32_t>(jv[sidx < MAXR ? sidx : 0]);
                        w = wv[sidx < MAXR ? sidx : 0];
                    }
                } else if (sidx == kd) {
                    w = live ? dw : 0.0;
                } else if (sidx - 1 < len) {
                    o = 8u * static_cast<uint32_t>(jv[sidx >= 1 ? sidx - 1 : 0]);
                    w = wv[sidx >= 1 ? sidx - 1 : 0];
                }
                if (kRegs) {
                    ro[sidx < NSR ? sidx : 0] = o;
                    rw[sidx < NSR ? sidx : 0] = w;
                } else {
                    so[sidx * 32 + lane] = o;
                    sw[sidx * 32 + lane] = w;
                }
            }
        }
        if (!kRegs) __syncwarp();
        // ---- columns, CB per pass: CB independent accumulation chains with all
        // CB*NS gathers and the own-row / H loads issued before the chains
        constexpr int CB = kRegs ? CBT : 1;
        for (int c0 = 0; c0 < m; c0 += CB) {
            const char* xcol[CB];
            bool on[CB];
            double xi[CB], hv[CB], acc[CB];
#pragma unroll
            for (int q = 0; q < CB; ++q) {
                on[q] = c0 + q < m;
                xcol[q] = xbase + static_cast<uint64_t>(on[q] ? c0 + q : c0) * ldx8;
                xi[q] = ldx<HF>(reinterpret_cast<const double*>(xcol[q] + grow8));
                hv[q] = 0.0;
                if (EPI == EPI_POLY && !ea.first && ea.h_terms && live && on[q])
                    hv[q] = ta.H[static_cast<int64_t>(c0 + q) * ta.ldh + row];
                acc[q] = 0.0;
            }
#pragma unroll
            for (int sidx = 0; sidx < NS; ++sidx) {
                const uint32_t o = kRegs ? ro[sidx < NSR ? sidx : 0] : so[sidx * 32 + lane];
                const double w = kRegs ? rw[sidx < NSR ? sidx : 0] : sw[sidx * 32 + lane];
#pragma unroll
                for (int q = 0; q < CB; ++q) {
                    const double g = ldx<HF>(reinterpret_cast<const double*>(xcol[q] + o));
                    acc[q] = __dadd_rn(acc[q], __dmul_rn(w, g));
                }
            }
#pragma unroll
            for (int q = 0; q < CB; ++q) {
                double sq = 0.0;
                if (live && on[q]) {
                    const int c = c0 + q;
                    const int64_t yo = static_cast<int64_t>(c) * ta.ldy + row;
                    if (EPI == EPI_STORE) {
                        ta.Y[yo] = acc[q];
                    } else if (EPI == EPI_RESIDUAL) {
                        const double bx = ea.bdiag ? __dmul_rn(ea.bdiag[row], xi[q]) : xi[q];
                        const double r = __dsub_rn(acc[q], __dmul_rn(s_theta[c], bx));
                        ta.Y[yo] = r;
                        sq = r * r;
                    } else {
                        const double pn = __dsub_rn(xi[q], __dmul_rn(ea.inv_cur, acc[q]));
                        ta.Y[yo] = pn;
                        if (ea.h_terms)
                            ta.H[static_cast<int64_t>(c) * ta.ldh + row] = poly_h(ea, hv[q], xi[q], pn);
                    }
                }
                if (EPI == EPI_RESIDUAL) {
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
                    if (lane == 0 && on[q]) s_sq[warp][c0 + q] += sq;
                }
            }
        }
        if (!kRegs) __syncwarp();
    }
    if (EPI == EPI_RESIDUAL) {
        __syncthreads();
        for (int c = threadIdx.x; c < m; c += kThreads) {
            double s = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) s += s_sq[w][c];
            ea.partial[static_cast<int64_t>(blockIdx.x) * m + c] = s;
        }
    }
}

// One CTA per long row (power-law hubs). Warp w takes entries k0+w, k0+w+8, ...
// (unrolled by 4 for memory-level parallelism); lane c accumulates column c0+c,
// so every entry is one coalesced read of the X row. The 8 warp partials are
// summed in a fixed order.
template <int MODE, int EPI>
__global__ void __launch_bounds__(kThreads) spmm_long_kernel(const DevOp op, const View X,
                                                             const EpiArgs ea, const int m,
                                                             const int partial_base) {
    const int64_t row = op.long_rows[blockIdx.x];
    const int64_t grow = op.row0 + row;
    const int64_t k0 = op.offs[row], k1 = op.offs[row + 1];
    constexpr int NW = kThreads / 32;
    __shared__ double red[NW][32];
    __shared__ double sqs[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double isdi = 0.0;
    if (MODE == OP_NORMAL_UNIT) isdi = op.isd[grow];
    for (int c0 = 0; c0 < m; c0 += 32) {
        const int mc = min(32, m - c0);
        const bool act = lane < mc;
        const int c = c0 + (act ? lane : 0);
        double acc = 0.0;
        int64_t k = k0 + warp;
        for (; k + 3 * NW < k1; k += 4 * NW) {
            int j[4];
            double v[4], x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                j[u] = op.cols[k + u * NW];
                if (MODE == OP_EXPLICIT) v[u] = op.vals[k + u * NW];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (MODE == OP_NORMAL_UNIT) v[u] = __dmul_rn(-isdi, op.isd[j[u]]);
                else if (MODE == OP_LAPLACE_UNIT) v[u] = -1.0;
                x[u] = act ? X.at(j[u], c) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) acc = __dadd_rn(acc, __dmul_rn(v[u], x[u]));
        }
        for (; k < k1; k += NW) {
            const int j = op.cols[k];
            double v;
            if (MODE == OP_EXPLICIT) v = op.vals[k];
            else if (MODE == OP_NORMAL_UNIT) v = __dmul_rn(-isdi, op.isd[j]);
            else v = -1.0;
            const double x = act ? X.at(j, c) : 0.0;
            acc = __dadd_rn(acc, __dmul_rn(v, x));
        }
        red[warp][lane] = acc;
        __syncthreads();
        if (threadIdx.x < mc) {
            const int cc = threadIdx.x;
            double s = 0.0;
            for (int w = 0; w < NW; ++w) s += red[w][cc];
            const double xi = X.at(grow, c0 + cc);
            if (MODE == OP_LAPLACE_UNIT) s = __dadd_rn(s, __dmul_rn(op.diag[row], xi));
            if (MODE == OP_NORMAL_UNIT) s = __dadd_rn(s, xi);
            double sq = 0.0;
            epilogue<EPI>(ea, row, c0 + cc, s, xi, sq);
            sqs[cc] = sq;
        }
        __syncthreads();
        if (EPI == EPI_RESIDUAL && threadIdx.x < mc)
            ea.partial[static_cast<int64_t>(partial_base + blockIdx.x) * m + c0 + threadIdx.x] =
                sqs[threadIdx.x];
        __syncthreads();
    }
}

template <int KL, int KU, int EPI, int CB, int MINB, bool HF, bool PAT = false>
__global__ void __launch_bounds__(kThreads, MINB) spmm_ell_kernel(const DevOp op, const TileArgs ta, const EpiArgs ea,
                                                                   const HaloFuse hf) {
    constexpr int W = KL + KU;
    __shared__ double s_sq[kThreads / 32][kMaxCols];
    __shared__ double s_theta[kMaxCols];
    // pattern-compressed slots (ellpat.cu): table of per-pattern column offsets and degrees
    __shared__ int32_t s_tab[PAT ? 256 * W : 1];
    __shared__ double s_deg[PAT ? 256 : 1];
    if (PAT) {
        for (int e = threadIdx.x; e < op.ell_npat * W; e += kThreads) s_tab[e] = op.ell_pat_tab[e];
        for (int e = threadIdx.x; e < op.ell_npat; e += kThreads) s_deg[e] = op.ell_pat_deg[e];
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int m = ta.m;
    // HF: the halo rows were sent by the copy engine (halo_ce_start); warps wait
    // for the peers' flags before their first halo tile
    if (HF && hf.probe && threadIdx.x == 0) atomicMin(&hf.probe[0], global_ns());
    if (EPI == EPI_RESIDUAL) {
        for (int c = threadIdx.x; c < m; c += kThreads) s_theta[c] = ea.theta[c];
        for (int c = lane; c < m; c += 32) s_sq[warp][c] = 0.0;
        __syncthreads();
    }
    const int64_t ntiles = (op.n + 31) / 32;
    const int64_t gwarp = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + warp;
    const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
    const uint32_t zrow = static_cast<uint32_t>(op.ell_zero_row);
    // the next tile's slot indices and diagonal are loaded one tile ahead, so
    // the index -> gather dependency does not serialize two memory latencies
    // (wide stencils skip the look-ahead: their W indices already fill the registers)
    constexpr bool kAhead = W <= 8;
    // logical -> physical tile (see HaloFuse::bnd)
    const int64_t nb = ntiles - hf.n_int;
    // each loop segment maps logical lt to physical (lt + koff + rot) mod ntiles
    int64_t koff = 0;
    auto phys = [&](int64_t lt) {
        if (!HF) return lt;
        const int64_t p = lt + koff + hf.rot;
        return p >= ntiles ? p - ntiles : p;
    };
    uint32_t jn[W];
    double dwn = 0.0;
    auto load_slots = [&](int64_t lt) {
        const int64_t row = phys(lt) * 32 + lane;
        const bool live = lt < ntiles && row < op.n;
        if (PAT) {
            const int p = live ? static_cast<int>(__ldg(op.ell_pat + row)) : 0;
            const int32_t* tp = s_tab + p * W;
#pragma unroll
            for (int sidx = 0; sidx < W; ++sidx) {
                const int32_t d = tp[sidx];
                jn[sidx] = (live && d != kEllPad) ? static_cast<uint32_t>(row + d) : zrow;
            }
            dwn = live ? s_deg[p] : 0.0;
        } else {
#pragma unroll
            for (int sidx = 0; sidx < W; ++sidx)
                jn[sidx] = live ? static_cast<uint32_t>(__ldg(op.ell + static_cast<int64_t>(sidx) * op.ell_ld + row)) : zrow;
            dwn = live ? __ldg(op.diag + row) : 0.0;
        }
    };
    if (kAhead) load_slots(gwarp);
    // two loops: logical tiles before the halo segment, then (after this warp's
    // one wait, if it has halo tiles) the rest — no flag logic inside the loops
    const int64_t lt_split = HF ? hf.bnd : ntiles;
    auto tile_loop = [&](int64_t lt_begin, int64_t lt_end) {
    for (int64_t lt = lt_begin; lt < lt_end; lt += nwarps) {
        const int64_t tile = phys(lt);
        const int64_t row = tile * 32 + lane;
        const bool live = row < op.n;
        if (!kAhead) load_slots(lt);
        uint32_t j[W];
#pragma unroll
        for (int sidx = 0; sidx < W; ++sidx) j[sidx] = jn[sidx];
        const double dw = dwn;
        if (kAhead) load_slots(lt + nwarps);
        const uint32_t own = live ? static_cast<uint32_t>(row) : zrow;
        for (int c0 = 0; c0 < m; c0 += CB) {
            const double* xc[CB];
            bool on[CB];
            double xi[CB], hv[CB], acc[CB];
#pragma unroll
            for (int q = 0; q < CB; ++q) {
                on[q] = c0 + q < m;
                xc[q] = ta.X + static_cast<int64_t>(on[q] ? c0 + q : c0) * ta.ldx;
                xi[q] = ldx<HF>(xc[q] + own);
                hv[q] = 0.0;
                if (EPI == EPI_POLY && !ea.first && ea.h_terms && live && on[q])
                    hv[q] = ta.H[static_cast<int64_t>(c0 + q) * ta.ldh + row];
                acc[q] = 0.0;
            }
            // gathers in chunks of CH slots, each chunk issued before its ordered adds
            constexpr int CH = 8;
#pragma unroll
            for (int s0 = 0; s0 < KL; s0 += CH) {
                double gv[CB][CH];
#pragma unroll
                for (int u = 0; u < CH; ++u)
                    if (s0 + u < KL)
#pragma unroll
                        for (int q = 0; q < CB; ++q) gv[q][u] = ldx<HF>(xc[q] + j[s0 + u]);
#pragma unroll
                for (int u = 0; u < CH; ++u)
                    if (s0 + u < KL)
#pragma unroll
                        for (int q = 0; q < CB; ++q) acc[q] = __dsub_rn(acc[q], gv[q][u]);
            }
#pragma unroll
            for (int q = 0; q < CB; ++q) acc[q] = __dadd_rn(acc[q], __dmul_rn(dw, xi[q]));
#pragma unroll
            for (int s0 = KL; s0 < W; s0 += CH) {
                double gv[CB][CH];
#pragma unroll
                for (int u = 0; u < CH; ++u)
                    if (s0 + u < W)
#pragma unroll
                        for (int q = 0; q < CB; ++q) gv[q][u] = ldx<HF>(xc[q] + j[s0 + u]);
#pragma unroll
                for (int u = 0; u < CH; ++u)
                    if (s0 + u < W)
#pragma unroll
                        for (int q = 0; q < CB; ++q) acc[q] = __dsub_rn(acc[q], gv[q][u]);
            }
#pragma unroll
            for (int q = 0; q < CB; ++q) {
                double sq = 0.0;
                if (live && on[q]) {
                    const int c = c0 + q;
                    const int64_t yo = static_cast<int64_t>(c) * ta.ldy + row;
                    if (EPI == EPI_STORE) {
                        ta.Y[yo] = acc[q];
                    } else if (EPI == EPI_RESIDUAL) {
                        const double bx = ea.bdiag ? __dmul_rn(ea.bdiag[row], xi[q]) : xi[q];
                        const double r = __dsub_rn(acc[q], __dmul_rn(s_theta[c], bx));
                        ta.Y[yo] = r;
                        sq = r * r;
                    } else {
                        const double pn = __dsub_rn(xi[q], __dmul_rn(ea.inv_cur, acc[q]));
                        ta.Y[yo] = pn;
                        if (ea.h_terms)
                            ta.H[static_cast<int64_t>(c) * ta.ldh + row] = poly_h(ea, hv[q], xi[q], pn);
                    }
                }
                if (EPI == EPI_RESIDUAL) {
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, off);
                    if (lane == 0 && on[q]) s_sq[warp][c0 + q] += sq;
                }
            }
        }
    }
    };
    tile_loop(gwarp, lt_split);
    if (HF) {
        // first logical tile of this warp at or after lt0
        auto first_from = [&](int64_t lt0) {
            int64_t lt = gwarp;
            if (lt < lt0) lt += ((lt0 - lt + nwarps - 1) / nwarps) * nwarps;
            return lt;
        };
        // halo segment [bnd, bnd + nb): physical k = n_int + (lt - bnd)
        int64_t lt = first_from(hf.bnd);
        const int64_t hend = hf.bnd + nb;
        if (lt < hend) {
            halo_wait_warp(hf);
            koff = hf.n_int - hf.bnd;
            if (kAhead) load_slots(lt);
            tile_loop(lt, hend);
        }
        // remaining interior [bnd + nb, ntiles): physical k = lt - nb
        lt = first_from(hend);
        if (lt < ntiles) {
            koff = -nb;
            if (kAhead) load_slots(lt);
            tile_loop(lt, ntiles);
        }
    }
    if (HF && hf.probe && lane == 0) atomicMax(&hf.probe[4], global_ns());
    if (EPI == EPI_RESIDUAL) {
        __syncthreads();
        for (int c = threadIdx.x; c < m; c += kThreads) {
            double s = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) s += s_sq[w][c];
            ea.partial[static_cast<int64_t>(blockIdx.x) * m + c] = s;
        }
    }
}

// PAT instantiations exist only for the pattern-compressed stencil classes.
// Launch shape (profiles/r01_cfg2_pat_variants.json): two columns per pass at
// 4 CTAs/SM for 5/7-point stencils.
template <int KL, int KU, int EPI>
auto pat_ell_kernel(bool hf) -> decltype(&spmm_ell_kernel<KL, KU, EPI, 2, 4, false>) {
    if constexpr (KL == KU && (KL == 2 || KL == 3)) {
        if (hf) return &spmm_ell_kernel<KL, KU, EPI, 2, 4, true, true>;
        return &spmm_ell_kernel<KL, KU, EPI, 2, 4, false, true>;
    } else {
        return nullptr;
    }
}

template <int MODE, int EPI>
int launch_mode_epi(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s, const HaloFuse* hf) {
    int G = 1;
    while (G < m && G < 32) G <<= 1;
    // column-major blocks (regular graphs): row per lane
    if (MODE != OP_DIAGONAL && spmm_col_path(op, X, m, ea)) {
        TileArgs ta;
        ta.X = X.ptr;
        ta.ldx = static_cast<int>(m > 1 ? X.cs : 0);
        ta.Y = ea.Y.ptr;
        ta.ldy = static_cast<int>(m > 1 ? ea.Y.cs : 0);
        ta.H = ea.H.ptr;
        ta.ldh = static_cast<int>(ea.mode == EPI_POLY && m > 1 ? ea.H.cs : 0);
        ta.m = m;
        const int64_t ntiles = (op.n + 31) / 32;
        const int mr = op.max_row;
        int grid = 0;
        auto go = [&](auto kern, int maxr) {
            const size_t smem = maxr <= 8 ? 0 : (kThreads / 32) * (maxr + 1) * 32 * (sizeof(uint32_t) + sizeof(double));
            // one wave of co-resident CTAs (grid-stride loop inside)
            static std::vector<std::pair<const void*, int>> occ;
            const void* key = reinterpret_cast<const void*>(kern);
            int per_sm = 0;
            for (auto& e : occ)
                if (e.first == key) per_sm = e.second;
            if (!per_sm) {
                if (smem > 48 * 1024)
                    SPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                SPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem));
                per_sm = std::max(per_sm, 1);
                occ.emplace_back(key, per_sm);
            }
            grid = grid_for(ntiles, kThreads / 32, per_sm);
            kern<<<grid, kThreads, smem, s>>>(op, ta, ea, hf ? *hf : HaloFuse{});
        };
        if (MODE == OP_LAPLACE_UNIT && (!hf || hf->nopush) && spmm_mesh_ok(op, X, m, ea))
            return spmm_mesh_launch(op, X, m, ea, s, hf);
        if (MODE == OP_LAPLACE_UNIT && op.ell) {
            // fixed-slot ELL (meshes), pattern-compressed when the solver found the patterns
            const bool pat = op.ell_pat != nullptr;
#define SPB_ELL(KL_, KU_)                                                                                   \
    do {                                                                                                    \
        if (pat && pat_ell_kernel<KL_, KU_, EPI>(hf != nullptr) != nullptr)                                 \
            go(pat_ell_kernel<KL_, KU_, EPI>(hf != nullptr), 0);                                           \
        else if (hf) go(spmm_ell_kernel<KL_, KU_, EPI, 2, 4, true>, 0);                                     \
        else go(spmm_ell_kernel<KL_, KU_, EPI, 2, 4, false>, 0);                                            \
    } while (0)
            switch (op.ell_kl * 100 + op.ell_ku) {
            case 202: SPB_ELL(2, 2); break;
            case 303: SPB_ELL(3, 3); break;
            case 404: SPB_ELL(4, 4); break;
            case 1313:
                // cfg4 A/B (profiles/r01_cfg4_pat_variants.json): one column per pass at
                // 3 CTAs/SM (80 registers) 1.318 ms/launch, 4 CTAs/SM 1.348, two columns 1.765
                if (pat && !hf) go(spmm_ell_kernel<13, 13, EPI, 1, 3, false, true>, 0);
                else if (pat) go(spmm_ell_kernel<13, 13, EPI, 1, 4, true, true>, 0);
                else if (hf) go(spmm_ell_kernel<13, 13, EPI, 1, 4, true>, 0);
                else go(spmm_ell_kernel<13, 13, EPI, 1, 4, false>, 0);
                break;
            default:
                if (op.ell_kl == 8 && op.ell_ku == 8) SPB_ELL(8, 8);
                else SPB_ELL(16, 16);
                break;
            }
#undef SPB_ELL
            SPB_LAUNCH_CHECK();
            return grid;
        }
        if (mr <= 8) go(hf ? spmm_col_kernel<8, MODE, EPI, 2, 5, true> : spmm_col_kernel<8, MODE, EPI, 2, 5>, 8);
        else if (mr <= 16) go(hf ? spmm_col_kernel<16, MODE, EPI, 2, 1, true> : spmm_col_kernel<16, MODE, EPI>, 16);
        else go(hf ? spmm_col_kernel<32, MODE, EPI, 2, 1, true> : spmm_col_kernel<32, MODE, EPI>, 32);
        SPB_LAUNCH_CHECK();
        return grid;
    }
    const bool rowmajor_ok = (m == 1 || (X.cs == 1 && ea.Y.cs == 1 && (ea.mode != EPI_POLY || ea.H.cs == 1))) &&
                             X.rs * 8 < (int64_t(1) << 32) && (op.row0 + op.n) < (int64_t(1) << 32) &&
                             op.n * ea.Y.rs < (int64_t(1) << 31);
    if (MODE != OP_DIAGONAL && op.max_row <= 32 && op.n_long == 0 && rowmajor_ok) {
        // row-major addressing: element (r, c) at r*ld + c (m == 1 column views use ld = rs)
        TileArgs ta;
        ta.X = X.ptr;
        ta.ldx = static_cast<int>(X.rs);
        ta.Y = ea.Y.ptr;
        ta.ldy = static_cast<int>(ea.Y.rs);
        ta.H = ea.H.ptr;
        ta.ldh = static_cast<int>(ea.H.rs);
        ta.m = m;
        // STORE: 8-wide column chunks keep 4 rows per warp for wide blocks; fused
        // epilogues need one chunk per row (column = lane)
        int Gt = G;
        if (ea.mode == EPI_STORE && m > 8) Gt = 8;
        const int64_t ntiles = (op.n + kTileRows - 1) / kTileRows;
        const int grid = grid_for(ntiles, kThreads / 32, 8);
        const size_t smem = (kThreads / 32) * kTileCap *
                            (sizeof(int32_t) + ((MODE == OP_EXPLICIT || MODE == OP_NORMAL_UNIT) ? sizeof(double) : 0));
        auto go = [&](auto kern) {
            // every instantiation has the same function-pointer type: key the
            // one-time attribute call by address
            static std::vector<const void*> done;
            const void* key = reinterpret_cast<const void*>(kern);
            if (std::find(done.begin(), done.end(), key) == done.end()) {
                SPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
                done.push_back(key);
            }
            kern<<<grid, kThreads, smem, s>>>(op, ta, ea);
        };
        const int mr = op.max_row;
#define SPB_TILE_CASES(GG)                                                                     \
    if (mr <= 8) go(spmm_tile_kernel<GG, 8, 2, MODE, EPI>);                                    \
    else if (mr <= 16) go(spmm_tile_kernel<GG, 16, 1, MODE, EPI>);                            \
    else go(spmm_tile_kernel<GG, 32, 1, MODE, EPI>);
        switch (Gt) {
        case 1: SPB_TILE_CASES(1) break;
        case 2: SPB_TILE_CASES(2) break;
        case 4: SPB_TILE_CASES(4) break;
        case 8: SPB_TILE_CASES(8) break;
        case 16: SPB_TILE_CASES(16) break;
        default: SPB_TILE_CASES(32) break;
        }
#undef SPB_TILE_CASES
        SPB_LAUNCH_CHECK();
        return grid;
    }
    if (MODE != OP_DIAGONAL && spmm_vec_ok(op, X, m, ea)) {
        // binned vector kernels + chunked long rows (solver path on irregular graphs)
        return spmm_vec_launch(op, X, m, ea, s);
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
int launch_epi(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s, const HaloFuse* hf) {
    switch (op.mode) {
    case OP_EXPLICIT: return launch_mode_epi<OP_EXPLICIT, EPI>(op, X, m, ea, s, hf);
    case OP_LAPLACE_UNIT: return launch_mode_epi<OP_LAPLACE_UNIT, EPI>(op, X, m, ea, s, hf);
    case OP_NORMAL_UNIT: return launch_mode_epi<OP_NORMAL_UNIT, EPI>(op, X, m, ea, s, hf);
    default: return launch_mode_epi<OP_DIAGONAL, EPI>(op, X, m, ea, s, hf);
    }
}

__global__ void reduce_partials_kernel(const double* partial, int rows, int m, double* out) {
    const int c = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (c >= m) return;
    double s = 0.0;
    for (int r = lane; r < rows; r += 32) s += partial[static_cast<int64_t>(r) * m + c];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) out[c] = s;
}

} // namespace

int spmm_launch(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s, const HaloFuse* hf) {
    if (m <= 0) return 0;
    if (ea.mode != EPI_STORE && m > 32)
        throw_dimension("spmm: fused epilogues support at most 32 columns");
    if (hf && !spmm_col_path(op, X, m, ea)) throw SpError(1, "spmm: fused halo exchange needs the column kernel");
    switch (ea.mode) {
    case EPI_STORE: return launch_epi<EPI_STORE>(op, X, m, ea, s, hf);
    case EPI_RESIDUAL: return launch_epi<EPI_RESIDUAL>(op, X, m, ea, s, hf);
    default: return launch_epi<EPI_POLY>(op, X, m, ea, s, hf);
    }
}

namespace {
__device__ __forceinline__ int ell_lower(const DevOp& op, int64_t i, int64_t k0, int len) {
    if (op.dpos) return op.dpos[i];
    int c = 0;
    for (int t = 0; t < len; ++t) c += op.cols[k0 + t] < op.row0 + i ? 1 : 0;
    return c;
}
__global__ void ell_count_kernel(const DevOp op, unsigned* klku) {
    unsigned kl = 0, ku = 0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < op.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k0 = op.offs[i];
        const int len = static_cast<int>(op.offs[i + 1] - k0);
        const int lo = ell_lower(op, i, k0, len);
        kl = max(kl, static_cast<unsigned>(lo));
        ku = max(ku, static_cast<unsigned>(len - lo));
    }
    atomicMax(&klku[0], kl);
    atomicMax(&klku[1], ku);
}
__global__ void ell_fill_kernel(const DevOp op, int KL, int KU, int64_t ld, int32_t zrow, int32_t* ell) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < op.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t k0 = op.offs[i];
        const int len = static_cast<int>(op.offs[i + 1] - k0);
        const int lo = ell_lower(op, i, k0, len);
        const int up = len - lo;
        for (int s = 0; s < KL - lo; ++s) ell[s * ld + i] = zrow;
        for (int t = 0; t < lo; ++t) ell[(KL - lo + t) * ld + i] = op.cols[k0 + t];
        for (int t = 0; t < up; ++t) ell[(KL + t) * ld + i] = op.cols[k0 + lo + t];
        for (int s = KL + up; s < KL + KU; ++s) ell[s * ld + i] = zrow;
    }
}
} // namespace

bool build_ell(DevOp& op, int64_t zero_row, DBuf<int32_t>& store, cudaStream_t s) {
    if (op.mode != OP_LAPLACE_UNIT || op.n <= 0 || op.n_long > 0 || op.max_row > 32) return false;
    DBuf<unsigned> klku(2);
    SPB_CUDA(cudaMemsetAsync(klku.p, 0, 2 * sizeof(unsigned), s));
    ell_count_kernel<<<grid_for(op.n, 256, 4), 256, 0, s>>>(op, klku.p);
    SPB_LAUNCH_CHECK();
    unsigned h[2];
    SPB_CUDA(cudaMemcpyAsync(h, klku.p, sizeof(h), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    int KL, KU;
    const unsigned kl = h[0], ku = h[1];
    if ((kl == 2 && ku == 2) || (kl == 3 && ku == 3) || (kl == 4 && ku == 4) || (kl == 13 && ku == 13)) {
        KL = static_cast<int>(kl);
        KU = static_cast<int>(ku);
    } else if (kl <= 8 && ku <= 8) {
        KL = KU = 8;
    } else if (kl <= 16 && ku <= 16) {
        KL = KU = 16;
    } else {
        return false;
    }
    store.alloc(static_cast<size_t>(KL + KU) * op.n);
    ell_fill_kernel<<<grid_for(op.n, 256, 4), 256, 0, s>>>(op, KL, KU, op.n, static_cast<int32_t>(zero_row), store.p);
    SPB_LAUNCH_CHECK();
    op.ell = store.p;
    op.ell_kl = KL;
    op.ell_ku = KU;
    op.ell_ld = op.n;
    op.ell_zero_row = zero_row;
    return true;
}

bool spmm_col_path(const DevOp& op, const View& X, int m, const EpiArgs& ea) {
    const bool colmajor = m > 1 ? (X.rs == 1 && ea.Y.rs == 1 && (ea.mode != EPI_POLY || ea.H.rs == 1))
                                : (X.rs == 1 && ea.Y.rs == 1);
    return op.mode != OP_DIAGONAL && op.max_row <= 32 && op.n_long == 0 && colmajor &&
           std::max(op.x_rows, op.row0 + op.n) * 8 < (int64_t(1) << 32) && m <= kMaxCols;
}

void reduce_partials(const double* partial, int rows, int m, double* out, cudaStream_t s) {
    reduce_partials_kernel<<<ceil_div(m, 4), 128, 0, s>>>(partial, rows, m, out);
    SPB_LAUNCH_CHECK();
}

} // namespace spb
