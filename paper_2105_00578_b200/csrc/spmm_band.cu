// spmm_band.cu — band-staged SpMM for structured meshes (pattern-compressed ELL).
//
// Same operator, slots, summation order and epilogues as spmm_ell_kernel
// (spmm.cu), hence the same bit-exact result as kernels::spmv_block
// (src/kernels.cpp:36-62) on L_C; only the data movement differs.
//
// On a naturally ordered mesh every column offset (col - row) of every row
// pattern falls into a few narrow bands: {-nx*ny}, [-nx-1, nx+1], {+nx*ny} for
// a 7-point stencil, three bands of width 2*nx+3 for 27 points, one for a 2-D
// grid. For a tile of T consecutive rows the X rows a band can touch are one
// contiguous range [r0 + lo, r0 + T + hi). A producer warp stages those ranges
// of one column with one cp.async.bulk each (non-tensor TMA) into a ring of
// shared-memory stages tracked by mbarriers; the eight consumer warps read
// every neighbour from shared memory (conflict-free: consecutive threads own
// consecutive rows), so the per-element L1 gathers of spmm_ell_kernel (7–27
// per output, ~2.5 wavefronts each) become ~3.3 bulk-copied doubles per
// output from L2 and plain shared-memory loads. A stage is (tile, column):
// the whole block streams column after column through the ring.
#include "bulk.cuh"
#include "ops.cuh"
#include "spmm_epilogue.cuh"

#include <algorithm>
#include <vector>

namespace spb {

namespace {

constexpr int kConsumers = 256;              // 8 consumer warps
constexpr int kBandThreads = kConsumers + 32;  // + 1 producer warp

struct BandGeo {
    int nb;                  // bands
    int lo[kMaxBands];       // band b holds offsets [lo, hi]; tile r0 stages rows [r0 + lo, r0 + T + hi), lo even
    int hi[kMaxBands];
    int sb[kMaxBands];       // smem offset (doubles) of band b inside a stage
    int stage;               // doubles per stage (multiple of 2)
    int nst;                 // stages in the ring
};

// One (tile, column) per stage. T = kConsumers * RPT rows per tile; thread t
// owns rows t, t + 256, ... of the tile.
template <int KL, int KU, int EPI, int RPT>
__global__ void __launch_bounds__(kBandThreads, 2) spmm_band_kernel(const DevOp op, const View X, const EpiArgs ea,
                                                                    const int m, const BandGeo geo) {
    constexpr int W = KL + KU;
    constexpr int T = kConsumers * RPT;
    constexpr bool kRegIdx = W * RPT <= 32;  // slot indices in registers across the columns
    extern __shared__ __align__(128) double smem[];
    __shared__ uint64_t full[8], empty[8];
    __shared__ int16_t s_idx[256 * W];       // per (pattern, slot): smem index - row, or -1 (padding)
    __shared__ int16_t s_own;                // smem index - row of the row itself (offset 0)
    __shared__ double s_deg[256];
    __shared__ double s_theta[kMaxCols];
    __shared__ double s_sq[kConsumers / 32][kMaxCols];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int s = 0; s < geo.nst; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kConsumers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        int own = -1;
        for (int b = 0; b < geo.nb; ++b)
            if (geo.lo[b] <= 0 && 0 <= geo.hi[b]) own = geo.sb[b] - geo.lo[b];
        s_own = static_cast<int16_t>(own);
    }
    for (int e = tid; e < op.ell_npat * W; e += kBandThreads) {
        const int32_t d = op.ell_pat_tab[e];
        int v = -1;
        if (d != kEllPad)
            for (int b = 0; b < geo.nb; ++b)
                if (geo.lo[b] <= d && d <= geo.hi[b]) v = geo.sb[b] + d - geo.lo[b];
        s_idx[e] = static_cast<int16_t>(v);
    }
    for (int e = tid; e < op.ell_npat; e += kBandThreads) s_deg[e] = op.ell_pat_deg[e];
    if (EPI == EPI_RESIDUAL) {
        for (int c = tid; c < m; c += kBandThreads) s_theta[c] = ea.theta[c];
        for (int e = tid; e < (kConsumers / 32) * kMaxCols; e += kBandThreads) (&s_sq[0][0])[e] = 0.0;
    }
    __syncthreads();

    const int64_t ntiles = (op.n + T - 1) / T;
    const int64_t my_tiles = ntiles > blockIdx.x ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const int64_t items = my_tiles * m;
    // rows staged per column: up to the zero row (row n), never past the block's leading dimension
    const int64_t xend = (op.n + 1) & ~int64_t(1);

    if (warp == kConsumers / 32) {
        // ---- producer: one elected lane issues the bulk copies of each stage
        if (lane == 0) {
            for (int64_t it = 0; it < items; ++it) {
                const int s = static_cast<int>(it % geo.nst);
                const int64_t round = it / geo.nst;
                if (round > 0) mbar_wait(empty + s, static_cast<unsigned>((round - 1) & 1));
                const int64_t tile = blockIdx.x + (it / m) * gridDim.x;
                const int c = static_cast<int>(it % m);
                const int64_t r0 = tile * T;
                const double* col = X.ptr + static_cast<int64_t>(c) * X.cs;
                double* st = smem + static_cast<size_t>(s) * geo.stage;
                auto range = [&](int b, int64_t& gs, int64_t& ge) {
                    gs = r0 + geo.lo[b] > 0 ? r0 + geo.lo[b] : 0;
                    ge = (r0 + T + geo.hi[b] + 1) & ~int64_t(1);
                    if (ge > xend) ge = xend;
                };
                unsigned bytes = 0;
                for (int b = 0; b < geo.nb; ++b) {
                    int64_t gs, ge;
                    range(b, gs, ge);
                    if (ge > gs) bytes += static_cast<unsigned>(ge - gs) * 8u;
                }
                mbar_expect_tx(full + s, bytes);
                for (int b = 0; b < geo.nb; ++b) {
                    int64_t gs, ge;
                    range(b, gs, ge);
                    if (ge > gs)
                        bulk_g2s(st + geo.sb[b] + (gs - (r0 + geo.lo[b])), col + gs, static_cast<unsigned>(ge - gs) * 8u,
                                 full + s);
                }
            }
        }
        return;
    }

    // ---- consumers
    int64_t it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t r0 = tile * T;
        int pid[RPT];
        double dw[RPT];
        bool live[RPT];
        int16_t idx[kRegIdx ? RPT : 1][kRegIdx ? W : 1];
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
            const int64_t row = r0 + tid + k * kConsumers;
            live[k] = row < op.n;
            pid[k] = live[k] ? static_cast<int>(__ldg(op.ell_pat + row)) : 0;
            dw[k] = s_deg[pid[k]];
            if (kRegIdx) {
#pragma unroll
                for (int sl = 0; sl < W; ++sl) idx[kRegIdx ? k : 0][kRegIdx ? sl : 0] = s_idx[pid[k] * W + sl];
            }
        }
        const int own = s_own;
        for (int c = 0; c < m; ++c, ++it) {
            const int s = static_cast<int>(it % geo.nst);
            const unsigned ph = static_cast<unsigned>((it / geo.nst) & 1);
            // epilogue operands not in the stage: issue before the wait
            double hv[RPT], bd[RPT];
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                const int64_t row = r0 + tid + k * kConsumers;
                hv[k] = 0.0;
                bd[k] = 1.0;
                if (EPI == EPI_POLY && !ea.first && ea.h_terms && live[k]) hv[k] = ea.H.at(row, c);
                if (EPI == EPI_RESIDUAL && ea.bdiag && live[k]) bd[k] = ea.bdiag[row];
            }
            mbar_wait(full + s, ph);
            const double* st = smem + static_cast<size_t>(s) * geo.stage;
#pragma unroll
            for (int k = 0; k < RPT; ++k) {
                const int rl = tid + k * kConsumers;
                const double xi = st[rl + own];
                double acc = 0.0;
                // acc -= x_j over the lower slots, += deg * x_i, -= x_j over the upper slots:
                // the storage order of build_combinatorial's row (bit-identical to spmv_block)
#pragma unroll
                for (int sl = 0; sl < KL; ++sl) {
                    const int v = kRegIdx ? idx[kRegIdx ? k : 0][kRegIdx ? sl : 0] : s_idx[pid[k] * W + sl];
                    if (v >= 0) acc = __dsub_rn(acc, st[rl + v]);
                }
                acc = __dadd_rn(acc, __dmul_rn(dw[k], xi));
#pragma unroll
                for (int sl = KL; sl < W; ++sl) {
                    const int v = kRegIdx ? idx[kRegIdx ? k : 0][kRegIdx ? sl : 0] : s_idx[pid[k] * W + sl];
                    if (v >= 0) acc = __dsub_rn(acc, st[rl + v]);
                }
                double sq = 0.0;
                if (live[k]) {
                    const int64_t row = r0 + rl;
                    if (EPI == EPI_STORE) {
                        ea.Y.at(row, c) = acc;
                    } else if (EPI == EPI_RESIDUAL) {
                        const double bx = ea.bdiag ? __dmul_rn(bd[k], xi) : xi;
                        const double r = __dsub_rn(acc, __dmul_rn(s_theta[c], bx));
                        ea.Y.at(row, c) = r;
                        sq = r * r;
                    } else {
                        const double pn = __dsub_rn(xi, __dmul_rn(ea.inv_cur, acc));
                        ea.Y.at(row, c) = pn;
                        if (ea.h_terms) ea.H.at(row, c) = poly_h(ea, hv[k], xi, pn);
                    }
                }
                if (EPI == EPI_RESIDUAL) {
                    double v = sq;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                    if (lane == 0) s_sq[warp][c] += v;
                }
            }
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + s)) : "memory");
        }
    }
    if (EPI == EPI_RESIDUAL) {
        asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
        for (int c = tid; c < m; c += kConsumers) {
            double v = 0.0;
            for (int w = 0; w < kConsumers / 32; ++w) v += s_sq[w][c];
            ea.partial[static_cast<int64_t>(blockIdx.x) * m + c] = v;
        }
    }
}

constexpr int kRpt = 4;  // T = 1024 rows per tile

BandGeo geometry(const DevOp& op, int T, int nst) {
    BandGeo g{};
    g.nb = op.band_n;
    int off = 0;
    for (int b = 0; b < g.nb; ++b) {
        g.lo[b] = op.band_lo[b];
        g.hi[b] = op.band_hi[b];
        g.sb[b] = off;
        off += (T + g.hi[b] - g.lo[b] + 2) & ~1;  // rows [r0+lo, r0+T+hi), end rounded up to even
    }
    g.stage = (off + 15) & ~15;  // 128-byte aligned stages
    g.nst = nst;
    return g;
}

template <int KL, int KU, int EPI>
int launch_band(const DevOp& op, const View& X, int m, const EpiArgs& ea, cudaStream_t s) {
    constexpr int T = kConsumers * kRpt;
    const BandGeo g0 = geometry(op, T, 1);
    // ring depth: as many stages as fit next to a second CTA on the SM
    const size_t per_stage = sizeof(double) * g0.stage;
    int nst = static_cast<int>(std::min<size_t>(6, (100 * 1024) / per_stage));
    nst = std::max(nst, 2);
    const BandGeo g = geometry(op, T, nst);
    const size_t smem = per_stage * nst;
    auto kern = spmm_band_kernel<KL, KU, EPI, kRpt>;
    static bool attr = false;
    if (!attr) {
        SPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        attr = true;
    }
    int per_sm = 0;
    SPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBandThreads, smem));
    per_sm = std::max(per_sm, 1);
    const int64_t ntiles = (op.n + T - 1) / T;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(ntiles, int64_t(device_sm_count()) * per_sm)));
    kern<<<grid, kBandThreads, smem, s>>>(op, X, ea, m, g);
    SPB_LAUNCH_CHECK();
    return grid;
}

} // namespace

bool band_plan(DevOp& op, cudaStream_t s) {
    op.band_n = 0;
    if (!op.ell_pat || op.ell_npat <= 0) return false;
    const int W = op.ell_kl + op.ell_ku;
    std::vector<int32_t> tab(static_cast<size_t>(op.ell_npat) * W);
    SPB_CUDA(cudaMemcpyAsync(tab.data(), op.ell_pat_tab, sizeof(int32_t) * tab.size(), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> offs{0};
    for (int32_t d : tab)
        if (d != kEllPad) offs.push_back(d);
    std::sort(offs.begin(), offs.end());
    offs.erase(std::unique(offs.begin(), offs.end()), offs.end());
    // cluster offsets whose gap is at most kBandGap rows into one band
    constexpr int64_t kBandGap = 1024;
    std::vector<std::pair<int64_t, int64_t>> bands;
    for (int64_t d : offs) {
        if (!bands.empty() && d - bands.back().second <= kBandGap) bands.back().second = d;
        else bands.push_back({d, d});
    }
    if (static_cast<int>(bands.size()) > kMaxBands) return false;
    int64_t width = 0;
    for (auto& b : bands) width += b.second - b.first;
    if (width > 8192) return false;  // stages would not fit next to a second CTA
    op.band_n = static_cast<int>(bands.size());
    for (int b = 0; b < op.band_n; ++b) {
        op.band_lo[b] = static_cast<int>(bands[b].first & ~int64_t(1));  // even: 16-byte aligned bulk copies
        op.band_hi[b] = static_cast<int>(bands[b].second);
    }
    return true;
}

bool spmm_band_ok(const DevOp& op, const View& X, int m, const EpiArgs& ea) {
    if (op.band_n <= 0 || !op.ell_pat || op.mode != OP_LAPLACE_UNIT || op.row0 != 0 || op.dpos) return false;
    // column-major blocks whose columns hold the zero row, 16-byte aligned column starts
    auto cm = [&](const View& v) { return v.rs == 1 && (m == 1 || v.cs >= op.n + 1); };
    if (!cm(X) || !cm(ea.Y) || (ea.mode == EPI_POLY && !cm(ea.H))) return false;
    if (X.cs < op.n + 1) return false;
    if (reinterpret_cast<uintptr_t>(X.ptr) % 16 != 0 || (m > 1 && X.cs % 2 != 0)) return false;
    return m <= kMaxCols;
}

int spmm_band_launch(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s) {
    const int kk = op.ell_kl * 100 + op.ell_ku;
    switch (ea.mode) {
#define SPB_BAND(EPI_)                                                                  \
    switch (kk) {                                                                     \
    case 202: return launch_band<2, 2, EPI_>(op, X, m, ea, s);                        \
    case 303: return launch_band<3, 3, EPI_>(op, X, m, ea, s);                        \
    default: return launch_band<13, 13, EPI_>(op, X, m, ea, s);                       \
    }
    case EPI_STORE: SPB_BAND(EPI_STORE)
    case EPI_RESIDUAL: SPB_BAND(EPI_RESIDUAL)
    default: SPB_BAND(EPI_POLY)
#undef SPB_BAND
    }
}

} // namespace spb
