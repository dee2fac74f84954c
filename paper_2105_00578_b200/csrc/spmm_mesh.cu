// spmm_mesh.cu — SpMM on naturally ordered structured meshes: TMA 3-D tiles, z-marching.
//
// Same operator, slots, summation order and epilogues as spmm_ell_kernel (spmm.cu),
// hence the same bit-exact result as kernels::spmv_block (src/kernels.cpp:36-62) on
// L_C; only the data movement differs.
//
// The graphs of generators.cpp:126-162 (grid2d, stencil3d 7/27) number vertex
// (x, y, z) as (z*ny + y)*nx + x, so every row's neighbours are the in-bounds
// points of a 3x3x3 box around it. mesh_plan recognises that structure from the
// pattern-compressed ELL (the offsets decompose as dz*nx*ny + dy*nx + dx and
// every row's pattern is exactly its in-bounds stencil, verified on the device).
//
// A CTA owns a 32x32 (x, y) tile of one block column and marches a chunk of z
// planes. A producer warp loads each plane of X as one 36x34 box (the tile plus
// its x/y halo; the x start is moved to x0 - 2 because a box must start on a
// 16-byte boundary of the innermost dimension) with a 4-D tensor-map TMA copy
// (out-of-range halo is zero-filled by the TMA unit), plus the 32x32 box of H the POLY epilogue reads, into a ring
// of shared-memory stages tracked by mbarriers. Consumer warps compute plane z
// from the stages of planes z-1, z, z+1 — each X element crosses L2 -> SM about
// 1.2x (the halo) instead of the ~3x of per-plane gathers (z-1, z, z+1 reads of
// the same element from three different tiles) — and write Y (and H) with
// coalesced 256-byte warp stores.
//
// Multi-GPU: a rank whose rows are whole z planes (mesh_plan_slab, on the global ids before
// localization) runs the same kernel on its slab; the neighbours' boundary planes, which the
// halo plan puts after the own rows, come through a second tensor map once the copy engine's
// flags arrived. spmm_mesh_poly2_kernel fuses two polynomial steps per pass (5/7-point
// meshes; on slabs with a two-plane halo), bit-identical to two single steps.
#include "bulk.cuh"
#include "ops.cuh"
#include "spmm_epilogue.cuh"

#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace spb {

namespace {

constexpr int kTile = 32;                 // x and y extent of a tile
constexpr int kHaloW = kTile + 4;         // 36: x extent of an X box (its start must be 16-byte aligned: x0 - 2)
constexpr int kHaloH = kTile + 2;         // 34: y extent (one halo row each side)
constexpr int kConsumers = 256;           // 8 consumer warps; warp w owns tile rows w, w+8, w+16, w+24
constexpr int kMeshThreads = kConsumers + 32;
constexpr int kXPlane = kHaloW * kHaloH;                       // doubles of an X box
constexpr int kXPlanePad = ((kXPlane * 8 + 127) / 128) * 16;   // 128-byte aligned (in doubles)
constexpr int kHPlane = kTile * kTile;
constexpr int kMaxStages = 8;

struct MeshGeo {
    int nx, ny, nz;
    int ntx, nty;       // tiles per plane
    int zc, nzc;        // z planes per chunk, chunks
    int nst;            // ring stages
    int h_stage;        // stages carry the H box (POLY with an H read)
    int stage;          // doubles per stage
    // z-slab of a multi-GPU row block: global z of local plane 0, global planes, the
    // halo map's plane of the neighbour below / above (-1: none, the TMA zero-fills
    // and the stencil presence excludes them), chunk rotation (boundary chunks last)
    int z0, nzg, hlo, hhi, zrot;
    // copy-engine halo: the producer waits for these flags before its first halo plane
    const uint64_t* flags;
    unsigned long long epoch;
    uint32_t recv_mask;
    int world;
    int* err;
};

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
            smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

template <bool BOX27, int EPI>
__global__ void __launch_bounds__(kMeshThreads, 2)
    spmm_mesh_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap hmap,
                     const __grid_constant__ CUtensorMap lmap, const DevOp op, const EpiArgs ea, const int m,
                     const MeshGeo geo) {
    extern __shared__ __align__(128) double smem[];
    __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
    __shared__ double s_theta[kMaxCols];
    __shared__ double s_sq[EPI == EPI_RESIDUAL ? kConsumers / 32 : 1][kMaxCols];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int s = 0; s < geo.nst; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kConsumers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (EPI == EPI_RESIDUAL) {
        for (int c = tid; c < m; c += kMeshThreads) s_theta[c] = ea.theta[c];
        for (int e = tid; e < (kConsumers / 32) * kMaxCols; e += kMeshThreads) (&s_sq[0][0])[e] = 0.0;
    }
    __syncthreads();

    const int64_t items = static_cast<int64_t>(geo.ntx) * geo.nty * geo.nzc * m;
    // item -> (column, z chunk, tile y, tile x); columns innermost so concurrent CTAs share planes in L2
    auto decode = [&](int64_t it, int& c, int& tx, int& ty, int& z0, int& z1) {
        c = static_cast<int>(it % m);
        int64_t r = it / m;
        tx = static_cast<int>(r % geo.ntx);
        r /= geo.ntx;
        ty = static_cast<int>(r % geo.nty);
        int zq = static_cast<int>(r / geo.nty);
        if (geo.zrot) zq = zq + 1 == geo.nzc ? 0 : zq + 1;  // the slab's first chunk (lower halo) last
        z0 = zq * geo.zc;
        z1 = min(geo.nz, z0 + geo.zc);
    };
    const unsigned xbytes = kXPlane * 8u, hbytes = geo.h_stage ? kHPlane * 8u : 0u;

    if (warp == kConsumers / 32) {
        if (lane == 0) {
            int s = 0;
            unsigned eph = 0;
            int64_t g = 0;  // stage sequence number
            bool waited = geo.flags == nullptr;
            for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
                int c, tx, ty, z0, z1;
                decode(it, c, tx, ty, z0, z1);
                // stage p carries X plane p and (POLY) the H box of output plane p - 1
                for (int p = z0 - 1; p <= z1; ++p, ++g) {
                    // planes past the slab: the neighbours' boundary planes (halo rows)
                    const CUtensorMap* mp = &xmap;
                    int pz = p;
                    if (p < 0 && geo.hlo >= 0) {
                        mp = &lmap;
                        pz = geo.hlo;
                    } else if (p >= geo.nz && geo.hhi >= 0) {
                        mp = &lmap;
                        pz = geo.hhi;
                    }
                    if (mp == &lmap && !waited) {
                        // the peers' copy engines wrote these rows, then raised our flags
                        for (int q = 0; q < geo.world; ++q)
                            if ((geo.recv_mask >> q) & 1u) wait_flag(geo.flags + q, geo.epoch, geo.err);
                        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic -> TMA reads
                        waited = true;
                    }
                    if (g >= geo.nst) mbar_wait(empty + s, eph);
                    double* st = smem + static_cast<size_t>(s) * geo.stage;
                    mbar_expect_tx(full + s, xbytes + hbytes);
                    tma_load_4d(st, mp, tx * kTile - 2, ty * kTile - 1, pz, c, full + s);
                    if (geo.h_stage) tma_load_4d(st + kXPlanePad, &hmap, tx * kTile, ty * kTile, p - 1, c, full + s);
                    if (++s == geo.nst) {
                        s = 0;
                        if (g >= geo.nst) eph ^= 1u;
                    }
                }
            }
        }
        return;
    }

    // ---- consumers: (slot, phase) of the next stage in sequence, advanced without divisions
    int qs = 0;
    unsigned qph = 0;
    auto advance = [&](int& sl, unsigned& ph) {
        if (++sl == geo.nst) {
            sl = 0;
            ph ^= 1u;
        }
    };
    auto release = [&](int sl) {
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + sl)) : "memory");
    };
    const int64_t nxny = static_cast<int64_t>(geo.nx) * geo.ny;
    // tile rows of this thread: 27-point: four consecutive rows (the (dy, dx) neighbours of
    // the four outputs share registers: 18 shared-memory loads per plane instead of 36);
    // 7-point: rows warp, warp + 8, ...
    auto row_of = [&](int j) { return BOX27 ? 4 * warp + j : warp + 8 * j; };
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        int c, tx, ty, z0, z1;
        decode(it, c, tx, ty, z0, z1);
        const int x = tx * kTile + lane;
        const bool xin = x < geo.nx;
        // per item: this thread's rows of one plane (offsets within a plane), y neighbours
        int64_t roff[4];
        bool live[4], ym[4], yp[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int y = ty * kTile + row_of(j);
            live[j] = xin && y < geo.ny;
            ym[j] = y > 0;
            yp[j] = y + 1 < geo.ny;
            roff[j] = static_cast<int64_t>(y) * geo.nx + x;
        }
        const bool xm = xin && x > 0, xp = x + 1 < geo.nx;
        double* ycol = ea.Y.ptr + static_cast<int64_t>(c) * ea.Y.cs;  // column-major (rs == 1)
        double* hcol = EPI == EPI_POLY ? ea.H.ptr + static_cast<int64_t>(c) * ea.H.cs : nullptr;
        // planes z0 - 1 and z0 first
        int sp = qs;
        unsigned pp = qph;
        int sc = sp;
        unsigned pc = pp;
        advance(sc, pc);
        mbar_wait(full + sp, pp);
        mbar_wait(full + sc, pc);
        for (int z = z0; z < z1; ++z) {
            int sn = sc;
            unsigned pn2 = pc;
            advance(sn, pn2);
            const int64_t zoff = static_cast<int64_t>(z) * nxny;
            double bd[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                bd[j] = (EPI == EPI_RESIDUAL && ea.bdiag && live[j]) ? ea.bdiag[zoff + roff[j]] : 1.0;
            mbar_wait(full + sn, pn2);
            const double* p0 = smem + static_cast<size_t>(sp) * geo.stage;  // plane z - 1
            const double* p1 = smem + static_cast<size_t>(sc) * geo.stage;  // plane z
            const double* p2 = smem + static_cast<size_t>(sn) * geo.stage;  // plane z + 1
            const double* hs = p2 + kXPlanePad;
            const int zg = geo.z0 + z;  // global plane: stencil presence
            const bool zm = zg > 0, zp = zg + 1 < geo.nzg;
            // the rows' entries in storage (= ascending column = lexicographic (dz, dy, dx))
            // order: acc -= x_j before the diagonal, += deg * x_i, -= x_j after it —
            // build_combinatorial's order, so each sum is bit-identical to spmv_block
            double accv[4], xiv[4];
            if constexpr (BOX27) {
                int deg[4];
                const int cx = 1 + xm + xp, cz = 1 + zm + zp;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    deg[j] = cx * (1 + ym[j] + yp[j]) * cz - 1;
                    accv[j] = 0.0;
                    xiv[j] = p1[(row_of(j) + 1) * kHaloW + lane + 2];
                }
                const int r0 = 4 * warp;  // box row of tile row r0 - 1
                // warp-uniform: every output of the warp has all 26 neighbours (no presence tests;
                // the same operations in the same order as the general path)
                bool in = zm && zp && xm && xp && live[0];
#pragma unroll
                for (int j = 0; j < 4; ++j) in = in && ym[j] && yp[j] && live[j];
                const bool all_in = __all_sync(0xffffffffu, in);
#pragma unroll
                for (int dzi = 0; dzi < 3; ++dzi) {
                    const double* pl = dzi == 0 ? p0 : dzi == 1 ? p1 : p2;
                    const bool zon = dzi == 0 ? zm : dzi == 2 ? zp : true;
                    double v[6][3];  // box rows r0 .. r0 + 5 (tile rows r0 - 1 .. r0 + 4), x - 1 .. x + 1
#pragma unroll
                    for (int r = 0; r < 6; ++r)
#pragma unroll
                        for (int d = 0; d < 3; ++d) v[r][d] = pl[(r0 + r) * kHaloW + lane + 1 + d];
                    if (all_in) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
#pragma unroll
                            for (int dyi = 0; dyi < 3; ++dyi)
#pragma unroll
                                for (int dxi = 0; dxi < 3; ++dxi) {
                                    if (dzi == 1 && dyi == 1 && dxi == 1)
                                        accv[j] = __dadd_rn(accv[j], __dmul_rn(26.0, xiv[j]));
                                    else
                                        accv[j] = __dsub_rn(accv[j], v[j + dyi][dxi]);
                                }
                        continue;
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j)
#pragma unroll
                        for (int dyi = 0; dyi < 3; ++dyi)
#pragma unroll
                            for (int dxi = 0; dxi < 3; ++dxi) {
                                if (dzi == 1 && dyi == 1 && dxi == 1) {
                                    accv[j] = __dadd_rn(accv[j], __dmul_rn(static_cast<double>(deg[j]), xiv[j]));
                                    continue;
                                }
                                const bool on = zon && (dyi == 0 ? ym[j] : dyi == 2 ? yp[j] : true) &&
                                                (dxi == 0 ? xm : dxi == 2 ? xp : true);
                                if (on) accv[j] = __dsub_rn(accv[j], v[j + dyi][dxi]);
                            }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int ctr = (row_of(j) + 1) * kHaloW + lane + 2;  // this row's element in its plane box
                    const double xi = p1[ctr];
                    double acc = 0.0;
                    const int deg = zm + ym[j] + xm + xp + yp[j] + zp;
                    if (zm) acc = __dsub_rn(acc, p0[ctr]);
                    if (ym[j]) acc = __dsub_rn(acc, p1[ctr - kHaloW]);
                    if (xm) acc = __dsub_rn(acc, p1[ctr - 1]);
                    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(deg), xi));
                    if (xp) acc = __dsub_rn(acc, p1[ctr + 1]);
                    if (yp[j]) acc = __dsub_rn(acc, p1[ctr + kHaloW]);
                    if (zp) acc = __dsub_rn(acc, p2[ctr]);
                    accv[j] = acc;
                    xiv[j] = xi;
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int ly = row_of(j);
                const double acc = accv[j], xi = xiv[j];
                double sq = 0.0;
                if (live[j]) {
                    const int64_t r = zoff + roff[j];
                    if (EPI == EPI_STORE) {
                        ycol[r] = acc;
                    } else if (EPI == EPI_RESIDUAL) {
                        const double bx = ea.bdiag ? __dmul_rn(bd[j], xi) : xi;
                        const double rr = __dsub_rn(acc, __dmul_rn(s_theta[c], bx));
                        ycol[r] = rr;
                        sq = rr * rr;
                    } else {
                        const double pn = __dsub_rn(xi, __dmul_rn(ea.inv_cur, acc));
                        ycol[r] = pn;
                        if (ea.h_terms) hcol[r] = poly_h(ea, geo.h_stage ? hs[ly * kTile + lane] : 0.0, xi, pn);
                    }
                }
                if (EPI == EPI_RESIDUAL) {
                    double v = sq;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
                    if (lane == 0) s_sq[warp][c] += v;
                }
            }
            release(sp);  // plane z - 1 is no longer needed by this item
            sp = sc;
            pp = pc;
            sc = sn;
            pc = pn2;
        }
        release(sp);  // planes z1 - 1 and z1
        release(sc);
        qs = sc;
        qph = pc;
        advance(qs, qph);
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

// ---- two polynomial steps per pass (5/7-point meshes, one GPU) ----
// Step i: q = p_i - inv_cur * A p_i is computed on the tile plus a one-point ring (34 x 34)
// into a 4-plane shared-memory ring; step i + 1: r = q - inv_next * A q on the 32 x 32 tile
// of the plane behind it. X boxes are 36 x 36 (two-point ring). Only p_i is read, r (p_{i+2})
// and H written: H = (first ? inv_cur p_i : H + inv_cur p_i) + inv_next q (+ inv_after r when
// last) — the operations, and their order, of the two single steps (bit-identical).
constexpr int kBox2 = kTile + 4;                   // 36
constexpr int kXPlane2 = kBox2 * kBox2;            // 1296 doubles (10368 B, a multiple of 128 B)
constexpr int kQW = kTile + 2;                     // 34
constexpr int kQPlane = ((kQW * kQW + 15) / 16) * 16;  // 1168 doubles
constexpr int kQPts = kQW * kQW;                   // 1156 points of q per plane

__global__ void __launch_bounds__(kMeshThreads, 2)
    spmm_mesh_poly2_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap lmap,
                           const DevOp op, const EpiArgs ea, const int m, const MeshGeo geo) {
    extern __shared__ __align__(128) double smem[];
    __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    double* qring = smem + static_cast<size_t>(geo.nst) * kXPlane2;
    if (tid == 0) {
        for (int s = 0; s < geo.nst; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kConsumers / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t items = static_cast<int64_t>(geo.ntx) * geo.nty * geo.nzc * m;
    auto decode = [&](int64_t it, int& c, int& tx, int& ty, int& z0, int& z1) {
        c = static_cast<int>(it % m);
        int64_t r = it / m;
        tx = static_cast<int>(r % geo.ntx);
        r /= geo.ntx;
        ty = static_cast<int>(r % geo.nty);
        int zq = static_cast<int>(r / geo.nty);
        if (geo.zrot) zq = zq + 1 == geo.nzc ? 0 : zq + 1;  // the slab's first chunk (lower halo) last
        z0 = zq * geo.zc;
        z1 = min(geo.nz, z0 + geo.zc);
    };
    if (warp == kConsumers / 32) {
        if (lane == 0) {
            int s = 0;
            unsigned eph = 0;
            int64_t g = 0;
            bool waited = geo.flags == nullptr;
            for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
                int c, tx, ty, z0, z1;
                decode(it, c, tx, ty, z0, z1);
                for (int p = z0 - 2; p <= z1 + 1; ++p, ++g) {
                    // z-slab: planes -2, -1 and nz, nz + 1 are the neighbours' (4-plane halo map)
                    const CUtensorMap* mp = &xmap;
                    int pz = p;
                    if (p < 0 && geo.hlo >= 0) {
                        mp = &lmap;
                        pz = p + 2;
                    } else if (p >= geo.nz && geo.hhi >= 0) {
                        mp = &lmap;
                        pz = 2 + p - geo.nz;
                    }
                    if (mp == &lmap && !waited) {
                        for (int q = 0; q < geo.world; ++q)
                            if ((geo.recv_mask >> q) & 1u) wait_flag(geo.flags + q, geo.epoch, geo.err);
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        waited = true;
                    }
                    if (g >= geo.nst) mbar_wait(empty + s, eph);
                    double* st = smem + static_cast<size_t>(s) * kXPlane2;
                    mbar_expect_tx(full + s, kXPlane2 * 8u);
                    tma_load_4d(st, mp, tx * kTile - 2, ty * kTile - 2, pz, c, full + s);
                    if (++s == geo.nst) {
                        s = 0;
                        if (g >= geo.nst) eph ^= 1u;
                    }
                }
            }
        }
        return;
    }
    int qs = 0;
    unsigned qph = 0;
    auto advance = [&](int& sl, unsigned& ph) {
        if (++sl == geo.nst) {
            sl = 0;
            ph ^= 1u;
        }
    };
    auto release = [&](int sl) {
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(empty + sl)) : "memory");
    };
    auto cbar = [] { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); };
    const int64_t nxny = static_cast<int64_t>(geo.nx) * geo.ny;
    for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
        int c, tx, ty, z0, z1;
        decode(it, c, tx, ty, z0, z1);
        double* ycol = ea.Y.ptr + static_cast<int64_t>(c) * ea.Y.cs;
        double* hcol = ea.H.ptr + static_cast<int64_t>(c) * ea.H.cs;
        // X stages of planes zA - 1, zA, zA + 1 (zA = the plane step i computes next)
        int sm = qs, sc = qs;
        unsigned pm = qph, pc = qph;
        advance(sc, pc);
        mbar_wait(full + sm, pm);
        mbar_wait(full + sc, pc);
        cbar();  // the previous item's step-2 reads of the q ring are done
        for (int zA = z0 - 1; zA <= z1; ++zA) {
            int sn = sc;
            unsigned pn = pc;
            advance(sn, pn);
            mbar_wait(full + sn, pn);
            const double* x0p = smem + static_cast<size_t>(sm) * kXPlane2;  // plane zA - 1
            const double* x1p = smem + static_cast<size_t>(sc) * kXPlane2;  // plane zA
            const double* x2p = smem + static_cast<size_t>(sn) * kXPlane2;  // plane zA + 1
            const int zB = zA - 1;
            const bool doB = zB >= z0;
            // H of the step-2 outputs, loaded before step 1 runs (latency hidden behind it)
            double hv[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int x = tx * kTile + lane, y = ty * kTile + warp + 8 * j;
                hv[j] = (doB && !ea.first && x < geo.nx && y < geo.ny)
                            ? hcol[static_cast<int64_t>(zB) * nxny + static_cast<int64_t>(y) * geo.nx + x]
                            : 0.0;
            }
            // step i on plane zA, tile + one-point ring
            {
                double* q = qring + static_cast<size_t>((zA - z0 + 1) & 3) * kQPlane;
                const int zg = geo.z0 + zA;
                const bool zm = zg > 0, zp = zg + 1 < geo.nzg;
                for (int p = tid; p < kQPts; p += kConsumers) {
                    const int rr = p / kQW, cc = p - rr * kQW;
                    const int x = tx * kTile - 1 + cc, y = ty * kTile - 1 + rr;
                    const bool xm = x > 0, xp = x + 1 < geo.nx, ym = y > 0, yp = y + 1 < geo.ny;
                    const int ctr = (rr + 1) * kBox2 + cc + 1;
                    const double xi = x1p[ctr];
                    double acc = 0.0;
                    const int deg = zm + ym + xm + xp + yp + zp;
                    if (zm) acc = __dsub_rn(acc, x0p[ctr]);
                    if (ym) acc = __dsub_rn(acc, x1p[ctr - kBox2]);
                    if (xm) acc = __dsub_rn(acc, x1p[ctr - 1]);
                    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(deg), xi));
                    if (xp) acc = __dsub_rn(acc, x1p[ctr + 1]);
                    if (yp) acc = __dsub_rn(acc, x1p[ctr + kBox2]);
                    if (zp) acc = __dsub_rn(acc, x2p[ctr]);
                    q[p] = __dsub_rn(xi, __dmul_rn(ea.inv_cur, acc));
                }
            }
            cbar();
            if (doB) {
                // step i + 1 on plane zB = zA - 1 from q planes zB - 1, zB, zB + 1
                const double* q0 = qring + static_cast<size_t>((zB - z0) & 3) * kQPlane;
                const double* q1 = qring + static_cast<size_t>((zB - z0 + 1) & 3) * kQPlane;
                const double* q2 = qring + static_cast<size_t>((zB - z0 + 2) & 3) * kQPlane;
                const int zg = geo.z0 + zB;
                const bool zm = zg > 0, zp = zg + 1 < geo.nzg;
                const int x = tx * kTile + lane;
                const bool xm = x > 0, xp = x + 1 < geo.nx;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int ly = warp + 8 * j;
                    const int y = ty * kTile + ly;
                    const bool ym = y > 0, yp = y + 1 < geo.ny;
                    const int qc = (ly + 1) * kQW + lane + 1;
                    const double qi = q1[qc];
                    double acc = 0.0;
                    const int deg = zm + ym + xm + xp + yp + zp;
                    if (zm) acc = __dsub_rn(acc, q0[qc]);
                    if (ym) acc = __dsub_rn(acc, q1[qc - kQW]);
                    if (xm) acc = __dsub_rn(acc, q1[qc - 1]);
                    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(deg), qi));
                    if (xp) acc = __dsub_rn(acc, q1[qc + 1]);
                    if (yp) acc = __dsub_rn(acc, q1[qc + kQW]);
                    if (zp) acc = __dsub_rn(acc, q2[qc]);
                    const double r = __dsub_rn(qi, __dmul_rn(ea.inv_next, acc));
                    if (x < geo.nx && y < geo.ny) {
                        const int64_t row = static_cast<int64_t>(zB) * nxny + static_cast<int64_t>(y) * geo.nx + x;
                        ycol[row] = r;
                        const double pi = x0p[(ly + 2) * kBox2 + lane + 2];  // p_i on plane zB
                        double h = ea.first ? __dmul_rn(ea.inv_cur, pi) : __dadd_rn(hv[j], __dmul_rn(ea.inv_cur, pi));
                        h = __dadd_rn(h, __dmul_rn(ea.inv_next, qi));
                        if (ea.last) h = __dadd_rn(h, __dmul_rn(ea.inv_after, r));
                        hcol[row] = h;
                    }
                }
            }
            release(sm);  // plane zA - 1: steps i (zA) and i + 1 (zA - 1) are done with it
            sm = sc;
            pm = pc;
            sc = sn;
            pc = pn;
        }
        release(sm);  // planes z1 and z1 + 1
        release(sc);
        qs = sc;
        qph = pc;
        advance(qs, qph);
    }
}

// ---- tensor maps (driver entry point: the library links only the runtime) ----
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess) {
            cudaGetLastError();
            return static_cast<EncodeTiledFn>(nullptr);
        }
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// the block as a 4-D tensor (x, y, z, column) of doubles; planes from row `row_off`
void make_map(CUtensorMap* map, const View& v, int m, const DevOp& op, int box_x, int box_y, int nz = 0,
              int64_t row_off = 0) {
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(op.mesh_nx), static_cast<cuuint64_t>(op.mesh_ny),
                                static_cast<cuuint64_t>(nz > 0 ? nz : op.mesh_nz), static_cast<cuuint64_t>(m)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(op.mesh_nx) * 8,
                                   static_cast<cuuint64_t>(op.mesh_nx) * op.mesh_ny * 8,
                                   static_cast<cuuint64_t>(m > 1 ? v.cs : (op.n + 1) & ~int64_t(1)) * 8};
    const cuuint32_t box[4] = {static_cast<cuuint32_t>(box_x), static_cast<cuuint32_t>(box_y), 1, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, v.ptr + row_off, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw SpError(8, "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
}

template <bool BOX27, int EPI>
int launch_mesh(const DevOp& op, const View& X, int m, const EpiArgs& ea, cudaStream_t s, const HaloFuse* hf) {
    MeshGeo geo{};
    geo.nx = op.mesh_nx;
    geo.ny = op.mesh_ny;
    geo.nz = op.mesh_nz;
    geo.z0 = op.mesh_z0;
    geo.nzg = op.mesh_nzg > 0 ? op.mesh_nzg : op.mesh_nz;
    const int64_t nxny = static_cast<int64_t>(op.mesh_nx) * op.mesh_ny;
    const bool lo = op.mesh_halo_lo >= 0, hi = op.mesh_halo_hi >= 0;
    // one map over the halo planes: [below | above] as the halo plan numbers them
    const int64_t hrow = lo ? op.mesh_halo_lo : op.mesh_halo_hi;
    geo.hlo = lo ? 0 : -1;
    geo.hhi = hi ? static_cast<int>((op.mesh_halo_hi - hrow) / nxny) : -1;
    geo.zrot = (lo || hi) ? 1 : 0;
    if (hf && hf->on) {
        geo.flags = hf->my_flags;
        geo.epoch = hf->epoch;
        geo.recv_mask = hf->recv_mask;
        geo.world = hf->world;
        geo.err = hf->err;
    }
    geo.ntx = (geo.nx + kTile - 1) / kTile;
    geo.nty = (geo.ny + kTile - 1) / kTile;
    geo.h_stage = (EPI == EPI_POLY && !ea.first && ea.h_terms) ? 1 : 0;
    geo.stage = kXPlanePad + (geo.h_stage ? kHPlane : 0);
    auto kern = spmm_mesh_kernel<BOX27, EPI>;
    static bool attr = false;
    if (!attr) {
        SPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    // ring: up to 6 stages within 100 KB, two CTAs per SM
    const size_t per_stage = sizeof(double) * geo.stage;
    const size_t budget = 100 * 1024;
    geo.nst = static_cast<int>(std::min<size_t>(6, budget / per_stage));
    const size_t smem = per_stage * geo.nst;
    int per_sm = 0;
    SPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMeshThreads, smem));
    const int ctas = device_sm_count() * std::max(per_sm, 1);
    // z chunks: enough work items for ~4 per CTA, at least 8 planes per chunk (the two
    // halo planes of a chunk are re-read from L2)
    const int64_t per_chunk = static_cast<int64_t>(geo.ntx) * geo.nty * m;
    int nzc = static_cast<int>(std::min<int64_t>(geo.nz, std::max<int64_t>(1, (4LL * ctas + per_chunk - 1) / per_chunk)));
    nzc = std::min(nzc, std::max(1, geo.nz / 8));
    geo.zc = (geo.nz + nzc - 1) / nzc;
    geo.nzc = (geo.nz + geo.zc - 1) / geo.zc;
    const int64_t items = per_chunk * geo.nzc;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(items, ctas)));
    CUtensorMap xmap, hmap, lmap;
    make_map(&xmap, X, m, op, kHaloW, kHaloH);
    if (geo.h_stage) make_map(&hmap, ea.H, m, op, kTile, kTile);
    else hmap = xmap;
    if (lo || hi) make_map(&lmap, X, m, op, kHaloW, kHaloH, (lo ? 1 : 0) + (hi ? 1 : 0), hrow);
    else lmap = xmap;
    kern<<<grid, kMeshThreads, smem, s>>>(xmap, hmap, lmap, op, ea, m, geo);
    SPB_LAUNCH_CHECK();
    return grid;
}

int launch_mesh_poly2(const DevOp& op, const View& X, int m, const EpiArgs& ea, cudaStream_t s, const HaloFuse* hf) {
    MeshGeo geo{};
    geo.nx = op.mesh_nx;
    geo.ny = op.mesh_ny;
    geo.nz = op.mesh_nz;
    geo.z0 = op.mesh_z0;
    geo.nzg = op.mesh_nzg > 0 ? op.mesh_nzg : op.mesh_nz;
    const bool slab = op.mesh_halo2 >= 0;
    geo.hlo = slab && op.mesh_halo_lo >= 0 ? 0 : -1;
    geo.hhi = slab && op.mesh_halo_hi >= 0 ? 2 : -1;
    geo.zrot = slab ? 1 : 0;
    if (hf && hf->on) {
        geo.flags = hf->my_flags;
        geo.epoch = hf->epoch;
        geo.recv_mask = hf->recv_mask;
        geo.world = hf->world;
        geo.err = hf->err;
    }
    geo.ntx = (geo.nx + kTile - 1) / kTile;
    geo.nty = (geo.ny + kTile - 1) / kTile;
    auto kern = spmm_mesh_poly2_kernel;
    static bool attr = false;
    if (!attr) {
        SPB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    // X ring + the 4-plane q ring, two CTAs per SM
    const size_t qbytes = sizeof(double) * 4 * kQPlane;
    geo.nst = static_cast<int>(std::min<size_t>(6, (108 * 1024 - qbytes) / (sizeof(double) * kXPlane2)));
    const size_t smem = sizeof(double) * kXPlane2 * geo.nst + qbytes;
    int per_sm = 0;
    SPB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kMeshThreads, smem));
    const int ctas = device_sm_count() * std::max(per_sm, 1);
    const int64_t per_chunk = static_cast<int64_t>(geo.ntx) * geo.nty * m;
    int nzc = static_cast<int>(std::min<int64_t>(geo.nz, std::max<int64_t>(1, (4LL * ctas + per_chunk - 1) / per_chunk)));
    nzc = std::min(nzc, std::max(1, geo.nz / 8));
    geo.zc = (geo.nz + nzc - 1) / nzc;
    geo.nzc = (geo.nz + geo.zc - 1) / geo.zc;
    const int64_t items = per_chunk * geo.nzc;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(items, ctas)));
    CUtensorMap xmap, lmap;
    make_map(&xmap, X, m, op, kBox2, kBox2);
    if (slab) make_map(&lmap, X, m, op, kBox2, kBox2, 4, op.mesh_halo2);  // [z0-2, z0-1 | z1, z1+1]
    else lmap = xmap;
    kern<<<grid, kMeshThreads, smem, s>>>(xmap, lmap, op, ea, m, geo);
    SPB_LAUNCH_CHECK();
    return grid;
}

__global__ void mesh_verify_kernel(const DevOp op, int nx, int ny, int nz, int W, bool box27, int* bad) {
    const int64_t nxny = static_cast<int64_t>(nx) * ny;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < op.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int x = static_cast<int>(i % nx), y = static_cast<int>((i / nx) % ny), z = static_cast<int>(i / nxny);
        const int p = op.ell_pat[i];
        int cnt = 0;
        bool ok = true;
        for (int s = 0; s < W && ok; ++s) {
            const int32_t d = op.ell_pat_tab[p * W + s];
            if (d == kEllPad) continue;
            const int dz = d > nxny / 2 ? 1 : (d < -nxny / 2 ? -1 : 0);
            const int64_t r = d - dz * nxny;
            const int dy = r > nx / 2 ? 1 : (r < -nx / 2 ? -1 : 0);
            const int dx = static_cast<int>(r - static_cast<int64_t>(dy) * nx);
            ok = dx >= -1 && dx <= 1 && x + dx >= 0 && x + dx < nx && y + dy >= 0 && y + dy < ny && z + dz >= 0 &&
                 z + dz < nz && (box27 || (dx != 0) + (dy != 0) + (dz != 0) == 1);
            ++cnt;
        }
        // the row holds every in-bounds point of its stencil (offsets are sorted and distinct)
        const int cx = 1 + (x > 0) + (x + 1 < nx), cy = 1 + (y > 0) + (y + 1 < ny), cz = 1 + (z > 0) + (z + 1 < nz);
        const int want = box27 ? cx * cy * cz - 1 : (cx - 1) + (cy - 1) + (cz - 1);
        if (!ok || cnt != want) atomicExch(bad, 1);
    }
}

// the rank's rows [row0, row0 + n) of the global mesh: every row's global columns are
// exactly the in-bounds points of its stencil, ascending, no diagonal
__global__ void mesh_verify_csr_kernel(const DevOp op, int nx, int ny, int nzg, bool box27, int* bad) {
    const int64_t nxny = static_cast<int64_t>(nx) * ny;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < op.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t gi = op.row0 + i;
        const int x = static_cast<int>(gi % nx), y = static_cast<int>((gi / nx) % ny), z = static_cast<int>(gi / nxny);
        const int64_t k0 = op.offs[i], k1 = op.offs[i + 1];
        bool ok = true;
        int64_t prev = -1;
        for (int64_t k = k0; k < k1 && ok; ++k) {
            const int64_t j = op.cols[k];
            const int64_t d = j - gi;
            const int jx = static_cast<int>(j % nx), jy = static_cast<int>((j / nx) % ny),
                      jz = static_cast<int>(j / nxny);
            const int dx = jx - x, dy = jy - y, dz = jz - z;
            ok = j > prev && d != 0 && j >= 0 && jz < nzg && dx >= -1 && dx <= 1 && dy >= -1 && dy <= 1 && dz >= -1 &&
                 dz <= 1 && (box27 || (dx != 0) + (dy != 0) + (dz != 0) == 1);
            prev = j;
        }
        const int cx = 1 + (x > 0) + (x + 1 < nx), cy = 1 + (y > 0) + (y + 1 < ny), cz = 1 + (z > 0) + (z + 1 < nzg);
        const int want = box27 ? cx * cy * cz - 1 : (cx - 1) + (cy - 1) + (cz - 1);
        if (!ok || k1 - k0 != want) atomicExch(bad, 1);
    }
}

} // namespace

bool no_mesh_kernel() {
    static const bool off = [] {
        const char* e = std::getenv("SPB_MESH");
        return e && e[0] == '0';
    }();
    return off;
}

bool mesh_plan(DevOp& op, cudaStream_t s) {
    op.mesh_nx = op.mesh_ny = op.mesh_nz = 0;
    if (!op.ell_pat || op.ell_npat <= 0 || op.row0 != 0 || op.dpos || !encode_fn()) return false;
    const int W = op.ell_kl + op.ell_ku;
    if (W != 4 && W != 6 && W != 26) return false;
    std::vector<int32_t> tab(static_cast<size_t>(op.ell_npat) * W);
    SPB_CUDA(cudaMemcpyAsync(tab.data(), op.ell_pat_tab, sizeof(int32_t) * tab.size(), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    std::vector<int64_t> pos;
    for (int32_t d : tab)
        if (d != kEllPad && d > 0) pos.push_back(d);
    std::sort(pos.begin(), pos.end());
    pos.erase(std::unique(pos.begin(), pos.end()), pos.end());
    // positive offsets: 5/7-point {1, nx[, nx*ny]}; 27-point {1, nx-1, nx, nx+1[, nx*ny-nx-1 .. nx*ny+nx+1]}
    int64_t nx = 0, nxny = 0;
    const bool box27 = W == 26;
    if (!box27 && (pos.size() == 2 || pos.size() == 3) && pos[0] == 1) {
        nx = pos[1];
        nxny = pos.size() == 3 ? pos[2] : op.n;
    } else if (box27 && (pos.size() == 4 || pos.size() == 13) && pos[0] == 1) {
        nx = pos[2];
        nxny = pos.size() == 13 ? pos[8] : op.n;
    } else {
        return false;
    }
    if (nx < 4 || nxny % nx || op.n % nxny) return false;
    const int64_t ny = nxny / nx, nz = op.n / nxny;
    if (nx % 2 || nx > (1 << 30) || ny > (1 << 30) || nz > (1 << 30)) return false;  // TMA: 16-byte strides
    DBuf<int> bad(1);
    SPB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    mesh_verify_kernel<<<grid_for(op.n, 256, 8), 256, 0, s>>>(op, static_cast<int>(nx), static_cast<int>(ny),
                                                              static_cast<int>(nz), W, box27, bad.p);
    SPB_LAUNCH_CHECK();
    int hb = 1;
    SPB_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    if (hb) return false;
    op.mesh_nx = static_cast<int>(nx);
    op.mesh_ny = static_cast<int>(ny);
    op.mesh_nz = static_cast<int>(nz);
    op.mesh_z0 = 0;
    op.mesh_nzg = static_cast<int>(nz);
    op.mesh_box27 = box27 ? 1 : 0;
    op.mesh_halo_lo = op.mesh_halo_hi = -1;
    return true;
}

bool mesh_plan_slab(DevOp& op, int64_t n_global, cudaStream_t s) {
    op.mesh_nx = op.mesh_ny = op.mesh_nz = 0;
    if (op.mode != OP_LAPLACE_UNIT || op.n <= 0 || op.max_row > 26 || op.n_long > 0 || !encode_fn()) return false;
    // candidate geometry from the positive offsets of a few rows near the middle of the block
    const int64_t cand[3] = {op.n / 2, op.n / 2 + 7, op.n / 3 + 13};
    for (int64_t ci : cand) {
        const int64_t i = std::min<int64_t>(std::max<int64_t>(ci, 0), op.n - 1);
        int64_t k[2];
        SPB_CUDA(cudaMemcpyAsync(k, op.offs + i, sizeof(k), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        const int len = static_cast<int>(k[1] - k[0]);
        if (len <= 0 || len > 26) continue;
        std::vector<int32_t> c(len);
        SPB_CUDA(cudaMemcpyAsync(c.data(), op.cols + k[0], sizeof(int32_t) * len, cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        std::vector<int64_t> pos;
        for (int32_t j : c)
            if (j > op.row0 + i) pos.push_back(j - (op.row0 + i));
        int64_t nx = 0, nxny = 0;
        bool box27 = false;
        if (pos.size() == 3 && pos[0] == 1) {
            nx = pos[1];
            nxny = pos[2];
        } else if (pos.size() == 13 && pos[0] == 1) {
            nx = pos[2];
            nxny = pos[8];
            box27 = true;
        } else {
            continue;
        }
        if (nx < 4 || nx % 2 || nxny % nx || n_global % nxny || op.row0 % nxny || op.n % nxny) continue;
        const int64_t ny = nxny / nx, nzg = n_global / nxny;
        if (ny > (1 << 30) || nzg > (1 << 30)) continue;
        DBuf<int> bad(1);
        SPB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
        mesh_verify_csr_kernel<<<grid_for(op.n, 256, 8), 256, 0, s>>>(op, static_cast<int>(nx), static_cast<int>(ny),
                                                                      static_cast<int>(nzg), box27, bad.p);
        SPB_LAUNCH_CHECK();
        int hb = 1;
        SPB_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        if (hb) continue;
        op.mesh_nx = static_cast<int>(nx);
        op.mesh_ny = static_cast<int>(ny);
        op.mesh_nz = static_cast<int>(op.n / nxny);
        op.mesh_z0 = static_cast<int>(op.row0 / nxny);
        op.mesh_nzg = static_cast<int>(nzg);
        op.mesh_box27 = box27 ? 1 : 0;
        op.mesh_halo_lo = op.mesh_halo_hi = -1;  // set once the halo plan exists (Solver)
        return true;
    }
    return false;
}

bool spmm_mesh_ok(const DevOp& op, const View& X, int m, const EpiArgs& ea) {
    if (op.mesh_nx <= 0 || op.mode != OP_LAPLACE_UNIT || op.row0 != 0 || m > kMaxCols)
        return false;
    // column-major blocks, 16-byte aligned bases and column strides (TMA global address rules)
    auto ok = [&](const View& v) {
        return v.rs == 1 && reinterpret_cast<uintptr_t>(v.ptr) % 16 == 0 && (m == 1 || (v.cs % 2 == 0 && v.cs >= op.n));
    };
    if (!ok(X) || ea.Y.rs != 1 || (ea.mode == EPI_POLY && ea.h_terms && ea.H.rs != 1)) return false;
    if (ea.mode == EPI_POLY && ea.h_terms && !ea.first && !ok(ea.H)) return false;
    return true;
}

bool spmm_mesh_poly2_ok(const DevOp& op, const View& X, int m, const EpiArgs& ea) {
    static const bool off = [] {  // SPB_POLY2=0: one step per launch (the bit-exactness test's reference)
        const char* e = std::getenv("SPB_POLY2");
        return e && e[0] == '0';
    }();
    if (off || !spmm_mesh_ok(op, X, m, ea) || op.mesh_box27 || ea.mode != EPI_POLY) return false;
    // one GPU, or a z-slab with the two-plane halo set up; H column-major
    const bool one = op.mesh_halo_lo < 0 && op.mesh_halo_hi < 0 && op.mesh_z0 == 0 && op.mesh_nzg == op.mesh_nz;
    return (one || op.mesh_halo2 >= 0) && ea.H.rs == 1 && ea.Y.rs == 1;
}

int spmm_mesh_poly2_launch(const DevOp& op, const View& X, int m, const EpiArgs& ea, cudaStream_t s,
                           const HaloFuse* hf) {
    return launch_mesh_poly2(op, X, m, ea, s, hf);
}

int spmm_mesh_launch(const DevOp& op, const View& X, int m, EpiArgs& ea, cudaStream_t s, const HaloFuse* hf) {
    const bool box27 = op.mesh_box27 != 0;
    switch (ea.mode) {
#define SPB_MESH(EPI_)                                                                  \
    return box27 ? launch_mesh<true, EPI_>(op, X, m, ea, s, hf) : launch_mesh<false, EPI_>(op, X, m, ea, s, hf);
    case EPI_STORE: SPB_MESH(EPI_STORE)
    case EPI_RESIDUAL: SPB_MESH(EPI_RESIDUAL)
    default: SPB_MESH(EPI_POLY)
#undef SPB_MESH
    }
}

} // namespace spb
