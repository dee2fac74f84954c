// halo.cu — halo exchange for the row-partitioned operator.
//
// The reference is single-node; its SpMM reads x_j for every stored
// column j (kernels.cpp:20-48). With rows split over GPUs, rank k needs x_j
// only for the columns of its rows that it does not own — two z-slabs for a
// 3-D mesh, a scattered set for R-MAT. Setup (once per operator):
//   1. bitmap of referenced foreign ids -> sorted halo list (per-word popcount
//      scan, so the list is ascending and therefore grouped by owner rank);
//   2. columns rewritten to local ids: own j -> j-row0, halo j -> nloc+slot;
//   3. dpos[i] = number of stored columns with global id < i: the slot where
//      the reference's laplacian.cpp:53-79 splices the diagonal, which local
//      ids no longer encode;
//   4. counts all-gathered, halo id lists sent to their owners (grouped
//      ncclSend/ncclRecv), which become the owners' send lists.
// Per SpMM: pack the rows peers need, one grouped send/recv round, unpack into
// the halo rows of the input block. Results are bit-identical to the one-GPU
// operator: the accumulation order of every row is unchanged.
#include "context.hpp"

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <vector>

namespace spb {

namespace {

__global__ void mark_foreign_kernel(int64_t nnz, const int32_t* cols, int64_t lo, int64_t hi, uint32_t* bm) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = cols[k];
        if (j < lo || j >= hi) atomicOr(&bm[j >> 5], 1u << (j & 31));
    }
}

__global__ void popc_kernel(int64_t words, const uint32_t* bm, int32_t* cnt) {
    for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < words;
         w += static_cast<int64_t>(gridDim.x) * blockDim.x)
        cnt[w] = __popc(bm[w]);
}

__global__ void emit_halo_kernel(int64_t words, const uint32_t* bm, const int32_t* off, int32_t* halo) {
    for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < words;
         w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint32_t b = bm[w];
        int32_t o = off[w];
        while (b) {
            const int bit = __ffs(b) - 1;
            halo[o++] = static_cast<int32_t>(w * 32 + bit);
            b &= b - 1;
        }
    }
}

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* a, int64_t n, int64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void remap_cols_kernel(int64_t nnz, const int32_t* cols, int64_t lo, int64_t hi, const int32_t* halo,
                                  int64_t nhalo, int64_t base, int32_t* out) {
    for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < nnz;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t j = cols[k];
        out[k] = static_cast<int32_t>((j >= lo && j < hi) ? j - lo : base + lower_bound_i32(halo, nhalo, j));
    }
}

// interior rows: [P, Q) with P = 1 + last row referencing a lower rank, Q = first
// row referencing a higher rank (a slab partition of a banded mesh)
__global__ void interior_kernel(int64_t n, const int64_t* offs, const int32_t* cols, int64_t lo, int64_t hi,
                                unsigned long long* pq) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        bool below = false, above = false;
        for (int64_t k = offs[i]; k < offs[i + 1]; ++k) {
            below |= cols[k] < lo;
            above |= cols[k] >= hi;
        }
        if (below) atomicMax(&pq[0], static_cast<unsigned long long>(i + 1));
        if (above) atomicMin(&pq[1], static_cast<unsigned long long>(i));
    }
}

__global__ void dpos_kernel(int64_t n, int64_t row0, const int64_t* offs, const int32_t* cols, int32_t* dpos) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        int32_t c = 0;
        for (int64_t k = offs[i]; k < offs[i + 1]; ++k) c += cols[k] < row0 + i ? 1 : 0;
        dpos[i] = c;
    }
}

__global__ void isd_halo_kernel(int64_t nloc, int64_t base, int64_t row0, const int32_t* halo, int64_t nhalo,
                                const double* isd, double* out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < base + nhalo;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = i < nloc ? isd[row0 + i] : (i < base ? 0.0 : isd[halo[i - base]]);
}

__global__ void owner_bounds_kernel(const int32_t* halo, int64_t nhalo, int64_t n_pad, int world, int64_t* b) {
    const int p = threadIdx.x;
    if (p <= world) b[p] = lower_bound_i32(halo, nhalo, static_cast<int64_t>(p) * n_pad);
}

__global__ void to_local_kernel(int64_t n, int32_t* ids, int64_t row0) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        ids[i] = static_cast<int32_t>(ids[i] - row0);
}

__global__ void halo_pack_kernel(int64_t rows, const int32_t* idx, View X, int m, double* out) {
    const int64_t total = rows * m;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t t = e / m;
        const int c = static_cast<int>(e - t * m);
        out[e] = X.at(idx[t], c);
    }
}

__global__ void halo_unpack_kernel(int64_t rows, int64_t nloc, const double* in, int m, View X) {
    const int64_t total = rows * m;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t t = e / m;
        const int c = static_cast<int>(e - t * m);
        X.at(nloc + t, c) = in[e];
    }
}

} // namespace

void localize_operator(Comm& cm, const DevGraph& g, DevLaplacian& L, cudaStream_t s) {
    HaloPlan& hp = cm.halo;
    hp = HaloPlan{};
    if (!cm.active()) return;
    DevOp& op = L.op;
    const int64_t nloc = g.n_local, lo = g.row0, hi = g.row0 + g.n_local;
    const int64_t n = cm.n_global, nnz = op.mode == OP_DIAGONAL ? 0 : op.nnz;
    const int world = cm.world;

    // 1. foreign-id bitmap -> ascending halo list
    const int64_t words = (n + 31) / 32;
    DBuf<uint32_t> bm(std::max<int64_t>(words, 1));
    DBuf<int32_t> wcnt(std::max<int64_t>(words, 1) + 1), woff(std::max<int64_t>(words, 1) + 1);
    SPB_CUDA(cudaMemsetAsync(bm.p, 0, sizeof(uint32_t) * std::max<int64_t>(words, 1), s));
    if (nnz > 0) {
        mark_foreign_kernel<<<grid_for(nnz, 256, 8), 256, 0, s>>>(nnz, op.cols, lo, hi, bm.p);
        SPB_LAUNCH_CHECK();
    }
    popc_kernel<<<grid_for(words, 256, 8), 256, 0, s>>>(words, bm.p, wcnt.p);
    SPB_LAUNCH_CHECK();
    SPB_CUDA(cudaMemsetAsync(wcnt.p + words, 0, sizeof(int32_t), s));
    size_t tmp_bytes = 0;
    SPB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, wcnt.p, woff.p, words + 1, s));
    DBuf<unsigned char> tmp(std::max<size_t>(tmp_bytes, 1));
    SPB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, wcnt.p, woff.p, words + 1, s));
    int32_t nh = 0;
    SPB_CUDA(cudaMemcpyAsync(&nh, woff.p + words, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    hp.nhalo = nh;
    DBuf<int32_t> halo(std::max<int64_t>(nh, 1));
    emit_halo_kernel<<<grid_for(words, 256, 8), 256, 0, s>>>(words, bm.p, woff.p, halo.p);
    SPB_LAUNCH_CHECK();

    // 2./3. local column ids, diagonal slots, isd over own + halo rows; halo
    // rows start at a 32-row boundary so no cache line holds own and halo rows
    const int64_t base = (nloc + 1 + 31) / 32 * 32;  // row nloc stays zero (ELL padding)
    hp.halo_base = base;
    {
        DBuf<unsigned long long> pq(2);
        const unsigned long long init[2] = {0ull, static_cast<unsigned long long>(nloc)};
        SPB_CUDA(cudaMemcpyAsync(pq.p, init, sizeof(init), cudaMemcpyHostToDevice, s));
        if (nnz > 0 && nloc > 0) {
            interior_kernel<<<grid_for(nloc, 256, 8), 256, 0, s>>>(nloc, op.offs, op.cols, lo, hi, pq.p);
            SPB_LAUNCH_CHECK();
        }
        unsigned long long h[2];
        SPB_CUDA(cudaMemcpyAsync(h, pq.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        const int64_t ntiles = (nloc + 31) / 32;
        const int64_t P = static_cast<int64_t>(h[0]), Q = static_cast<int64_t>(h[1]);
        hp.rot_tiles = ntiles > 0 ? std::min<int64_t>((P + 31) / 32, ntiles) % ntiles : 0;
        const int64_t q_t = Q >= nloc ? ntiles : Q / 32;
        hp.n_int_tiles = (P <= Q && ntiles > 0) ? std::max<int64_t>(0, q_t - (P + 31) / 32) : 0;
    }
    if (nnz > 0) {
        L.cols_halo.alloc(nnz);
        remap_cols_kernel<<<grid_for(nnz, 256, 8), 256, 0, s>>>(nnz, op.cols, lo, hi, halo.p, nh, base,
                                                               L.cols_halo.p);
        SPB_LAUNCH_CHECK();
        if (op.mode == OP_LAPLACE_UNIT || op.mode == OP_NORMAL_UNIT) {
            L.dpos.alloc(std::max<int64_t>(nloc, 1));
            dpos_kernel<<<grid_for(std::max<int64_t>(nloc, 1), 256, 8), 256, 0, s>>>(nloc, lo, op.offs, op.cols,
                                                                                   L.dpos.p);
            SPB_LAUNCH_CHECK();
            op.dpos = L.dpos.p;
        }
        op.cols = L.cols_halo.p;
    }
    if (op.isd) {
        L.isd_halo.alloc(std::max<int64_t>(base + nh, 1));
        isd_halo_kernel<<<grid_for(std::max<int64_t>(base + nh, 1), 256, 8), 256, 0, s>>>(nloc, base, lo, halo.p,
                                                                                        nh, op.isd, L.isd_halo.p);
        SPB_LAUNCH_CHECK();
        op.isd = L.isd_halo.p;
    }
    op.row0 = 0;
    op.x_rows = base + nh;

    // 4. per-owner counts, all-gathered; halo id lists to their owners
    DBuf<int64_t> bounds(world + 1), cnt(world), allcnt(static_cast<size_t>(world) * world);
    owner_bounds_kernel<<<1, 64 * ((world + 64) / 64), 0, s>>>(halo.p, nh, cm.n_pad, world, bounds.p);
    SPB_LAUNCH_CHECK();
    std::vector<int64_t> hb(world + 1);
    SPB_CUDA(cudaMemcpyAsync(hb.data(), bounds.p, sizeof(int64_t) * (world + 1), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    hp.recv_cnt.assign(world, 0);
    hp.recv_off.assign(world, 0);
    for (int p = 0; p < world; ++p) {
        hp.recv_off[p] = hb[p];
        hp.recv_cnt[p] = hb[p + 1] - hb[p];
    }
    SPB_CUDA(cudaMemcpyAsync(cnt.p, hp.recv_cnt.data(), sizeof(int64_t) * world, cudaMemcpyHostToDevice, s));
    SPB_NCCL(::spb::nccl().AllGather(cnt.p, allcnt.p, world, ncclInt64, cm.nccl, s));
    std::vector<int64_t> M(static_cast<size_t>(world) * world);
    SPB_CUDA(cudaMemcpyAsync(M.data(), allcnt.p, sizeof(int64_t) * M.size(), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    hp.send_cnt.assign(world, 0);
    hp.send_off.assign(world, 0);
    int64_t off = 0;
    for (int p = 0; p < world; ++p) {
        hp.send_cnt[p] = M[static_cast<size_t>(p) * world + cm.rank];  // rows p needs from me
        hp.send_off[p] = off;
        off += hp.send_cnt[p];
    }
    hp.total_send = off;
    hp.send_idx.alloc(std::max<int64_t>(off, 1));
    SPB_NCCL(::spb::nccl().GroupStart());
    for (int p = 0; p < world; ++p) {
        if (p == cm.rank) continue;
        if (hp.recv_cnt[p] > 0)
            SPB_NCCL(::spb::nccl().Send(halo.p + hp.recv_off[p], hp.recv_cnt[p], ncclInt32, p, cm.nccl, s));
        if (hp.send_cnt[p] > 0)
            SPB_NCCL(::spb::nccl().Recv(hp.send_idx.p + hp.send_off[p], hp.send_cnt[p], ncclInt32, p, cm.nccl, s));
    }
    SPB_NCCL(::spb::nccl().GroupEnd());
    if (off > 0) {
        to_local_kernel<<<grid_for(off, 256, 8), 256, 0, s>>>(off, hp.send_idx.p, lo);
        SPB_LAUNCH_CHECK();
    }
    // P2P push targets: destination rank and row of every send entry; the
    // common block height (max over ranks of own + halo rows)
    {
        std::vector<int32_t> dpeer(std::max<int64_t>(off, 1)), drow(std::max<int64_t>(off, 1));
        int64_t maxrows = 0;
        for (int p = 0; p < world; ++p) {
            const int64_t r0p = static_cast<int64_t>(p) * cm.n_pad;
            const int64_t nlp = (((r0p >= n ? 0 : std::min<int64_t>(cm.n_pad, n - r0p))) + 1 + 31) / 32 * 32;
            int64_t nhp = 0, before_me = 0;
            for (int q = 0; q < world; ++q) {
                nhp += M[static_cast<size_t>(p) * world + q];
                if (q < cm.rank) before_me += M[static_cast<size_t>(p) * world + q];
            }
            maxrows = std::max(maxrows, nlp + nhp);
            for (int64_t t = 0; t < hp.send_cnt[p]; ++t) {
                dpeer[hp.send_off[p] + t] = p;
                drow[hp.send_off[p] + t] = static_cast<int32_t>(nlp + before_me + t);
            }
            if (hp.send_cnt[p] > 0) hp.send_mask |= 1u << p;
            if (hp.recv_cnt[p] > 0) hp.recv_mask |= 1u << p;
        }
        hp.max_rows = maxrows;
        // 16-byte pushes need every even entry paired with the next one
        {
            std::vector<int32_t> srow(std::max<int64_t>(off, 1));
            if (off > 0)
                SPB_CUDA(cudaMemcpyAsync(srow.data(), hp.send_idx.p, sizeof(int32_t) * off, cudaMemcpyDeviceToHost, s));
            SPB_CUDA(cudaStreamSynchronize(s));
            bool ok = off > 0 && off % 2 == 0;
            for (int64_t t = 0; ok && t < off; t += 2)
                ok = dpeer[t] == dpeer[t + 1] && srow[t] % 2 == 0 && drow[t] % 2 == 0 && srow[t + 1] == srow[t] + 1 &&
                     drow[t + 1] == drow[t] + 1;
            hp.vec2 = ok;
            // copy-engine plan: every destination's entries form one contiguous source
            // run and one contiguous destination run
            hp.ce.clear();
            bool ce = off > 0;
            for (int p = 0; p < world && ce; ++p) {
                const int64_t t0 = hp.send_off[p], c = hp.send_cnt[p];
                if (c == 0) continue;
                for (int64_t t = t0 + 1; t < t0 + c && ce; ++t)
                    ce = srow[t] == srow[t0] + (t - t0) && drow[t] == drow[t0] + (t - t0);
                hp.ce.push_back({p, srow[t0], drow[t0], c});
            }
            hp.ce_ok = ce;
        }
        hp.dst_peer.alloc(dpeer.size());
        hp.dst_row.alloc(drow.size());
        SPB_CUDA(cudaMemcpyAsync(hp.dst_peer.p, dpeer.data(), sizeof(int32_t) * dpeer.size(), cudaMemcpyHostToDevice, s));
        SPB_CUDA(cudaMemcpyAsync(hp.dst_row.p, drow.data(), sizeof(int32_t) * drow.size(), cudaMemcpyHostToDevice, s));
    }
    SPB_CUDA(cudaStreamSynchronize(s));  // halo/bm/tmp are freed on return
    cm.sym_init(s);
    hp.on = true;
}

void Comm::halo_exchange(const View& X, int m, cudaStream_t s) {
    if (!active() || !halo.on) return;
    if (halo_push(*this, X, m, s)) return;  // NVLink peer writes (symm.cu)
    HaloPlan& hp = halo;
    hp.sendbuf.alloc(std::max<int64_t>(hp.total_send * m, 1));
    hp.recvbuf.alloc(std::max<int64_t>(hp.nhalo * m, 1));
    if (hp.total_send > 0) {
        halo_pack_kernel<<<grid_for(hp.total_send * m, 256, 8), 256, 0, s>>>(hp.total_send, hp.send_idx.p, X, m,
                                                                             hp.sendbuf.p);
        SPB_LAUNCH_CHECK();
    }
    SPB_NCCL(::spb::nccl().GroupStart());
    for (int p = 0; p < world; ++p) {
        if (p == rank) continue;
        if (hp.send_cnt[p] > 0)
            SPB_NCCL(::spb::nccl().Send(hp.sendbuf.p + hp.send_off[p] * m, hp.send_cnt[p] * m, ncclDouble, p, nccl,
                                        s));
        if (hp.recv_cnt[p] > 0)
            SPB_NCCL(::spb::nccl().Recv(hp.recvbuf.p + hp.recv_off[p] * m, hp.recv_cnt[p] * m, ncclDouble, p, nccl,
                                        s));
    }
    SPB_NCCL(::spb::nccl().GroupEnd());
    bytes_moved += hp.nhalo * m * 8;
    if (hp.nhalo > 0) {
        halo_unpack_kernel<<<grid_for(hp.nhalo * m, 256, 8), 256, 0, s>>>(hp.nhalo, hp.halo_base, hp.recvbuf.p, m, X);
        SPB_LAUNCH_CHECK();
    }
}

} // namespace spb
