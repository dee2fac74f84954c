// symm.cu — symmetric peer memory over NVLink for the row-partitioned solver.
//
// The NCCL halo round (pack kernel, grouped send/recv, unpack kernel) and the
// NCCL all-gather behind every small reduction cost ~20-30 us each, longer
// than the SpMM itself once rows are split 4-8 ways. Here the ranks of one
// box map each other's solver blocks (CUDA IPC, once per context) and
//   * halo_push: one kernel writes the boundary rows every peer needs straight
//     into the halo rows of that peer's copy of the input block, the last CTA
//     raises a flag on each destination, then waits for its own sources;
//   * sum_p2p: one CTA writes its partial vector into slot [rank] of every
//     peer, flags, waits, and sums the slots in rank order (the same order as
//     the NCCL path, so results are bit-identical to it on every rank).
// Write-after-read safety: a push into block B on a peer can only start after
// this rank consumed the peer's previous push, which the peer issued after
// finishing every earlier kernel, so the peer is no longer reading B unless B
// was the input of the immediately preceding exchange — that case is detected
// and preceded by a barrier. Sum slots alternate by epoch parity for the same
// reason. Every peer wait has a 30 s timeout that sets an error word (checked
// by the host) instead of hanging the GPU.
#include "context.hpp"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace spb {

namespace {

__global__ void halo_push_kernel(View X, int m, HaloFuse hf) {
    halo_push_part(hf, m, [&](int64_t r, int c) { return &X.at(r, c); });
    if (blockIdx.x == 0 && threadIdx.x < 32) halo_wait_warp(hf);
}

__global__ void halo_wait_kernel(HaloFuse hf) {
    if (threadIdx.x < 32) halo_wait_warp(hf);
}

__global__ void sum_p2p_kernel(double* dev, int count, int world, int me, PeerAddr slot, const double* my_slots,
                               PeerAddr remote_flag, const uint64_t* my_flags, uint64_t epoch, int* err) {
    for (int p = 0; p < world; ++p) {
        double* dst = reinterpret_cast<double*>(slot.p[p]);
        for (int e = threadIdx.x; e < count; e += blockDim.x) dst[e] = dev[e];
    }
    __syncthreads();
    if (threadIdx.x == 0) __threadfence_system();
    __syncthreads();
    const int p = threadIdx.x;
    if (p < world && p != me) {
        st_release_sys(reinterpret_cast<uint64_t*>(remote_flag.p[p]), epoch);
        wait_flag(my_flags + p, epoch, err);
    }
    __syncthreads();
    for (int e = threadIdx.x; e < count; e += blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < world; ++r) s += __ldcg(my_slots + static_cast<size_t>(r) * kSumMax + e);
        dev[e] = s;
    }
}

__global__ void barrier_kernel(int world, int me, PeerAddr remote_flag, const uint64_t* my_flags, uint64_t epoch,
                               int* err) {
    const int p = threadIdx.x;
    if (p < world && p != me) {
        __threadfence_system();
        st_release_sys(reinterpret_cast<uint64_t*>(remote_flag.p[p]), epoch);
        wait_flag(my_flags + p, epoch, err);
    }
}

} // namespace

// ---------------------------------------------------------------------------

static SymSeg map_segment(Comm& cm, size_t bytes, cudaStream_t s) {
    SymSeg seg;
    seg.size = bytes;
    SPB_CUDA(cudaMalloc(&seg.base, bytes));
    SPB_CUDA(cudaMemsetAsync(seg.base, 0, bytes, s));
    cudaIpcMemHandle_t h;
    SPB_CUDA(cudaIpcGetMemHandle(&h, seg.base));
    DBuf<unsigned char> mine(sizeof(h)), all(sizeof(h) * cm.world);
    SPB_CUDA(cudaMemcpyAsync(mine.p, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    SPB_NCCL(::spb::nccl().AllGather(mine.p, all.p, sizeof(h), ncclUint8, cm.nccl, s));
    std::vector<cudaIpcMemHandle_t> hs(cm.world);
    SPB_CUDA(cudaMemcpyAsync(hs.data(), all.p, sizeof(h) * cm.world, cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    seg.peer.assign(cm.world, nullptr);
    for (int p = 0; p < cm.world; ++p) {
        if (p == cm.rank) {
            seg.peer[p] = seg.base;
            continue;
        }
        void* q = nullptr;
        SPB_CUDA(cudaIpcOpenMemHandle(&q, hs[p], cudaIpcMemLazyEnablePeerAccess));
        seg.peer[p] = static_cast<char*>(q);
    }
    return seg;
}

bool Comm::sym_init(cudaStream_t s) {
    if (!active()) return false;
    if (sym.tried) return sym.on;
    sym.tried = true;
    const char* env = std::getenv("SPB_P2P");
    int ok = (env && env[0] == '0') || world > kMaxPeers ? 0 : 1;
    if (ok) {
        try {
            sym.ctrl = map_segment(*this, kCtrlBytes, s);
            sym.counter.alloc(1);
            sym.err.alloc(1);
            SPB_CUDA(cudaMemsetAsync(sym.counter.p, 0, sizeof(int), s));
            SPB_CUDA(cudaMemsetAsync(sym.err.p, 0, sizeof(int), s));
        } catch (const SpError&) {
            ok = 0;
            cudaGetLastError();
        }
    }
    // every rank must agree (a single failure sends everyone down the NCCL paths)
    DBuf<int> one(1), all(world);
    SPB_CUDA(cudaMemcpyAsync(one.p, &ok, sizeof(int), cudaMemcpyHostToDevice, s));
    SPB_NCCL(::spb::nccl().AllGather(one.p, all.p, 1, ncclInt32, nccl, s));
    std::vector<int> h(world);
    SPB_CUDA(cudaMemcpyAsync(h.data(), all.p, sizeof(int) * world, cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    sym.on = true;
    for (int v : h) sym.on = sym.on && v;
    return sym.on;
}

double* Comm::sym_alloc(size_t elems, cudaStream_t s) {
    const size_t bytes = ((elems * sizeof(double) + 255) / 256) * 256;
    while (sym.seg_i < sym.segs.size()) {
        SymSeg& g = sym.segs[sym.seg_i];
        if (sym.off + bytes <= g.size) {
            double* p = reinterpret_cast<double*>(g.base + sym.off);
            sym.off += bytes;
            return p;
        }
        ++sym.seg_i;
        sym.off = 0;
    }
    // new segment (collective: every rank reaches this point with the same sizes)
    const size_t seg_bytes = std::max<size_t>(bytes, size_t(256) << 20);
    sym.segs.push_back(map_segment(*this, seg_bytes, s));
    sym.seg_i = sym.segs.size() - 1;
    sym.off = bytes;
    return reinterpret_cast<double*>(sym.segs.back().base);
}

int64_t Comm::sym_delta(const void* p, int peer) const {
    const char* c = static_cast<const char*>(p);
    for (const SymSeg& g : sym.segs)
        if (c >= g.base && c < g.base + g.size) return static_cast<int64_t>(g.peer[peer] - g.base);
    return INT64_MIN;
}

void Comm::sym_check(cudaStream_t s) {
    if (!sym.on) return;
    int e = 0;
    SPB_CUDA(cudaMemcpyAsync(&e, sym.err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    if (e) SPB_CUDA(cudaMemsetAsync(sym.err.p, 0, sizeof(int), s));
    if (e) throw SpError(9, "P2P: timed out waiting for a peer rank (a rank failed or diverged)");
}

static PeerAddr flag_addrs(const Comm& cm, size_t flag_off) {
    PeerAddr a{};
    for (int p = 0; p < cm.world; ++p)
        a.p[p] = cm.sym.ctrl.peer[p] + flag_off + sizeof(uint64_t) * cm.rank;  // my slot on p
    return a;
}

void Comm::barrier_p2p(cudaStream_t s) {
    ++sym.bar_epoch;
    barrier_kernel<<<1, 32, 0, s>>>(world, rank, flag_addrs(*this, kFlBar),
                                    reinterpret_cast<const uint64_t*>(sym.ctrl.base + kFlBar), sym.bar_epoch,
                                    sym.err.p);
    SPB_LAUNCH_CHECK();
}

static void fill_fuse(Comm& cm, const View& X, HaloFuse& hf) {
    HaloPlan& hp = cm.halo;
    hf.on = 1;
    hf.world = cm.world;
    hf.rot = hp.rot_tiles;
    hf.n_int = hp.n_int_tiles;
    // halo tiles after 60% of the interior (the peers' rows arrive ~10-15 us after
    // launch), interior work after them keeps the tail free of waits
    hf.bnd = hp.n_int_tiles * 60 / 100;
    hf.total = hp.total_send;
    // pairs are 16-byte aligned only in column-major blocks with even leading dimension
    hf.vec2 = (hp.vec2 && X.rs == 1 && (X.cols == 1 || X.cs % 2 == 0) &&
               reinterpret_cast<uintptr_t>(X.ptr) % 16 == 0) ? 1 : 0;
    hf.src_row = hp.send_idx.p;
    hf.dst_peer = hp.dst_peer.p;
    hf.dst_row = hp.dst_row.p;
    for (int p = 0; p < cm.world; ++p) hf.xd.d[p] = cm.sym_delta(X.ptr, p);
    hf.counter = cm.sym.counter.p;
    hf.epoch = ++cm.sym.halo_epoch;
    hf.remote_flag = flag_addrs(cm, kFlHalo);
    hf.send_mask = hp.send_mask;
    hf.recv_mask = hp.recv_mask;
    hf.my_flags = reinterpret_cast<const uint64_t*>(cm.sym.ctrl.base + kFlHalo);
    hf.err = cm.sym.err.p;
}

bool halo_fuse_prepare(Comm& cm, const View& X, int m, HaloFuse& hf, cudaStream_t s) {
    if (!cm.sym.on || !cm.halo.on) return false;
    if (cm.sym_delta(X.ptr, cm.rank) == INT64_MIN) return false;
    if (cm.sym.last_halo_src == X.ptr) cm.barrier_p2p(s);
    cm.sym.last_halo_src = X.ptr;
    fill_fuse(cm, X, hf);
    cm.bytes_moved += cm.halo.total_send * m * 8;
    return true;
}

using WriteValue64Fn = int (*)(cudaStream_t, unsigned long long, unsigned long long, unsigned int);

bool halo_ce_start(Comm& cm, const View& X, int m, HaloFuse& hf, cudaStream_t s,
                   const std::vector<HaloPlan::CeSeg>* segs) {
    static const bool off = [] {
        const char* e = std::getenv("SPB_HALO_CE");
        return e && e[0] == '0';
    }();
    if (!segs && off) return false;
    if (!cm.sym.on || !cm.halo.on || (!segs && !cm.halo.ce_ok) || X.rs != 1) return false;
    if (cm.sym_delta(X.ptr, cm.rank) == INT64_MIN) return false;
    if (!cm.sym.side) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) {
            cudaGetLastError();
            return false;
        }
        cm.sym.write_value64 = fn;
        SPB_CUDA(cudaStreamCreateWithFlags(&cm.sym.side, cudaStreamNonBlocking));
        SPB_CUDA(cudaEventCreateWithFlags(&cm.sym.ev_ready, cudaEventDisableTiming));
        SPB_CUDA(cudaEventCreateWithFlags(&cm.sym.ev_done, cudaEventDisableTiming));
    }
    if (cm.sym.last_halo_src == X.ptr) cm.barrier_p2p(s);
    cm.sym.last_halo_src = X.ptr;
    HaloPlan& hp = cm.halo;
    fill_fuse(cm, X, hf);
    hf.nopush = 1;
    hf.total = 0;
    SPB_CUDA(cudaEventRecord(cm.sym.ev_ready, s));
    SPB_CUDA(cudaStreamWaitEvent(cm.sym.side, cm.sym.ev_ready, 0));
    int64_t sent = 0;
    for (const auto& sg : segs ? *segs : hp.ce) {
        sent += sg.rows;
        // one column: any pitch >= the width (cudaMemcpy2D requires width <= pitch)
        const size_t pitch = sizeof(double) * static_cast<size_t>(m > 1 ? X.cs : sg.rows);
        const double* src = X.ptr + sg.src_row;
        char* dst = reinterpret_cast<char*>(X.ptr + sg.dst_row) + hf.xd.d[sg.peer];
        SPB_CUDA(cudaMemcpy2DAsync(dst, pitch, src, pitch, sizeof(double) * sg.rows, m, cudaMemcpyDeviceToDevice,
                                   cm.sym.side));
    }
    auto wv = reinterpret_cast<WriteValue64Fn>(cm.sym.write_value64);
    for (int p = 0; p < cm.world; ++p)
        if ((hp.send_mask >> p) & 1u) {
            const int r = wv(cm.sym.side, reinterpret_cast<unsigned long long>(hf.remote_flag.p[p]), hf.epoch, 0);
            if (r != 0) throw SpError(8, "cuStreamWriteValue64 failed: " + std::to_string(r));
        }
    SPB_CUDA(cudaEventRecord(cm.sym.ev_done, cm.sym.side));
    cm.bytes_moved += sent * m * 8;
    return true;
}

void halo_ce_finish(Comm& cm, cudaStream_t s) { SPB_CUDA(cudaStreamWaitEvent(s, cm.sym.ev_done, 0)); }

void halo_wait_flags(const HaloFuse& hf, cudaStream_t s) {
    halo_wait_kernel<<<1, 32, 0, s>>>(hf);
    SPB_LAUNCH_CHECK();
}

// P2P halo push (called by Comm::halo_exchange when X lives in the heap)
bool halo_push(Comm& cm, const View& X, int m, cudaStream_t s) {
    if (!cm.sym.on) return false;
    if (cm.sym_delta(X.ptr, cm.rank) == INT64_MIN) return false;
    HaloPlan& hp = cm.halo;
    if (cm.sym.last_halo_src == X.ptr) cm.barrier_p2p(s);  // same block twice in a row
    cm.sym.last_halo_src = X.ptr;
    HaloFuse hf;
    fill_fuse(cm, X, hf);
    const int64_t elems = hp.total_send * m;
    const int grid = elems > 0 ? static_cast<int>(std::min<int64_t>(ceil_div(elems, 256), device_sm_count())) : 1;
    halo_push_kernel<<<grid, 256, 0, s>>>(X, m, hf);
    SPB_LAUNCH_CHECK();
    cm.bytes_moved += hp.total_send * m * 8;
    return true;
}

// P2P deterministic small sum (called by Comm::sum_small)
bool sum_p2p(Comm& cm, double* dev, int count, cudaStream_t s) {
    if (!cm.sym.on || count > kSumMax) return false;
    const uint64_t epoch = ++cm.sym.sum_epoch;
    const size_t par = static_cast<size_t>(epoch & 1) * kMaxPeers * kSumMax * sizeof(double);
    PeerAddr slot{};
    for (int p = 0; p < cm.world; ++p)
        slot.p[p] = cm.sym.ctrl.peer[p] + kSumSlots + par + sizeof(double) * kSumMax * cm.rank;
    const double* mine = reinterpret_cast<const double*>(cm.sym.ctrl.base + kSumSlots + par);
    sum_p2p_kernel<<<1, 1024, 0, s>>>(dev, count, cm.world, cm.rank, slot, mine, flag_addrs(cm, kFlSum),
                                      reinterpret_cast<const uint64_t*>(cm.sym.ctrl.base + kFlSum), epoch,
                                      cm.sym.err.p);
    SPB_LAUNCH_CHECK();
    return true;
}

void sym_release(Comm& cm) {
    auto drop = [&](SymSeg& g) {
        for (int p = 0; p < static_cast<int>(g.peer.size()); ++p)
            if (p != cm.rank && g.peer[p]) cudaIpcCloseMemHandle(g.peer[p]);
        if (g.base) cudaFree(g.base);
        g = SymSeg{};
    };
    if (cm.sym.side) cudaStreamSynchronize(cm.sym.side);
    if (cm.sym.ev_ready) cudaEventDestroy(cm.sym.ev_ready);
    if (cm.sym.ev_done) cudaEventDestroy(cm.sym.ev_done);
    if (cm.sym.side) cudaStreamDestroy(cm.sym.side);
    cm.sym.side = nullptr;
    cm.sym.ev_ready = cm.sym.ev_done = nullptr;
    for (SymSeg& g : cm.sym.segs) drop(g);
    cm.sym.segs.clear();
    drop(cm.sym.ctrl);
    cm.sym.on = false;
}

} // namespace spb
