// p2p.cuh — peer-memory (NVLink) signalling primitives shared by the halo push
// kernel (symm.cu) and the SpMM kernel with the fused halo exchange (spmm.cu).
#pragma once

#include <cstdint>

namespace spb {

constexpr int kMaxPeers = 8;

struct PeerAddr {
    char* p[kMaxPeers];
};
struct PeerDelta {
    long long d[kMaxPeers];
};

// Arguments of an SpMM with its halo exchange fused in (spmm_col/ell_kernel): the
// CTAs first write the boundary rows every peer needs into the peers' copies of
// X (byte delta xd[p] from the local address), raise one flag per destination
// (last CTA), and process the row tiles in an order that starts with interior
// tiles (no halo row read); a warp waits for the peers' flags before its first
// halo tile. Physical tiles (rot + k) mod ntiles, k < n_int, are interior.
struct HaloFuse {
    int on = 0;
    int world = 1;
    int64_t rot = 0;
    int64_t n_int = 0;
    // logical order: interior tiles [0, bnd), halo tiles [bnd, bnd + ntiles - n_int),
    // then the remaining interior tiles — the halo tiles run early enough for the
    // peers' rows to have arrived, and the kernel's tail is interior work
    int64_t bnd = 0;
    int64_t total = 0;  // send entries
    int vec2 = 0;       // entries pair up (consecutive even src/dst rows, same peer): 16-byte pushes
    int nopush = 0;     // the rows were sent by the copy engine (symm.cu halo_ce_start): wait only
    const int32_t* src_row = nullptr;
    const int32_t* dst_peer = nullptr;
    const int32_t* dst_row = nullptr;
    PeerDelta xd{};
    int* counter = nullptr;
    unsigned long long epoch = 0;
    PeerAddr remote_flag{};
    uint32_t send_mask = 0, recv_mask = 0;
    const uint64_t* my_flags = nullptr;
    int* err = nullptr;
    // SPB_HALO_PROBE diagnostics: [0] kernel start (min), [1] push fenced (max over
    // CTAs), [2] sum of warp wait ns, [3] waits, [4] kernel end (max)
    unsigned long long* probe = nullptr;
};

#ifdef __CUDACC__
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// spins until *f >= epoch; after 30 s sets *err and gives up (no GPU hang)
__device__ __forceinline__ void wait_flag(const uint64_t* f, uint64_t epoch, int* err) {
    const uint64_t t0 = global_ns();
    while (ld_acquire_sys(f) < epoch) {
        if (global_ns() - t0 > 30ull * 1000000000ull) {
            atomicExch(err, 1);
            return;
        }
    }
}
// The push half of a halo exchange, run by every thread of the grid; the last
// CTA to finish raises the destination flags. Column-major element order so a
// warp's reads and remote writes are contiguous for slab halos.
template <class XAt>
__device__ __forceinline__ void halo_push_part(const HaloFuse& hf, int m, XAt xat) {
    if (hf.vec2) {
        // column-major pairs of rows: one 16-byte load and one 16-byte remote store
        const int64_t pairs = hf.total / 2;
        const int64_t elems = pairs * m;
        for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < elems;
             e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int c = static_cast<int>(e / pairs);
            const int64_t t = 2 * (e - static_cast<int64_t>(c) * pairs);
            const double2 v = *reinterpret_cast<const double2*>(xat(hf.src_row[t], c));
            char* dst = reinterpret_cast<char*>(xat(hf.dst_row[t], c)) + hf.xd.d[hf.dst_peer[t]];
            *reinterpret_cast<double2*>(dst) = v;
        }
    } else {
        const int64_t elems = hf.total * m;
        for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < elems;
             e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int c = static_cast<int>(e / hf.total);
            const int64_t t = e - static_cast<int64_t>(c) * hf.total;
            const double v = *xat(hf.src_row[t], c);
            char* dst = reinterpret_cast<char*>(xat(hf.dst_row[t], c)) + hf.xd.d[hf.dst_peer[t]];
            *reinterpret_cast<double*>(dst) = v;
        }
    }
    // one system-scope fence per CTA, by thread 0 only: the barrier makes the
    // CTA's stores observed by thread 0, whose fence is cumulative over them.
    // The other warps go straight on to their interior rows; the last CTA's
    // thread 0 raises the destination flags.
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        if (hf.probe) atomicMax(&hf.probe[1], global_ns());
        if (atomicAdd(hf.counter, 1) == static_cast<int>(gridDim.x) - 1) {
            __threadfence_system();
            for (int p = 0; p < hf.world; ++p)
                if ((hf.send_mask >> p) & 1u) st_release_sys(reinterpret_cast<uint64_t*>(hf.remote_flag.p[p]), hf.epoch);
            *hf.counter = 0;
        }
    }
}
// wait for every source peer's data (one lane per peer), then the warp proceeds
__device__ __forceinline__ void halo_wait_warp(const HaloFuse& hf) {
    const int lane = threadIdx.x & 31;
    const uint64_t t0 = hf.probe ? global_ns() : 0;
    if (lane < hf.world && ((hf.recv_mask >> lane) & 1u)) wait_flag(hf.my_flags + lane, hf.epoch, hf.err);
    __syncwarp();
    if (hf.probe && lane == 0) {
        const uint64_t t1 = global_ns();
        atomicAdd(&hf.probe[2], t1 - t0);
        atomicAdd(&hf.probe[3], 1ull);
        atomicMin(&hf.probe[5], t0);  // first warp to reach a halo tile
        atomicMax(&hf.probe[6], t1);  // last warp released
    }
}
#endif

} // namespace spb
