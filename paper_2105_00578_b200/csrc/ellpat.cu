// ellpat.cu — pattern compression of the fixed-slot ELL (structured meshes).
//
// On a mesh almost every row has the same slot vector of column offsets
// (col - row): interior rows share one, faces / edges / corners a few dozen
// more, and the diagonal of a unit-cost Laplacian is the row's neighbour count.
// Storing one byte per row (the pattern id) plus a <= 256-entry table replaces
// 4·W bytes of column indices and 8 bytes of diagonal per row — the index
// stream of every SpMM shrinks from 24+8 B/row to 1 B/row for a 7-point mesh.
// The slots, their order and the arithmetic are unchanged (bit-identical).
#include "ops.cuh"

#include <algorithm>
#include <vector>

namespace spb {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h *= 0xbf58476d1ce4e5b9ull;
    return h ^ (h >> 31);
}

__global__ void pat_hash_kernel(const DevOp op, int W, uint64_t* hash) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < op.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint64_t h = 0x1234567ull;
        for (int s = 0; s < W; ++s) {
            const int64_t j = op.ell[s * op.ell_ld + i];
            const int64_t d = j == op.ell_zero_row ? static_cast<int64_t>(kEllPad) : j - i;
            h = mix64(h, static_cast<uint64_t>(d));
        }
        hash[i] = h == 0ull ? 1ull : h;
    }
}

// distinct hashes per CTA in a shared-memory open-addressing set, then appended
// to a short global list (deduplicated and sorted on the host: pattern ids are
// deterministic)
constexpr int kSetSize = 1024;
__global__ void pat_collect_kernel(int64_t n, const uint64_t* hash, int* count, uint64_t* list, int* list_row,
                                   int list_cap, int* overflow) {
    __shared__ unsigned long long set[kSetSize];
    __shared__ int setrow[kSetSize];  // a row having that hash (the inserting one)
    for (int e = threadIdx.x; e < kSetSize; e += blockDim.x) set[e] = 0ull;
    __syncthreads();
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        unsigned long long h = hash[i];
        if (h == 0ull) h = 1ull;
        int slot = static_cast<int>(h % kSetSize), probes = 0;
        while (true) {
            const unsigned long long cur = set[slot];
            if (cur == h) break;
            if (cur == 0ull) {
                const unsigned long long old = atomicCAS(&set[slot], 0ull, h);
                if (old == 0ull) setrow[slot] = static_cast<int>(i);
                if (old == 0ull || old == h) break;
            }
            slot = (slot + 1) % kSetSize;
            if (++probes >= kSetSize) {
                atomicExch(overflow, 1);
                break;
            }
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kSetSize; e += blockDim.x)
        if (set[e]) {
            const int pos = atomicAdd(count, 1);
            if (pos < list_cap) {
                list[pos] = set[e];
                list_row[pos] = setrow[e];
            } else {
                atomicExch(overflow, 1);
            }
        }
}

__global__ void pat_assign_kernel(const DevOp op, const uint64_t* hash, const uint64_t* uniq, int npat,
                                  uint8_t* pid) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < op.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t h = hash[i];
        int lo = 0, hi = npat - 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (uniq[mid] < h) lo = mid + 1;
            else hi = mid;
        }
        pid[i] = static_cast<uint8_t>(lo);
    }
}

__global__ void pat_table_kernel(const DevOp op, int W, const int* rep, int npat, int32_t* tab, double* deg) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= npat) return;
    const int64_t i = rep[p];
    int cnt = 0;
    for (int s = 0; s < W; ++s) {
        const int64_t j = op.ell[s * op.ell_ld + i];
        const bool pad = j == op.ell_zero_row;
        tab[p * W + s] = pad ? kEllPad : static_cast<int32_t>(j - i);
        cnt += pad ? 0 : 1;
    }
    deg[p] = static_cast<double>(cnt);
}

// every row must reproduce its own slots and diagonal from its pattern
__global__ void pat_verify_kernel(const DevOp op, int W, const uint8_t* pid, const int32_t* tab, const double* deg,
                                  int* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < op.n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int p = pid[i];
        bool ok = op.diag[i] == deg[p];
        for (int s = 0; s < W && ok; ++s) {
            const int64_t j = op.ell[s * op.ell_ld + i];
            const int32_t d = tab[p * W + s];
            ok = (d == kEllPad) ? (j == op.ell_zero_row) : (j == i + d);
        }
        if (!ok) atomicExch(bad, 1);
    }
}

} // namespace

bool build_ell_patterns(DevOp& op, EllPatStore& st, cudaStream_t s) {
    if (!op.ell || op.mode != OP_LAPLACE_UNIT || op.n <= 0) return false;
    const int W = op.ell_kl + op.ell_ku;
    const int64_t n = op.n;
    DBuf<uint64_t> hash(n), uniq(256);
    DBuf<int> cnt(1), rep(256), bad(1);
    pat_hash_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(op, W, hash.p);
    SPB_LAUNCH_CHECK();
    const int list_cap = 1 << 16;
    DBuf<uint64_t> list(list_cap);
    DBuf<int> list_row(list_cap);
    DBuf<int> overflow(1);
    SPB_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(int), s));
    SPB_CUDA(cudaMemsetAsync(overflow.p, 0, sizeof(int), s));
    pat_collect_kernel<<<grid_for(n, 256, 2), 256, 0, s>>>(n, hash.p, cnt.p, list.p, list_row.p, list_cap, overflow.p);
    SPB_LAUNCH_CHECK();
    int hc[2] = {0, 0};
    SPB_CUDA(cudaMemcpyAsync(&hc[0], cnt.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaMemcpyAsync(&hc[1], overflow.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    if (hc[1] || hc[0] < 1) return false;
    int npat = 0;
    {
        std::vector<uint64_t> u(hc[0]);
        std::vector<int> ur(hc[0]);
        SPB_CUDA(cudaMemcpyAsync(u.data(), list.p, sizeof(uint64_t) * hc[0], cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaMemcpyAsync(ur.data(), list_row.p, sizeof(int) * hc[0], cudaMemcpyDeviceToHost, s));
        SPB_CUDA(cudaStreamSynchronize(s));
        std::vector<std::pair<uint64_t, int>> kv(hc[0]);
        for (int e = 0; e < hc[0]; ++e) kv[e] = {u[e], ur[e]};
        std::sort(kv.begin(), kv.end());  // any row of a pattern represents it (all are verified)
        std::vector<uint64_t> keys;
        std::vector<int> reps;
        for (const auto& e : kv)
            if (keys.empty() || keys.back() != e.first) {
                keys.push_back(e.first);
                reps.push_back(e.second);
            }
        if (keys.size() > 256) return false;
        npat = static_cast<int>(keys.size());
        SPB_CUDA(cudaMemcpyAsync(uniq.p, keys.data(), sizeof(uint64_t) * npat, cudaMemcpyHostToDevice, s));
        SPB_CUDA(cudaMemcpyAsync(rep.p, reps.data(), sizeof(int) * npat, cudaMemcpyHostToDevice, s));
        SPB_CUDA(cudaStreamSynchronize(s));  // host vectors go out of scope
    }
    st.pid.alloc(n);
    st.tab.alloc(static_cast<size_t>(npat) * W);
    st.deg.alloc(npat);
    pat_assign_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(op, hash.p, uniq.p, npat, st.pid.p);
    SPB_LAUNCH_CHECK();
    pat_table_kernel<<<ceil_div(npat, 64), 64, 0, s>>>(op, W, rep.p, npat, st.tab.p, st.deg.p);
    SPB_LAUNCH_CHECK();
    SPB_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), s));
    pat_verify_kernel<<<grid_for(n, 256, 8), 256, 0, s>>>(op, W, st.pid.p, st.tab.p, st.deg.p, bad.p);
    SPB_LAUNCH_CHECK();
    int b = 0;
    SPB_CUDA(cudaMemcpyAsync(&b, bad.p, sizeof(int), cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    if (b) return false;  // hash collision or non-unit diagonal: keep the plain ELL
    op.ell_pat = st.pid.p;
    op.ell_pat_tab = st.tab.p;
    op.ell_pat_deg = st.deg.p;
    op.ell_npat = npat;
    return true;
}

} // namespace spb
