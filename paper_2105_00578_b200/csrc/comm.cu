// comm.cu — NCCL plumbing for the 1-D row partition.
//
// The reference has no communication layer (single-node OpenMP). The
// B200 build shards rows over the GPUs of one box: SpMM inputs are all-gathered
// over NVLink (halo = everything for R-MAT; a superset of the 2 z-slab halos for
// meshes), and every block inner product is an all-gather of per-rank partials
// followed by a rank-order sum, which keeps results bit-identical on every rank
// and run to run at a fixed GPU count.
#include "context.hpp"

#include <chrono>
#include <dlfcn.h>

#include <algorithm>
#include <vector>
#include <cstdio>

namespace spb {

namespace {

__global__ void pack_kernel(int64_t n, View in, double* out, int m) {
    const int64_t total = n * m;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = idx / m;
        const int c = static_cast<int>(idx - r * m);
        out[idx] = in.at(r, c);
    }
}

__global__ void ordered_sum_kernel(const double* parts, int world, int count, double* out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    double s = 0.0;
    for (int r = 0; r < world; ++r) s += parts[static_cast<int64_t>(r) * count + e];
    out[e] = s;
}

__global__ void ordered_sum_i64_kernel(const int64_t* parts, int world, int count, int64_t* out) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= count) return;
    int64_t s = 0;
    for (int r = 0; r < world; ++r) s += parts[static_cast<int64_t>(r) * count + e];
    out[e] = s;
}

} // namespace

const NcclApi& nccl() {
    static NcclApi api;
    static bool loaded = false;
    if (loaded) return api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw SpError(9, std::string("NCCL: cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* name) {
        void* f = dlsym(h, name);
        if (!f) throw SpError(9, std::string("NCCL: missing symbol ") + name);
        return f;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    loaded = true;
    return api;
}

double PhaseProf::now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
void PhaseProf::start(cudaStream_t s) {
    if (!on) return;
    cudaStreamSynchronize(s);
    acc.clear();
    last = now();
}
void PhaseProf::mark(cudaStream_t s, const char* name) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const double t = now();
    for (auto& kv : acc)
        if (kv.first == name) {
            kv.second += t - last;
            last = t;
            return;
        }
    acc.emplace_back(name, t - last);
    last = t;
}
void PhaseProf::dump(const char* title) {
    if (!on) return;
    double tot = 0.0;
    for (auto& kv : acc) tot += kv.second;
    std::fprintf(stderr, "[spb-profile] %s total %.3f ms\n", title, tot * 1e3);
    for (auto& kv : acc) std::fprintf(stderr, "[spb-profile]   %-22s %9.3f ms\n", kv.first.c_str(), kv.second * 1e3);
}

View Comm::gather_rows(const View& local, int m, cudaStream_t s) {
    if (!active()) return local;
    const int64_t nl = nloc();
    stage.alloc(static_cast<size_t>(n_pad) * m);
    full.alloc(static_cast<size_t>(n_pad) * world * m);
    if (nl > 0) {
        pack_kernel<<<grid_for(nl * m, 256, 8), 256, 0, s>>>(nl, local, stage.p, m);
        SPB_LAUNCH_CHECK();
    }
    SPB_NCCL(::spb::nccl().AllGather(stage.p, full.p, static_cast<size_t>(n_pad) * m, ncclDouble, nccl, s));
    bytes_moved += static_cast<int64_t>(n_pad) * m * 8 * (world - 1);
    return rowmajor(full.p, m, m);
}

void Comm::sum_small(double* dev, int count, cudaStream_t s) {
    if (!active() || count <= 0) return;
    if (sum_p2p(*this, dev, count, s)) return;  // NVLink slots (symm.cu), same rank order
    small.alloc(static_cast<size_t>(count) * world);
    SPB_NCCL(::spb::nccl().AllGather(dev, small.p, count, ncclDouble, nccl, s));
    ordered_sum_kernel<<<ceil_div(count, 128), 128, 0, s>>>(small.p, world, count, dev);
    SPB_LAUNCH_CHECK();
}

void Comm::sum_i64(int64_t* dev, int count, cudaStream_t s) {
    if (!active() || count <= 0) return;
    DBuf<int64_t> tmp(static_cast<size_t>(count) * world);
    SPB_NCCL(::spb::nccl().AllGather(dev, tmp.p, count, ncclInt64, nccl, s));
    ordered_sum_i64_kernel<<<ceil_div(count, 128), 128, 0, s>>>(tmp.p, world, count, dev);
    SPB_LAUNCH_CHECK();
    SPB_CUDA(cudaStreamSynchronize(s));
}

double Comm::max_f64(double v, cudaStream_t s) {
    if (!active()) return v;
    DBuf<double> one(1), all(world);
    SPB_CUDA(cudaMemcpyAsync(one.p, &v, sizeof(double), cudaMemcpyHostToDevice, s));
    SPB_NCCL(::spb::nccl().AllGather(one.p, all.p, 1, ncclDouble, nccl, s));
    std::vector<double> h(world);
    SPB_CUDA(cudaMemcpyAsync(h.data(), all.p, sizeof(double) * world, cudaMemcpyDeviceToHost, s));
    SPB_CUDA(cudaStreamSynchronize(s));
    double m = h[0];
    for (double x : h) m = std::max(m, x);
    return m;
}

void Comm::gather_i32(const int32_t* local, int32_t* global, cudaStream_t s) {
    if (!active()) {
        SPB_CUDA(cudaMemcpyAsync(global, local, sizeof(int32_t) * n_global, cudaMemcpyDeviceToDevice, s));
        return;
    }
    // local must hold n_pad entries (the tail beyond nloc() is ignored by readers)
    SPB_NCCL(::spb::nccl().AllGather(local, global, n_pad, ncclInt32, nccl, s));
}

void Comm::gather_f64(const double* local, double* global, cudaStream_t s) {
    if (!active()) {
        SPB_CUDA(cudaMemcpyAsync(global, local, sizeof(double) * n_global, cudaMemcpyDeviceToDevice, s));
        return;
    }
    SPB_NCCL(::spb::nccl().AllGather(local, global, n_pad, ncclDouble, nccl, s));
}

} // namespace spb
