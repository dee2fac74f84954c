// common.cuh — shared device/host plumbing for the specpart B200 path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <atomic>
#include <stdexcept>
#include <string>
#include <vector>

namespace spb {

// ---- errors: one C++ exception per reference error type (errors.hpp:10-54) ----
struct SpError : std::runtime_error {
    int code;
    SpError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
struct BreakdownErr : SpError {
    int iteration;
    bool retried;
    BreakdownErr(int it, bool r)
        : SpError(3, "eigensolver breakdown at iteration " + std::to_string(it) +
                         (r ? " (after retry without search directions)" : "")),
          iteration(it), retried(r) {}
};
inline void throw_infeasible(const std::string& m) { throw SpError(4, m); }
inline void throw_degenerate(const std::string& m) { throw SpError(5, m); }
inline void throw_dimension(const std::string& m) { throw SpError(6, m); }
inline void throw_invalid(const std::string& m) { throw SpError(7, m); }

#define SPB_CUDA(call)                                                                       \
    do {                                                                                     \
        cudaError_t _e = (call);                                                             \
        if (_e != cudaSuccess)                                                               \
            throw ::spb::SpError(8, std::string("CUDA: ") + cudaGetErrorString(_e) + " at " + \
                                        __FILE__ + ":" + std::to_string(__LINE__));          \
    } while (0)

// Every kernel launch of the library is followed by SPB_LAUNCH_CHECK, which
// also counts it (reported as gpu_launches).
long long& launch_counter();
#define SPB_LAUNCH_CHECK()                      \
    do {                                        \
        ++::spb::launch_counter();              \
        SPB_CUDA(cudaGetLastError());           \
    } while (0)

// ---- device buffers ----
// Stream-ordered allocation from the device's default memory pool (release
// threshold raised at context creation, so freed blocks stay cached): the many
// per-call scratch buffers cost no cudaMalloc/cudaFree and no implicit device
// synchronization. Allocations and frees are ordered on the stream of the
// entry point running on this thread (set by guarded() in abi.cu).
inline cudaStream_t& alloc_stream() {
    static thread_local cudaStream_t s = nullptr;
    return s;
}
struct AllocStreamScope {
    cudaStream_t prev;
    explicit AllocStreamScope(cudaStream_t s) : prev(alloc_stream()) { alloc_stream() = s; }
    ~AllocStreamScope() { alloc_stream() = prev; }
};

// Guard mode (SPECPART_B200_GUARD=1 in the environment, read once): every DBuf carries
// 64 KiB guard bands before and after it, filled with a byte pattern and checked when
// the buffer is released (and by sp_debug_guard_check), so an out-of-bounds store
// into a neighbouring pool allocation — which raises no fault — is reported. The
// memory-safety check this library uses on the B200 pool (guard.cu).
bool guard_on();
void* guard_alloc(size_t bytes, cudaStream_t s);
void guard_free(void* p, cudaStream_t s);
long long guard_check_all(long long* checked);  // bytes overwritten so far

template <class T> struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    explicit DBuf(size_t count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(size_t count) {
        if (count <= n && p) return;
        release();
        if (count) {
            if (guard_on()) p = static_cast<T*>(guard_alloc(count * sizeof(T), alloc_stream()));
            else SPB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), alloc_stream()));
        }
        n = count;
    }
    void release() {
        if (p && guard_on()) guard_free(p, alloc_stream());
        else if (p) cudaFreeAsync(p, alloc_stream());
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
};

// ---- a strided 2-D view of a tall block: element (r, c) = ptr[r*rs + c*cs] ----
// Row-major blocks (the device default): rs = ld, cs = 1. Column-major (the
// Arnoldi basis, host exchange): rs = 1, cs = ld.
struct View {
    double* ptr = nullptr;
    int64_t rs = 0;
    int64_t cs = 1;
    int cols = 0;
    __host__ __device__ double& at(int64_t r, int c) const { return ptr[r * rs + c * cs]; }
    __host__ __device__ View sub(int c0, int ncols) const {
        View v = *this;
        v.ptr = ptr + c0 * cs;
        v.cols = ncols;
        return v;
    }
};
inline View rowmajor(double* p, int64_t ld, int cols) { return View{p, ld, 1, cols}; }
inline View colmajor(double* p, int64_t ld, int cols) { return View{p, 1, ld, cols}; }

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

// Persistent-style grid sizing: a multiple of the SM count (148 on B200).
int device_sm_count();
inline int grid_for(int64_t work_items, int per_block, int blocks_per_sm = 4) {
    const int64_t need = (work_items + per_block - 1) / per_block;
    const int64_t cap = static_cast<int64_t>(device_sm_count()) * blocks_per_sm;
    return static_cast<int>(need < cap ? (need > 0 ? need : 1) : cap);
}

} // namespace spb
