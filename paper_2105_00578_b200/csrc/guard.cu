// guard.cu — guard bands around every device buffer (SPECPART_B200_GUARD=1).
//
// compute-sanitizer is not available on the GPU pool, and an out-of-bounds store into
// a neighbouring stream-ordered pool allocation raises no fault. In guard mode each
// DBuf is allocated with kGuard bytes before and after the caller's range, both bands
// filled with kPattern; release (and sp_debug_guard_check, for every live buffer)
// waits for the device, reads both bands back and counts every changed byte. The
// tests run the library in a guard-mode process over every kernel family and require
// zero violations (tests/test_gpu_guard.py).
#include "common.cuh"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

namespace spb {

namespace {
constexpr size_t kGuard = 64 << 10;
constexpr unsigned char kPattern = 0xA5;

struct Registry {
    std::mutex mu;
    std::unordered_map<void*, size_t> live;  // caller pointer -> caller bytes
    long long violations = 0;
    long long checked = 0;
};
Registry& reg() {
    static Registry* r = new Registry;  // never destroyed: buffers may be released at exit
    return *r;
}

// both bands of one buffer; returns the number of bytes that changed
long long check_bands(void* user, size_t bytes) {
    std::vector<unsigned char> h(2 * kGuard);  // not a static: buffers are also released at exit
    unsigned char* base = static_cast<unsigned char*>(user) - kGuard;
    if (cudaMemcpy(h.data(), base, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
    if (cudaMemcpy(h.data() + kGuard, static_cast<unsigned char*>(user) + bytes, kGuard, cudaMemcpyDeviceToHost) !=
        cudaSuccess)
        return 0;
    long long bad = 0;
    size_t first = SIZE_MAX;
    for (size_t i = 0; i < 2 * kGuard; ++i)
        if (h[i] != kPattern) {
            ++bad;
            if (first == SIZE_MAX) first = i;
        }
    if (bad) {
        const bool before = first < kGuard;
        std::fprintf(stderr, "[specpart_b200 guard] %lld byte(s) overwritten %s a %zu-byte buffer (first at %s%zu)\n",
                     bad, before ? "before" : "after", bytes, before ? "-" : "+",
                     before ? kGuard - first : first - kGuard);
    }
    return bad;
}
} // namespace

bool guard_on() {
    static const bool on = [] {
        const char* e = std::getenv("SPECPART_B200_GUARD");
        return e && e[0] == '1';
    }();
    return on;
}

void* guard_alloc(size_t bytes, cudaStream_t s) {
    unsigned char* base = nullptr;
    SPB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&base), bytes + 2 * kGuard, s));
    SPB_CUDA(cudaMemsetAsync(base, kPattern, kGuard, s));
    SPB_CUDA(cudaMemsetAsync(base + kGuard + bytes, kPattern, kGuard, s));
    void* user = base + kGuard;
    Registry& r = reg();
    std::lock_guard<std::mutex> lk(r.mu);
    r.live[user] = bytes;
    return user;
}

void guard_free(void* p, cudaStream_t s) {
    Registry& r = reg();
    size_t bytes = 0;
    {
        std::lock_guard<std::mutex> lk(r.mu);
        auto it = r.live.find(p);
        if (it == r.live.end()) return;
        bytes = it->second;
        r.live.erase(it);
    }
    // every stream's work on this buffer must have finished before its bands are read
    if (cudaDeviceSynchronize() == cudaSuccess) {
        const long long bad = check_bands(p, bytes);
        std::lock_guard<std::mutex> lk(r.mu);
        r.violations += bad;
        ++r.checked;
    }
    cudaFreeAsync(static_cast<unsigned char*>(p) - kGuard, s);
}

// every live buffer now, plus the released ones so far
long long guard_check_all(long long* checked) {
    Registry& r = reg();
    std::vector<std::pair<void*, size_t>> bufs;
    {
        std::lock_guard<std::mutex> lk(r.mu);
        bufs.assign(r.live.begin(), r.live.end());
    }
    SPB_CUDA(cudaDeviceSynchronize());
    long long bad = 0;
    for (auto& b : bufs) bad += check_bands(b.first, b.second);
    std::lock_guard<std::mutex> lk(r.mu);
    r.violations += bad;
    r.checked += static_cast<long long>(bufs.size());
    if (checked) *checked = r.checked;
    return r.violations;
}

} // namespace spb
