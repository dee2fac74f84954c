// rng.cu — std::mt19937_64 streams generated on the GPU, bit-identical.
//
// The reference fills its initial LOBPCG block column-major from
// std::mt19937_64(seed) (eigensolver.cpp:20-33) and the GMRES seed vector the
// same way (preconditioners.cpp:82-87): x = 2*((r >> 11) * 2^-53) - 1. On the
// host this is a sequential 5 ns/draw loop (14.7M draws for cfg2, 151M for
// cfg4). Here the output stream is cut into chunks of J = 2^18 draws; CTA k
// jumps the seeded state ahead by k*J with the precomputed polynomials
// z^(J*2^b) mod phi (tools/mt_jump_gen.cpp; each jump = 20k-word sequence in
// shared memory + an XOR correlation), then runs the standard twist/temper
// for its chunk and scatters the doubles to their (row, column) slots.
#include "ops.cuh"

#include "mt_jump_table.inc"

#include <algorithm>
#include <vector>

namespace spb {

namespace {

constexpr int NN = 312, MM = 156, DEG = 19937;
constexpr int SEQ = DEG + NN + 2;      // words kept for one jump
constexpr int kThreads = 320;
constexpr int64_t kChunk = int64_t(1) << SPB_MT_LOG2_CHUNK;
constexpr uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL, UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;

__device__ __forceinline__ uint64_t next_word(uint64_t y0, uint64_t y1, uint64_t y156) {
    const uint64_t x = (y0 & UM) | (y1 & LM);
    return y156 ^ (x >> 1) ^ ((x & 1) ? MATRIX_A : 0);
}

__device__ __forceinline__ uint64_t temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= (z >> 43);
    return z;
}

struct FillArgs {
    uint64_t seed;
    int64_t total;       // n * d draws
    int64_t n;           // rows of the column-major block
    int64_t row0, nloc;  // local row range written
    View out;            // nloc x d
    const int64_t* chunks;
    const int* exp_off;
    const unsigned short* exps;
};

__global__ void __launch_bounds__(kThreads, 1) mt_fill_kernel(const FillArgs a) {
    extern __shared__ uint64_t Y[];           // SEQ words
    unsigned short* E = reinterpret_cast<unsigned short*>(Y + SEQ);  // staged exponent list
    const int tid = threadIdx.x;
    const int64_t k = a.chunks[blockIdx.x];

    if (tid == 0) {
        Y[0] = a.seed;
        for (int i = 1; i < NN; ++i) Y[i] = 6364136223846793005ULL * (Y[i - 1] ^ (Y[i - 1] >> 62)) + i;
    }
    __syncthreads();

    // S_{kJ} = prod_b (z^{J 2^b})^{bit b of k} S_0
    for (int b = 0; b < SPB_MT_NJUMPS; ++b) {
        if (!((k >> b) & 1)) continue;
        for (int base = NN; base < SEQ; base += MM) {
            const int t = base + tid;
            if (tid < MM && t < SEQ) Y[t] = next_word(Y[t - NN], Y[t - NN + 1], Y[t - MM]);
            __syncthreads();
        }
        const int e0 = a.exp_off[b], ne = a.exp_off[b + 1] - e0;
        for (int i = tid; i < ne; i += kThreads) E[i] = a.exps[e0 + i];
        __syncthreads();
        uint64_t acc = 0;
        if (tid < NN)
            for (int i = 0; i < ne; ++i) acc ^= Y[E[i] + tid];
        __syncthreads();
        if (tid < NN) Y[tid] = acc;
        __syncthreads();
    }

    // twist/temper: after each twist W[i] = y_{t+312+i} = draw (kJ + q0 + i). Thread t < 156
    // keeps words t and t + 156 in registers; word t + 1 comes from the next lane (shuffle), or
    // across a warp boundary / the wrap-around through a small double-buffered exchange, so a
    // round costs two barriers instead of four and no shared-memory round trips of the state
    __shared__ uint64_t xlo[2][8], xhi[2][8], xnew0[2];
    uint64_t ylo = 0, yhi = 0;
    if (tid < MM) {
        ylo = Y[tid];
        yhi = Y[tid + MM];
    }
    __syncthreads();
    if (tid >= 160) return;  // warps 0-4 hold the 156 state threads (named barrier 1)
    const bool live = tid < MM;
    const int lane = tid & 31, warp = tid >> 5;
    const int64_t o_begin = k * kChunk;
    const int64_t o_end = min(a.total, o_begin + kChunk);
    // (column, row) of this thread's two draws, advanced by NN draws per round without a division
    int64_t oj1 = (o_begin + tid) / a.n, oi1 = (o_begin + tid) - oj1 * a.n;
    int64_t oj2 = (o_begin + tid + MM) / a.n, oi2 = (o_begin + tid + MM) - oj2 * a.n;
    auto emit = [&](uint64_t y, int64_t o, int64_t oi, int64_t oj) {
        if (o < o_end && oi >= a.row0 && oi < a.row0 + a.nloc) {
            const uint64_t r = temper(y);
            const double u = __dmul_rn(static_cast<double>(r >> 11), 0x1.0p-53);
            a.out.at(oi - a.row0, static_cast<int>(oj)) = __dsub_rn(__dmul_rn(2.0, u), 1.0);
        }
    };
    auto step = [&](int64_t& oi, int64_t& oj) {
        oi += NN;
        while (oi >= a.n) {
            oi -= a.n;
            ++oj;
        }
    };
    const unsigned mask = warp == MM / 32 ? ((1u << (MM % 32)) - 1u) : 0xffffffffu;  // 156 = 4 * 32 + 28
    int par = 0;
    for (int64_t q0 = o_begin; q0 < o_end; q0 += NN, par ^= 1) {
        if (lane == 0) {
            xlo[par][warp] = ylo;
            xhi[par][warp] = yhi;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(160) : "memory");  // warps 0-4
        // old words t + 1 and t + 157
        uint64_t n_lo = 0, n_hi = 0, new_lo = 0;
        if (live) {
            n_lo = __shfl_down_sync(mask, ylo, 1);
            n_hi = __shfl_down_sync(mask, yhi, 1);
            if (lane == 31 && tid + 1 < MM) {
                n_lo = xlo[par][warp + 1];
                n_hi = xhi[par][warp + 1];
            }
            if (tid == MM - 1) n_lo = xhi[par][0];  // word 156 = thread 0's upper word
            new_lo = next_word(ylo, n_lo, yhi);
            if (tid == 0) xnew0[par] = new_lo;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(160) : "memory");
        if (live) {
            if (tid == MM - 1) n_hi = xnew0[par];  // word 312 wraps to the new word 0
            const uint64_t new_hi = next_word(yhi, n_hi, new_lo);
            ylo = new_lo;
            yhi = new_hi;
            emit(ylo, q0 + tid, oi1, oj1);
            emit(yhi, q0 + MM + tid, oi2, oj2);
            step(oi1, oj1);
            step(oi2, oj2);
        }
    }
}

struct Tables {
    DBuf<int> off;
    DBuf<unsigned short> exps;
    int device = -1;
};

Tables& tables() {
    static Tables t;
    int dev = 0;
    SPB_CUDA(cudaGetDevice(&dev));
    if (t.device != dev) {
        const size_t ne = sizeof(kMtJumpExps) / sizeof(kMtJumpExps[0]);
        t.off.alloc(SPB_MT_NJUMPS + 1);
        t.exps.alloc(ne);
        SPB_CUDA(cudaMemcpy(t.off.p, kMtJumpOffset, sizeof(kMtJumpOffset), cudaMemcpyHostToDevice));
        SPB_CUDA(cudaMemcpy(t.exps.p, kMtJumpExps, sizeof(kMtJumpExps), cudaMemcpyHostToDevice));
        t.device = dev;
    }
    return t;
}

} // namespace

// Draws [0, n*d) of std::mt19937_64(seed) mapped to uniform(-1, 1) in the
// reference's column-major order; rows [row0, row0+nloc) of every column are
// written to out (nloc x d).
void mt_uniform_block(uint64_t seed, int64_t n, int d, int64_t row0, int64_t nloc, const View& out,
                      cudaStream_t s) {
    if (nloc <= 0 || d <= 0) return;
    const int64_t total = n * d;
    if ((total - 1) / kChunk >= (int64_t(1) << SPB_MT_NJUMPS))
        throw_dimension("mt_uniform_block: stream longer than the jump table covers");
    std::vector<int64_t> chunks;
    for (int j = 0; j < d; ++j) {
        const int64_t lo = j * n + row0, hi = j * n + row0 + nloc;  // [lo, hi)
        for (int64_t c = lo / kChunk; c * kChunk < hi; ++c)
            if (chunks.empty() || chunks.back() < c) chunks.push_back(c);
    }
    std::sort(chunks.begin(), chunks.end());
    chunks.erase(std::unique(chunks.begin(), chunks.end()), chunks.end());
    Tables& t = tables();
    AllocStreamScope scope(s);  // the chunk list lives and dies on s (which may be a side stream)
    DBuf<int64_t> dch(chunks.size());
    SPB_CUDA(cudaMemcpyAsync(dch.p, chunks.data(), sizeof(int64_t) * chunks.size(), cudaMemcpyHostToDevice, s));
    FillArgs a{seed, total, n, row0, nloc, out, dch.p, t.off.p, t.exps.p};
    int maxe = 0;
    for (int b = 0; b < SPB_MT_NJUMPS; ++b) maxe = std::max(maxe, kMtJumpOffset[b + 1] - kMtJumpOffset[b]);
    const size_t smem = sizeof(uint64_t) * SEQ + sizeof(unsigned short) * (maxe + 8);
    SPB_CUDA(cudaFuncSetAttribute(mt_fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    mt_fill_kernel<<<static_cast<int>(chunks.size()), kThreads, smem, s>>>(a);
    SPB_LAUNCH_CHECK();
}  // dch: stream-ordered free on s

} // namespace spb
