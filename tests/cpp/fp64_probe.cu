// Diagnostic: FP64 throughput of this GPU — DFMA (CUDA cores) and DMMA.8x8x4 (mma.sync f64),
// independent chains per warp, and a 1-column dot product at full occupancy.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 1e-9;
    for (int i = 0; i < iters; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int CH>
__global__ void dmma_kernel(double* out, int iters) {
    double d0[CH], d1[CH];
    for (int c = 0; c < CH; ++c) d0[c] = d1[c] = 0.0;
    double a = threadIdx.x * 1e-3, b = 1.0;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(d0[c], d1[c], a, b);
    double s = 0;
    for (int c = 0; c < CH; ++c) s += d0[c] + d1[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dot_kernel(const double* x, long n, double* out) {
    double s = 0;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) s += x[i] * x[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float ms;
    const int iters = 4096;
    dfma_kernel<<<sms * 4, 256>>>(out, 16);
    cudaEventRecord(e0); dfma_kernel<<<sms * 4, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * sms * 4 * 256;
    printf("DFMA: %.3f ms, %.2f TFLOP/s\n", ms, flops / ms / 1e9);
    for (int rep = 0; rep < 2; ++rep) {
        dmma_kernel<8><<<sms * 4, 256>>>(out, 16);
        cudaEventRecord(e0); dmma_kernel<8><<<sms * 4, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 256 * 8 * (double)iters * sms * 4 * 8;  // per warp: 8 chains x iters DMMA, 256 FMA each
        printf("DMMA 8 chains: %.3f ms, %.2f TFLOP/s\n", ms, flops / ms / 1e9);
    }
    cudaEventRecord(e0); dmma_kernel<1><<<sms * 4, 256>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DMMA 1 chain: %.3f ms, latency %.1f ns per DMMA\n", ms, ms * 1e6 / iters);
    long n = 1L << 21;
    double* x; cudaMalloc(&x, sizeof(double) * n); cudaMemset(x, 0, sizeof(double) * n);
    dot_kernel<<<sms * 8, 256>>>(x, n, out);
    cudaEventRecord(e0); for (int r = 0; r < 10; ++r) dot_kernel<<<sms * 8, 256>>>(x, n, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("dot 16 MB: %.1f us, %.0f GB/s\n", ms * 100, n * 8.0 / (ms / 10 * 1e-3) / 1e9);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
