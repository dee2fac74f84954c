// Diagnostic: one 4-D tensor-map TMA box load (the spmm_mesh.cu pattern) checked on the host.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include "bulk.cuh"
using namespace spb;

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 :: "r"(smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar)) : "memory");
}

__global__ void probe(const __grid_constant__ CUtensorMap map, int bx, int by, int x0, int y0, int z, int c, double* out, int manual) {
    extern __shared__ __align__(128) double sm[];
    __shared__ uint64_t bar;
    double* dst = sm;
    if (manual) dst = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(sm) + 127) & ~uintptr_t(127));
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        out[bx * by] = static_cast<double>(smem_u32(sm) % 128);
        mbar_expect_tx(&bar, bx * by * 8);
        tma_load_4d(dst, &map, x0, y0, z, c, &bar);
    }
    mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < bx * by; i += blockDim.x) out[i] = dst[i];
}

using EncFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
    const int arg_box = argc > 1 ? atoi(argv[1]) : 34, arg_manual = argc > 2 ? atoi(argv[2]) : 0, arg_x0 = argc > 3 ? atoi(argv[3]) : -1;
    const int nx = 40, ny = 12, nz = 10, m = 2;
    const int64_t n = int64_t(nx) * ny * nz, ld = ((n + 1 + 63) / 64) * 64;
    std::vector<double> h(ld * m);
    for (int64_t i = 0; i < ld * m; ++i) h[i] = double(i);
    double *X, *out;
    cudaMalloc(&X, ld * m * 8);
    cudaMalloc(&out, 34 * 34 * 8 + 8);
    cudaMemcpy(X, h.data(), ld * m * 8, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q{};
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<EncFn>(fp);
    int fails = 0;
    for (int bxy : {arg_box}) {
        for (int manual : {arg_manual}) {
            CUtensorMap map;
            const cuuint64_t dims[4] = {nx, ny, nz, m};
            const cuuint64_t strides[3] = {nx * 8ull, uint64_t(nx) * ny * 8ull, uint64_t(ld) * 8ull};
            const cuuint32_t box[4] = {cuuint32_t(bxy), cuuint32_t(bxy), 1, 1}, es[4] = {1, 1, 1, 1};
            CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, X, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            const int x0 = arg_x0, y0 = arg_x0, z = 3, c = 1;
            cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
            probe<<<1, 128, 34 * 34 * 8 + 256>>>(map, bxy, bxy, x0, y0, z, c, out, manual);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<double> o(bxy * bxy + 1);
            if (e == cudaSuccess) cudaMemcpy(o.data(), out, (bxy * bxy + 1) * 8, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int yy = 0; yy < bxy && e == cudaSuccess; ++yy)
                for (int xx = 0; xx < bxy; ++xx) {
                    const int gx = x0 + xx, gy = y0 + yy;
                    const double want = (gx < 0 || gx >= nx || gy < 0 || gy >= ny) ? 0.0 : h[c * ld + (int64_t(z) * ny + gy) * nx + gx];
                    bad += o[yy * bxy + xx] != want;
                }
            std::printf("box %d manual %d: encode %d, kernel %s, smem base %% 128 = %g, mismatches %d\n", bxy, manual, int(r),
                        cudaGetErrorString(e), e == cudaSuccess ? o[bxy * bxy] : -1.0, bad);
            fails += (e != cudaSuccess) || bad;
            if (e != cudaSuccess) return 1;
        }
    }
    return fails ? 1 : 0;
}
