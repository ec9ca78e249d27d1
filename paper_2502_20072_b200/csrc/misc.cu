// misc.cu -- FP64 pipe microbenchmark: the roofline denominator bench.py reports.
//
// MEASURED_PEAKS.json carries HBM and bf16 figures only, so the fp64 peak is
// measured here: 8 independent DFMA chains per thread, enough warps to cover
// the pipe latency on every SM, timed with CUDA events.
#include <cuda.h>

#include "../../include/l0search.h"
#include "common.cuh"
#include "kernels.h"

namespace l0s {
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link).
bool make_tma_2d(TmaDesc* out, const double* G, unsigned long long cols, unsigned long long rows, unsigned bx,
                 unsigned by) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            return false;
        fn = (Fn)p;
    }
    static_assert(sizeof(TmaDesc) == sizeof(CUtensorMap), "descriptor size");
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * sizeof(double)};
    const cuuint32_t box[2] = {bx, by};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)G, dims, strides,
                    box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_tma_i8_3d(TmaDesc* out, const void* base, unsigned long long cols, unsigned long long rows,
                    unsigned long long planes, unsigned bx, unsigned by) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                            CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static Fn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            return false;
        fn = (Fn)p;
    }
    const cuuint64_t dims[3] = {cols, rows, planes};
    const cuuint64_t strides[2] = {cols, cols * rows};
    const cuuint32_t box[3] = {bx, by, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(reinterpret_cast<CUtensorMap*>(out), CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}
}  // namespace l0s

namespace l0s {
namespace {
__global__ void __launch_bounds__(256) k_dfma_peak(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = s;
}
}  // namespace

double fp64_peak_tflops(int dev) {
    cudaSetDevice(dev);
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, dev);
    double* out;
    cudaMalloc(&out, 8);
    int blocks = prop.multiProcessorCount * 8;
    const int iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma_peak<<<blocks, 256>>>(out, 64, 0.999999, 1e-7);  // warm-up
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        k_dfma_peak<<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFree(out);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    double flops = 2.0 * 8 * 16 * (double)iters * (double)blocks * 256.0;
    return flops / (best * 1e-3) / 1e12;
}
}  // namespace l0s

extern "C" int l0s_fp64_peak(l0s_ctx* ctx, double* out_tflops) {
    (void)ctx;
    int dev = 0;
    cudaGetDevice(&dev);
    *out_tflops = l0s::fp64_peak_tflops(dev);
    return cudaGetLastError() == cudaSuccess ? L0S_OK : L0S_ECUDA;
}

// Accuracy of rcp_fast_abs (MUFU.RCP64H on the high word) over `count` doubles whose
// mantissas and exponents are spread by a hash; returns max |r*d - 1|.
namespace l0s {
namespace {
__global__ void k_rcp_check(int64_t count, double* out) {
    double worst = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
        h ^= h >> 29;
        h *= 0xBF58476D1CE4E5B9ull;
        h ^= h >> 32;
        // mantissa random, exponent in [-600, 600]
        long long e = (long long)(h % 1200ull) - 600 + 1023;
        unsigned long long bits = ((unsigned long long)e << 52) | (h & 0xFFFFFFFFFFFFFull);
        double d = __longlong_as_double((long long)bits);
        if (i & 1) d = -d;
        double r = rcp_fast_abs(d);
        double err = fabs(fma(r, fabs(d), -1.0));
        worst = fmax(worst, err);
        r = fabs(rcp_sweep(d));
        err = fabs(fma(r, fabs(d), -1.0));
        worst = fmax(worst, err);
    }
    for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(L0S_FULL, worst, o));
    if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)out, (unsigned long long)__double_as_longlong(worst));
}
}  // namespace
}  // namespace l0s

extern "C" int l0s_rcp_check(int64_t count, double* out_max_rel) {
    double* d;
    if (cudaMalloc(&d, 8) != cudaSuccess) return L0S_ECUDA;
    cudaMemset(d, 0, 8);
    l0s::k_rcp_check<<<1184, 256>>>(count, d);
    cudaMemcpy(out_max_rel, d, 8, cudaMemcpyDeviceToHost);
    cudaFree(d);
    return cudaGetLastError() == cudaSuccess ? L0S_OK : L0S_ECUDA;
}
