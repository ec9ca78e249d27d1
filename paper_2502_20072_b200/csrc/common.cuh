// common.cuh -- device helpers shared by the l0 search kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define L0S_FULL 0xffffffffu

namespace l0s {

constexpr double kEps = 1.1102230246251565e-16;  // 2^-53, unit roundoff of fp64

// Order-preserving map double -> uint64 (NaN excluded) so that a global
// threshold can be lowered with one atomicMin on an integer.
__host__ __device__ inline unsigned long long ord_enc(double x) {
#ifdef __CUDA_ARCH__
    unsigned long long u = (unsigned long long)__double_as_longlong(x);
#else
    unsigned long long u;
    __builtin_memcpy(&u, &x, 8);
#endif
    return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ inline double ord_dec(unsigned long long u) {
    u = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double x;
    __builtin_memcpy(&x, &u, 8);
    return x;
#endif
}

#ifdef __CUDACC__
// 1/|d| from the MUFU.RCP64H unit: one integer LOP (sign clear, low word
// dropped) and one MUFU op, no FP64-pipe instruction.  Relative error is
// bounded by kRcpRel (measured exhaustively over mantissas by
// tests/test_gpu_kernels.py::test_rcp_fast_bound); the screen absorbs it by
// shrinking its threshold, so a tuple is never dropped because of it.
constexpr double kRcpRel = 1.0 / 131072.0;  // 2^-17, conservative
__device__ __forceinline__ double rcp_fast_abs(double d) {
    int hi = __double2hiint(d) & 0x7fffffff;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(__hiloint2double(hi, 0)));
    return r;
}

// Same for d known to be positive: MUFU.RCP64H straight on the high word.
__device__ __forceinline__ double rcp_fast_pos(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    return r;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
#endif

}  // namespace l0s
