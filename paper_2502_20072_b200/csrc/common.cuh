// common.cuh -- device helpers shared by the l0 search kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define L0S_FULL 0xffffffffu

namespace l0s {

constexpr double kEps = 1.1102230246251565e-16;  // 2^-53, unit roundoff of fp64
constexpr double kEps32 = 5.9604644775390625e-08;  // 2^-24, unit roundoff of fp32

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
// Lexicographic unranking (search.unrank_tuple, search.py:66-85) on the device's binomial
// table (C(a, k) at binom[k * (m + 1) + a]).  Position k takes the largest e with
// sum_{e0 <= e' < e} C(m-1-e', rem) <= r; by the hockey-stick identity that sum is
// C(m-e0, rem+1) - C(m-e, rem+1), so e is found by binary search: O(n log m) dependent
// loads instead of a scan over e.  (A saturated table entry falls back to the scan.)
__device__ __forceinline__ void unrank_lex(int64_t rank, int64_t m, int n, const int64_t* __restrict__ binom,
                                          int64_t* out) {
    int64_t r = rank, e0 = 0;
    for (int k = 0; k < n; ++k) {
        const int rem = n - k - 1;
        const int64_t* B = binom + (int64_t)(rem + 1) * (m + 1);
        const int64_t top = B[m - e0];
        int64_t e;
        if (top == INT64_MAX) {
            e = e0;
            for (;;) {
                const int64_t c = binom[(int64_t)rem * (m + 1) + (m - 1 - e)];
                if (r < c) break;
                r -= c;
                ++e;
            }
        } else {
            const int64_t target = top - r;
            int64_t lo = e0, hi = m - 1 - rem;
            while (lo < hi) {
                const int64_t mid = (lo + hi + 1) >> 1;
                if (B[m - mid] >= target)
                    lo = mid;
                else
                    hi = mid - 1;
            }
            e = lo;
            r -= top - B[m - e];
        }
        out[k] = e;
        e0 = e + 1;
    }
}

// 1/|d| from the MUFU.RCP64H unit: one integer LOP (sign clear, low word
// dropped) and one MUFU op, no FP64-pipe instruction.  Relative error is
// bounded by kRcpRel (measured exhaustively over mantissas by
// tests/test_gpu_parity.py::test_rcp_fast_bound); the screen absorbs it by
// shrinking its threshold, so a tuple is never dropped because of it.
constexpr double kRcpRel = 1.0 / 65536.0;  // 2^-16, conservative (measured < 2^-17)
__device__ __forceinline__ double rcp_fast_abs(double d) {
    int hi = __double2hiint(d) & 0x7fffffff;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(__hiloint2double(hi, 0)));
    return r;
}

// The sweep's form of the same: MUFU.RCP64H on d's high word, with d's own low word kept
// as the result's low word (a < 2^-20 relative perturbation, inside kRcpRel), so ptxas
// writes the result in place -- no zeroing move.  The sign is d's: callers take fabs() of
// the result inside their FMA, a free DFMA operand modifier (one MUFU per reciprocal, no
// integer op).
__device__ __forceinline__ double rcp_sweep(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    return __hiloint2double(__double2hiint(r), __double2loint(d));
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

// ---- mbarrier + TMA (cp.async.bulk.tensor) ----
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// generic-proxy accesses to shared memory are ordered before later async-proxy (TMA) writes
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// 2-D tile load, (x = innermost coordinate, y = row), completion counted on `bar`
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(tmap)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
#endif

}  // namespace l0s
