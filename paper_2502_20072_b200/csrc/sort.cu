// sort.cu -- device sort of (score/bound, rank) pairs by (value, rank), ascending.
//
// Replaces the reference's per-chunk selection (np.argpartition + sort by (score, rank),
// search.py:186-199 and :303-304) on the device.  The composite key is
//     hi = order-preserving encoding of the double (NaN sorts with +inf),
//     lo = rank with its sign bit flipped (signed order),
// so equal values fall back to the smaller rank exactly like the reference's (score, rank)
// order, and every key is distinct for distinct ranks (the sort needs no stability).
//
//  * n <= 8192: one CTA sorts the whole list in shared memory (bitonic network, 1024 threads).
//  * larger: 8192-element blocks are sorted the same way, then log2(n / 8192) merge rounds
//    (merge path: each thread binary-searches its output diagonal and merges 16 outputs).
// Keys travel as 16-byte (hi, lo) pairs; the last pass decodes them back in place.
#include "common.cuh"
#include "kernels.h"

namespace l0s {

namespace {

constexpr int SB = 8192;   // elements per shared-memory block sort
constexpr int ST = 1024;   // threads of the block sort
constexpr int MPT = 16;    // outputs per thread in a merge round

struct K2 {
    unsigned long long hi, lo;
};

__device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ bool k_less(const K2& a, const K2& b) { return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo); }

__device__ __forceinline__ K2 make_key(double v, int64_t r) {
    K2 k;
    k.hi = ord_enc(v == v ? v : __longlong_as_double(0x7ff0000000000000ll));
    k.lo = (unsigned long long)r ^ 0x8000000000000000ull;
    return k;
}

// Bitonic sort of the block's slice in shared memory (padded to a power of two with the
// largest key).  Source: (v, r) arrays (src_kv == nullptr) or encoded keys; destination:
// decoded (v, r) arrays (dst_kv == nullptr) or encoded keys.
// (in place when out_v == v: every element is read before the first barrier, written after the last)
__global__ void __launch_bounds__(ST) k_block_sort(const double* v, const int64_t* r, const K2* __restrict__ src_kv,
                                                   int64_t n, K2* __restrict__ dst_kv, double* out_v, int64_t* out_r) {
    extern __shared__ K2 sk[];
    const int64_t base = (int64_t)blockIdx.x * SB;
    const int cnt = (int)(n - base < SB ? n - base : SB);
    int np = 1;
    while (np < cnt) np <<= 1;
    for (int x = threadIdx.x; x < np; x += ST) {
        K2 k{~0ull, ~0ull};
        if (x < cnt) k = src_kv ? src_kv[base + x] : make_key(v[base + x], r[base + x]);
        sk[x] = k;
    }
    __syncthreads();
    for (int k = 2; k <= np; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int x = threadIdx.x; x < np; x += ST) {
                const int y = x ^ j;
                if (y > x) {
                    const K2 a = sk[x], b = sk[y];
                    const bool up = (x & k) == 0;
                    if (k_less(b, a) == up) {
                        sk[x] = b;
                        sk[y] = a;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int x = threadIdx.x; x < cnt; x += ST) {
        const K2 k = sk[x];
        if (dst_kv) {
            dst_kv[base + x] = k;
        } else {
            out_v[base + x] = ord_dec(k.hi);
            out_r[base + x] = (int64_t)(k.lo ^ 0x8000000000000000ull);
        }
    }
}

// One merge round: runs of `w` sorted keys are merged pairwise into runs of 2w.
__global__ void __launch_bounds__(256) k_merge(const K2* __restrict__ in, int64_t n, int64_t w, K2* __restrict__ out,
                                               double* __restrict__ out_v, int64_t* __restrict__ out_r) {
    const int64_t o0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * MPT;
    if (o0 >= n) return;
    const int64_t pair = o0 / (2 * w);
    const int64_t lo = pair * 2 * w;
    const int64_t la = imin(w, n - lo);                   // left run length
    const int64_t lb = imax(0, imin(w, n - lo - w));      // right run length
    const K2* A = in + lo;
    const K2* B = A + la;
    const int64_t d = o0 - lo;  // output diagonal inside the pair
    // merge path: the number i of left elements among the first d outputs
    int64_t ilo = imax(0, d - lb), ihi = imin(d, la);
    while (ilo < ihi) {
        const int64_t i = (ilo + ihi) >> 1;
        // take A[i] before B[d - 1 - i]?  (keys are distinct)
        if (k_less(A[i], B[d - 1 - i]))
            ilo = i + 1;
        else
            ihi = i;
    }
    int64_t i = ilo, j = d - ilo;
    const int64_t end = imin(MPT, imin(n, lo + 2 * w) - o0);
    for (int64_t e = 0; e < end; ++e) {
        K2 k;
        if (j >= lb || (i < la && k_less(A[i], B[j])))
            k = A[i++];
        else
            k = B[j++];
        if (out) {
            out[o0 + e] = k;
        } else {
            out_v[o0 + e] = ord_dec(k.hi);
            out_r[o0 + e] = (int64_t)(k.lo ^ 0x8000000000000000ull);
        }
    }
}

}  // namespace

size_t sort_pairs_temp_bytes(int64_t n) { return (size_t)(n > SB ? 2 * n : 0) * sizeof(K2) + 256; }

// Sorts (v, rank) ascending by (v, rank) in place; NaN values come back as +inf.
// temp: sort_pairs_temp_bytes(n) bytes.  v_tmp / rank_tmp are unused (kept for the callers'
// buffer bookkeeping).  Launches: 1 for n <= 8192, else 1 + ceil(log2(n / 8192)).
int sort_pairs(double* v, int64_t* rank, double* v_tmp, int64_t* rank_tmp, int64_t n, void* temp, size_t temp_bytes,
               cudaStream_t st) {
    (void)v_tmp;
    (void)rank_tmp;
    if (n <= 1) return 0;
    const size_t smem = sizeof(K2) * SB;
    cudaFuncSetAttribute(k_block_sort, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);  // per device
    if (n <= SB) {
        k_block_sort<<<1, ST, smem, st>>>(v, rank, nullptr, n, nullptr, v, rank);
        return 1;
    }
    if (temp_bytes < sort_pairs_temp_bytes(n)) return -1;
    K2* a = reinterpret_cast<K2*>(temp);
    K2* b = a + n;
    const unsigned nb = (unsigned)((n + SB - 1) / SB);
    k_block_sort<<<nb, ST, smem, st>>>(v, rank, nullptr, n, a, nullptr, nullptr);
    int launches = 1;
    for (int64_t w = SB; w < n; w *= 2) {
        const bool last = 2 * w >= n;
        const int64_t threads = (n + MPT - 1) / MPT;
        k_merge<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(a, n, w, last ? nullptr : b, v, rank);
        ++launches;
        K2* t = a;
        a = b;
        b = t;
    }
    return launches;
}

}  // namespace l0s
