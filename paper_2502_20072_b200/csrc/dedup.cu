// dedup.cu -- the streamed last rung's value dedup on the device (generation.py:364-385).
//
// The reference walks the candidates of every operator in order and drops one whose rounded
// value vector was seen before (its blake2b fingerprint is in a set that starts with the pool's
// and grows by every kept candidate).  Here the fingerprints (128 bits, gen.cu) go into a device
// hash table whose entries remember their first owner: candidate x of chunk e inserts
// (e << 32 | x) with atomicMin, so after a chunk every fingerprint is owned by its earliest
// occurrence in stream order -- pool entries (epoch 0) and earlier chunks first, then the
// smallest index of this chunk -- and a candidate is kept iff it owns its fingerprint.  The
// decisions are the ordered walk's, independent of thread timing.
#include "common.cuh"
#include "kernels.h"

namespace l0s {

namespace {

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z ^= z >> 33;
    z *= 0xff51afd7ed558ccdull;
    z ^= z >> 33;
    z *= 0xc4ceb9fe1a85ec53ull;
    z ^= z >> 33;
    return z;
}

// Insert (or find) key (lo, hi) and lower its owner to `own`.  state: 0 empty, 1 being written,
// 2 ready.  Returns the slot.
__device__ __forceinline__ unsigned long long table_put(DedupTable t, unsigned long long lo, unsigned long long hi,
                                                        unsigned long long own) {
    unsigned long long slot = mix64(lo ^ (hi * 0x9e3779b97f4a7c15ull)) & t.mask;
    for (;;) {
        unsigned st = *(volatile unsigned*)&t.state[slot];
        if (st == 0u) {
            if (atomicCAS(&t.state[slot], 0u, 1u) == 0u) {
                t.lo[slot] = lo;
                t.hi[slot] = hi;
                t.owner[slot] = own;
                __threadfence();
                atomicExch(&t.state[slot], 2u);
                atomicAdd(t.used, 1ull);
                return slot;
            }
            continue;  // lost the race for this slot: read it again
        }
        while (st == 1u) {
            __nanosleep(32);
            st = *(volatile unsigned*)&t.state[slot];
        }
        __threadfence();
        if (*(volatile unsigned long long*)&t.lo[slot] == lo && *(volatile unsigned long long*)&t.hi[slot] == hi) {
            atomicMin(&t.owner[slot], own);
            return slot;
        }
        slot = (slot + 1) & t.mask;
    }
}

__device__ __forceinline__ unsigned long long table_find(DedupTable t, unsigned long long lo, unsigned long long hi) {
    unsigned long long slot = mix64(lo ^ (hi * 0x9e3779b97f4a7c15ull)) & t.mask;
    while (!(t.state[slot] == 2u && t.lo[slot] == lo && t.hi[slot] == hi)) {
        if (t.state[slot] == 0u) return ~0ull;  // not in the table
        slot = (slot + 1) & t.mask;
    }
    return slot;
}

__global__ void k_dedup_insert(DedupTable t, const unsigned char* __restrict__ valid,
                               const unsigned long long* __restrict__ hash, int64_t count, unsigned long long epoch) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= count || (valid && !valid[x])) return;
    table_put(t, hash[2 * x], hash[2 * x + 1], (epoch << 32) | (unsigned long long)x);
}

__global__ void k_dedup_mark(DedupTable t, const unsigned char* __restrict__ valid,
                             const unsigned long long* __restrict__ hash, int64_t count, unsigned long long epoch,
                             unsigned char* __restrict__ kept) {
    const int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= count) return;
    unsigned char k = 0;
    if (valid[x]) {
        const unsigned long long slot = table_find(t, hash[2 * x], hash[2 * x + 1]);
        k = slot != ~0ull && t.owner[slot] == ((epoch << 32) | (unsigned long long)x);
    }
    kept[x] = k;
}

// every ready entry of `from` into `to` (growth); owners move unchanged
__global__ void k_dedup_rehash(DedupTable from, DedupTable to) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s > (int64_t)from.mask || from.state[s] != 2u) return;
    table_put(to, from.lo[s], from.hi[s], from.owner[s]);
}

}  // namespace

void launch_dedup_insert(DedupTable t, const unsigned char* valid, const unsigned long long* hash, int64_t count,
                         unsigned long long epoch, cudaStream_t st) {
    if (count > 0) k_dedup_insert<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(t, valid, hash, count, epoch);
}

void launch_dedup_mark(DedupTable t, const unsigned char* valid, const unsigned long long* hash, int64_t count,
                       unsigned long long epoch, unsigned char* kept, cudaStream_t st) {
    if (count > 0) k_dedup_mark<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(t, valid, hash, count, epoch, kept);
}

void launch_dedup_rehash(DedupTable from, DedupTable to, cudaStream_t st) {
    const int64_t n = (int64_t)from.mask + 1;
    k_dedup_rehash<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(from, to);
}

}  // namespace l0s
