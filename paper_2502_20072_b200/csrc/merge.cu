// merge.cu -- global merge of the per-warp candidate lists.
//
// The union of the warp lists contains the K' smallest lower bounds over all
// tuples (each warp keeps its own K' best; the shared threshold theta_g is the
// smallest per-warp K'-th bound).  Entries above theta_g cannot be among the
// global K' and are dropped here; the survivors are sorted by (lb) on the
// device (CUB radix sort on an order-preserving integer key).
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.h"

namespace l0s {

namespace {
__global__ void k_gather_cand(const double* __restrict__ wl_lb, const int64_t* __restrict__ wl_rank,
                              const int* __restrict__ wl_cnt, int slots, int kc,
                              const unsigned long long* __restrict__ theta_g, double* __restrict__ out_lb,
                              int64_t* __restrict__ out_rank, unsigned long long* __restrict__ out_cnt) {
    const double th = ord_dec(*theta_g);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)slots * kc;
         e += (int64_t)gridDim.x * blockDim.x) {
        int slot = (int)(e / kc), x = (int)(e % kc);
        if (x >= wl_cnt[slot]) continue;
        double lb = wl_lb[e];
        if (!(lb <= th)) continue;
        unsigned long long pos = atomicAdd(out_cnt, 1ull);
        out_lb[pos] = lb;
        out_rank[pos] = wl_rank[e];
    }
}

__global__ void k_enc(const double* __restrict__ lb, unsigned long long* __restrict__ key, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        double x = lb[i];
        key[i] = ord_enc(x == x ? x : __longlong_as_double(0x7ff0000000000000ll));  // NaN sorts with +inf
    }
}
__global__ void k_dec(const unsigned long long* __restrict__ key, double* __restrict__ lb, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) lb[i] = ord_dec(key[i]);
}
}  // namespace

void launch_gather_candidates(const double* wl_lb, const int64_t* wl_rank, const int* wl_cnt, int slots, int kc,
                              const unsigned long long* theta_g, double* out_lb, int64_t* out_rank,
                              unsigned long long* out_cnt, cudaStream_t st) {
    int64_t total = (int64_t)slots * kc;
    unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 4096);
    if (blocks == 0) blocks = 1;
    k_gather_cand<<<blocks, 256, 0, st>>>(wl_lb, wl_rank, wl_cnt, slots, kc, theta_g, out_lb, out_rank, out_cnt);
}

size_t sort_pairs_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const unsigned long long*)nullptr,
                                    (unsigned long long*)nullptr, (const int64_t*)nullptr, (int64_t*)nullptr,
                                    (int)n);
    return bytes + 2 * sizeof(unsigned long long) * (size_t)n + 256;
}

// Sorts (lb, rank) ascending by lb; lb_tmp/rank_tmp receive the sorted result and are copied back.
void sort_pairs(double* lb, int64_t* rank, double* lb_tmp, int64_t* rank_tmp, int64_t n, void* temp,
                size_t temp_bytes, cudaStream_t st) {
    if (n <= 1) return;
    unsigned long long* k_in = (unsigned long long*)temp;
    unsigned long long* k_out = k_in + n;
    void* cub_tmp = (void*)(k_out + n);
    size_t cub_bytes = temp_bytes - 2 * sizeof(unsigned long long) * (size_t)n - 256;
    unsigned blocks = (unsigned)((n + 255) / 256);
    k_enc<<<blocks, 256, 0, st>>>(lb, k_in, n);
    cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, k_in, k_out, rank, rank_tmp, (int)n, 0, 64, st);
    k_dec<<<blocks, 256, 0, st>>>(k_out, lb_tmp, n);
    cudaMemcpyAsync(lb, lb_tmp, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(rank, rank_tmp, sizeof(int64_t) * n, cudaMemcpyDeviceToDevice, st);
}

}  // namespace l0s
