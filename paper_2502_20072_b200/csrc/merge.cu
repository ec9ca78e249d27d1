// merge.cu -- global merge of the per-warp candidate lists.
//
// The union of the warp lists contains the K' smallest lower bounds over all
// tuples (each warp keeps its own K' best; the shared threshold theta_g is the
// smallest per-warp K'-th bound).  Entries above theta_g cannot be among the
// global K' and are dropped here; the survivors are sorted by (lb, rank) on
// the device (sort.cu).
#include <algorithm>

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

}  // namespace

void launch_gather_candidates(const double* wl_lb, const int64_t* wl_rank, const int* wl_cnt, int slots, int kc,
                              const unsigned long long* theta_g, double* out_lb, int64_t* out_rank,
                              unsigned long long* out_cnt, cudaStream_t st) {
    int64_t total = (int64_t)slots * kc;
    unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 4096);
    if (blocks == 0) blocks = 1;
    k_gather_cand<<<blocks, 256, 0, st>>>(wl_lb, wl_rank, wl_cnt, slots, kc, theta_g, out_lb, out_rank, out_cnt);
}

}  // namespace l0s
