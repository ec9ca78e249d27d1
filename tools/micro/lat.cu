// Dependent-chain latency of FP64 ops on this GPU (one thread): cycles per op.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, int n, double x0, double y) {
    double acc = x0, acc2 = x0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, y);
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) acc2 = __dadd_rn(acc2, __dmul_rn(y, acc2));
    long long t2 = clock64();
    double a3 = x0;
    for (int i = 0; i < n; ++i) a3 = fma(a3, y, y);
    long long t3 = clock64();
    out[0] = acc + acc2 + a3;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2;
}
__global__ void kl(const double* s_in, double* out, long long* cyc, int n) {
    __shared__ double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = s_in[i];
    __syncthreads();
    if (threadIdx.x) return;
    double acc = 0;
    long long t0 = clock64();
    for (int r = 0; r < n / 4096; ++r)
        for (int i = 0; i < 4096; i += 8) {
            double px[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) px[u] = s[i + u];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, __dmul_rn(px[u], px[u]));
        }
    long long t1 = clock64();
    out[1] = acc;
    cyc[3] = t1 - t0;
}
int main() {
    double* out; long long* cyc; double* sin_;
    cudaMalloc(&out, 16); cudaMalloc(&cyc, 64); cudaMalloc(&sin_, 4096 * 8); cudaMemset(sin_, 0, 4096 * 8);
    int n = 1 << 20;
    k<<<1, 1>>>(out, cyc, n, 1.0, 1e-9);
    kl<<<1, 128>>>(sin_, out, cyc, n);
    long long h[4]; cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    printf("DADD chain %.2f cyc/op, DMUL+DADD chain %.2f, DFMA chain %.2f, smem seq_dot %.2f cyc/elem\n",
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n);
    return 0;
}
