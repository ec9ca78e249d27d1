// Host copy bandwidth probe for the pageable -> pinned staging ring (hostcopy.cu):
// memcpy vs AVX2 non-temporal stores, 1..N threads, 160 MB source (C3's matrix).
//   gcc -O3 -mavx2 -pthread tools/micro/hostbw.c -o /tmp/hostbw && /tmp/hostbw [threads...]
#include <immintrin.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static char *src, *dst;
static size_t total = (size_t)160 << 20;
static int mode;

typedef struct { size_t a, b; } Job;

static void nt_copy(char* d, const char* s, size_t n) {
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        __m256i x0 = _mm256_loadu_si256((const __m256i*)(s + i));
        __m256i x1 = _mm256_loadu_si256((const __m256i*)(s + i + 32));
        __m256i x2 = _mm256_loadu_si256((const __m256i*)(s + i + 64));
        __m256i x3 = _mm256_loadu_si256((const __m256i*)(s + i + 96));
        _mm256_stream_si256((__m256i*)(d + i), x0);
        _mm256_stream_si256((__m256i*)(d + i + 32), x1);
        _mm256_stream_si256((__m256i*)(d + i + 64), x2);
        _mm256_stream_si256((__m256i*)(d + i + 96), x3);
    }
    if (i < n) memcpy(d + i, s + i, n - i);
    _mm_sfence();
}

static void* work(void* p) {
    Job* j = (Job*)p;
    if (mode == 0)
        memcpy(dst + j->a, src + j->a, j->b - j->a);
    else
        nt_copy(dst + j->a, src + j->a, j->b - j->a);
    return NULL;
}

static double now(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec + 1e-9 * t.tv_nsec;
}

int main(int argc, char** argv) {
    src = aligned_alloc(4096, total);
    dst = aligned_alloc(4096, total);
    memset(src, 1, total);
    memset(dst, 2, total);
    int th[] = {1, 4, 8, 12, 16, 24, 32};
    for (mode = 0; mode < 2; ++mode)
        for (int k = 0; k < 7; ++k) {
            int n = th[k];
            pthread_t t[64];
            Job jb[64];
            double best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                double t0 = now();
                for (int i = 0; i < n; ++i) {
                    size_t per = (total / n + 63) / 64 * 64;
                    jb[i].a = (size_t)i * per < total ? (size_t)i * per : total;
                    jb[i].b = jb[i].a + per < total ? jb[i].a + per : total;
                    pthread_create(&t[i], NULL, work, &jb[i]);
                }
                for (int i = 0; i < n; ++i) pthread_join(t[i], NULL);
                double dt = now() - t0;
                if (dt < best) best = dt;
            }
            printf("%s threads %2d: %.2f ms, %.1f GB/s\n", mode ? "nt   " : "memcpy", n, best * 1e3, total / best / 1e9);
        }
    return 0;
}
