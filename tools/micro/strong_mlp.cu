// Memory-level parallelism of strong (relaxed.gpu) loads in one warp:
// time for a batch of N independent loads to distinct lines, strong vs weak,
// with and without a strong store issued before each batch (publish + fetch).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ld_s(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_w(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.global.cv.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_tex(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_s(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int N, int KIND, bool STORE>
__global__ void k(unsigned long long *g, unsigned long long *out, int iters) {
    unsigned long long acc = 0;
    unsigned long long *p = g + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (STORE) st_s(g + (1 << 20) + threadIdx.x + (i & 63) * 16, i);
        unsigned long long v[N];
#pragma unroll
        for (int j = 0; j < N; j++) {
            const unsigned long long *q = p + (((i * N + j) * 16 + acc) & ((1 << 18) - 1));
            v[j] = KIND == 0 ? ld_s(q) : KIND == 1 ? ld_w(q) : ld_tex(q);
        }
#pragma unroll
        for (int j = 0; j < N; j++) acc += v[j];
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[1] = acc; }
}

template <int N, int KIND, bool STORE>
void run(unsigned long long *g, unsigned long long *out, const char *name) {
    k<N, KIND, STORE><<<1, 32>>>(g, out, 2000);
    cudaDeviceSynchronize();
    k<N, KIND, STORE><<<1, 32>>>(g, out, 2000);
    cudaDeviceSynchronize();
    printf("%-14s N=%d store=%d : %llu cycles per batch\n", name, N, (int)STORE, out[0]);
}

int main() {
    unsigned long long *g, *out;
    cudaMalloc(&g, 8ull << 22);
    cudaMemset(g, 0, 8ull << 22);
    cudaMallocManaged(&out, 64);
    run<1, 0, false>(g, out, "relaxed.gpu");
    run<4, 0, false>(g, out, "relaxed.gpu");
    run<8, 0, false>(g, out, "relaxed.gpu");
    run<1, 0, true>(g, out, "relaxed.gpu");
    run<4, 0, true>(g, out, "relaxed.gpu");
    run<1, 1, false>(g, out, "ld.cv");
    run<4, 1, false>(g, out, "ld.cv");
    run<1, 2, false>(g, out, "ld.weak");
    run<4, 2, false>(g, out, "ld.weak");
    run<4, 2, true>(g, out, "ld.weak");
    return 0;
}
