// Cross-SM latency microbenchmark: two CTAs ping-pong a counter through
// global memory with st.relaxed.gpu / ld.relaxed.gpu (the wavefront halo
// protocol).  Reports ns per one-way hop.  Also: same with __nanosleep backoff,
// and with the two CTAs far apart (blockIdx 0 and gridDim-1).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ldr(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void str(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    return g;
}

__global__ void pp(unsigned long long *buf, int iters, int a, int b, int sleep,
                   unsigned long long *out, unsigned *smid) {
    int me = blockIdx.x;
    if (threadIdx.x != 0) return;
    unsigned sm;
    asm("mov.u32 %0, %%smid;" : "=r"(sm));
    if (me == a) smid[0] = sm;
    if (me == b) smid[1] = sm;
    if (me != a && me != b) return;
    unsigned long long *ping = buf, *pong = buf + 32;
    unsigned long long t0 = gt();
    for (int i = 1; i <= iters; i++) {
        if (me == a) {
            str(ping, i);
            unsigned ns = 20;
            while (ldr(pong) != (unsigned long long)i)
                if (sleep) { __nanosleep(ns); ns = ns < 320 ? 2 * ns : ns; }
        } else {
            unsigned ns = 20;
            while (ldr(ping) != (unsigned long long)i)
                if (sleep) { __nanosleep(ns); ns = ns < 320 ? 2 * ns : ns; }
            str(pong, i);
        }
    }
    if (me == a) out[0] = gt() - t0;
}

int main() {
    unsigned long long *buf, *out;
    unsigned *smid;
    cudaMalloc(&buf, 4096);
    cudaMallocManaged(&out, 64);
    cudaMallocManaged(&smid, 64);
    const int iters = 20000;
    int nb = 148;
    int pairs[][2] = {{0, 1}, {0, 2}, {0, 74}, {0, 147}, {0, 75}, {0, 10}};
    for (int sleep = 0; sleep < 2; sleep++)
        for (auto &p : pairs) {
            cudaMemset(buf, 0, 4096);
            pp<<<nb, 32>>>(buf, iters, p[0], p[1], sleep, out, smid);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            printf("sleep %d blocks %3d,%3d  sm %3u,%3u : %.1f ns per one-way hop\n", sleep, p[0],
                   p[1], smid[0], smid[1], out[0] / (2.0 * iters));
        }
    return 0;
}
