// Does a warp with outstanding global loads slow another warp's shared-memory
// loads on the same SM?  Warp 1 keeps 4 loads in flight to L2-resident lines
// (kind: 0 none, 1 ld.relaxed.gpu, 2 ld.global (weak), 3 ld.global.cg,
// 4 ld.volatile); warp 0 times a chain of dependent LDS.
#include <cstdio>
#include <cuda_runtime.h>

template <int KIND>
__device__ __forceinline__ unsigned long long gload(const unsigned long long *p) {
    unsigned long long v = 0;
    if (KIND == 1) asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if (KIND == 2) asm volatile("ld.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if (KIND == 3) asm volatile("ld.global.cg.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if (KIND == 4) asm volatile("ld.volatile.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <int KIND>
__global__ void k(const unsigned long long *g, unsigned long long *out, int iters) {
    __shared__ unsigned idx[1024];
    __shared__ volatile int stop;
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    if (w == 0) {
        unsigned j = lane;
        long long t0 = clock64();
        for (int i = 0; i < iters; i++) j = idx[j];
        long long t1 = clock64();
        if (lane == 0) { out[blockIdx.x * 2] = (t1 - t0) / iters; out[blockIdx.x * 2 + 1] = j; }
        stop = 1;
    } else if (KIND != 0) {
        unsigned long long acc = 0;
        const unsigned long long *p = g + (blockIdx.x * 4096) + lane;
        int r = 0;
        while (!stop) {
            unsigned long long a = gload<KIND>(p + ((r + 0) & 1023) * 16);
            unsigned long long b = gload<KIND>(p + ((r + 1) & 1023) * 16);
            unsigned long long c = gload<KIND>(p + ((r + 2) & 1023) * 16);
            unsigned long long d = gload<KIND>(p + ((r + 3) & 1023) * 16);
            acc += a + b + c + d;
            r += 4;
        }
        if (acc == 12345) out[0] = acc;
    }
}

int main() {
    unsigned long long *g, *out;
    cudaMalloc(&g, 8ull << 24);
    cudaMemset(g, 0, 8ull << 24);
    cudaMallocManaged(&out, 8 * 2 * 148);
    const char *names[] = {"none", "ld.relaxed.gpu", "ld.global", "ld.global.cg", "ld.volatile"};
    for (int kind = 0; kind < 5; kind++) {
        for (int nb : {1, 148}) {
            switch (kind) {
                case 0: k<0><<<nb, 64>>>(g, out, 20000); break;
                case 1: k<1><<<nb, 64>>>(g, out, 20000); break;
                case 2: k<2><<<nb, 64>>>(g, out, 20000); break;
                case 3: k<3><<<nb, 64>>>(g, out, 20000); break;
                case 4: k<4><<<nb, 64>>>(g, out, 20000); break;
            }
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            printf("%-16s blocks %3d: dependent LDS latency %llu cycles\n", names[kind], nb, out[0]);
        }
    }
    return 0;
}
