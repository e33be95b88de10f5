// k_mic_cl step-cost detail: which part of "+ops" (operands from a shared
// chunk, row test, 8-byte STG of the output) costs cycles, and does
// loading step s+1's operands during step s hide it?
#include <cstdio>
#include <cuda_runtime.h>

template <int LD, int ST, int PF>
__global__ void __launch_bounds__(288) k(int steps, double *dst, unsigned long long *cyc) {
    constexpr int KC = 4, TP = 256;
    __shared__ double sval[2][18][18];
    __shared__ __align__(16) double opb[2][KC][TP];
    const int t = threadIdx.x;
    for (int q = t; q < 2 * 18 * 18; q += blockDim.x) (&sval[0][0][0])[q] = 0.0;
    for (int q = t; q < 2 * KC * TP; q += blockDim.x) (&opb[0][0][0])[q] = 1.0 + q;
    __syncthreads();
    if (t >= 256) { for (int s = 0; s < steps; s++) __syncthreads(); return; }
    const int jj = t & 15, kk = t >> 4;
    double pv = 0.0, sc = 0.25;
    double *d = dst + (size_t)blockIdx.x * steps * TP + t;
    double na = opb[0][0][t], npr = opb[1][0][t];
    long long c0 = clock64();
    for (int s = 0; s < steps; s++) {
        __syncthreads();
        const int cur = s & 1, prv = cur ^ 1, u = s % KC;
        double a = 1e-3 * t, pr = 0.5;
        if (LD) {
            if (PF) { a = na; pr = npr; const int un = (s + 1) % KC; na = opb[0][un][t]; npr = opb[1][un][t]; }
            else { a = opb[0][u][t]; pr = opb[1][u][t]; }
        }
        double yv = sval[prv][kk + 1][jj], zv = sval[prv][kk][jj + 1];
        double tt = ((a + pv) + yv) + zv;
        double q = tt * pr;
        if (ST && a != 12345.0) d[(size_t)s * TP] = q;
        double o = (sc * pr) * q;
        sval[cur][kk + 1][jj + 1] = o;
        pv = o;
    }
    long long c1 = clock64();
    if (t == 0 && blockIdx.x == 0) cyc[0] = (c1 - c0) / steps;
}

template <int LD, int ST, int PF>
void run(const char *name, double *dst, unsigned long long *cyc, int steps) {
    for (int r = 0; r < 2; r++) { k<LD, ST, PF><<<296, 288>>>(steps, dst, cyc); cudaDeviceSynchronize(); }
    printf("%-26s %llu cycles/step\n", name, cyc[0]);
}

int main() {
    const int steps = 512;
    double *dst; unsigned long long *cyc;
    cudaMalloc(&dst, (size_t)296 * steps * 256 * 8);
    cudaMallocManaged(&cyc, 64);
    run<0, 0, 0>("skeleton (+helper)", dst, cyc, steps);
    run<1, 0, 0>("+LDS operands", dst, cyc, steps);
    run<1, 0, 1>("+LDS operands prefetched", dst, cyc, steps);
    run<0, 1, 0>("+STG output", dst, cyc, steps);
    run<1, 1, 0>("+LDS +STG", dst, cyc, steps);
    run<1, 1, 1>("+LDS prefetched +STG", dst, cyc, steps);
    return 0;
}
