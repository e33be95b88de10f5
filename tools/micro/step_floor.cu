// Floor of one wavefront step in the k_mic_lane2 / k_mic_cl shape: 256
// compute threads (+ an idle 32-thread warp), each step = barrier, two
// shared-memory neighbour loads, the MIC(0) forward chain
// (((a+pv)+y)+z)*pr then *(sc*pr), one shared store.  Reports cycles/step
// for 1 CTA on the GPU and for 148 / 296 CTAs (one / two per SM).
#include <cstdio>
#include <cuda_runtime.h>

template <int EXTRA>
__global__ void k(int steps, double *out, unsigned long long *cyc) {
    __shared__ double sval[2][18][18];
    const int t = threadIdx.x;
    for (int q = t; q < 2 * 18 * 18; q += blockDim.x) (&sval[0][0][0])[q] = 0.0;
    __syncthreads();
    const int jj = t & 15, kk = (t >> 4) & 15;
    double pv = 0.0, a = 1e-3 * t, pr = 0.5, sc = 0.25;
    long long c0 = clock64();
    for (int s = 0; s < steps; s++) {
        __syncthreads();
        const int cur = s & 1, prv = cur ^ 1;
        if (t < 256) {
            double yv = sval[prv][kk + 1][jj], zv = sval[prv][kk][jj + 1];
            double tt = ((a + pv) + yv) + zv;
            double q = tt * pr;
            double o = (sc * pr) * q;
            if (EXTRA) o = o * 0.999;
            sval[cur][kk + 1][jj + 1] = o;
            pv = o;
        }
    }
    long long c1 = clock64();
    if (t == 0 && blockIdx.x == 0) cyc[0] = (c1 - c0) / steps;
    if (t == 0) out[blockIdx.x] = pv;
}

int main() {
    double *out;
    unsigned long long *cyc;
    cudaMalloc(&out, 8 * 4096);
    cudaMallocManaged(&cyc, 64);
    for (int nb : {1, 148, 296}) {
        k<0><<<nb, 288>>>(20000, out, cyc);
        cudaDeviceSynchronize();
        k<0><<<nb, 288>>>(20000, out, cyc);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        printf("CTAs %3d: %llu cycles per step\n", nb, cyc[0]);
    }
    return 0;
}
