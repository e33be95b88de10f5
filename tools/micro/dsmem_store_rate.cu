// Throughput of remote shared-memory stores (st.shared::cluster) from one
// warp: N "steps", each storing one 128-byte face row (16 lanes x 8 B, or 8
// lanes x v2, or 1 lane bulk copy), then a cluster-scope fence.  Reports
// cycles per step.
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(const void *p, unsigned r) {
    unsigned o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(sa(p)), "r"(r)); return o;
}

template <int MODE>
__global__ void k(int steps, unsigned long long *out) {
    __shared__ __align__(128) double ring[64 * 16];
    cg::cluster_group cl = cg::this_cluster();
    unsigned me = cl.block_rank();
    for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) ring[i] = 0;
    cl.sync();
    if (me == 0 && threadIdx.x < 32) {
        int lane = threadIdx.x;
        unsigned rbase = mapa(ring, 1);
        long long t0 = clock64();
        for (int s = 0; s < steps; s++) {
            unsigned row = rbase + (unsigned)((s & 63) * 128);
            double v = s + lane;
            if (MODE == 0) {           // 16 lanes x 8 B
                if (lane < 16)
                    asm volatile("st.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(row + lane * 8), "d"(v) : "memory");
            } else if (MODE == 1) {    // 8 lanes x 16 B
                if (lane < 8)
                    asm volatile("st.relaxed.cluster.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(row + lane * 16), "d"(v), "d"(v) : "memory");
            } else if (MODE == 2) {    // 4 lanes x 32 B (two v2 each)
                if (lane < 4) {
                    asm volatile("st.relaxed.cluster.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(row + lane * 32), "d"(v), "d"(v) : "memory");
                    asm volatile("st.relaxed.cluster.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(row + lane * 32 + 16), "d"(v), "d"(v) : "memory");
                }
            } else {                   // 2 lanes x 8 B (the y-face pattern per warp)
                if (lane == 0 || lane == 16)
                    asm volatile("st.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(row + (lane & 15) * 8), "d"(v) : "memory");
            }
        }
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        long long t1 = clock64();
        if (lane == 0) out[0] = (t1 - t0) / steps;
    }
    cl.sync();
}

int main() {
    unsigned long long *out;
    cudaMallocManaged(&out, 64);
    const char *names[] = {"16 lanes x b64", "8 lanes x v2.f64", "4 lanes x 2 v2.f64", "2 lanes x b64"};
    for (int mode = 0; mode < 4; mode++) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2);
        cfg.blockDim = dim3(64);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        cudaError_t e;
        switch (mode) {
            case 0: e = cudaLaunchKernelEx(&cfg, k<0>, 20000, out); break;
            case 1: e = cudaLaunchKernelEx(&cfg, k<1>, 20000, out); break;
            case 2: e = cudaLaunchKernelEx(&cfg, k<2>, 20000, out); break;
            default: e = cudaLaunchKernelEx(&cfg, k<3>, 20000, out); break;
        }
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        printf("%-22s: %llu cycles per step\n", names[mode], out[0]);
    }
    return 0;
}
