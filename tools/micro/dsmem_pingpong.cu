// One-way latency of a value pushed into a neighbour CTA's shared memory
// (st.shared::cluster) and spotted by the neighbour polling its own smem,
// vs the global-memory ping-pong (pingpong.cu).  Cluster of 2 (and of 8,
// ranks 0 <-> 7).
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ void st_remote(unsigned addr, unsigned long long v) {
    asm volatile("st.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_local(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.cluster.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ unsigned mapa(const void *p, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(rank));
    return r;
}

__global__ void pp(int iters, int other, unsigned long long *out) {
    __shared__ unsigned long long box;
    cg::cluster_group cl = cg::this_cluster();
    unsigned me = cl.block_rank();
    if (threadIdx.x == 0) box = 0;
    cl.sync();
    if (threadIdx.x == 0 && (me == 0 || me == (unsigned)other)) {
        unsigned peer = me == 0 ? other : 0;
        unsigned raddr = mapa(&box, peer);
        long long t0 = clock64();
        for (int i = 1; i <= iters; i++) {
            if (me == 0) {
                st_remote(raddr, 2 * i - 1);
                while (ld_local(&box) != (unsigned long long)(2 * i)) {}
            } else {
                while (ld_local(&box) != (unsigned long long)(2 * i - 1)) {}
                st_remote(raddr, 2 * i);
            }
        }
        if (me == 0) out[0] = (clock64() - t0) / (2 * iters);
    }
    cl.sync();
}

int main() {
    unsigned long long *out;
    cudaMallocManaged(&out, 64);
    for (int cs : {2, 8}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 16);
        cfg.blockDim = dim3(32);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, pp, 20000, cs - 1, out);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        printf("cluster %d, rank 0 <-> %d: %llu cycles one-way\n", cs, cs - 1, out[0]);
    }
    return 0;
}
