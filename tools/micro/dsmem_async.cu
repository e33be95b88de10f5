// One-way latency through distributed shared memory with st.async +
// mbarrier complete_tx (the receiver waits on its own mbarrier with
// try_wait.parity instead of polling the value), next to the relaxed
// st.shared::cluster + polling ping-pong of dsmem_pingpong.cu.
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned smem(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(const void *p, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async(unsigned addr, unsigned long long v, unsigned bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                 ::"r"(addr), "l"(v), "r"(bar) : "memory");
}
__device__ __forceinline__ void arm(unsigned long long *bar) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8;" ::"r"(smem(bar)) : "memory");
}
__device__ __forceinline__ void wait_phase(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra W;\n}" ::"r"(smem(bar)), "r"(parity) : "memory");
}

__global__ void pp(int iters, int other, unsigned long long *out) {
    __shared__ unsigned long long box;
    __shared__ __align__(8) unsigned long long bar;
    cg::cluster_group cl = cg::this_cluster();
    unsigned me = cl.block_rank();
    if (threadIdx.x == 0) {
        box = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl.sync();
    if (threadIdx.x == 0 && (me == 0 || me == (unsigned)other)) {
        unsigned peer = me == 0 ? other : 0;
        unsigned rbox = mapa(&box, peer), rbar = mapa(&bar, peer);
        unsigned phase = 0;
        long long t0 = clock64();
        for (int i = 1; i <= iters; i++) {
            if (me == 0) {
                arm(&bar);                       // expect the reply
                st_async(rbox, 2 * i - 1, rbar);
                wait_phase(&bar, phase);
            } else {
                arm(&bar);
                wait_phase(&bar, phase);
                st_async(rbox, 2 * i, rbar);
            }
            phase ^= 1;
        }
        if (me == 0) out[0] = (clock64() - t0) / (2 * iters);
        if (box == 0) out[1] = 1;                // keep the value live
    }
    cl.sync();
}

int main() {
    unsigned long long *out;
    cudaMallocManaged(&out, 64);
    for (int cs : {2, 8, 16}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs * 8);
        cfg.blockDim = dim3(32);
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cs > 8) cudaFuncSetAttribute(pp, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaError_t e = cudaLaunchKernelEx(&cfg, pp, 20000, cs - 1, out);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        printf("st.async + mbarrier, cluster %d, rank 0 <-> %d: %llu cycles one-way\n", cs, cs - 1, out[0]);
    }
    return 0;
}
