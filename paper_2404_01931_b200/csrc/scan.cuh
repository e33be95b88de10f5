// scan.cuh — deterministic device-wide exclusive prefix sum over int32
// (reduce-then-scan, 3 kernels).  Integer sums are exact, so this equals
// flipsim.binning.exclusive_scan (binning.py:45-79) for any input whose total
// fits int32.  Templated on a functor so callers fuse the producer
// (e.g. "is this cell a pressure row") into the scan read.
#pragma once
#include "common.cuh"

namespace flip {

constexpr int kScanItems = 16;
constexpr int kScanTile = kThreads * kScanItems;  // 4096 elements per block

__device__ __forceinline__ int warp_incl_scan(int v) {
    int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += t;
    }
    return v;
}

// Exclusive block scan of one int per thread; returns the block total in *total.
__device__ __forceinline__ int block_excl_scan(int v, int *smem_warps, int *total) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int incl = warp_incl_scan(v);
    if (lane == 31) smem_warps[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int s = lane < nw ? smem_warps[lane] : 0;
        int si = warp_incl_scan(s);
        if (lane < nw) smem_warps[lane] = si - s;
        if (lane == nw - 1) smem_warps[32] = si;
    }
    __syncthreads();
    int res = smem_warps[wid] + incl - v;
    *total = smem_warps[32];
    __syncthreads();
    return res;
}

template <class In>
__global__ void k_scan_reduce(In in, int64_t n, int *partials) {
    __shared__ int sw[33];
    int64_t base = (int64_t)blockIdx.x * kScanTile;
    int s = 0;
#pragma unroll
    for (int it = 0; it < kScanItems; it++) {
        int64_t i = base + it * kThreads + threadIdx.x;
        if (i < n) s += in(i);
    }
    int tot;
    block_excl_scan(s, sw, &tot);
    if (threadIdx.x == 0) partials[blockIdx.x] = tot;
}

// single block: exclusive scan of the block partials (nb <= 65536), total -> *total
__global__ void k_scan_partials(int *partials, int nb, int *total);

template <class In>
__global__ void k_scan_down(In in, int64_t n, const int *partials, int *out) {
    __shared__ int sw[33];
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    int vals[kScanItems];
    int s = 0;
#pragma unroll
    for (int it = 0; it < kScanItems; it++) {
        int64_t i = base + it;
        vals[it] = i < n ? in(i) : 0;
        s += vals[it];
    }
    int tot;
    int run = block_excl_scan(s, sw, &tot) + partials[blockIdx.x];
#pragma unroll
    for (int it = 0; it < kScanItems; it++) {
        int64_t i = base + it;
        if (i < n) out[i] = run;
        run += vals[it];
    }
}

struct ArrayIn {
    const int *a;
    __device__ int operator()(int64_t i) const { return a[i]; }
};

// out[0..n) = exclusive scan, *total_dev = sum (out may alias nothing of in).
// tmp must hold ceil(n / kScanTile) ints.
template <class In>
void exclusive_scan(In in, int64_t n, int *out, int *total_dev, int *tmp, cudaStream_t st) {
    int nb = (int)((n + kScanTile - 1) / kScanTile);
    if (nb == 0) {
        cudaMemsetAsync(total_dev, 0, sizeof(int), st);
        return;
    }
    k_scan_reduce<<<nb, kThreads, 0, st>>>(in, n, tmp);
    k_scan_partials<<<1, 1024, 0, st>>>(tmp, nb, total_dev);
    k_scan_down<<<nb, kThreads, 0, st>>>(in, n, tmp, out);
}

inline int64_t scan_tmp_ints(int64_t n) { return (n + kScanTile - 1) / kScanTile + 1; }

}  // namespace flip
