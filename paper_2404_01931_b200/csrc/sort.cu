// sort.cu — stable LSD radix sort of (cell key, particle index) pairs, the
// GPU counting sort behind bin_particles (flipsim/binning.py:82-97,
// flipsim/_kernels/_core.pyx:179-193).  A stable sort by cell yields the
// unique permutation the reference's sequential cursor scatter produces, so
// the particle order is byte-identical.  Plus the scan partials kernel and
// the six-array gather of ParticleSet.reorder (particles.py:54-64).
#include <cstdlib>

#include "ops.cuh"

namespace flip {

__global__ void k_scan_partials(int *partials, int nb, int *total) {
    __shared__ int sw[33];
    int per = (nb + blockDim.x - 1) / blockDim.x;
    int b0 = threadIdx.x * per;
    int s = 0;
    for (int i = 0; i < per; i++)
        if (b0 + i < nb) s += partials[b0 + i];
    int tot;
    int run = block_excl_scan(s, sw, &tot);
    for (int i = 0; i < per; i++)
        if (b0 + i < nb) {
            int v = partials[b0 + i];
            partials[b0 + i] = run;
            run += v;
        }
    if (threadIdx.x == 0) *total = tot;
}

constexpr int kSortItems = 16;                       // keys per thread
constexpr int kSortWarps = kThreads / 32;            // 8
constexpr int kSortTile = kThreads * kSortItems;     // 4096 keys per tile
constexpr int kWarpSpan = 32 * kSortItems;           // 512 consecutive keys per warp

// Per-tile digit histogram -> hist[digit * ntiles + tile] (digit-major so one
// exclusive scan gives every (digit, tile) its global output base).
__global__ void k_radix_hist(const int *__restrict__ keys, int64_t n, int shift, int nbits,
                             int ntiles, int *__restrict__ hist) {
    extern __shared__ int sh[];
    int nb = 1 << nbits, mask = nb - 1;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    int64_t base = (int64_t)blockIdx.x * kSortTile;
    for (int it = 0; it < kSortItems; it++) {
        int64_t i = base + it * kThreads + threadIdx.x;
        if (i < n) atomicAdd(&sh[(keys[i] >> shift) & mask], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nb; i += blockDim.x) hist[(int64_t)i * ntiles + blockIdx.x] = sh[i];
}

// Stable scatter of one tile.  Warp w owns keys [w*512, (w+1)*512) of the
// tile and walks them in 16 rounds of 32 in index order; peers with the same
// digit are ranked by lane with __match_any_sync, so each warp's ranks are
// stable; per-(warp, digit) counts are then prefix-summed across warps in
// warp order, which keeps the whole tile stable.
template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
k_radix_scatter(const int *__restrict__ keys_in, const int *__restrict__ vals_in,
                                int64_t n, int shift, int nbits, int ntiles,
                                const int *__restrict__ hist_scanned, int *__restrict__ keys_out,
                                int *__restrict__ vals_out) {
    extern __shared__ int sh[];
    int nb = 1 << nbits, mask = nb - 1;
    int *wcnt = sh;                       // [kSortWarps][nb]
    int *tbase = sh + kSortWarps * nb;    // [nb]
    for (int i = threadIdx.x; i < kSortWarps * nb; i += blockDim.x) wcnt[i] = 0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x)
        tbase[i] = hist_scanned[(int64_t)i * ntiles + blockIdx.x];
    __syncthreads();
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned lt = (1u << lane) - 1u;
    int64_t base = (int64_t)blockIdx.x * kSortTile + (int64_t)w * kWarpSpan;
    int kv[kSortItems], vv[kSortItems], pos[kSortItems];
#pragma unroll
    for (int it = 0; it < kSortItems; it++) {
        int64_t i = base + it * 32 + lane;
        bool valid = i < n;
        int key = valid ? keys_in[i] : 0;
        int val = valid ? (vals_in ? vals_in[i] : (int)i) : 0;
        int digit = valid ? ((key >> shift) & mask) : nb;  // invalid lanes form their own group
        unsigned peers = __match_any_sync(0xffffffffu, digit);
        int before = __popc(peers & lt);
        int leader = 31 - __clz(peers);
        int cnt = 0;
        if (valid) cnt = wcnt[w * nb + digit];
        __syncwarp();
        if (valid && lane == leader) wcnt[w * nb + digit] = cnt + __popc(peers);
        __syncwarp();
        kv[it] = key;
        vv[it] = val;
        pos[it] = valid ? cnt + before : -1;
    }
    __syncthreads();
    for (int d = threadIdx.x; d < nb; d += blockDim.x) {
        int run = 0;
        for (int ww = 0; ww < kSortWarps; ww++) {
            int t = wcnt[ww * nb + d];
            wcnt[ww * nb + d] = run;
            run += t;
        }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kSortItems; it++) {
        if (pos[it] < 0) continue;
        int digit = (kv[it] >> shift) & mask;
        int p = tbase[digit] + wcnt[w * nb + digit] + pos[it];
        keys_out[p] = kv[it];
        vals_out[p] = vv[it];
    }
}

static int bits_for(int64_t ncells) {
    int b = 0;
    while (((int64_t)1 << b) < ncells) b++;
    return b;
}

int64_t radix_hist_ints(int64_t cap, int64_t ncells) {
    int bits = bits_for(ncells);
    int passes = bits == 0 ? 0 : (bits + 8) / 9;
    int nbits = passes ? (bits + passes - 1) / passes : 0;
    int64_t ntiles = (cap + kSortTile - 1) / kSortTile;
    return ((int64_t)1 << nbits) * (ntiles + 1) + 1;
}

// Sorts keys[0..n) (values in [0, ncells)) stably; returns the permutation
// (old index per new slot) in *perm_out and the sorted keys in *keys_sorted.
// Buffers k0/k1/v0/v1 hold n ints each; pointers returned alias two of them.
int radix_sort_cells(int *k0, int *k1, int *v0, int *v1, int64_t n, int64_t ncells, int *hist,
                     int *scan_tmp, int *scan_total, cudaStream_t st, int **keys_sorted,
                     int **perm_out, int64_t *launches) {
    int bits = bits_for(ncells);
    if (n == 0) {
        *keys_sorted = k0;
        *perm_out = v0;
        return 0;
    }
    int passes = bits == 0 ? 0 : (bits + 8) / 9;
    if (passes == 0) {  // single cell: identity permutation
        k_iota<<<(int)((n + kThreads - 1) / kThreads), kThreads, 0, st>>>(v0, n);
        *launches += 1;
        *keys_sorted = k0;
        *perm_out = v0;
        return 0;
    }
    int nbits = (bits + passes - 1) / passes;
    int ntiles = (int)((n + kSortTile - 1) / kSortTile);
    int nb = 1 << nbits;
    size_t sh_hist = sizeof(int) * nb, sh_scat = sizeof(int) * (kSortWarps + 1) * nb;
    int *kin = k0, *kout = k1, *vin = nullptr, *vout = v0;
    for (int p = 0; p < passes; p++) {
        int shift = p * nbits;
        k_radix_hist<<<ntiles, kThreads, sh_hist, st>>>(kin, n, shift, nbits, ntiles, hist);
        exclusive_scan(ArrayIn{hist}, (int64_t)nb * ntiles, hist, scan_total, scan_tmp, st);
        // 4 CTAs/SM (64 registers, 64 B spilled): BIN 1.536 -> 1.463 ms (2: 1.77)
        static const int minb = getenv("FLIPB200_SCATTER_MINB") ? atoi(getenv("FLIPB200_SCATTER_MINB")) : 4;
        auto ks = minb == 4 ? k_radix_scatter<4> : minb == 2 ? k_radix_scatter<2> : k_radix_scatter<3>;
        ks<<<ntiles, kThreads, sh_scat, st>>>(kin, vin, n, shift, nbits, ntiles, hist, kout, vout);
        *launches += 5;
        int *tk = kin;
        kin = kout;
        kout = tk;
        // value buffers ping-pong between v0 and v1 (the first pass reads the
        // implicit identity permutation)
        vin = vout;
        vout = (vout == v0) ? v1 : v0;
    }
    *keys_sorted = kin;
    *perm_out = vin;
    return 0;
}

__global__ void k_iota(int *a, int64_t n) {
    for (int64_t i = gtid(); i < n; i += gstride()) a[i] = (int)i;
}

// k_gather6 that also writes the P2G records rec[comp][i] = {x, y, z, v_comp}
// (three 32-byte stores per particle).
__global__ void k_gather6_rec(ParticlePtrs src, ParticlePtrs dst, const int *__restrict__ perm,
                              int64_t n, double *__restrict__ rec, int64_t ld) {
    for (int64_t i = gtid(); i < n; i += gstride()) {
        const int j = perm[i];
        double v[6];
#pragma unroll
        for (int a = 0; a < 6; a++) {
            v[a] = __ldg(src.a[a] + j);
            dst.a[a][i] = v[a];
        }
#pragma unroll
        for (int c = 0; c < 3; c++) {
            double *r = rec + ((int64_t)c * ld + i) * 4;
            asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(r), "d"(v[0]), "d"(v[1]),
                         "d"(v[2]), "d"(v[3 + c])
                         : "memory");
        }
    }
}

// ParticleSet.reorder: dst[a][i] = src[a][perm[i]] for the six SoA arrays.
__global__ void k_gather6(ParticlePtrs src, ParticlePtrs dst, const int *__restrict__ perm,
                          int64_t n) {
    for (int64_t i = gtid(); i < n; i += gstride()) {
        int j = perm[i];
#pragma unroll
        for (int a = 0; a < 6; a++) dst.a[a][i] = __ldg(src.a[a] + j);
    }
}

}  // namespace flip
