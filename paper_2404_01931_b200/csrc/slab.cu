// slab.cu — z-slab decomposition of the step (north star:
// "slab-decomposed ... ghost-layer pressure/velocity halo exchange and
// particle migration ... the CG dot products are allreduced").
//
// Rank r owns the cell planes [k0, k1).  The flat index is x-fastest with z
// slowest (flipsim/grid.py:47-72), so the rank's cells, the faces of its
// planes, the pressure rows of its cells (rows ascend with the cell index,
// pressure.py:76-166) and its cell-sorted particles are each ONE contiguous
// range of the global arrays.  Every array keeps its full-grid size and the
// global indexing; a rank computes only its own range and the boundary
// planes travel through the host transport (flip_comm callbacks: NCCL on the
// ctx stream in production, gloo in the CPU/one-GPU tests).  Nothing here
// changes an arithmetic order, so the sharded step is bit-identical to one
// GPU (tests/test_dist_gpu.py).
#include <algorithm>
#include <cstring>

#include "ops.cuh"

namespace flip {

// ------------------------------------------------------------ transport --
static int comm_fail(const char *what) {
    set_error(std::string("slab exchange failed: ") + what);
    return FLIP_E_CUDA;
}

int slab_neighbors(Ctx &c, const void *slo, int64_t nslo, const void *shi, int64_t nshi,
                   void *rlo, int64_t nrlo, void *rhi, int64_t nrhi) {
    Slab &S = c.slab;
    if (S.rank == 0) nslo = nrlo = 0;
    if (S.rank == S.world - 1) nshi = nrhi = 0;
    S.bytes += nslo + nshi;
    S.calls++;
    if (S.comm.neighbors(S.comm.user, (void *)c.st, slo, nslo, shi, nshi, rlo, nrlo, rhi, nrhi))
        return comm_fail("neighbors");
    return 0;
}

int slab_allreduce(Ctx &c, int64_t *buf, int64_t n, int op) {
    Slab &S = c.slab;
    S.bytes += 8 * n;
    S.calls++;
    if (S.comm.allreduce(S.comm.user, (void *)c.st, buf, n, op)) return comm_fail("allreduce");
    return 0;
}

int slab_allgatherv(Ctx &c, void *buf, const int64_t *offsets) {
    Slab &S = c.slab;
    S.bytes += offsets[S.rank + 1] - offsets[S.rank];
    S.calls++;
    if (S.comm.allgatherv(S.comm.user, (void *)c.st, buf, offsets)) return comm_fail("allgatherv");
    return 0;
}

char *slab_xbuf(Ctx &c, size_t bytes) {
    Slab &S = c.slab;
    if (bytes > S.xcap) {
        const size_t cap = std::max<size_t>(bytes, 2 * S.xcap);
        cudaStreamSynchronize(c.st);
        cudaFree(S.xbuf);
        S.xbuf = nullptr;
        S.xcap = 0;
        if (cudaMalloc(&S.xbuf, cap) != cudaSuccess) return nullptr;
        S.xcap = cap;
    }
    return S.xbuf;
}

int slab_free(Ctx &c) {
    Slab &S = c.slab;
    if (S.xbuf) cudaFree(S.xbuf);
    if (S.mig) cudaFree(S.mig);
    if (S.kstart_dev) cudaFree(S.kstart_dev);
    if (S.cnt_dev) cudaFree(S.cnt_dev);
    if (S.dotbuf) cudaFree(S.dotbuf);
    if (S.gscan) cudaFree(S.gscan);
    S.gscan = nullptr;
    S.dotbuf = nullptr;
    S.dotcap = 0;
    S.xbuf = nullptr;
    S.mig = nullptr;
    S.kstart_dev = nullptr;
    S.cnt_dev = nullptr;
    return 0;
}

static int64_t plane_faces(const Dims &d, int comp) {
    return comp == 0 ? (int64_t)(d.nx + 1) * d.ny
                     : comp == 1 ? (int64_t)d.nx * (d.ny + 1) : (int64_t)d.nx * d.ny;
}

void slab_face_range(const Ctx &c, int comp, int64_t *lo, int64_t *hi) {
    const int64_t pf = plane_faces(c.d, comp);
    const int64_t nplanes = comp == 2 ? c.d.nz + 1 : c.d.nz;
    if (!c.slab.on) {
        *lo = 0;
        *hi = pf * nplanes;
        return;
    }
    int64_t k1 = c.slab.k1;
    if (comp == 2 && c.slab.rank == c.slab.world - 1) k1 += 1;  // the top w plane
    *lo = c.slab.k0 * pf;
    *hi = k1 * pf;
}

// --------------------------------------------------------- migration ----
// Particles whose cell left the slab after advect go to the owning rank.
// The new local set is [from rank 0 | ... | stayers | ... | from rank W-1]
// with every source's particles in their original order: a subsequence of
// the 1-GPU particle array in its order, so the stable binning sort that
// follows reproduces the 1-GPU order exactly (binning.py:82-97).
__device__ __forceinline__ int owner_of(const int *kstart, int world, int plane) {
    int q = 0;
    while (q + 1 < world && plane >= kstart[q + 1]) q++;
    return q;
}

__global__ void k_mig_count(ParticlePtrs P, int64_t n, Dims d, const int *kstart, int world,
                            long long *cnt) {
    __shared__ int sc[64];
    for (int i = threadIdx.x; i < world; i += blockDim.x) sc[i] = 0;
    __syncthreads();
    const int64_t pc = (int64_t)d.nx * d.ny;
    for (int64_t t = gtid(); t < n; t += gstride()) {
        const int plane = (int)(cell_of(d, P.a[0][t], P.a[1][t], P.a[2][t]) / pc);
        atomicAdd(&sc[owner_of(kstart, world, plane)], 1);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < world; i += blockDim.x)
        if (sc[i]) atomicAdd((unsigned long long *)&cnt[i], (unsigned long long)sc[i]);
}

__global__ void k_mig_flag(ParticlePtrs P, int64_t n, Dims d, const int *kstart, int world,
                           int rank, int *dest, int *leave) {
    const int64_t pc = (int64_t)d.nx * d.ny;
    for (int64_t t = gtid(); t < n; t += gstride()) {
        const int plane = (int)(cell_of(d, P.a[0][t], P.a[1][t], P.a[2][t]) / pc);
        const int q = owner_of(kstart, world, plane);
        dest[t] = q;
        leave[t] = q != rank;
    }
}

// stayers -> Q[stay_base + stay index]; leavers -> (index, dest) lists
__global__ void k_mig_split(ParticlePtrs P, ParticlePtrs Q, int64_t n, const int *__restrict__ dest,
                            const int *__restrict__ leave, const int *__restrict__ lpos,
                            int64_t stay_base, int *__restrict__ lidx, int *__restrict__ ldest) {
    for (int64_t t = gtid(); t < n; t += gstride()) {
        const int l = lpos[t];
        if (leave[t]) {
            lidx[l] = (int)t;
            ldest[l] = dest[t];
        } else {
            const int64_t o = stay_base + (t - l);
#pragma unroll
            for (int a = 0; a < 6; a++) Q.a[a][o] = P.a[a][t];
        }
    }
}

struct Blocks {  // per-rank particle blocks of an all-to-all buffer
    long long start[64];  // first particle of block q (prefix of the counts)
    long long cnt[64];
};

// send buffer: block q = the leavers for rank q as 6 SoA arrays of cnt[q]
__global__ void k_mig_pack(ParticlePtrs P, int64_t m, const int *__restrict__ perm,
                           const int *__restrict__ lidx, const int *__restrict__ qsorted, Blocks B,
                           double *__restrict__ buf) {
    for (int64_t i = gtid(); i < m; i += gstride()) {
        const int q = qsorted[i];
        const int64_t t = lidx[perm[i]];
        const int64_t w = i - B.start[q];
        double *blk = buf + 6 * B.start[q];
#pragma unroll
        for (int a = 0; a < 6; a++) blk[a * B.cnt[q] + w] = P.a[a][t];
    }
}

// received blocks (sources in rank order, own rank's block empty) ->
// Q[dst_start[q] + i]
__global__ void k_mig_unpack(const double *__restrict__ buf, Blocks B, Blocks D, int world,
                             int64_t m, ParticlePtrs Q) {
    for (int64_t i = gtid(); i < m; i += gstride()) {
        int q = 0;
        while (q + 1 < world && i >= B.start[q + 1]) q++;
        const int64_t w = i - B.start[q];
        const double *blk = buf + 6 * B.start[q];
#pragma unroll
        for (int a = 0; a < 6; a++) Q.a[a][D.start[q] + w] = blk[a * B.cnt[q] + w];
    }
}

int slab_migrate(Ctx &c) {
    Slab &S = c.slab;
    const int W = S.world, r = S.rank;
    cudaStream_t st = c.st;
    // 1. per-destination counts, all-gathered into the W x W matrix
    int64_t *mat = S.cnt_dev;  // [W][W]: row q = rank q's send counts
    FLIP_CUDA_OK(cudaMemsetAsync(mat, 0, sizeof(int64_t) * W * W, st));
    if (c.n > 0) {
        k_mig_count<<<nblocks(c.n), kThreads, 0, st>>>(c.P, c.n, c.d, S.kstart_dev, W,
                                                       (long long *)(mat + (int64_t)r * W));
        c.launches++;
    }
    std::vector<int64_t> off(W + 1);
    for (int q = 0; q <= W; q++) off[q] = (int64_t)q * W * 8;
    if (int rc = slab_allgatherv(c, mat, off.data())) return rc;
    std::vector<int64_t> M((size_t)W * W);
    FLIP_CUDA_OK(cudaMemcpyAsync(M.data(), mat, sizeof(int64_t) * W * W, cudaMemcpyDeviceToHost, st));
    FLIP_CUDA_OK(cudaStreamSynchronize(st));
    const int64_t n_stay = M[(size_t)r * W + r];
    const int64_t n_leave = c.n - n_stay;
    Blocks sendB{}, recvB{}, dstB{};
    int64_t s_acc = 0, r_acc = 0, d_acc = 0;
    std::vector<int64_t> sbytes(W), rbytes(W);
    for (int q = 0; q < W; q++) {
        const int64_t sq = q == r ? 0 : M[(size_t)r * W + q];   // I send to q
        const int64_t rq = q == r ? 0 : M[(size_t)q * W + r];   // q sends to me
        sendB.start[q] = s_acc;
        sendB.cnt[q] = sq;
        recvB.start[q] = r_acc;
        recvB.cnt[q] = rq;
        dstB.start[q] = d_acc;  // final position of source q's block (mine: stayers)
        dstB.cnt[q] = q == r ? n_stay : rq;
        s_acc += sq;
        r_acc += rq;
        d_acc += dstB.cnt[q];
        sbytes[q] = 48 * sq;
        rbytes[q] = 48 * rq;
    }
    const int64_t n_new = d_acc;
    int64_t crossing = 0;  // the same on every rank: all skip the all-to-all or none
    for (int q = 0; q < W; q++)
        for (int p = 0; p < W; p++)
            if (p != q) crossing += M[(size_t)q * W + p];
    if (crossing == 0) return 0;
    if (int rc = reserve_particles(c, std::max(n_new, c.n))) return rc;
    // 2. stable split: stayers into Q at their final place, leavers listed
    if (S.mig_cap < std::max<int64_t>(n_leave, 1) || S.mig_cap < c.n) {
        cudaFree(S.mig);
        S.mig = nullptr;
        S.mig_cap = std::max<int64_t>(c.cap, 1);
        const int64_t hist = radix_hist_ints(S.mig_cap, 64);
        FLIP_CUDA_OK(cudaMalloc(&S.mig, sizeof(int) * (7 * S.mig_cap + hist)));
    }
    int *dest = S.mig, *leave = dest + S.mig_cap, *lpos = leave + S.mig_cap,
        *lidx = lpos + S.mig_cap, *ldest = lidx + S.mig_cap, *k1 = ldest + S.mig_cap,
        *v1 = k1 + S.mig_cap, *hist = v1 + S.mig_cap;
    if (c.n > 0) {
        k_mig_flag<<<nblocks(c.n), kThreads, 0, st>>>(c.P, c.n, c.d, S.kstart_dev, W, r, dest, leave);
        exclusive_scan(ArrayIn{leave}, c.n, lpos, &c.sc->total, c.scan_tmp, st);
        k_mig_split<<<nblocks(c.n), kThreads, 0, st>>>(c.P, c.Q, c.n, dest, leave, lpos,
                                                        dstB.start[r], lidx, ldest);
        c.launches += 5;
    }
    // 3. leavers grouped by destination, stably (LSD radix on the rank)
    char *buf = slab_xbuf(c, (size_t)48 * (s_acc + r_acc) + 64);
    if (!buf) return comm_fail("staging buffer allocation");
    double *sendbuf = (double *)buf, *recvbuf = sendbuf + 6 * s_acc;
    if (n_leave > 0) {
        int *ks = nullptr, *perm = nullptr;
        radix_sort_cells(ldest, k1, lpos /* scratch: free after the split */, v1, n_leave, W, hist,
                         c.scan_tmp, &c.sc->total, st, &ks, &perm, &c.launches);
        k_mig_pack<<<nblocks(n_leave), kThreads, 0, st>>>(c.P, n_leave, perm, lidx, ks, sendB,
                                                          sendbuf);
        c.launches++;
    }
    // 4. all-to-all, then the received blocks into Q
    S.bytes += 48 * s_acc;
    S.calls++;
    if (S.comm.alltoallv(S.comm.user, (void *)st, sendbuf, sbytes.data(), recvbuf, rbytes.data()))
        return comm_fail("alltoallv");
    if (r_acc > 0) {
        k_mig_unpack<<<nblocks(r_acc), kThreads, 0, st>>>(recvbuf, recvB, dstB, W, r_acc, c.Q);
        c.launches++;
    }
    std::swap(c.P, c.Q);
    c.n = n_new;
    c.keys_valid = 0;
    return 0;
}

// ------------------------------------------------------------- labels ----
// classify_cells (grid.py:185-190) ran on the rank's planes; the sealed-
// region labelling of the assembly (pressure.py:109-130) is global, so every
// rank receives all planes (1 byte per cell).
int slab_labels(Ctx &c) {
    const int64_t pc = (int64_t)c.d.nx * c.d.ny;
    std::vector<int64_t> off(c.slab.world + 1);
    for (int q = 0; q <= c.slab.world; q++) off[q] = c.slab.kstart[q] * pc;
    c.box_valid = 1;  // SOLID cells are unchanged by the exchange
    return slab_allgatherv(c, c.label, off.data());
}

// ------------------------------------------------------- ghost particles --
// P2G of a face in plane k0 (k1-1) reads the particles of cell plane k0-1
// (k1): the neighbours send their boundary planes.  Ghosts are placed so the
// cell segments stay back to back around the own particles -- plane k0-1 at
// [-g_lo, 0) (front slack of the particle buffers), plane k1 at [n, n+g_hi)
// -- so the CONTIG P2G kernel runs unchanged.
__global__ void k_ghost_offsets(int *__restrict__ count, int *__restrict__ offset, int64_t c0,
                                int64_t pc, int base, const int *__restrict__ scan) {
    for (int64_t i = gtid(); i < pc; i += gstride()) offset[c0 + i] = base + scan[i];
}

__global__ void k_pack_planes(ParticlePtrs P, int64_t s0, int64_t m, double *__restrict__ buf) {
    for (int64_t i = gtid(); i < m; i += gstride())
#pragma unroll
        for (int a = 0; a < 6; a++) buf[a * m + i] = P.a[a][s0 + i];
}

__global__ void k_unpack_planes(ParticlePtrs P, int64_t d0, int64_t m, const double *__restrict__ buf) {
    for (int64_t i = gtid(); i < m; i += gstride())
#pragma unroll
        for (int a = 0; a < 6; a++) P.a[a][d0 + i] = buf[a * m + i];
}

__global__ void k_fill_int(int *a, int64_t n, int v) {
    for (int64_t i = gtid(); i < n; i += gstride()) a[i] = v;
}

int slab_ghosts(Ctx &c) {
    Slab &S = c.slab;
    cudaStream_t st = c.st;
    const int64_t pc = (int64_t)c.d.nx * c.d.ny;
    const bool has_lo = S.rank > 0, has_hi = S.rank < S.world - 1;
    // (1) the boundary planes' per-cell counts (fixed size)
    if (int rc = slab_neighbors(c, c.count + S.k0 * pc, 4 * pc, c.count + (S.k1 - 1) * pc, 4 * pc,
                                c.count + (S.k0 - 1) * pc, 4 * pc, c.count + S.k1 * pc, 4 * pc))
        return rc;
    // (2) sizes: what I send (own offsets) and what I got (received counts);
    // the ghost planes' prefix sums live in a buffer of their own (gscan)
    int *scan_lo = S.gscan, *scan_hi = S.gscan + pc, *tot = S.gscan + 2 * pc;
    FLIP_CUDA_OK(cudaMemsetAsync(tot, 0, 8 * sizeof(int), st));
    if (has_lo) exclusive_scan(ArrayIn{c.count + (S.k0 - 1) * pc}, pc, scan_lo, tot, c.scan_tmp, st);
    if (has_hi) exclusive_scan(ArrayIn{c.count + S.k1 * pc}, pc, scan_hi, tot + 1, c.scan_tmp, st);
    int h[2] = {0, 0}, o[4] = {0, 0, 0, 0};
    FLIP_CUDA_OK(cudaMemcpyAsync(h, tot, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    FLIP_CUDA_OK(cudaMemcpyAsync(&o[0], c.offset + S.k0 * pc, sizeof(int), cudaMemcpyDeviceToHost, st));
    FLIP_CUDA_OK(cudaMemcpyAsync(&o[1], c.offset + (S.k0 + 1) * pc, sizeof(int), cudaMemcpyDeviceToHost, st));
    FLIP_CUDA_OK(cudaMemcpyAsync(&o[2], c.offset + (S.k1 - 1) * pc, sizeof(int), cudaMemcpyDeviceToHost, st));
    FLIP_CUDA_OK(cudaMemcpyAsync(&o[3], c.offset + S.k1 * pc, sizeof(int), cudaMemcpyDeviceToHost, st));
    FLIP_CUDA_OK(cudaStreamSynchronize(st));
    const int64_t g_lo = has_lo ? h[0] : 0, g_hi = has_hi ? h[1] : 0;
    const int64_t s_lo = has_lo ? o[1] - o[0] : 0, s_hi = has_hi ? o[3] - o[2] : 0;
    // (3) room: g_lo entries before index 0, n + g_hi after
    if (g_lo > c.pfront || c.n + g_hi > c.cap) {
        const int64_t front = std::max(c.pfront, g_lo + g_lo / 2 + 1024);
        const int64_t cap = std::max(c.cap, c.n + g_hi + (c.n + g_hi) / 4);
        if (int rc = realloc_particles(c, cap, front)) return rc;
    }
    // (4) payload: 6 SoA arrays per plane, staged
    const int64_t pay = s_lo + s_hi + g_lo + g_hi;
    char *xb = slab_xbuf(c, 48 * pay + 64);
    if (!xb) return comm_fail("staging buffer allocation");
    double *pb = (double *)xb;
    double *send_lo = pb, *send_hi = send_lo + 6 * s_lo, *recv_lo = send_hi + 6 * s_hi,
           *recv_hi = recv_lo + 6 * g_lo;
    if (s_lo) k_pack_planes<<<nblocks(s_lo), kThreads, 0, st>>>(c.P, o[0], s_lo, send_lo);
    if (s_hi) k_pack_planes<<<nblocks(s_hi), kThreads, 0, st>>>(c.P, o[2], s_hi, send_hi);
    if (int rc = slab_neighbors(c, send_lo, 48 * s_lo, send_hi, 48 * s_hi, recv_lo, 48 * g_lo,
                                recv_hi, 48 * g_hi))
        return rc;
    if (g_lo) k_unpack_planes<<<nblocks(g_lo), kThreads, 0, st>>>(c.P, -g_lo, g_lo, recv_lo);
    if (g_hi) k_unpack_planes<<<nblocks(g_hi), kThreads, 0, st>>>(c.P, c.n, g_hi, recv_hi);
    // (5) offsets of the ghost planes around the own segments
    if (has_lo)
        k_ghost_offsets<<<nblocks(pc), kThreads, 0, st>>>(c.count, c.offset, (S.k0 - 1) * pc, pc,
                                                          (int)-g_lo, scan_lo);
    if (has_hi) {
        k_ghost_offsets<<<nblocks(pc), kThreads, 0, st>>>(c.count, c.offset, S.k1 * pc, pc,
                                                          (int)c.n, scan_hi);
        k_fill_int<<<1, 32, 0, st>>>(c.offset + (S.k1 + 1) * pc, 1, (int)(c.n + g_hi));
    }
    c.launches += 7;
    S.g_lo = g_lo;
    S.g_hi = g_hi;
    return 0;
}

// The hash back to the own particles only (reseed and the accessors read it).
void slab_ghosts_clear(Ctx &c) {
    Slab &S = c.slab;
    const int64_t pc = (int64_t)c.d.nx * c.d.ny;
    if (S.rank > 0) {
        cudaMemsetAsync(c.count + (S.k0 - 1) * pc, 0, sizeof(int) * pc, c.st);
        cudaMemsetAsync(c.offset + (S.k0 - 1) * pc, 0, sizeof(int) * pc, c.st);
    }
    if (S.rank < S.world - 1) {
        cudaMemsetAsync(c.count + S.k1 * pc, 0, sizeof(int) * pc, c.st);
        k_fill_int<<<nblocks(pc + 1), kThreads, 0, c.st>>>(c.offset + S.k1 * pc, pc + 1, (int)c.n);
        c.launches++;
    }
    S.g_lo = S.g_hi = 0;
}

// ------------------------------------------------------------ face halos --
// One face plane per side of every selected array: my first own plane goes
// to rank-1 (its plane k1), my last own plane to rank+1 (its plane k0-1).
int slab_face_halo(Ctx &c, int what) {
    Slab &S = c.slab;
    cudaStream_t st = c.st;
    struct Arr {
        void *p;
        int comp;
        int esz;
    };
    std::vector<Arr> arrs;
    double *g[3] = {c.u, c.v, c.w}, *o[3] = {c.uo, c.vo, c.wo};
    uint8_t *k[3] = {c.ku, c.kv, c.kw};
    uint8_t *s0[3] = {c.ku1, c.kv1, c.kw1};
    uint8_t *s1[3] = {c.ku1 + c.nfu, c.kv1 + c.nfv, c.kw1 + c.nfw};
    for (int a = 0; a < 3; a++) {
        if (what & SLAB_H_GRID) arrs.push_back({g[a], a, 8});
        if (what & SLAB_H_OLD) arrs.push_back({o[a], a, 8});
        if (what & SLAB_H_KNOWN) arrs.push_back({k[a], a, 1});
        if (what & SLAB_H_SCRATCH0) arrs.push_back({s0[a], a, 1});
        if (what & SLAB_H_SCRATCH1) arrs.push_back({s1[a], a, 1});
    }
    int64_t total = 0;
    for (const Arr &a : arrs) total += plane_faces(c.d, a.comp) * a.esz;
    const bool has_lo = S.rank > 0, has_hi = S.rank < S.world - 1;
    char *xb = slab_xbuf(c, 4 * total + 64);
    if (!xb) return comm_fail("staging buffer allocation");
    char *send_lo = xb, *send_hi = xb + total, *recv_lo = xb + 2 * total, *recv_hi = xb + 3 * total;
    int64_t at = 0;
    for (const Arr &a : arrs) {
        const int64_t pb = plane_faces(c.d, a.comp) * a.esz;
        char *base = (char *)a.p;
        if (has_lo) cudaMemcpyAsync(send_lo + at, base + S.k0 * pb, pb, cudaMemcpyDeviceToDevice, st);
        if (has_hi) cudaMemcpyAsync(send_hi + at, base + (S.k1 - 1) * pb, pb, cudaMemcpyDeviceToDevice, st);
        at += pb;
    }
    if (int rc = slab_neighbors(c, send_lo, total, send_hi, total, recv_lo, total, recv_hi, total))
        return rc;
    at = 0;
    for (const Arr &a : arrs) {
        const int64_t pb = plane_faces(c.d, a.comp) * a.esz;
        char *base = (char *)a.p;
        if (has_lo) cudaMemcpyAsync(base + (S.k0 - 1) * pb, recv_lo + at, pb, cudaMemcpyDeviceToDevice, st);
        if (has_hi) cudaMemcpyAsync(base + S.k1 * pb, recv_hi + at, pb, cudaMemcpyDeviceToDevice, st);
        at += pb;
    }
    FLIP_CUDA_OK(cudaGetLastError());
    return 0;
}

// -------------------------------------------------------------- row ranges --
__global__ void k_rowscan_at(const int *__restrict__ rowscan, Blocks idx, int m, int64_t nc,
                             const DevScalars *sc, long long *out) {
    for (int i = threadIdx.x; i < m; i += blockDim.x)
        out[i] = idx.start[i] >= nc ? (long long)sc->nrows : (long long)rowscan[idx.start[i]];
}

// rstart[q] = first global row of rank q (rows of cell planes [kstart[q],
// kstart[q+1])), and the row ranges of my boundary and halo planes.
int slab_rows(Ctx &c) {
    Slab &S = c.slab;
    const int W = S.world;
    const int64_t pc = (int64_t)c.d.nx * c.d.ny, nc = c.ncells;
    Blocks idx{};
    int m = 0;
    for (int q = 0; q <= W; q++) idx.start[m++] = S.kstart[q] * pc;
    const int64_t extra[4] = {std::max<int64_t>(S.k0 - 1, 0) * pc, std::min<int64_t>(S.k0 + 1, c.d.nz) * pc,
                              std::max<int64_t>(S.k1 - 1, 0) * pc, std::min<int64_t>(S.k1 + 1, c.d.nz) * pc};
    for (int t = 0; t < 4; t++) idx.start[m++] = extra[t];
    k_rowscan_at<<<1, 128, 0, c.st>>>(c.rowscan, idx, m, nc, c.sc, (long long *)S.cnt_dev);
    c.launches++;
    std::vector<int64_t> v(m);
    FLIP_CUDA_OK(cudaMemcpyAsync(v.data(), S.cnt_dev, sizeof(int64_t) * m, cudaMemcpyDeviceToHost, c.st));
    FLIP_CUDA_OK(cudaStreamSynchronize(c.st));
    S.rstart.assign(v.begin(), v.begin() + W + 1);
    S.R0 = S.rstart[S.rank];
    S.R1 = S.rstart[S.rank + 1];
    S.Rlo = S.rank > 0 ? v[W + 1] : S.R0;
    S.R0f = v[W + 2];
    S.R1l = v[W + 3];
    S.Rhi = S.rank < W - 1 ? v[W + 4] : S.R1;
    return 0;
}

// ------------------------------------------------------------- row halo --
// Rows ascend with the cell index, so the rows of my first (last) plane are
// one contiguous range [R0, R0f) ([R1l, R1)), and so are the halo rows of
// planes k0-1 ([Rlo, R0)) and k1 ([R1, Rhi)).
int slab_row_halo(Ctx &c, double *vec) {
    Slab &S = c.slab;
    return slab_neighbors(c, vec + S.R0, 8 * (S.R0f - S.R0), vec + S.R1l, 8 * (S.R1 - S.R1l),
                          vec + S.Rlo, 8 * (S.R0 - S.Rlo), vec + S.R1, 8 * (S.Rhi - S.R1));
}

}  // namespace flip

using namespace flip;

extern "C" int flip_set_slab_comm(flip_ctx *ctx, int32_t rank, int32_t world,
                                  const int64_t *plane_start, const flip_comm *comm) {
    Ctx &c = *reinterpret_cast<Ctx *>(ctx);
    cudaSetDevice(c.device);
    Slab &S = c.slab;
    if (!comm || world <= 1) {
        S.on = false;
        return 0;
    }
    if (world > 32 || rank < 0 || rank >= world) {
        set_error("slab: 1 <= world <= 32 and 0 <= rank < world");
        return FLIP_E_ARG;
    }
    if (!comm->neighbors || !comm->allreduce || !comm->allgatherv || !comm->alltoallv) {
        set_error("slab: every flip_comm callback is required");
        return FLIP_E_ARG;
    }
    if (plane_start[0] != 0 || plane_start[world] != c.d.nz) {
        set_error("slab: plane_start must run from 0 to nz");
        return FLIP_E_ARG;
    }
    for (int q = 0; q < world; q++)
        if (plane_start[q + 1] - plane_start[q] < 1) {
            set_error("slab: every rank needs at least one cell plane");
            return FLIP_E_ARG;
        }
    S.on = true;
    S.rank = rank;
    S.world = world;
    S.comm = *comm;
    S.kstart.assign(plane_start, plane_start + world + 1);
    S.k0 = plane_start[rank];
    S.k1 = plane_start[rank + 1];
    if (!S.kstart_dev) FLIP_CUDA_OK(cudaMalloc(&S.kstart_dev, sizeof(int) * 65));
    if (!S.cnt_dev) FLIP_CUDA_OK(cudaMalloc(&S.cnt_dev, sizeof(int64_t) * 64 * 64 + 64));
    if (!S.gscan)
        FLIP_CUDA_OK(cudaMalloc(&S.gscan, sizeof(int) * (2 * (int64_t)c.d.nx * c.d.ny + 16)));
    std::vector<int> ks(S.kstart.begin(), S.kstart.end());
    FLIP_CUDA_OK(cudaMemcpy(S.kstart_dev, ks.data(), sizeof(int) * ks.size(), cudaMemcpyHostToDevice));
    const int64_t pc = (int64_t)c.d.nx * c.d.ny;
    c.slab_c0 = S.k0 * pc;  // reseed refills only the own cells
    c.slab_c1 = S.k1 * pc;
    S.bytes = S.calls = 0;
    return 0;
}

extern "C" int flip_slab_bytes(flip_ctx *ctx, int64_t *sent, int64_t *calls) {
    Ctx &c = *reinterpret_cast<Ctx *>(ctx);
    *sent = c.slab.bytes;
    *calls = c.slab.calls;
    c.slab.bytes = c.slab.calls = 0;
    return 0;
}
