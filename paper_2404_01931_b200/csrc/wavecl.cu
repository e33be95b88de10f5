// wavecl.cu — MIC(0) forward/backward substitution (_core.pyx:311-347) as the
// tiled wavefront of k_mic_lane2, with tile faces exchanged through
// distributed shared memory inside thread-block clusters.
//
// A cluster is a CY x CZ block of 16x16 tiles (one CTA each).  Inside it, a
// face lane of the producing tile stores each step's output straight into
// the consuming CTA's face ring (st.shared::cluster); the consumer's face
// lanes poll their own shared memory.  Rings hold the whole sweep
// (face[step][lane]) and are pre-filled with the pending marker before the
// cluster barrier, so no flow control is needed.  Faces that cross a
// cluster boundary use the global step-major halo of k_mic_lane2 through
// the helper warp.  Cross-SM visibility through DSMEM measured ~195 ns vs
// ~450 ns through L2 (tools/micro/), and the consumer issues no global
// loads for those faces.
//
// Operands stream through a 16-step register ring (lane-major layout, one
// coalesced 8-byte load per thread per step), which leaves shared memory to
// the rings so two CTAs fit on an SM.
//
// Arithmetic and operation order are k_mic_lane2's (absent neighbours are
// -0.0, an exact no-op), so results are bit-identical.
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "ops.cuh"
#include "wavefront.cuh"

namespace flip {

namespace {

constexpr int CT = 16;   // tile edge: TY = TZ = 16

// global-halo prefetch depth (steps).  Measured at 256^3 (bench, ms/step):
// UH 1: 72.8, 2: 71.6*, 4: 74.9, 8: 75.9*, no prefetch: 81 (*warm single
// step).  A consumer runs close behind its producer, so a slot read several
// steps early is mostly still pending and only adds a wasted global load.
constexpr int UH = 1;

__device__ __forceinline__ unsigned smem_addr(const void *p) { return smem_u32(p); }
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned map_rank(const void *p, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ void st_remote(unsigned addr, double v) {
    asm volatile("st.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(addr),
                 "l"(__double_as_longlong(v))
                 : "memory");
}
__device__ __forceinline__ int ld_remote_int(unsigned addr) {
    int v;
    asm volatile("ld.relaxed.cluster.shared::cluster.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ double poll_local(const double *p) {
    unsigned long long v;
    const unsigned a = smem_addr(p);
    do {
        asm volatile("ld.relaxed.cluster.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    } while (v == WAVE_PENDING);
    return __longlong_as_double((long long)v);
}

// Global face slot, polled without back-off: on this path a consumer waits
// for a value its producer has just published, so every sleep quantum lands
// on the sweep's critical path.
__device__ __forceinline__ double poll_spin_gpu(const double *p) {
    unsigned long long v;
    do {
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    } while (v == WAVE_PENDING);
    return __longlong_as_double((long long)v);
}

// one non-blocking read of a ring slot (the pending marker if not yet stored)
__device__ __forceinline__ double peek_local(const double *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.cluster.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"(smem_addr(p)) : "memory");
    return __longlong_as_double((long long)v);
}

// Face value for this step from a slot read one step earlier: the read's
// latency overlaps the previous step, and only a slot that was still
// pending then is polled again.
__device__ __forceinline__ double take_face(double pre, const double *p) {
    return is_pending(pre) ? poll_local(p) : pre;
}

// cluster ticket -> (bq, cq) in anti-diagonal order over the cluster grid
__device__ __forceinline__ void cluster_tile(int t, int CB, int CC, int &bq, int &cq) {
    int d = 0;
    while (true) {
        int blo = max(0, d - (CC - 1)), bhi = min(CB - 1, d);
        int cnt = bhi - blo + 1;
        if (t < cnt) {
            bq = blo + t;
            cq = d - bq;
            return;
        }
        t -= cnt;
        d++;
    }
}

}  // namespace

template <bool REV, int CY, int CZ, int KC, int NB, int L2AHEAD>
__global__ void __launch_bounds__(CT *CT + 32) k_mic_cl(LaneArgs A) {
    constexpr int TY = CT, TZ = CT, TP = TY * TZ;
    constexpr int DY = TY - 1, DZ = TZ - 1;
    __shared__ double sval[2][TZ + 2][TY + 2];
    __shared__ int s_tile;
    __shared__ __align__(8) unsigned long long mbar[NB > 0 ? NB : 1];
    // yring[nsteps][TZ], zring[nsteps][TY], then the operand chunks
    extern __shared__ __align__(128) double ring[];
    const int t = threadIdx.x;
    pdl_wait();
    if (A.sc && A.sc->done) return;  // same value in every CTA of the launch
    const WaveGeom G = A.geom;
    const int nsteps = G.nsteps;
    double *yring = ring, *zring = ring + (int64_t)nsteps * TZ;
    const unsigned cr = cluster_rank();
    const int ry = (int)cr / CZ, rz = (int)cr % CZ;
    const double nz0 = -0.0;
    const double pend = __longlong_as_double((long long)WAVE_PENDING);
    for (int q = t; q < 2 * (TZ + 2) * (TY + 2); q += blockDim.x) (&sval[0][0][0])[q] = nz0;
    for (int q = t; q < nsteps * (TY + TZ); q += blockDim.x) ring[q] = pend;
    if (cr == 0 && t == 0) s_tile = atomicAdd(A.ticket, 1);
    if (t == 0) {
        for (int q = 0; q < NB; q++) mbar_init(&mbar[q], 1);
        mbar_fence_init();
    }
    unsigned long long t_start = 0;
    if (A.trace && t == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    cluster_sync_all();  // rings pre-filled everywhere, rank 0's ticket visible
    const int tk = cr == 0 ? s_tile : ld_remote_int(map_rank(&s_tile, 0));
    int bq, cq;
    cluster_tile(tk, G.TB / CY, G.TC / CZ, bq, cq);
    int b = bq * CY + ry, c = cq * CZ + rz;
    if (REV) {
        b = G.TB - 1 - b;
        c = G.TC - 1 - c;
    }
    const int tile = b * G.TC + c;
    if (A.trace && !REV && t == 0) A.trace[4 * tile + 0] = t_start;
    auto lstep = [&](int s) { return REV ? nsteps - 1 - s : s; };
    // In rank space the producer is always the previous rank along an axis
    // and the consumer the next one, in both sweep directions.
    const bool ydin = ry > 0, ydout = ry < CY - 1;
    const bool zdin = rz > 0, zdout = rz < CZ - 1;

    // operands: KC-step chunks through the bulk-copy engine into an NB-deep
    // ring after the face rings (opb[buf][src|precon][KC][TP]).  The helper
    // warp's lane 0 issues them, off the compute warps' critical path.
    double *opb = ring + (int64_t)nsteps * (TY + TZ);
    const int nch = (nsteps + KC - 1) / KC;
    auto issue = [&](int ch) {
        if (ch >= nch) return;
        const int64_t tbase = (int64_t)tile * nsteps * TP;
        const int s0 = ch * KC, cnt = min(KC, nsteps - s0);
        const int lo = REV ? nsteps - s0 - cnt : s0;
        const int buf = ch % (NB > 0 ? NB : 1);
        const unsigned bytes = (unsigned)(cnt * TP * 8);
        mbar_expect_tx(&mbar[buf], 2 * bytes);
        bulk_g2s(opb + (buf * 2 + 0) * KC * TP, A.src + tbase + (int64_t)lo * TP, bytes, &mbar[buf]);
        bulk_g2s(opb + (buf * 2 + 1) * KC * TP, A.precon + tbase + (int64_t)lo * TP, bytes,
                 &mbar[buf]);
        // stage a later chunk in L2 so the smem ring only has to hide L2 latency
        const int pf = ch + L2AHEAD;
        if (L2AHEAD > 0 && pf < nch) {
            const int p0 = pf * KC, pc = min(KC, nsteps - p0);
            const int plo = REV ? nsteps - p0 - pc : p0;
            const unsigned pb = (unsigned)(pc * TP * 8);
            bulk_prefetch_l2(A.src + tbase + (int64_t)plo * TP, pb);
            bulk_prefetch_l2(A.precon + tbase + (int64_t)plo * TP, pb);
        }
    };

    if (t >= TP) {
        // -------------------- helper warp: faces across cluster boundaries
        const int l = t - TP;
        const bool yface = l < TZ, zface = l >= TZ && l < TZ + TY;
        const int kk = yface ? l : 0, jj = zface ? l - TZ : 0;
        const int W = yface ? TZ : TY;
        const int D = yface ? DY : DZ;
        const double *in = nullptr;  // producing lanes publish their own faces
        int in_row = 0, in_col = 0, cons_j = 0, cons_k = 0;
        if (yface) {
            cons_j = REV ? TY - 1 : 0;
            cons_k = kk;
            const bool has = REV ? b + 1 < G.TB : b > 0;
            if (has && !ydin)
                in = A.halo_y + (int64_t)(REV ? tile + G.TC : tile - G.TC) * nsteps * TZ + kk;
            in_row = kk + 1;
            in_col = REV ? TY + 1 : 0;
        } else if (zface) {
            cons_j = jj;
            cons_k = REV ? TZ - 1 : 0;
            const bool has = REV ? c + 1 < G.TC : c > 0;
            if (has && !zdin)
                in = A.halo_z + (int64_t)(REV ? tile + 1 : tile - 1) * nsteps * TY + jj;
            in_row = REV ? TZ + 1 : 0;
            in_col = jj + 1;
        }
        const bool cvalid = G.jlo + b * TY + cons_j <= G.jhi && G.klo + c * TZ + cons_k <= G.khi;
        if (!cvalid) in = nullptr;
        if (NB > 0 && l == 0)
            for (int q = 0; q < NB; q++) issue(q);
        double hr[UH];
        auto fetch = [&](int s, int u) {
            const int sp = s + D;
            hr[u] = (in && sp < nsteps) ? ld_relaxed(in + (int64_t)sp * W) : nz0;
        };
#pragma unroll
        for (int u = 0; u < UH; u++) fetch(u + 1, u);
        if (in) sval[1][in_row][in_col] = D < nsteps ? poll_spin_gpu(in + (int64_t)D * W) : nz0;
        for (int s0 = 0; s0 < nsteps; s0 += UH) {
#pragma unroll
            for (int u = 0; u < UH; u++) {
                const int s = s0 + u;
                if (s >= nsteps) break;
                __syncthreads();
                if (NB > 0 && l == 0 && s > 0 && s % KC == 0) {
                    // every compute thread finished chunk s/KC - 1 before this barrier
                    fence_proxy_async();
                    issue(s / KC - 1 + NB);
                }
                const int cur = s & 1, prv = cur ^ 1;
                if (in) {
                    double v = hr[u];
                    if (is_pending(v)) v = poll_spin_gpu(in + (int64_t)(s + 1 + D) * W);
                    sval[cur][in_row][in_col] = v;
                    fetch(s + 1 + UH, u);
                }
            }
        }
        __syncthreads();
    } else {
        // ------------------------------------------------- compute warps
        const int jj = t % TY, kk = t / TY;
        const bool valid = G.jlo + b * TY + jj <= G.jhi && G.klo + c * TZ + kk <= G.khi;
        const int cons_j = REV ? TY - 1 : 0, cons_k = REV ? TZ - 1 : 0;
        const int prod_j = REV ? 0 : TY - 1, prod_k = REV ? 0 : TZ - 1;
        const bool yin = ydin && jj == cons_j && valid;
        const bool zin = zdin && kk == cons_k && valid;
        // consumer ranks: (ry+1, rz) = cr + CZ, (ry, rz+1) = cr + 1
        const unsigned yout = (ydout && jj == prod_j) ? map_rank(yring + kk, cr + CZ) : 0u;
        const unsigned zout = (zdout && kk == prod_k) ? map_rank(zring + jj, cr + 1) : 0u;
        // faces leaving the cluster: the producing lanes publish to the global
        // halo themselves (one store per step, no helper round trip)
        double *gy = (!ydout && jj == prod_j)
                         ? A.halo_y + (int64_t)tile * nsteps * TZ + kk : nullptr;
        double *gz = (!zdout && kk == prod_k)
                         ? A.halo_z + (int64_t)tile * nsteps * TY + jj : nullptr;
        const int yr = kk + 1, yc = REV ? jj + 2 : jj, zr = REV ? kk + 2 : kk, zc = jj + 1;
        const int64_t base = (int64_t)tile * nsteps * TP + t;
        double *dstL = A.dst + base;
        double pv = nz0;
        // face slots of the next step, read one step ahead (take_face)
        double ypre = yin && DY < nsteps ? peek_local(yring + DY * TZ + kk) : pend;
        double zpre = zin && DZ < nsteps ? peek_local(zring + DZ * TY + jj) : pend;
        const double sc = A.scale;
        if constexpr (NB == 0) {
            // operands straight into registers KC steps ahead (coalesced 8-byte
            // loads from the lane-major layout), no shared-memory round trip
            const int64_t base = (int64_t)tile * nsteps * TP + t;
            const double *srcL = A.src + base, *preL = A.precon + base;
            double av[KC], bv[KC];
            auto load = [&](int s, int u) {
                const int sl = max(min(lstep(s), nsteps - 1), 0);
                av[u] = __ldcs(srcL + (int64_t)sl * TP);
                bv[u] = __ldcs(preL + (int64_t)sl * TP);
            };
#pragma unroll
            for (int u = 0; u < KC; u++) load(u, u);
            for (int s0 = 0; s0 < nsteps; s0 += KC) {
#pragma unroll
                for (int u = 0; u < KC; u++) {
                    const int s = s0 + u;
                    if (s >= nsteps) break;
                    __syncthreads();
                    const int cur = s & 1, prv = cur ^ 1;
                    const double a = av[u], pr = bv[u];
                    load(s + KC, u);
                    double yv = sval[prv][yr][yc], zv = sval[prv][zr][zc];
                    if (yin) {
                        yv = s + DY < nsteps ? take_face(ypre, yring + (s + DY) * TZ + kk) : nz0;
                        if (s + 1 + DY < nsteps) ypre = peek_local(yring + (s + 1 + DY) * TZ + kk);
                    }
                    if (zin) {
                        zv = s + DZ < nsteps ? take_face(zpre, zring + (s + DZ) * TY + jj) : nz0;
                        if (s + 1 + DZ < nsteps) zpre = peek_local(zring + (s + 1 + DZ) * TY + jj);
                    }
                    const bool row = valid && present(a);
                    double o;
                    if (!REV) {  // _core.pyx:322-332
                        double tt = ((a + pv) + yv) + zv;
                        double q = tt * pr;
                        if (row) dstL[(int64_t)lstep(s) * TP] = q;
                        o = (sc * pr) * q;
                    } else {     // _core.pyx:333-346
                        double sp = sc * pr;
                        double tt = ((a + sp * pv) + sp * yv) + sp * zv;
                        o = tt * pr;
                        if (row) dstL[(int64_t)lstep(s) * TP] = o;
                    }
                    o = row ? o : nz0;
                    sval[cur][kk + 1][jj + 1] = o;
                    pv = o;
                    if (yout) st_remote(yout + (unsigned)(s * TZ * 8), o);
                    if (zout) st_remote(zout + (unsigned)(s * TY * 8), o);
                    if (gy) publish(gy + (int64_t)s * TZ, o);
                    if (gz) publish(gz + (int64_t)s * TY, o);
                }
            }
        }
        for (int ch = 0; NB > 0 && ch < nch; ch++) {
            const int s0 = ch * KC, cnt = min(KC, nsteps - s0);
            const int buf = ch % (NB > 0 ? NB : 1);
            mbar_wait(&mbar[buf], (unsigned)(ch / NB) & 1u);
            const double *ab = opb + (buf * 2 + 0) * KC * TP + t;
            const double *pb = opb + (buf * 2 + 1) * KC * TP + t;
#pragma unroll
            for (int u = 0; u < KC; u++) {
                if (u >= cnt) break;
                const int s = s0 + u;
                __syncthreads();
                const int cur = s & 1, prv = cur ^ 1;
                const int idx = REV ? cnt - 1 - u : u;
                const double a = ab[idx * TP], pr = pb[idx * TP];
                double yv = sval[prv][yr][yc], zv = sval[prv][zr][zc];
                if (yin) {
                    yv = s + DY < nsteps ? take_face(ypre, yring + (s + DY) * TZ + kk) : nz0;
                    if (s + 1 + DY < nsteps) ypre = peek_local(yring + (s + 1 + DY) * TZ + kk);
                }
                if (zin) {
                    zv = s + DZ < nsteps ? take_face(zpre, zring + (s + DZ) * TY + jj) : nz0;
                    if (s + 1 + DZ < nsteps) zpre = peek_local(zring + (s + 1 + DZ) * TY + jj);
                }
                if (A.trace && !REV && t == 0 && (s == 0 || (tile < 8 && s < 300))) {
                    unsigned long long g;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
                    if (tile < 8 && s < 300) A.trace[20000 + tile * 300 + s] = g;
                    if (s == 0) {
                        A.trace[4 * tile + 2] = g;
                        A.trace[4 * tile + 3] = (unsigned long long)b << 16 | (unsigned)c;
                    }
                }
                const bool row = valid && present(a);
                double o;
                if (!REV) {  // _core.pyx:322-332
                    double tt = ((a + pv) + yv) + zv;
                    double q = tt * pr;
                    if (row) dstL[(int64_t)lstep(s) * TP] = q;
                    o = (sc * pr) * q;
                } else {     // _core.pyx:333-346
                    double sp = sc * pr;
                    double tt = ((a + sp * pv) + sp * yv) + sp * zv;
                    o = tt * pr;
                    if (row) dstL[(int64_t)lstep(s) * TP] = o;
                }
                o = row ? o : nz0;
                sval[cur][kk + 1][jj + 1] = o;
                pv = o;
                if (yout) st_remote(yout + (unsigned)(s * TZ * 8), o);
                if (zout) st_remote(zout + (unsigned)(s * TY * 8), o);
                if (gy) publish(gy + (int64_t)s * TZ, o);
                if (gz) publish(gz + (int64_t)s * TY, o);
            }
        }
        __syncthreads();  // matches the helper's final barrier
        if (A.trace && !REV && t == 0) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            A.trace[4 * tile + 1] = g;
        }
    }
    // no CTA may leave while a cluster peer can still store into its rings
    cluster_sync_all();
}

// ------------------------------------------------------------- launching --
static int cluster_shape(int *cy, int *cz) {
    static int y = -1, z = -1;
    if (y < 0) {
        // default 4 x 4 tiles per cluster (fastest measured at 256^3);
        // FLIPB200_CLUSTER=CYxCZ picks another shape, =off disables
        y = z = 4;
        if (const char *e = getenv("FLIPB200_CLUSTER")) {
            int a = 0, b = 0;
            if (sscanf(e, "%dx%d", &a, &b) == 2) {
                y = a;
                z = b;
            } else {
                y = z = 0;
            }
        }
    }
    *cy = y;
    *cz = z;
    return y > 0 && z > 0;
}

int mic_cluster_pad(int *cy, int *cz) { return cluster_shape(cy, cz); }

// operand chunk ring: KC steps per bulk copy, NB chunks in flight, and an
// optional L2 prefetch L2AHEAD chunks further (FLIPB200_CL_CHUNKS=KCxNB[xL2]).
// Measured at 256^3 (project stage, 4x4 clusters): 4x3 65.8 ms, 4x8 69.8,
// 8x4 67.7, 4x3 + L2 prefetch 4 or 6 chunks ahead 65.8-65.9, "8x0" (no
// ring: operands loaded into registers 8 steps ahead) 87.4: deeper smem
// rings cost residency, registers expose the memory latency.
static int chunk_cfg() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("FLIPB200_CL_CHUNKS");  // "KCxNB" or "KCxNBxL2"
        int a = 4, b = 3, c = 0;
        if (e) sscanf(e, "%dx%dx%d", &a, &b, &c);
        v = c == 6 ? 4036 : (c == 4 ? 4034 : a * 100 + b);
    }
    return v;
}

template <bool REV, int CY, int CZ, int KC, int NB, int L2AHEAD>
static cudaError_t launch_cl_k(const LaneArgs &A, cudaStream_t st) {
    const int tiles = A.geom.TB * A.geom.TC;
    // face rings (2 x nsteps x 16) + operand chunks (NB x 2 x KC x 256), 128-B aligned
    const size_t rings = ((size_t)A.geom.nsteps * 2 * CT * sizeof(double) + 127) / 128 * 128;
    const size_t smem = rings + (size_t)NB * 2 * KC * CT * CT * sizeof(double);
    static cudaError_t attr = [] {
        cudaError_t e = cudaFuncSetAttribute(k_mic_cl<REV, CY, CZ, KC, NB, L2AHEAD>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             220 * 1024 - 6 * 1024);
        if (e == cudaSuccess && CY * CZ > 8)
            e = cudaFuncSetAttribute(k_mic_cl<REV, CY, CZ, KC, NB, L2AHEAD>,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return e;
    }();
    if (attr != cudaSuccess) return attr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)tiles);
    cfg.blockDim = dim3(CT * CT + 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CY * CZ;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // pdl_wait() in the kernel
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_mic_cl<REV, CY, CZ, KC, NB, L2AHEAD>, A);
    return e != cudaSuccess ? e : cudaPeekAtLastError();
}

template <bool REV, int CY, int CZ>
static cudaError_t launch_cl(const LaneArgs &A, cudaStream_t st) {
    switch (chunk_cfg()) {
        case 403: return launch_cl_k<REV, CY, CZ, 4, 3, 0>(A, st);
        case 804: return launch_cl_k<REV, CY, CZ, 8, 4, 0>(A, st);
        case 408: return launch_cl_k<REV, CY, CZ, 4, 8, 0>(A, st);
        case 4036: return launch_cl_k<REV, CY, CZ, 4, 3, 6>(A, st);
        case 4034: return launch_cl_k<REV, CY, CZ, 4, 3, 4>(A, st);
        case 800: return launch_cl_k<REV, CY, CZ, 8, 0, 0>(A, st);
        default: return launch_cl_k<REV, CY, CZ, 4, 3, 0>(A, st);
    }
}

// Returns cudaErrorNotSupported when no cluster shape is configured (the
// caller then uses k_mic_lane2).  Halos: step-major, halo_z after halo_y.
cudaError_t launch_mic_cluster(bool rev, const LaneArgs &A, cudaStream_t st) {
    int cy, cz;
    if (!cluster_shape(&cy, &cz) || A.geom.ty != CT || A.geom.tz != CT ||
        A.geom.TB % cy || A.geom.TC % cz)
        return cudaErrorNotSupported;
#define CL_CASE(a, b)                                                                \
    if (cy == a && cz == b) return rev ? launch_cl<true, a, b>(A, st) : launch_cl<false, a, b>(A, st);
    CL_CASE(2, 4)
    CL_CASE(4, 2)
    CL_CASE(2, 2)
    CL_CASE(4, 4)
    CL_CASE(1, 8)
    CL_CASE(8, 1)
    CL_CASE(1, 4)
    CL_CASE(2, 8)
    CL_CASE(1, 1)
#undef CL_CASE
    return cudaErrorNotSupported;
}

}  // namespace flip
