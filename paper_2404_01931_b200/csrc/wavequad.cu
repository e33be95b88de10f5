// wavequad.cu — MIC(0) forward/backward substitution (_core.pyx:311-347) as
// a tiled wavefront in which every thread owns a 2 x 2 block of x-pencils.
//
// k_mic_cl (wavecl.cu) gives each thread one pencil: a sweep then costs
// about ispan + jspan + kspan dependent steps (one CTA barrier each), ~529
// at 256^3.  Here thread (jj, kk) of a 16 x 16 tile owns pencils
// (2jj + a, 2kk + b), a, b in {0, 1}, and at step s visits i = ilo + s - jj
// - kk in all four.  Inside a step the four cells are evaluated in their
// dependency order (forward: (0,0); then (1,0) and (0,1); then (1,1) --
// each reads its in-thread -y / -z neighbour from the same step), so the
// dependent-step count drops to about ispan + jspan/2 + kspan/2 (~307 at
// 256^3) for a longer chain per step.  Tiles (32 x 32 pencils) exchange
// faces two values wide through DSMEM inside a cluster and through the
// step-major global halo across clusters, as in k_mic_cl.
//
// Arithmetic and operation order per cell are k_mic_cl's (absent
// neighbours are -0.0, an exact no-op), so results are bit-identical.
// Lane layout (k_lane_map with quad geometry): L[tile][step/4][q][thread]
// [step%4], q = a + 2b: 256 entries per tile-step, in groups of 4 steps so
// that consecutive rows of a pencil share a sector.
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "ops.cuh"
#include "wavefront.cuh"

namespace flip {

namespace {


__device__ __forceinline__ unsigned q_smem(const void *p) { return smem_u32(p); }
__device__ __forceinline__ unsigned q_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned q_map(const void *p, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(q_smem(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void q_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}
__device__ __forceinline__ void q_st_remote(unsigned addr, double v) {
    asm volatile("st.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(addr),
                 "l"(__double_as_longlong(v))
                 : "memory");
}
__device__ __forceinline__ int q_ld_remote_int(unsigned addr) {
    int v;
    asm volatile("ld.relaxed.cluster.shared::cluster.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ double q_poll(const double *p) {
    unsigned long long v;
    const unsigned a = q_smem(p);
    do {
        asm volatile("ld.relaxed.cluster.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    } while (v == WAVE_PENDING);
    return __longlong_as_double((long long)v);
}
__device__ __forceinline__ double q_peek(const double *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.cluster.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"(q_smem(p)) : "memory");
    return __longlong_as_double((long long)v);
}
__device__ __forceinline__ double q_take(double pre, const double *p) {
    return is_pending(pre) ? q_poll(p) : pre;
}
__device__ __forceinline__ double q_spin_gpu(const double *p) {
    unsigned long long v;
    do {
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    } while (v == WAVE_PENDING);
    return __longlong_as_double((long long)v);
}

__device__ __forceinline__ void q_cluster_tile(int t, int CB, int CC, int &bq, int &cq) {
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

// Stress mode (FLIPB200_QUAD_EXP=16, tests only): pseudo-random sleeps of
// up to ~2 us at ~1 in 8 (tile, step, thread) points perturb every
// producer/consumer timing of the face protocol; results must not change.
__device__ __forceinline__ void q_jitter(int X, int tile, int s, int t) {
    if (!(X & 16)) return;
    unsigned h = (unsigned)tile * 2654435761u ^ (unsigned)s * 40503u ^ (unsigned)t * 2246822519u;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    if ((h & 7u) == 0u) __nanosleep((h >> 16) & 2047u);
}

}  // namespace

// One cell of the substitution (k_mic_cl's arithmetic).  pv / yv / zv are
// the contributions of the -x / -y / -z (forward) or +x / +y / +z
// (backward) neighbours; returns the value passed on, -0.0 off the rows.
// The lane entry is written unconditionally (no branch): the value on a
// row, the ABSENT marker elsewhere (the next sweep's src keeps its markers;
// rows are only ever read back through posL).
template <bool REV>
__device__ __forceinline__ double mic_cell(double a, double pr, double pv, double yv, double zv,
                                           double sc, bool row, double *dst) {
    const double absent = __longlong_as_double((long long)WAVE_ABSENT);
    double o;
    if (!REV) {  // _core.pyx:322-332
        double tt = ((a + pv) + yv) + zv;
        double q = tt * pr;
        if (dst) __stcg(dst, row ? q : absent);
        o = (sc * pr) * q;
    } else {     // _core.pyx:333-346
        double sp = sc * pr;
        double tt = ((a + sp * pv) + sp * yv) + sp * zv;
        o = tt * pr;
        if (dst) __stcg(dst, row ? o : absent);
    }
    return row ? o : -0.0;
}

// mic_cell returning the lane-layout value (the row's result, or the ABSENT
// marker) instead of storing it: the quad kernel stores 4 steps at once.
template <bool REV>
__device__ __forceinline__ double mic_cell_v(double a, double pr, double pv, double yv, double zv,
                                             double sc, bool row, double &stored) {
    const double absent = __longlong_as_double((long long)WAVE_ABSENT);
    double o;
    if (!REV) {  // _core.pyx:322-332
        double tt = ((a + pv) + yv) + zv;
        double q = tt * pr;
        stored = row ? q : absent;
        o = (sc * pr) * q;
    } else {     // _core.pyx:333-346
        double sp = sc * pr;
        double tt = ((a + sp * pv) + sp * yv) + sp * zv;
        o = tt * pr;
        stored = row ? o : absent;
    }
    return row ? o : -0.0;
}

// One cell of the MIC(0) build (_core.pyx:291-307), the forward
// recurrence that produces precon.  a = diag (ABSENT off the rows), code =
// k_x + 3 k_y + 9 k_z with k_p the number of the lower neighbour's two
// "other" neighbours that are rows (o1/o2 of the pair), pv / yv / zv = the
// precon of the -x / -y / -z neighbour, or +-0.0 when that neighbour is not
// a row: with pq == 0 both updates of its pair subtract a zero, an exact
// no-op, as the reference's skipped pair (precon itself is never 0).
__device__ __forceinline__ double mic_build_v(double diag, double code, double pv, double yv,
                                              double zv, double scale, bool row, double &stored) {
    const double absent = __longlong_as_double((long long)WAVE_ABSENT);
    const double tau = 0.97, sigma = 0.25;  // mic0_build's defaults (_core.pyx:275-276)
    const int cd = row ? (int)code : 0;
    double e = diag * scale;
    const double pq3[3] = {pv, yv, zv};
    const int kp[3] = {cd % 3, (cd / 3) % 3, cd / 9};
#pragma unroll
    for (int p = 0; p < 3; p++) {
        const double pq = pq3[p];
        e = e - (scale * pq) * (scale * pq);
        double others = 0.0;
        if (kp[p] > 0) others = others - scale;
        if (kp[p] > 1) others = others - scale;
        e = e - (((tau * (-scale)) * others) * pq) * pq;
    }
    if (e < (sigma * diag) * scale) e = diag * scale;
    const double o = 1.0 / sqrt(e);
    stored = row ? o : absent;
    return row ? o : -0.0;
}

// QT threads per tile edge (16 or 8): a tile is 2QT x 2QT pencils, the
// faces are QW = 2QT values wide.
template <bool REV, int QT, int CY, int CZ, int KC, int NB, int PF, int HW = 1, int BUILD = 0>
__global__ void __launch_bounds__(QT * QT + 32 * HW) k_mic_quad(LaneArgs A) {
    constexpr int QP = QT * QT, QW = 2 * QT;
    constexpr int DY = QT - 1, DZ = QT - 1;
    // logical cell L (forward order (0,0), (1,0), (0,1), (1,1)) -> stored q
    // (pencil a + 2b); the backward sweep visits the block mirrored
    auto PQ = [](int L) { return REV ? 3 - L : L; };
    // sq[buf][q][kk + 1][jj + 1]: each thread's four outputs of a step
    // (q-planar, so a warp's loads and stores hit consecutive banks)
    __shared__ double sq[2][4][QT + 2][QT + 2];
    __shared__ int s_tile;
    __shared__ __align__(8) unsigned long long mbar[NB];
    // yring[nsteps][QW], zring[nsteps][QW], then the operand chunks
    extern __shared__ __align__(128) double ring[];
    const int t = threadIdx.x;
    pdl_wait();
    if (A.sc && A.sc->done) return;
    // probe: this launch's slot (the iteration counter is final before the
    // sweeps run: k_pcg_update advanced it)
    const int pslot = A.ts ? min(2 * (A.sc ? A.sc->iter : 0) + (REV ? 1 : 0), kProbeSlots - 1) : 0;
    if (A.ts && t == 0) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        atomicMin(A.ts + pslot, g);
    }
    const WaveGeom G = A.geom;
    const int nsteps = G.nsteps;
    // lane-layout entries and halo words per direction (checked build)
    const int64_t lane_n = (int64_t)G.TB * G.TC * nsteps * 4 * QP;
    const int64_t halo_n = (int64_t)G.TB * G.TC * nsteps * QW;
    (void)lane_n;
    (void)halo_n;
    double *yring = ring, *zring = ring + (int64_t)nsteps * QW;
    const unsigned cr = q_rank();
    const int ry = (int)cr / CZ, rz = (int)cr % CZ;
    const double nz0 = -0.0;
    const double pend = __longlong_as_double((long long)WAVE_PENDING);
    for (int q = t; q < 2 * 4 * (QT + 2) * (QT + 2); q += blockDim.x) (&sq[0][0][0][0])[q] = nz0;
    for (int q = t; q < nsteps * 2 * QW; q += blockDim.x) ring[q] = pend;
    if (cr == 0 && t == 0) s_tile = atomicAdd(A.ticket, 1);
    if (t == 0) {
        for (int q = 0; q < NB; q++) mbar_init(&mbar[q], 1);
        mbar_fence_init();
    }
    q_cluster_sync();
    const int tk = cr == 0 ? s_tile : q_ld_remote_int(q_map(&s_tile, 0));
    FLIP_CHECK_RANGE(tk, (int)(gridDim.x / (CY * CZ)), "quad cluster ticket");
    int bq, cq;
    q_cluster_tile(tk, G.TB / CY, G.TC / CZ, bq, cq);
    int b = bq * CY + ry, c = cq * CZ + rz;
    if (REV) {
        b = G.TB - 1 - b;
        c = G.TC - 1 - c;
    }
    const int tile = b * G.TC + c;
    unsigned long long *trace = (!REV && A.trace) ? A.trace : nullptr;  // FLIPB200_WAVE_TRACE
    if (trace && t == 0) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        trace[4 * tile + 0] = g;
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        trace[4 * tile + 3] = (unsigned long long)smid << 32 | (unsigned long long)b << 16 | (unsigned)c;
    }
    auto lstep = [&](int s) { return REV ? nsteps - 1 - s : s; };
    const bool ydin = ry > 0, ydout = ry < CY - 1;
    const bool zdin = rz > 0, zdout = rz < CZ - 1;
    constexpr int TS = 4 * QP;  // lane entries per tile-step
    double *opb = ring + (int64_t)nsteps * 2 * QW;
    const int nch = (nsteps + KC - 1) / KC;
    auto issue = [&](int ch) {
        if (ch >= nch) return;
        const int64_t tbase = (int64_t)tile * nsteps * TS;
        const int s0 = ch * KC, cnt = min(KC, nsteps - s0);
        const int lo = REV ? nsteps - s0 - cnt : s0;
        const int buf = ch % NB;
        const unsigned bytes = (unsigned)(cnt * TS * 8);
        mbar_expect_tx(&mbar[buf], 2 * bytes);
        FLIP_CHECK(lo >= 0 && lo + cnt <= nsteps && cnt % 4 == 0, "quad chunk", lo, nsteps);
        FLIP_CHECK_RANGE(tbase + (int64_t)(lo + cnt) * TS - 1, lane_n, "quad chunk source");
        bulk_g2s(opb + (buf * 2 + 0) * KC * TS, A.src + tbase + (int64_t)lo * TS, bytes, &mbar[buf]);
        bulk_g2s(opb + (buf * 2 + 1) * KC * TS, A.precon + tbase + (int64_t)lo * TS, bytes,
                 &mbar[buf]);
    };
    // neighbour-thread offsets in sq: forward reads jj-1 / kk-1, backward jj+1 / kk+1
    const int nbo = REV ? 2 : 0;

    if (t >= QP) {
        // ------------------- helper warp: faces across cluster boundaries
        // lane l carries y-face word l (consumer kk = l/2; e = 0 feeds
        // logical cell 0, e = 1 cell 2) and z-face word l (consumer jj =
        // l/2; e = 0 feeds cell 0, e = 1 cell 1)
        const int l = (t - QP) & 31;
        // y word ly and z word lz of this lane (-1: none).  HW = 2: one
        // helper warp per face (y: the first, z: the second), so a tile fed
        // on both faces does not run the two faces' waits one after the
        // other in divergent halves of one warp.
        const int hw = (t - QP) >> 5;
        const int ly = HW == 2 ? (hw == 0 && l < QW ? l : -1) : QW == 32 ? l : (l < QW ? l : -1);
        const int lz = HW == 2 ? (hw == 1 && l < QW ? l : -1)
                               : QW == 32 ? l : (l >= 32 - QW ? l - (32 - QW) : -1);
        // The helper also forwards the faces that arrive by DSMEM (from its
        // own rings), so no compute lane polls or diverges on face code
        // (measured: 176.4 -> 169.2 us per sweep at 256^3).
        const bool HF = true;
        const double *iny = nullptr, *inz = nullptr;
        const double *ly_ring = nullptr, *lz_ring = nullptr;
        {
            const bool has = REV ? b + 1 < G.TB : b > 0;
            if (has && !ydin && ly >= 0)
                iny = A.halo_y + (int64_t)(REV ? tile + G.TC : tile - G.TC) * nsteps * QW + ly;
            if (HF && ydin && ly >= 0) ly_ring = yring + ly;
            const bool hasz = REV ? c + 1 < G.TC : c > 0;
            if (hasz && !zdin && lz >= 0)
                inz = A.halo_z + (int64_t)(REV ? tile + 1 : tile - 1) * nsteps * QW + lz;
            if (HF && zdin && lz >= 0) lz_ring = zring + lz;
        }
        // where the value lands: the consumer reads its -y (-z) neighbour
        // thread's stored output of the producing logical cell
        const int ey = ly & 1, hy_ = ly >> 1, ez = lz & 1, hz_ = lz >> 1;
        const int y_row = hy_ + 1, y_col = REV ? QT + 1 : 0, y_q = PQ(ey == 0 ? 1 : 3);
        const int z_row = REV ? QT + 1 : 0, z_col = hz_ + 1, z_q = PQ(ez == 0 ? 2 : 3);
        // the consumer lanes must lie in the rows' box
        const int cons_j = REV ? QT - 1 : 0, cons_k = REV ? QT - 1 : 0;
        if (!(G.jlo + b * QW + 2 * cons_j <= G.jhi && G.klo + c * QW + 2 * hy_ <= G.khi)) iny = ly_ring = nullptr;
        if (!(G.jlo + b * QW + 2 * hz_ <= G.jhi && G.klo + c * QW + 2 * cons_k <= G.khi)) inz = lz_ring = nullptr;
        if (l == 0 && hw == 0)
            for (int q = 0; q < NB; q++) issue(q);
        // slot of producer step sp: global halo or local DSMEM ring
        auto peek_y = [&](int sp) {
            FLIP_CHECK_RANGE(sp, nsteps, "quad y face slot");
            if (iny) FLIP_CHECK_RANGE(iny + (int64_t)sp * QW - A.halo_y, halo_n, "quad y halo read");
            return iny ? ld_relaxed(iny + (int64_t)sp * QW) : q_peek(ly_ring + sp * QW);
        };
        auto spin_y = [&](int sp) { return iny ? q_spin_gpu(iny + (int64_t)sp * QW) : q_poll(ly_ring + sp * QW); };
        auto peek_z = [&](int sp) {
            FLIP_CHECK_RANGE(sp, nsteps, "quad z face slot");
            if (inz) FLIP_CHECK_RANGE(inz + (int64_t)sp * QW - A.halo_z, halo_n, "quad z halo read");
            return inz ? ld_relaxed(inz + (int64_t)sp * QW) : q_peek(lz_ring + sp * QW);
        };
        auto spin_z = [&](int sp) { return inz ? q_spin_gpu(inz + (int64_t)sp * QW) : q_poll(lz_ring + sp * QW); };
        const bool fy = iny || ly_ring, fz = inz || lz_ring;
        // lag (FLIPB200_QUAD_LAG, cross-cluster faces only): start only once
        // the producer is LAG steps further ahead than the skew requires, so
        // the face loads of later steps rarely find a pending slot
        if (A.lag > 0) {
            if (iny && DY + A.lag < nsteps) (void)spin_y(DY + A.lag);
            if (inz && DZ + A.lag < nsteps) (void)spin_z(DZ + A.lag);
        }
        if (fy) sq[1][y_q][y_row][y_col] = DY < nsteps ? spin_y(DY) : nz0;
        if (fz) sq[1][z_q][z_row][z_col] = DZ < nsteps ? spin_z(DZ) : nz0;
        // Face values of the next PF steps are loaded ahead: a global-halo
        // load takes ~0.6 us, longer than a step, so with one load in flight
        // a tile fed across a cluster boundary steps at the load latency
        // (trace: 0.55-0.65 us per step there vs 0.23-0.3 inside a
        // cluster).  The loop is unrolled by PF so every queued register is
        // read only when its slot is consumed (a rotating queue would wait
        // for all loads in flight at every step).
        double qy[PF], qz[PF];
#pragma unroll
        for (int u = 0; u < PF; u++) {
            qy[u] = (fy && 1 + u + DY < nsteps) ? peek_y(1 + u + DY) : nz0;
            qz[u] = (fz && 1 + u + DZ < nsteps) ? peek_z(1 + u + DZ) : nz0;
        }
        for (int s0 = 0; s0 < nsteps; s0 += PF) {
#pragma unroll
            for (int u = 0; u < PF; u++) {
                const int s = s0 + u;
                if (s >= nsteps) break;
                __syncthreads();
                if (l == 0 && hw == 0 && s > 0 && s % KC == 0 && !(A.dbg & 1)) {
                    fence_proxy_async();
                    issue(s / KC - 1 + NB);
                }
                const int cur = s & 1;
                q_jitter(A.dbg, tile, s, t);
                if (fy) {
                    double v = (s + 1 + DY < nsteps) ? qy[u] : nz0;
                    if (is_pending(v)) {
                        v = spin_y(s + 1 + DY);
                        const int trel = tile - A.trace_t0;
                        if (trace && trel >= 0 && trel < 8 && s < 300)
                            atomicOr(trace + 24000 + trel * 300 + s, iny ? 1ull : 4ull);
                    }
                    sq[cur][y_q][y_row][y_col] = v;
                    qy[u] = (s + 1 + PF + DY < nsteps) ? peek_y(s + 1 + PF + DY) : nz0;
                }
                if (fz) {
                    double v = (s + 1 + DZ < nsteps) ? qz[u] : nz0;
                    if (is_pending(v)) {
                        v = spin_z(s + 1 + DZ);
                        const int trel = tile - A.trace_t0;
                        if (trace && trel >= 0 && trel < 8 && s < 300)
                            atomicOr(trace + 24000 + trel * 300 + s, inz ? 2ull : 8ull);
                    }
                    sq[cur][z_q][z_row][z_col] = v;
                    qz[u] = (s + 1 + PF + DZ < nsteps) ? peek_z(s + 1 + PF + DZ) : nz0;
                }
            }
        }
        __syncthreads();
    } else {
        // ----------------------------------------------------- compute warps
        const int jj = t % QT, kk = t / QT;
        const int jbase = G.jlo + b * QW + 2 * jj, kbase = G.klo + c * QW + 2 * kk;
        // logical cell -> in the rows' box (pencil offsets mirrored backward)
        bool valid[4];
#pragma unroll
        for (int L = 0; L < 4; L++) {
            const int q = PQ(L);
            valid[L] = jbase + (q & 1) <= G.jhi && kbase + (q >> 1) <= G.khi;
        }
        const int cons_j = REV ? QT - 1 : 0, cons_k = REV ? QT - 1 : 0;
        const int prod_j = REV ? 0 : QT - 1, prod_k = REV ? 0 : QT - 1;
        // producing lanes: DSMEM into the next CTA of the cluster, or the
        // global halo when the face leaves the cluster
        const unsigned yout = (ydout && jj == prod_j) ? q_map(yring + 2 * kk, cr + CZ) : 0u;
        const unsigned zout = (zdout && kk == prod_k) ? q_map(zring + 2 * jj, cr + 1) : 0u;
        double *gy = (!ydout && jj == prod_j) ? A.halo_y + (int64_t)tile * nsteps * QW + 2 * kk : nullptr;
        double *gz = (!zdout && kk == prod_k) ? A.halo_z + (int64_t)tile * nsteps * QW + 2 * jj : nullptr;
        // lane layout, groups of 4 steps: entry ((g * TS + q * QP + t) * 4 + w)
        // for step 4g + w of the tile (k_lane_map), so 4 consecutive steps of
        // a pencil share one 32-byte sector (the PCG update's r scatter and
        // the z.r dot's gather touch a quarter of the sectors)
        double *dstL = A.dst + (int64_t)tile * nsteps * TS + 4 * t;
        double pv[4] = {nz0, nz0, nz0, nz0};
        const double sc = A.scale;
        const int yr = kk + 1, yc = jj + nbo, zr = kk + nbo, zc = jj + 1;
        const int X = A.dbg;  // timing experiments only (FLIPB200_QUAD_EXP): results differ
        // Per chunk, groups of 4 steps: a group's operands are in registers
        // before its first step (two 16-byte shared loads per cell and
        // array); the next group's are issued one cell per step during the
        // current group, behind that step's neighbour reads.  Outputs are
        // stored per group (16-byte stores).
        for (int ch = 0; ch < nch; ch++) {
            const int s0 = ch * KC, cnt = min(KC, nsteps - s0);  // cnt: a multiple of 4
            const int buf = ch % NB;
            if (!(X & 1) || ch < NB) mbar_wait(&mbar[buf], (unsigned)(ch / NB) & 1u);
            const double *ab = opb + (buf * 2 + 0) * KC * TS + 4 * t;
            const double *pb = opb + (buf * 2 + 1) * KC * TS + 4 * t;
            const int lo = REV ? nsteps - s0 - cnt : s0;  // the chunk holds logical steps [lo, lo + cnt)
            const int ng = cnt / 4;
            auto load_cell = [&](int gi, int L, double2 (&AA)[4][2], double2 (&PP)[4][2]) {
                const int g = REV ? ng - 1 - gi : gi;  // group in the buffer
                const double *pa = ab + (g * TS + PQ(L) * QP) * 4;
                const double *pp = pb + (g * TS + PQ(L) * QP) * 4;
                AA[L][0] = *reinterpret_cast<const double2 *>(pa);
                AA[L][1] = *reinterpret_cast<const double2 *>(pa + 2);
                PP[L][0] = *reinterpret_cast<const double2 *>(pp);
                PP[L][1] = *reinterpret_cast<const double2 *>(pp + 2);
            };
            double2 A2[4][2], P2[4][2], NA[4][2], NP[4][2];
            // the chunk's first group: only the half its first two steps use
            // is loaded before the first step, the other half during it
            const bool split = !(X & 256);  // (measured: 122.9 -> 121.6 us per sweep)
            const int h0 = REV ? 1 : 0;
            if (split) {
                const int g0 = REV ? ng - 1 : 0;
#pragma unroll
                for (int L = 0; L < 4; L++) {
                    A2[L][h0] = *reinterpret_cast<const double2 *>(ab + (g0 * TS + PQ(L) * QP) * 4 + 2 * h0);
                    P2[L][h0] = *reinterpret_cast<const double2 *>(pb + (g0 * TS + PQ(L) * QP) * 4 + 2 * h0);
                }
            } else {
#pragma unroll
                for (int L = 0; L < 4; L++) load_cell(0, L, A2, P2);
            }
#pragma unroll
            for (int gi = 0; gi < KC / 4; gi++) {
                if (gi >= ng) break;
                const int g = REV ? ng - 1 - gi : gi;  // group in the buffer
                if (gi > 0) {
#pragma unroll
                    for (int L = 0; L < 4; L++) {
                        A2[L][0] = NA[L][0];
                        A2[L][1] = NA[L][1];
                        P2[L][0] = NP[L][0];
                        P2[L][1] = NP[L][1];
                    }
                }
                double O[4][4];  // stored values [cell][step in the group, logical order]
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int s = s0 + 4 * gi + u;
                    const int w = REV ? 3 - u : u;  // logical step within the group
                    __syncthreads();
                    const int trel = tile - A.trace_t0;  // per-step stamps of 8 tiles
                    if (trace && t == 0 && (s == 0 || (trel >= 0 && trel < 8 && s < 300))) {
                        unsigned long long gt;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
                        if (trel >= 0 && trel < 8 && s < 300) trace[20000 + trel * 300 + s] = gt;
                        if (s == 0) trace[4 * tile + 2] = gt;
                    }
                    const int cur = s & 1, prv = cur ^ 1;
                    double a[4], pr[4];
#pragma unroll
                    for (int L = 0; L < 4; L++) {
                        const double2 av = A2[L][w >> 1], pv2 = P2[L][w >> 1];
                        a[L] = (w & 1) ? av.y : av.x;
                        pr[L] = (w & 1) ? pv2.y : pv2.x;
                    }
                    // neighbour contributions from the previous step: -y feeds
                    // logical cells 0 and 2 (the -y thread's cells 1 and 3), -z
                    // feeds cells 0 and 1 (the -z thread's cells 2 and 3)
                    const double y0 = sq[prv][PQ(1)][yr][yc], y2 = sq[prv][PQ(3)][yr][yc];
                    const double z0 = sq[prv][PQ(2)][zr][zc], z1 = sq[prv][PQ(3)][zr][zc];
                    if (split && gi == 0 && u == 0) {
                        const int g0 = REV ? ng - 1 : 0;
                        asm volatile("" ::: "memory");
#pragma unroll
                        for (int L = 0; L < 4; L++) {
                            A2[L][1 - h0] = *reinterpret_cast<const double2 *>(ab + (g0 * TS + PQ(L) * QP) * 4 + 2 * (1 - h0));
                            P2[L][1 - h0] = *reinterpret_cast<const double2 *>(pb + (g0 * TS + PQ(L) * QP) * 4 + 2 * (1 - h0));
                        }
                        asm volatile("" ::: "memory");
                    }
                    if (gi + 1 < ng) {
                        asm volatile("" ::: "memory");
                        load_cell(gi + 1, u, NA, NP);
                        asm volatile("" ::: "memory");
                    }
                    double o[4];
                    if (BUILD) {
                        o[0] = mic_build_v(a[0], pr[0], pv[0], y0, z0, sc, valid[0] && present(a[0]), O[0][w]);
                        o[1] = mic_build_v(a[1], pr[1], pv[1], o[0], z1, sc, valid[1] && present(a[1]), O[1][w]);
                        o[2] = mic_build_v(a[2], pr[2], pv[2], y2, o[0], sc, valid[2] && present(a[2]), O[2][w]);
                        o[3] = mic_build_v(a[3], pr[3], pv[3], o[2], o[1], sc, valid[3] && present(a[3]), O[3][w]);
                    } else {
                        o[0] = mic_cell_v<REV>(a[0], pr[0], pv[0], y0, z0, sc, valid[0] && present(a[0]), O[0][w]);
                        o[1] = mic_cell_v<REV>(a[1], pr[1], pv[1], o[0], z1, sc, valid[1] && present(a[1]), O[1][w]);
                        o[2] = mic_cell_v<REV>(a[2], pr[2], pv[2], y2, o[0], sc, valid[2] && present(a[2]), O[2][w]);
                        o[3] = mic_cell_v<REV>(a[3], pr[3], pv[3], o[2], o[1], sc, valid[3] && present(a[3]), O[3][w]);
                    }
#pragma unroll
                    for (int L = 0; L < 4; L++) {
                        sq[cur][PQ(L)][kk + 1][jj + 1] = o[L];
                        pv[L] = o[L];
                    }
                    if (X & 128) {  // per-step 8-byte stores instead of the group's
                        double *dd = dstL + (int64_t)((lo >> 2) + g) * TS * 4 + w;
#pragma unroll
                        for (int L = 0; L < 4; L++) __stcg(dd + PQ(L) * QP * 4, O[L][w]);
                    }
                    q_jitter(X, tile, s, t);
                    if (yout) {
                        FLIP_CHECK_RANGE(s, nsteps, "quad y DSMEM ring");
                        q_st_remote(yout + (unsigned)(s * QW * 8), o[1]);
                        q_st_remote(yout + (unsigned)(s * QW * 8 + 8), o[3]);
                    }
                    if (zout) {
                        q_st_remote(zout + (unsigned)(s * QW * 8), o[2]);
                        q_st_remote(zout + (unsigned)(s * QW * 8 + 8), o[3]);
                    }
                    if (gy) {
                        FLIP_CHECK_RANGE(gy + (int64_t)s * QW + 1 - A.halo_y, halo_n, "quad y halo publish");
                        publish(gy + (int64_t)s * QW, o[1]);
                        publish(gy + (int64_t)s * QW + 1, o[3]);
                    }
                    if (gz) {
                        FLIP_CHECK_RANGE(gz + (int64_t)s * QW + 1 - A.halo_z, halo_n, "quad z halo publish");
                        publish(gz + (int64_t)s * QW, o[2]);
                        publish(gz + (int64_t)s * QW + 1, o[3]);
                    }
                }
                if (!(X & 2) && !(X & 128)) {
                    double *d = dstL + (int64_t)((lo >> 2) + g) * TS * 4;
                    FLIP_CHECK_RANGE(d + PQ(3) * QP * 4 + 3 - A.dst, lane_n, "quad group store");
#pragma unroll
                    for (int L = 0; L < 4; L++) {
                        __stcg(reinterpret_cast<double2 *>(d + PQ(L) * QP * 4), make_double2(O[L][0], O[L][1]));
                        __stcg(reinterpret_cast<double2 *>(d + PQ(L) * QP * 4 + 2), make_double2(O[L][2], O[L][3]));
                    }
                }
            }
        }
        __syncthreads();  // matches the helper's final barrier
        if (trace && t == 0) {
            unsigned long long g;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
            trace[4 * tile + 1] = g;
        }
    }
    q_cluster_sync();  // no CTA leaves while a peer can still store into its rings
    if (A.ts && t == 0) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        atomicMax(A.ts + kProbeSlots + pslot, g);
    }
}

// ------------------------------------------------------------- launching --
int quad_threads();

// Helper warps per CTA (FLIPB200_QUAD_HW): 2 = one per face (measured at
// 256^3: 0.167 -> 0.118 ms per sweep), 1 = round-2's single helper warp.
static int hw_default() {
    static const int hw = getenv("FLIPB200_QUAD_HW") ? atoi(getenv("FLIPB200_QUAD_HW")) : 2;
    return hw == 1 ? 1 : 2;
}

int quad_cluster_shape(int *cy, int *cz) {
    static int y = -1, z = -1;
    if (y < 0) {
        y = quad_threads() == 16 ? 2 : 4;
        z = 4;
        if (const char *e = getenv("FLIPB200_QUAD_CLUSTER")) {
            int a = 0, b = 0;
            if (sscanf(e, "%dx%d", &a, &b) == 2) {
                y = a;
                z = b;
            }
        }
    }
    *cy = y;
    *cz = z;
    return 1;
}

bool mic_quad_enabled() {
    static const int on = [] {
        const char *e = getenv("FLIPB200_QUAD");
        return e ? atoi(e) : 1;
    }();
    return on != 0;
}

int quad_threads() {  // threads per tile edge (FLIPB200_QUAD_QT: 16 or 8)
    static const int q = [] {
        const char *e = getenv("FLIPB200_QUAD_QT");
        const int v = e ? atoi(e) : 8;
        return v == 16 ? 16 : 8;
    }();
    return q;
}

// Quad geometry: tiles of 2QT x 2QT pencils, QT x QT threads, padded to
// whole clusters; nsteps = ispan + 2 * (QT - 1).
WaveGeom quad_geom(const int lo[3], const int hi[3]) {
    int cy, cz;
    quad_cluster_shape(&cy, &cz);
    const int QT = quad_threads(), QW = 2 * QT;
    WaveGeom g{};
    g.ilo = lo[0];
    g.ihi = hi[0];
    g.jlo = lo[1];
    g.jhi = hi[1];
    g.klo = lo[2];
    g.khi = hi[2];
    g.ty = QW;
    g.tz = QW;
    g.TB = (hi[1] - lo[1] + QW) / QW;
    g.TC = (hi[2] - lo[2] + QW) / QW;
    g.TB = (g.TB + cy - 1) / cy * cy;
    g.TC = (g.TC + cz - 1) / cz * cz;
    g.ispan = hi[0] - lo[0] + 1;
    g.ispan_pad = (g.ispan + 1) & ~1;
    // a multiple of 4: the 4-step groups of the lane layout align with the
    // operand chunks in both sweep directions (chunks hold 8 or 4 steps)
    g.nsteps = (g.ispan + 2 * (QT - 1) + 3) / 4 * 4;
    g.quad = QT;
    return g;
}

template <bool REV, int QT, int CY, int CZ, int KC, int NB, int PF = 1, int HW = 1, int BUILD = 0>
static cudaError_t launch_quad_k(const LaneArgs &A, cudaStream_t st) {
    constexpr int QP = QT * QT, QW = 2 * QT;
    const int tiles = A.geom.TB * A.geom.TC;
    const size_t rings = ((size_t)A.geom.nsteps * 2 * QW * sizeof(double) + 127) / 128 * 128;
    static const size_t pad = getenv("FLIPB200_QUAD_PAD") ? (size_t)atoi(getenv("FLIPB200_QUAD_PAD")) * 1024 : 0;
    const size_t smem = rings + (size_t)NB * 2 * KC * 4 * QP * sizeof(double) + pad;
    static cudaError_t attr = [] {
        cudaError_t e = cudaFuncSetAttribute(k_mic_quad<REV, QT, CY, CZ, KC, NB, PF, HW, BUILD>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             227 * 1024 - 24 * 1024);
        if (e == cudaSuccess && CY * CZ > 8)
            e = cudaFuncSetAttribute(k_mic_quad<REV, QT, CY, CZ, KC, NB, PF, HW, BUILD>,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return e;
    }();
    if (attr != cudaSuccess) return attr;
    if (smem > 227 * 1024 - 24 * 1024) return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)tiles);
    cfg.blockDim = dim3(QP + 32 * HW);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CY * CZ;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_mic_quad<REV, QT, CY, CZ, KC, NB, PF, HW, BUILD>, A);
    return e != cudaSuccess ? e : cudaPeekAtLastError();
}

// Can the configured quad kernel's clusters be scheduled on this device
// (16-CTA clusters are non-portable)?  Checked once per process.
template <int QT, int CY, int CZ, int KC, int NB, int HW = 1>
static bool quad_fits(int nsteps) {
    constexpr int QP = QT * QT, QW = 2 * QT;
    const size_t rings = ((size_t)nsteps * 2 * QW * sizeof(double) + 127) / 128 * 128;
    const size_t smem = rings + (size_t)NB * 2 * KC * 4 * QP * sizeof(double);
    auto k = k_mic_quad<false, QT, CY, CZ, KC, NB, 1, HW>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024 - 24 * 1024) != cudaSuccess)
        return false;
    if (CY * CZ > 8 &&
        cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        return false;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CY * CZ);
    cfg.blockDim = dim3(QP + 32 * HW);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CY * CZ;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    const bool ok = cudaOccupancyMaxActiveClusters(&n, k, &cfg) == cudaSuccess && n > 0;
    cudaGetLastError();
    return ok;
}

static int quad_chunks() {
    static int v = -1;
    if (v < 0) {
        int a = 0, b = 0;
        if (const char *e = getenv("FLIPB200_QUAD_CHUNKS")) sscanf(e, "%dx%d", &a, &b);
        v = a * 100 + b;
    }
    return v;
}

template <bool REV, int CY, int CZ>
static cudaError_t launch_quad_c(const LaneArgs &A, cudaStream_t st) {
    if (A.geom.quad == 16) {
        switch (quad_chunks()) {
            case 204: return launch_quad_k<REV, 16, CY, CZ, 2, 4>(A, st);
            default:
                return A.hw == 2 ? launch_quad_k<REV, 16, CY, CZ, 2, 3, 1, 2>(A, st)
                                 : launch_quad_k<REV, 16, CY, CZ, 2, 3, 1, 1>(A, st);
        }
    }
    switch (quad_chunks()) {  // QT = 8: 2 KB of operands per array and step
        case 403: return A.hw == 2 ? launch_quad_k<REV, 8, CY, CZ, 4, 3, 1, 2>(A, st) : launch_quad_k<REV, 8, CY, CZ, 4, 3>(A, st);
        case 404: return A.hw == 2 ? launch_quad_k<REV, 8, CY, CZ, 4, 4, 1, 2>(A, st) : launch_quad_k<REV, 8, CY, CZ, 4, 4>(A, st);
        case 803: return launch_quad_k<REV, 8, CY, CZ, 8, 3>(A, st);
        case 1602: return launch_quad_k<REV, 8, CY, CZ, 16, 2>(A, st);
        default:
            switch (A.pf * 10 + A.hw) {  // FLIPB200_QUAD_PF, FLIPB200_QUAD_HW
                case 21: return launch_quad_k<REV, 8, CY, CZ, 8, 2, 2, 1>(A, st);
                case 31: return launch_quad_k<REV, 8, CY, CZ, 8, 2, 3, 1>(A, st);
                case 12: return launch_quad_k<REV, 8, CY, CZ, 8, 2, 1, 2>(A, st);
                case 22: return launch_quad_k<REV, 8, CY, CZ, 8, 2, 2, 2>(A, st);
                case 32: return launch_quad_k<REV, 8, CY, CZ, 8, 2, 3, 2>(A, st);
                default: return launch_quad_k<REV, 8, CY, CZ, 8, 2, 1, 1>(A, st);
            }
    }
}

cudaError_t launch_mic_quad(bool rev, const LaneArgs &A0, cudaStream_t st) {
    static const int exp_flags = getenv("FLIPB200_QUAD_EXP") ? atoi(getenv("FLIPB200_QUAD_EXP")) : 0;
    LaneArgs A = A0;
    A.dbg = exp_flags;
    static const int pf = [] {  // global-face prefetch depth (FLIPB200_QUAD_PF)
        const char *e = getenv("FLIPB200_QUAD_PF");
        return e ? atoi(e) : 1;
    }();
    A.pf = pf;
    A.hw = hw_default();
    static const int lag = getenv("FLIPB200_QUAD_LAG") ? atoi(getenv("FLIPB200_QUAD_LAG")) : 0;
    A.lag = lag;
    static const int t0 = getenv("FLIPB200_TRACE_TILE0") ? atoi(getenv("FLIPB200_TRACE_TILE0")) : 0;
    A.trace_t0 = t0;
    int cy, cz;
    quad_cluster_shape(&cy, &cz);
    if (!A.geom.quad || A.geom.TB % cy || A.geom.TC % cz) return cudaErrorNotSupported;
#define QCASE(a, b)                                                                          \
    if (cy == a && cz == b) return rev ? launch_quad_c<true, a, b>(A, st) : launch_quad_c<false, a, b>(A, st);
    QCASE(2, 4)
    QCASE(4, 4)
    QCASE(2, 2)
    QCASE(4, 2)
    QCASE(1, 4)
    QCASE(1, 1)
    QCASE(2, 8)
    QCASE(4, 8)
#undef QCASE
    return cudaErrorNotSupported;
}

// The MIC(0) build on the quad wavefront (forward order): A.src = diag and
// A.precon = pair codes in the lane layout, A.dst = precon (lane layout).
// Only the default shape (8 x 8 threads, 4 x 4 clusters, 8-step chunks).
cudaError_t launch_mic_quad_build(const LaneArgs &A0, cudaStream_t st) {
    LaneArgs A = A0;
    A.dbg = 0;
    A.pf = 1;
    A.hw = hw_default();
    A.trace = nullptr;
    A.ts = nullptr;
    int cy, cz;
    quad_cluster_shape(&cy, &cz);
    if (A.geom.quad != 8 || cy != 4 || cz != 4 || quad_chunks() != 0 || A.geom.TB % 4 || A.geom.TC % 4)
        return cudaErrorNotSupported;
    return A.hw == 2 ? launch_quad_k<false, 8, 4, 4, 8, 2, 1, 2, 1>(A, st)
                     : launch_quad_k<false, 8, 4, 4, 8, 2, 1, 1, 1>(A, st);
}

bool mic_quad_supported(int nsteps) {
    int cy, cz;
    quad_cluster_shape(&cy, &cz);
    const int key = cy * 100 + cz;
    // the default shape / chunking of each tile edge (what launch_quad_c picks)
    if (quad_threads() == 8 && key == 404 && (quad_chunks() == 0 || quad_chunks() == 802))
        return hw_default() == 2 ? quad_fits<8, 4, 4, 8, 2, 2>(nsteps) : quad_fits<8, 4, 4, 8, 2, 1>(nsteps);
    if (quad_threads() == 16 && key == 204)
        return hw_default() == 2 ? quad_fits<16, 2, 4, 2, 3, 2>(nsteps) : quad_fits<16, 2, 4, 2, 3, 1>(nsteps);
    return cy * cz <= 16;  // other (experimental) shapes: the launch reports misfits
}

}  // namespace flip
