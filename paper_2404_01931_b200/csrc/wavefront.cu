// wavefront.cu — pipelined hyperplane wavefront for the sequential row
// sweeps of the pressure solve on assembled (grid-structured) systems:
//   MIC(0) build  (_kernels/_core.pyx:275-308)
//   MIC(0) forward / backward substitution (_core.pyx:311-347)
//   lexicographic Gauss-Seidel (_core.pyx:237-252)
//
// Row r (cell i,j,k) reads only its -x/-y/-z rows (forward kinds) or its
// +x/+y/+z rows (backward), so the reference's sequential loop is reproduced
// exactly by any schedule that finishes a row's predecessors first; every
// row then performs the reference's arithmetic in the reference's order.
//
// Schedule.  A CTA owns a TY x TZ tile of x-pencils (one thread per pencil)
// spanning the rows' x range.  Thread (jj,kk) visits cell i = ilo+s-jj-kk at
// step s (mirrored for the backward sweep), so inside a tile the y/z
// predecessor was produced one step earlier by the neighbouring thread and
// arrives through shared memory (one __syncthreads per step); the x
// predecessor stays in a register.  Values crossing a tile face go through
// halo buffers indexed by (tile, lane, x): pre-filled with a pending-NaN
// marker, written once per sweep with one 8-byte store, so the consumer
// spins on exactly the word it needs — no counters, no fences.  Tiles are
// claimed in anti-diagonal order from an atomic ticket: a tile only waits on
// tiles already running, so any residency is deadlock-free.
//
// Latency hiding.  Every address a step needs is a function of the step
// index (cell -> rowscan/flags, row -> operands, (tile,lane,x) -> halo), so
// a two-level prefetch ring (level 1 two rounds ahead, level 2 one round
// ahead) is held in registers indexed statically inside an unrolled loop:
// no register is ever moved before its load has had U steps to land.
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "ops.cuh"
#include "wavefront.cuh"

namespace flip {

// tile ticket -> (b, c) in anti-diagonal order (b + c ascending, then b)
__device__ __forceinline__ void ticket_tile(int t, int TB, int TC, int &b, int &c) {
    int d = 0;
    while (true) {
        int blo = max(0, d - (TC - 1)), bhi = min(TB - 1, d);
        int cnt = bhi - blo + 1;
        if (t < cnt) {
            b = blo + t;
            c = d - b;
            return;
        }
        t -= cnt;
        d++;
    }
}

constexpr int U = 4;  // steps per unrolled round (prefetch distance U / 2U)
constexpr int LANE_NB = 3;  // k_mic_lane2 operand chunk ring depth

template <int MODE, int TY, int TZ>
__global__ void __launch_bounds__(TY *TZ) k_wave(WaveArgs A) {
    constexpr bool REV = (MODE == WV_MIC_BWD);  // backward substitution runs high -> low
    // sweep-direction predecessor flags in the per-cell CF_* word
    constexpr unsigned char PX = REV ? CF_PX : CF_MX, PY = REV ? CF_PY : CF_MY,
                            PZ = REV ? CF_PZ : CF_MZ;
    __shared__ double sval[2][TZ][TY];
    __shared__ unsigned char sflag[2][TZ][TY];
    __shared__ int s_tile;
    __shared__ unsigned long long s_spin;
    const int jj = threadIdx.x % TY, kk = threadIdx.x / TY;
    if (A.sc && A.sc->done) return;
    const WaveGeom G = A.geom;
    const Dims d = A.d;
    const int64_t sy = d.nx, sz = (int64_t)d.nx * d.ny;
    unsigned long long t_start = 0;
    if (threadIdx.x == 0) {
        s_tile = atomicAdd(A.ticket, 1);
        s_spin = 0;
        if (A.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    }
    __syncthreads();
    int b, c;
    ticket_tile(s_tile, G.TB, G.TC, b, c);
    const int tile = b * G.TC + c;
    const int j = REV ? G.jhi - (b * TY + jj) : G.jlo + b * TY + jj;
    const int k = REV ? G.khi - (c * TZ + kk) : G.klo + c * TZ + kk;
    const bool valid = j >= G.jlo && j <= G.jhi && k >= G.klo && k <= G.khi;
    const int64_t c0 = (int64_t)j * sy + (int64_t)k * sz;  // cell (0, j, k)
    const int64_t ny_off = REV ? sy : -sy, nz_off = REV ? sz : -sz;
    // halo lanes: I write mine if I sit on the tile's far face; I read the
    // predecessor tile's if I sit on the near face
    double *hy_out = (jj == TY - 1) ? A.halo_y + ((int64_t)tile * TZ + kk) * G.ispan_pad : nullptr;
    double *hz_out = (kk == TZ - 1) ? A.halo_z + ((int64_t)tile * TY + jj) * G.ispan_pad : nullptr;
    const double *hy_in =
        (jj == 0 && b > 0) ? A.halo_y + ((int64_t)(tile - G.TC) * TZ + kk) * G.ispan_pad : nullptr;
    const double *hz_in =
        (kk == 0 && c > 0) ? A.halo_z + ((int64_t)(tile - 1) * TY + jj) * G.ispan_pad : nullptr;

    // ---- two-level prefetch ring ----
    unsigned char l1f[U];
    bool l1in[U];  // step's cell inside the box (arithmetic, not loaded)
    int l1r[U];
    unsigned char l1fy[U], l1fz[U];  // BUILD: predecessor cells' flags
    int l1ox[U], l1oy[U], l1oz[U];   // GS: rows of the +x/+y/+z cells
    unsigned char l2f[U];
    int l2r[U];
    double l2a[U], l2b[U], l2hy[U], l2hz[U];
    unsigned char l2fy[U], l2fz[U];
    double l2ox[U], l2oy[U], l2oz[U];

    auto step_i = [&](int s) { return REV ? G.ihi - (s - jj - kk) : G.ilo + s - jj - kk; };
    // Level 1 never branches on the data it loads (that would stall the step
    // on a full memory latency): every load is issued unconditionally with a
    // clamped in-range address and only interpreted U steps later.
    const int64_t ncl = d.ncells() - 1;
    auto load1 = [&](int s, int u) {
        int i = step_i(s);
        bool in = valid && i >= G.ilo && i <= G.ihi;
        int64_t cell = in ? c0 + i : 0;
        l1f[u] = A.cflags[cell];  // raw: masked with l1in one round later
        l1in[u] = in;
        l1r[u] = A.rowscan[cell];
        if (MODE == WV_MIC_BUILD) {
            l1fy[u] = jj == 0 ? A.cflags[min(max(cell + ny_off, (int64_t)0), ncl)] : 0;
            l1fz[u] = kk == 0 ? A.cflags[min(max(cell + nz_off, (int64_t)0), ncl)] : 0;
        }
        if (MODE == WV_GS) {
            l1ox[u] = A.rowscan[min(cell + 1, ncl)];
            l1oy[u] = A.rowscan[min(cell + sy, ncl)];
            l1oz[u] = A.rowscan[min(cell + sz, ncl)];
        }
    };
    auto load2 = [&](int s, int u) {  // uses l1[u], which holds step s
        unsigned char f = l1in[u] ? l1f[u] : 0;
        l2f[u] = f;
        if (f & CF_ROW) {
            int row = l1r[u];
            l2r[u] = row;
            int x = step_i(s) - G.ilo;
            if (MODE == WV_MIC_FWD || MODE == WV_MIC_BWD) {
                l2a[u] = A.src[row];
                l2b[u] = A.precon[row];
            } else if (MODE == WV_MIC_BUILD) {
                l2a[u] = A.diag[row];
                l2fy[u] = l1fy[u];
                l2fz[u] = l1fz[u];
            } else {
                l2a[u] = A.rhs[row];
                l2b[u] = A.diag[row];
                if (f & CF_PX) l2ox[u] = A.src[l1ox[u]];
                if (f & CF_PY) l2oy[u] = A.src[l1oy[u]];
                if (f & CF_PZ) l2oz[u] = A.src[l1oz[u]];
            }
            if (hy_in && (f & PY)) l2hy[u] = ld_relaxed(hy_in + x);
            if (hz_in && (f & PZ)) l2hz[u] = ld_relaxed(hz_in + x);
        }
    };

#pragma unroll
    for (int u = 0; u < U; u++) load1(u, u);
#pragma unroll
    for (int u = 0; u < U; u++) load2(u, u);
#pragma unroll
    for (int u = 0; u < U; u++) load1(U + u, u);

    unsigned char pfl = 0;  // x predecessor: published flag / value
    double pv = 0.0;
    const double sc = A.scale;
    const int nsteps = G.nsteps;
    for (int s0 = 0; s0 < nsteps; s0 += U) {
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int s = s0 + u;
            if (s >= nsteps) break;  // uniform across the block
            __syncthreads();         // neighbours' step s-1 values are in shared memory
            const int cur = s & 1, prv = cur ^ 1;
            unsigned char ofl = 0;
            double ov = 0.0;
            const unsigned char f = l2f[u];
            if (f & CF_ROW) {
                const int row = l2r[u];
                const int x = step_i(s) - G.ilo;
                // y / z predecessors (flag 0 = not a row)
                unsigned char yfl = 0, zfl = 0;
                double yv = 0.0, zv = 0.0;
                if (f & PY) {
                    if (jj > 0) {
                        yfl = sflag[prv][kk][jj - 1];
                        yv = sval[prv][kk][jj - 1];
                    } else {
                        yv = l2hy[u];
                        if (is_pending(yv)) {
                            long long t0 = clock64();
                            yv = poll_ready(hy_in + x);
                            if (A.trace) atomicAdd(&s_spin, (unsigned long long)(clock64() - t0));
                        }
                        yfl = MODE == WV_MIC_BUILD ? (unsigned char)(l2fy[u] | CF_ROW) : CF_ROW;
                    }
                }
                if (f & PZ) {
                    if (kk > 0) {
                        zfl = sflag[prv][kk - 1][jj];
                        zv = sval[prv][kk - 1][jj];
                    } else {
                        zv = l2hz[u];
                        if (is_pending(zv)) {
                            long long t0 = clock64();
                            zv = poll_ready(hz_in + x);
                            if (A.trace) atomicAdd(&s_spin, (unsigned long long)(clock64() - t0));
                        }
                        zfl = MODE == WV_MIC_BUILD ? (unsigned char)(l2fz[u] | CF_ROW) : CF_ROW;
                    }
                }
                const bool xrow = (f & PX) != 0;  // == pfl != 0 for valid schedules
                if (MODE == WV_MIC_FWD) {  // _core.pyx:322-332 (published: scale*precon*q)
                    double t = l2a[u];
                    if (xrow) t += pv;
                    if (yfl) t += yv;
                    if (zfl) t += zv;
                    double pr = l2b[u];
                    double q = t * pr;
                    A.dst[row] = q;
                    ov = (sc * pr) * q;
                } else if (MODE == WV_MIC_BWD) {  // _core.pyx:333-346
                    double t = l2a[u];
                    double pr = l2b[u];
                    if (xrow) t += sc * pr * pv;
                    if (yfl) t += sc * pr * yv;
                    if (zfl) t += sc * pr * zv;
                    ov = t * pr;
                    A.dst[row] = ov;
                } else if (MODE == WV_GS) {  // _core.pyx:237-252 (src old x, dst new x)
                    double sum = 0.0;
                    if (xrow) sum += pv;
                    if (f & CF_PX) sum += l2ox[u];
                    if (yfl) sum += yv;
                    if (f & CF_PY) sum += l2oy[u];
                    if (zfl) sum += zv;
                    if (f & CF_PZ) sum += l2oz[u];
                    ov = (l2a[u] / sc + sum) / l2b[u];
                    A.dst[row] = ov;
                } else {  // WV_MIC_BUILD, _core.pyx:291-307
                    double dg = l2a[u];
                    double e = dg * sc;
                    const unsigned char fl3[3] = {pfl, yfl, zfl};
                    const double v3[3] = {pv, yv, zv};
                    const unsigned char o1[3] = {CF_PY, CF_PX, CF_PX}, o2[3] = {CF_PZ, CF_PZ, CF_PY};
#pragma unroll
                    for (int q = 0; q < 3; q++) {
                        if (!fl3[q]) continue;
                        double pq = v3[q];
                        e -= (sc * pq) * (sc * pq);
                        double others = 0.0;
                        if (fl3[q] & o1[q]) others -= sc;
                        if (fl3[q] & o2[q]) others -= sc;
                        e -= A.tau * (-sc) * others * pq * pq;
                    }
                    if (e < A.sigma * dg * sc) e = dg * sc;
                    ov = 1.0 / sqrt(e);
                    A.dst[row] = ov;
                }
                ofl = (unsigned char)(f & (CF_ROW | CF_PX | CF_PY | CF_PZ));
                if (hy_out) publish(hy_out + x, ov);
                if (hz_out) publish(hz_out + x, ov);
            }
            sval[cur][kk][jj] = ov;
            sflag[cur][kk][jj] = ofl;
            pfl = ofl;
            pv = ov;
            load2(s + U, u);
            load1(s + 2 * U, u);
        }
    }
    if (A.trace) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t_end;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            unsigned long long *tr = A.trace + 4 * (int64_t)tile;
            tr[0] = t_start;
            tr[1] = t_end;
            tr[2] = s_spin;
            tr[3] = ((unsigned long long)b << 32) | (unsigned)c;
        }
    }
}

// ---------------------------------------------------------------------------
// Lean kernel for the two hot sweeps, MIC(0) forward (REV=false) and backward
// (REV=true) substitution: 200 launches per 100-iteration solve.
//
// Row bookkeeping uses only the exclusive scan of the row mask: with
// E(t) = rowscan[cell(t) + REV], step t's cell is a row iff E(t+1) - E(t)
// (forward) or E(t) - E(t+1) (backward) is 1, and its row index is E(t)
// (forward) or E(t+1) (backward).  Consecutive steps are consecutive cells,
// so a single int load per step carries everything.  Non-rows publish the
// ABSENT marker (shared memory and halos alike), so a value and its presence
// travel in one 8-byte word and the step body is branch-light.


__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <bool REV, int TY, int TZ>
__global__ void __launch_bounds__(TY *TZ) k_mic_sweep(WaveArgs A) {
    constexpr int HR = 2 * U;  // halo ring (elements) per lane
    __shared__ double sval[2][TZ][TY];
    __shared__ __align__(16) double hyb[TZ][HR];  // y-face prefetch, lanes jj == 0
    __shared__ __align__(16) double hzb[TY][HR];  // z-face prefetch, lanes kk == 0
    __shared__ int s_tile, s_rows;
    const int jj = threadIdx.x % TY, kk = threadIdx.x / TY;
    if (A.sc && A.sc->done) return;
    const WaveGeom G = A.geom;
    const Dims d = A.d;
    if (threadIdx.x == 0) {
        s_tile = atomicAdd(A.ticket, 1);
        s_rows = 0;
    }
    __syncthreads();
    int b, c;
    ticket_tile(s_tile, G.TB, G.TC, b, c);
    const int tile = b * G.TC + c;
    const int j = REV ? G.jhi - (b * TY + jj) : G.jlo + b * TY + jj;
    const int k = REV ? G.khi - (c * TZ + kk) : G.klo + c * TZ + kk;
    const bool valid = j >= G.jlo && j <= G.jhi && k >= G.klo && k <= G.khi;
    const int64_t c0 = (int64_t)j * d.nx + (int64_t)k * d.nx * d.ny;
    const int lane_len = G.ispan_pad;  // halo lane stride (even => 16-byte aligned pairs)
    double *hy_out = (jj == TY - 1) ? A.halo_y + ((int64_t)tile * TZ + kk) * lane_len : nullptr;
    double *hz_out = (kk == TZ - 1) ? A.halo_z + ((int64_t)tile * TY + jj) * lane_len : nullptr;
    const double *hy_in =
        (jj == 0 && b > 0) ? A.halo_y + ((int64_t)(tile - G.TC) * TZ + kk) * lane_len : nullptr;
    const double *hz_in =
        (kk == 0 && c > 0) ? A.halo_z + ((int64_t)(tile - 1) * TY + jj) * lane_len : nullptr;
    const double absent = __longlong_as_double((long long)WAVE_ABSENT);
    if (valid) {
        int r0 = A.rowscan[c0 + G.ilo], r1 = A.rowscan[c0 + G.ihi + 1];
        if (r1 > r0) atomicAdd(&s_rows, r1 - r0);
    }
    __syncthreads();
    if (s_rows == 0) {  // no rows: publish "absent" along my faces and leave
        if (valid)
            for (int x = 0; x < G.ispan; x++) {
                if (hy_out) publish(hy_out + x, absent);
                if (hz_out) publish(hz_out + x, absent);
            }
        return;
    }
    auto step_i = [&](int s) { return REV ? G.ihi - (s - jj - kk) : G.ilo + s - jj - kk; };
    auto e_load = [&](int t) {  // E(t), address clamped to [ilo-1, ihi+1]
        int i = min(max(step_i(t), G.ilo - 1), G.ihi + 1);
        return valid ? A.rowscan[c0 + i + (REV ? 1 : 0)] : 0;
    };
    int e1[U];
    int rowv[U];
    double av[U], bv[U];
    // level 2 for step t (E(t) in e1[u], E(t+1) in e1[(u+1)%U]); halo pairs
    // go to shared memory through cp.async (one commit group per step)
    auto load2 = [&](int t, int u) {
        int ea = e1[u], eb = e1[(u + 1) % U];
        int i = step_i(t);
        bool in = valid && i >= G.ilo && i <= G.ihi;
        bool isrow = in && (REV ? ea - eb : eb - ea) == 1;
        int row = REV ? eb : ea;
        rowv[u] = isrow ? row : -1;
        int rr = isrow ? row : 0;
        av[u] = A.src[rr];
        bv[u] = A.precon[rr];
        int x = i - G.ilo;
        // first element of a 16-byte pair in sweep order, or the lane's first step
        bool first = in && (((x & 1) == (REV ? 1 : 0)) || x == (REV ? G.ispan - 1 : 0));
        if (first) {
            int pb = x & ~1;
            if (hy_in) cp_async16(&hyb[kk][pb % HR], hy_in + pb);
            if (hz_in) cp_async16(&hzb[jj][pb % HR], hz_in + pb);
        }
        cp_async_commit();
    };
#pragma unroll
    for (int u = 0; u < U; u++) e1[u] = e_load(u);
    {
        int e_u = e_load(U);
#pragma unroll
        for (int u = 0; u < U; u++) {
            int save = e1[(u + 1) % U];
            if (u == U - 1) e1[0] = e_u;
            load2(u, u);
            if (u == U - 1) e1[0] = save;
        }
    }
#pragma unroll
    for (int u = 0; u < U; u++) e1[u] = e_load(U + u);

    double pv = absent;
    const double sc = A.scale;
    double *const dst = A.dst;
    const int nsteps = G.nsteps;
    for (int s0 = 0; s0 < nsteps; s0 += U) {
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int s = s0 + u;
            if (s >= nsteps) break;  // uniform
            __syncthreads();
            const int cur = s & 1, prv = cur ^ 1;
            const int row = rowv[u];
            const int x = step_i(s) - G.ilo;
            double out = absent;
            if (row >= 0) {
                double yv = absent, zv = absent;
                if (jj > 0) {
                    yv = sval[prv][kk][jj - 1];
                } else if (hy_in) {
                    cp_async_wait<U - 1>();
                    yv = hyb[kk][x % HR];
                    if (is_pending(yv)) yv = poll_ready(hy_in + x);
                }
                if (kk > 0) {
                    zv = sval[prv][kk - 1][jj];
                } else if (hz_in) {
                    cp_async_wait<U - 1>();
                    zv = hzb[jj][x % HR];
                    if (is_pending(zv)) zv = poll_ready(hz_in + x);
                }
                const double a = av[u], pr = bv[u];
                if (!REV) {  // _core.pyx:322-332; publishes scale*precon*q
                    double t = a;
                    if (present(pv)) t += pv;
                    if (present(yv)) t += yv;
                    if (present(zv)) t += zv;
                    double q = t * pr;
                    dst[row] = q;
                    out = (sc * pr) * q;
                } else {  // _core.pyx:333-346
                    double t = a;
                    const double sp = sc * pr;
                    if (present(pv)) t += sp * pv;
                    if (present(yv)) t += sp * yv;
                    if (present(zv)) t += sp * zv;
                    out = t * pr;
                    dst[row] = out;
                }
            }
            sval[cur][kk][jj] = out;
            pv = out;
            if ((hy_out || hz_out) && x >= 0 && x < G.ispan && valid) {
                if (hy_out) publish(hy_out + x, out);
                if (hz_out) publish(hz_out + x, out);
            }
            load2(s + U, u);
            e1[u] = e_load(s + 2 * U);
        }
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// Lane-major MIC(0) substitution (the production sweep).  Operands live in a
// skewed tile-major layout L[tile][step][lane]: entry (t, s, p) is the cell
// lane p of tile t visits at forward step s (i = ilo + s - jj - kk).  A CTA
// step therefore reads/writes one contiguous TY*TZ*8-byte block per array
// (fully coalesced), instead of one cache line per lane.  The backward sweep
// visits the same entries in reverse step order with the same lanes
// (s' = nsteps-1-s), so one layout serves both sweeps.  Non-row cells hold
// the ABSENT marker in the input vector: row-ness comes with the data.
template <bool REV, int TY, int TZ>
__global__ void __launch_bounds__(TY *TZ) k_mic_lane(LaneArgs A) {
    constexpr int TP = TY * TZ;
    constexpr int HR = 2 * U;
    __shared__ double sval[2][TZ][TY];
    __shared__ __align__(16) double hyb[TZ][HR];
    __shared__ __align__(16) double hzb[TY][HR];
    __shared__ int s_tile;
    const int p = threadIdx.x, jj = p % TY, kk = p / TY;
    if (A.sc && A.sc->done) return;
    const WaveGeom G = A.geom;
    if (p == 0) s_tile = atomicAdd(A.ticket, 1);
    __syncthreads();
    int b, c;
    ticket_tile(s_tile, G.TB, G.TC, b, c);
    if (REV) {  // backward: far corner first, same tile partition
        b = G.TB - 1 - b;
        c = G.TC - 1 - c;
    }
    const int tile = b * G.TC + c;
    const int nsteps = G.nsteps;
    const int64_t base = (int64_t)tile * nsteps * TP + p;
    const double *srcL = A.src + base;
    const double *preL = A.precon + base;
    double *dstL = A.dst + base;
    const int LL = G.ispan_pad;
    // faces: forward consumes -y/-z and produces +y/+z; backward the reverse
    double *hy_out = REV ? (jj == 0 ? A.halo_y + ((int64_t)tile * TZ + kk) * LL : nullptr)
                         : (jj == TY - 1 ? A.halo_y + ((int64_t)tile * TZ + kk) * LL : nullptr);
    double *hz_out = REV ? (kk == 0 ? A.halo_z + ((int64_t)tile * TY + jj) * LL : nullptr)
                         : (kk == TZ - 1 ? A.halo_z + ((int64_t)tile * TY + jj) * LL : nullptr);
    const double *hy_in =
        REV ? ((jj == TY - 1 && b + 1 < G.TB) ? A.halo_y + ((int64_t)(tile + G.TC) * TZ + kk) * LL : nullptr)
            : ((jj == 0 && b > 0) ? A.halo_y + ((int64_t)(tile - G.TC) * TZ + kk) * LL : nullptr);
    const double *hz_in =
        REV ? ((kk == TZ - 1 && c + 1 < G.TC) ? A.halo_z + ((int64_t)(tile + 1) * TY + jj) * LL : nullptr)
            : ((kk == 0 && c > 0) ? A.halo_z + ((int64_t)(tile - 1) * TY + jj) * LL : nullptr);
    const bool y_local = REV ? jj + 1 < TY : jj > 0;
    const bool z_local = REV ? kk + 1 < TZ : kk > 0;
    const int yj = REV ? jj + 1 : jj - 1, zk = REV ? kk + 1 : kk - 1;
    const double absent = __longlong_as_double((long long)WAVE_ABSENT);
    const int jrow = G.jlo + b * TY + jj, krow = G.klo + c * TZ + kk;
    const bool valid = jrow <= G.jhi && krow <= G.khi;

    auto lstep = [&](int s) { return REV ? nsteps - 1 - s : s; };  // layout step
    auto xof = [&](int s) { return lstep(s) - jj - kk; };          // i - ilo
    double av[U], bv[U];
    auto load = [&](int s, int u) {
        int sl = min(lstep(s), nsteps - 1);
        sl = max(sl, 0);
        av[u] = srcL[(int64_t)sl * TP];
        bv[u] = preL[(int64_t)sl * TP];
        int x = xof(s);
        bool in = valid && s < nsteps && x >= 0 && x < G.ispan;
        bool first = in && (((x & 1) == (REV ? 1 : 0)) || x == (REV ? G.ispan - 1 : 0));
        if (first) {
            int pb = x & ~1;
            if (hy_in) cp_async16(&hyb[kk][pb % HR], hy_in + pb);
            if (hz_in) cp_async16(&hzb[jj][pb % HR], hz_in + pb);
        }
        cp_async_commit();
    };
#pragma unroll
    for (int u = 0; u < U; u++) load(u, u);

    double pv = absent;
    const double sc = A.scale;
    for (int s0 = 0; s0 < nsteps; s0 += U) {
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int s = s0 + u;
            if (s >= nsteps) break;  // uniform
            __syncthreads();
            if (A.trace && tile == 0 && p == 0 && s < 256) A.trace[s] = (unsigned long long)clock64();
            const int cur = s & 1, prv = cur ^ 1;
            const double a = av[u], pr = bv[u];
            const int x = xof(s);
            double out = absent;
            if (present(a) && valid && x >= 0 && x < G.ispan) {
                double yv = absent, zv = absent;
                if (y_local) {
                    yv = sval[prv][kk][yj];
                } else if (hy_in) {
                    cp_async_wait<U - 1>();
                    yv = hyb[kk][x % HR];
                    if (is_pending(yv)) yv = poll_ready(hy_in + x);
                }
                if (z_local) {
                    zv = sval[prv][zk][jj];
                } else if (hz_in) {
                    cp_async_wait<U - 1>();
                    zv = hzb[jj][x % HR];
                    if (is_pending(zv)) zv = poll_ready(hz_in + x);
                }
                if (!REV) {  // _core.pyx:322-332; publishes scale*precon*q
                    double t = a;
                    if (present(pv)) t += pv;
                    if (present(yv)) t += yv;
                    if (present(zv)) t += zv;
                    double q = t * pr;
                    dstL[(int64_t)lstep(s) * TP] = q;
                    out = (sc * pr) * q;
                } else {  // _core.pyx:333-346
                    double t = a;
                    const double sp = sc * pr;
                    if (present(pv)) t += sp * pv;
                    if (present(yv)) t += sp * yv;
                    if (present(zv)) t += sp * zv;
                    out = t * pr;
                    dstL[(int64_t)lstep(s) * TP] = out;
                }
            }
            sval[cur][kk][jj] = out;
            pv = out;
            if ((hy_out || hz_out) && valid && x >= 0 && x < G.ispan) {
                if (hy_out) publish(hy_out + x, out);
                if (hz_out) publish(hz_out + x, out);
            }
            load(s + U, u);
        }
    }
    cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// k_mic_lane2: warp-specialised lane-major MIC(0) substitution.
//
// Warps 0..TP/32-1 compute; one extra helper warp owns every cross-tile
// transfer, so the compute body is branch-light and never touches a halo.
// Absent neighbours (not a row, outside the box) are encoded as -0.0: for any
// t, t + (-0.0) == t bit for bit (IEEE), and in the backward sweep the
// multiplier scale*precon is strictly positive so (sp * -0.0) == -0.0 too —
// the reference's "if nb >= 0: t += ..." is reproduced exactly with no test.
// Shared exchange sval[slot][TZ+2][TY+2]: lane (jj,kk) lives at [kk+1][jj+1];
// the predecessor tile's face values land in the border row/column, written
// by the helper one step ahead.
template <bool REV, int TY, int TZ, int U, int KC>
__global__ void __launch_bounds__(TY *TZ + 32) k_mic_lane2(LaneArgs A) {
    constexpr int TP = TY * TZ;
    static_assert(TY + TZ <= 32, "one helper warp covers both faces");
    __shared__ double sval[2][TZ + 2][TY + 2];
    __shared__ int s_tile;
    const int t = threadIdx.x;
    if (A.sc && A.sc->done) return;
    const WaveGeom G = A.geom;
    unsigned long long t_start = 0;
    if (t == 0) {
        s_tile = atomicAdd(A.ticket, 1);
        if (A.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    }
    const double nz0 = -0.0;
    for (int q = t; q < 2 * (TZ + 2) * (TY + 2); q += blockDim.x) (&sval[0][0][0])[q] = nz0;
    __syncthreads();
    int b, c;
    ticket_tile(s_tile, G.TB, G.TC, b, c);
    if (REV) {
        b = G.TB - 1 - b;
        c = G.TC - 1 - c;
    }
    const int tile = b * G.TC + c;
    const int nsteps = G.nsteps;
    auto lstep = [&](int s) { return REV ? nsteps - 1 - s : s; };

    if (t >= TP) {
        // ------------------------------ helper warp ------------------------
        // Halo layout is step-major: face[tile][step][lane] holds the boundary
        // lane's output at that step.  A consumer at step s needs its
        // predecessor's step s + D (D = TY-1 across a y face, TZ-1 across a z
        // face, in both sweep directions), so every publish and every fetch is
        // one contiguous 16-lane access.
        const int l = t - TP;
        // lanes [0,TZ): y face, lane kk; lanes [TZ,TZ+TY): z face, lane jj
        const bool yface = l < TZ, zface = l >= TZ && l < TZ + TY;
        const bool active = yface || zface;
        const int kk = yface ? l : 0, jj = zface ? l - TZ : 0;
        const int W = yface ? TZ : TY;       // lanes per face row
        const int D = yface ? TY - 1 : TZ - 1;
        const double *in = nullptr;
        double *out = nullptr;
        int in_row = 0, in_col = 0, out_row = 0, out_col = 0, cons_j = 0, cons_k = 0;
        if (yface) {
            cons_j = REV ? TY - 1 : 0;
            cons_k = kk;
            const bool has = REV ? b + 1 < G.TB : b > 0;
            if (has) in = A.halo_y + (int64_t)(REV ? tile + G.TC : tile - G.TC) * nsteps * TZ + kk;
            out = A.halo_y + (int64_t)tile * nsteps * TZ + kk;
            in_row = kk + 1;
            in_col = REV ? TY + 1 : 0;
            out_row = kk + 1;
            out_col = (REV ? 0 : TY - 1) + 1;
        } else if (zface) {
            cons_j = jj;
            cons_k = REV ? TZ - 1 : 0;
            const bool has = REV ? c + 1 < G.TC : c > 0;
            if (has) in = A.halo_z + (int64_t)(REV ? tile + 1 : tile - 1) * nsteps * TY + jj;
            out = A.halo_z + (int64_t)tile * nsteps * TY + jj;
            in_row = REV ? TZ + 1 : 0;
            in_col = jj + 1;
            out_row = (REV ? 0 : TZ - 1) + 1;
            out_col = jj + 1;
        }
        // a consumer lane outside the box never computes: never wait on its face
        const bool cvalid = G.jlo + b * TY + cons_j <= G.jhi && G.klo + c * TZ + cons_k <= G.khi;
        if (!cvalid) in = nullptr;
        // prefetch ring: ring[u] holds the value consumed at step s0 + u + 1
        double ring[U];
        auto fetch = [&](int s, int u) {
            const int sp = s + D;
            ring[u] = (in && sp < nsteps) ? ld_relaxed(in + (int64_t)sp * W) : nz0;
        };
#pragma unroll
        for (int u = 0; u < U; u++) fetch(u + 1, u);
        if (in) {  // value consumed at step 0 lands in slot 1 (= prv of step 0)
            const double v = D < nsteps ? poll_ready(in + (int64_t)D * W) : nz0;
            sval[1][in_row][in_col] = v;
        }
        for (int s0 = 0; s0 < nsteps; s0 += U) {
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int s = s0 + u;
                if (s >= nsteps) break;
                __syncthreads();
                const int cur = s & 1, prv = cur ^ 1;
                if (active && s > 0) publish(out + (int64_t)(s - 1) * W, sval[prv][out_row][out_col]);
                if (in) {
                    double v = ring[u];
                    if (is_pending(v)) {
                        v = poll_ready(in + (int64_t)(s + 1 + D) * W);
                        if (A.trace && !REV && tile == A.dbg && s < 1000)
                            atomicAdd(&A.trace[16384 + 1024 + s], 1ULL);
                    }
                    sval[cur][in_row][in_col] = v;
                    fetch(s + 1 + U, u);
                }
            }
        }
        // final publish of the last step's output
        __syncthreads();
        if (active) publish(out + (int64_t)(nsteps - 1) * W, sval[(nsteps - 1) & 1][out_row][out_col]);
        return;
    }

    // ------------------------------- compute warps ---------------------------
    const int jj = t % TY, kk = t / TY;
    const int64_t base = (int64_t)tile * nsteps * TP + t;
    double *dstL = A.dst + base;
    const bool valid = G.jlo + b * TY + jj <= G.jhi && G.klo + c * TZ + kk <= G.khi;
    const int yr = kk + 1, yc = REV ? jj + 2 : jj, zr = REV ? kk + 2 : kk, zc = jj + 1;
    double pv = nz0;
    const double sc = A.scale;
    auto body_step = [&](int s, double a, double pr) {
        const int cur = s & 1, prv = cur ^ 1;
        const double yv = sval[prv][yr][yc], zv = sval[prv][zr][zc];
        const bool row = valid && present(a);
        double o;
        if (!REV) {  // _core.pyx:322-332 (absent terms are -0.0: exact no-ops)
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
    };
    if constexpr (KC == 0) {
        const double *srcL = A.src + base;
        const double *preL = A.precon + base;
        double av[U], bv[U];
        auto load = [&](int s, int u) {
            int sl = max(min(lstep(s), nsteps - 1), 0);
            av[u] = srcL[(int64_t)sl * TP];
            bv[u] = preL[(int64_t)sl * TP];
        };
#pragma unroll
        for (int u = 0; u < U; u++) load(u, u);
        for (int s0 = 0; s0 < nsteps; s0 += U) {
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int s = s0 + u;
                if (s >= nsteps) break;
                __syncthreads();
                body_step(s, av[u], bv[u]);
                load(s + U, u);
            }
        }
    } else {
        // operands arrive KC steps at a time through the bulk-copy engine into
        // a LANE_NB-deep smem ring (opb[buf][src|precon][KC][TP]), so the only
        // loads in this SM's LSU queue are the helper's halo polls
        extern __shared__ __align__(128) double opb[];
        __shared__ __align__(8) unsigned long long mbar[LANE_NB];
        const int nch = (nsteps + KC - 1) / KC;
        const int64_t tbase = (int64_t)tile * nsteps * TP;
        auto issue = [&](int ch) {  // thread 0 only
            if (ch >= nch) return;
            const int s0 = ch * KC, cnt = min(KC, nsteps - s0);
            const int lo = REV ? nsteps - s0 - cnt : s0;
            const int buf = ch % LANE_NB;
            const unsigned bytes = (unsigned)(cnt * TP * 8);
            mbar_expect_tx(&mbar[buf], 2 * bytes);
            bulk_g2s(opb + (buf * 2 + 0) * KC * TP, A.src + tbase + (int64_t)lo * TP, bytes,
                     &mbar[buf]);
            bulk_g2s(opb + (buf * 2 + 1) * KC * TP, A.precon + tbase + (int64_t)lo * TP, bytes,
                     &mbar[buf]);
        };
        if (t == 0) {
            for (int q = 0; q < LANE_NB; q++) mbar_init(&mbar[q], 1);
            mbar_fence_init();
            for (int q = 0; q < LANE_NB; q++) issue(q);
        }
        asm volatile("bar.sync 1, %0;" ::"r"(TP) : "memory");  // mbarrier init visible
        for (int ch = 0; ch < nch; ch++) {
            const int s0 = ch * KC, cnt = min(KC, nsteps - s0);
            const int buf = ch % LANE_NB;
            mbar_wait(&mbar[buf], (unsigned)(ch / LANE_NB) & 1u);

            const double *ab = opb + (buf * 2 + 0) * KC * TP + t;
            const double *pb = opb + (buf * 2 + 1) * KC * TP + t;
#pragma unroll
            for (int u = 0; u < KC; u++) {
                if (u >= cnt) break;
                const int s = s0 + u;
                __syncthreads();
                if (u == 0 && ch > 0 && t == 0) {
                    // every thread finished chunk ch-1 before this barrier
                    fence_proxy_async();
                    issue(ch - 1 + LANE_NB);
                }
                if (A.trace && !REV && ch == 0 && u == 0 && t == 0) {
                    // step-0 halo staged: the tile really starts here (LDS orders the stamp)
                    const double d = sval[1][0][0];
                    unsigned long long g;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
                    A.trace[4 * tile + 2] = g + (__double_as_longlong(d) == 1 ? 1 : 0);
                }
                const int idx = REV ? cnt - 1 - u : u;
                body_step(s, ab[idx * TP], pb[idx * TP]);
            }
        }
    }
    __syncthreads();  // matches the helper's final barrier
    if (A.trace && !REV && t == 0) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        A.trace[4 * tile + 0] = t_start;
        A.trace[4 * tile + 1] = g;
        A.trace[4 * tile + 3] = (unsigned long long)(b * 65536 + c);
    }
}

// L-layout maps: lrow[e] = row at entry e (or -1); posL[row] = e.
__global__ void k_lane_map(WaveGeom G, Dims d, int TY, int TZ, const uint8_t *__restrict__ isrow,
                           const int *__restrict__ rowscan, int *__restrict__ lrow,
                           int *__restrict__ posL, double *__restrict__ absent1,
                           double *__restrict__ absent2, int64_t nL) {
    const int TP = TY * TZ;
    const double ab = __longlong_as_double((long long)WAVE_ABSENT);
    for (int64_t e = gtid(); e < nL; e += gstride()) {
        // 32-bit decomposition: lane entries stay below 2^31 (lane_entries_max)
        const unsigned ue = (unsigned)e;
        int p, s, tile;
        if (G.quad) {  // ((tile * nsteps/4 + g) * TP + p) * 4 + w, step 4g + w
            const unsigned r = ue >> 2, tg = r / (unsigned)TP, ng = (unsigned)G.nsteps >> 2;
            p = (int)(r - tg * (unsigned)TP);
            const unsigned tq = tg / ng;
            s = 4 * (int)(tg - tq * ng) + (int)(ue & 3u);
            tile = (int)tq;
        } else {
            const unsigned ts = ue / (unsigned)TP;
            p = (int)(ue - ts * (unsigned)TP);
            const unsigned tq = ts / (unsigned)G.nsteps;
            s = (int)(ts - tq * (unsigned)G.nsteps);
            tile = (int)tq;
        }
        int b = tile / G.TC, c = tile % G.TC;
        int i, j, k;
        if (G.quad) {  // [q][thread]: thread (jj, kk) of QT x QT owns pencils (2jj + a, 2kk + b)
            const int QT = G.quad, QP = QT * QT;
            const int q = p / QP, th = p - q * QP, kk = th / QT, jj = th - kk * QT;
            i = G.ilo + s - jj - kk;
            j = G.jlo + b * TY + 2 * jj + (q & 1);
            k = G.klo + c * TZ + 2 * kk + (q >> 1);
        } else {
            int jj = p % TY, kk = p / TY;
            i = G.ilo + s - jj - kk, j = G.jlo + b * TY + jj, k = G.klo + c * TZ + kk;
        }
        int row = -1;
        if (i >= G.ilo && i <= G.ihi && j <= G.jhi && k <= G.khi) {
            int64_t cell = i + (int64_t)j * d.nx + (int64_t)k * d.nx * d.ny;
            if (isrow[cell]) row = rowscan[cell];
        }
        lrow[e] = row;
        FLIP_CHECK(e < (int64_t)INT_MAX, "lane entry index", e, INT_MAX);
        if (row >= 0) posL[row] = (int)e;
        absent1[e] = ab;
        absent2[e] = ab;
    }
}

// vec (compact rows) -> L layout, and back
__global__ void k_rows_to_lane(const double *__restrict__ v, const int *__restrict__ posL,
                               int64_t n, double *__restrict__ L, const DevScalars *sc) {
    if (sc && sc->done) return;
    for (int64_t r = gtid(); r < n; r += gstride()) L[posL[r]] = v[r];
}
__global__ void k_lane_to_rows(const double *__restrict__ L, const int *__restrict__ posL,
                               int64_t n, double *__restrict__ v, const DevScalars *sc) {
    if (sc && sc->done) return;
    for (int64_t r = gtid(); r < n; r += gstride()) v[r] = L[posL[r]];
}

// halo <- pending marker, ticket <- 0 (skipped after PCG convergence)
__global__ void k_wave_prep(double *halo, int64_t nh, int *ticket, const DevScalars *sc) {
    if (sc && sc->done) return;
    if (gtid() == 0) *ticket = 0;
    double m = __longlong_as_double((long long)WAVE_PENDING);
    for (int64_t i = gtid(); i < nh; i += gstride()) halo[i] = m;
}

// k_wave_prep for the cluster sweep: only tiles that publish across a
// cluster boundary use the global halo (y: tile rows b % cy == cy - 1 going
// forward, b % cy == 0 in reverse; z likewise with columns), a quarter of it
// for 4x4 clusters.  Each selected y row is one contiguous block of the
// step-major halo_y; each selected z tile one block of halo_z.
__global__ void k_wave_prep_cl(double *halo_y, double *halo_z, int TB, int TC, int nsteps, int ty,
                               int tz, int cy, int cz, int rev, int *ticket,
                               const DevScalars *sc) {
    pdl_wait();
    if (sc && sc->done) return;
    if (gtid() == 0) *ticket = 0;
    const double m = __longlong_as_double((long long)WAVE_PENDING);
    const int64_t yrow = (int64_t)TC * nsteps * tz;          // one tile row of halo_y
    const int64_t ny = (int64_t)(TB / cy) * yrow;
    const int64_t ztile = (int64_t)nsteps * ty;              // one tile of halo_z
    const int64_t nz = (int64_t)TB * (TC / cz) * ztile;
    for (int64_t e = gtid(); e < ny + nz; e += gstride()) {
        if (e < ny) {
            const int64_t q = e / yrow;
            const int64_t b = rev ? q * cy : q * cy + cy - 1;
            halo_y[b * yrow + e % yrow] = m;
        } else {
            const int64_t f = e - ny, t = f / ztile;
            const int64_t b = t / (TC / cz), qc = t % (TC / cz);
            const int64_t c = rev ? qc * cz : qc * cz + cz - 1;
            halo_z[(b * TC + c) * ztile + f % ztile] = m;
        }
    }
}

// CF_* flags per cell from the row mask (pressure rows = unpinned FLUID).
__global__ void k_cell_flags(Dims d, const uint8_t *__restrict__ isrow,
                             unsigned char *__restrict__ cf) {
    int64_t nc = d.ncells(), sy = d.nx, sz = (int64_t)d.nx * d.ny;
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        int i, j, k;
        cell_ijk(d, c, i, j, k);
        unsigned char f = 0;
        if (isrow[c]) {
            f = CF_ROW;
            if (i + 1 < d.nx && isrow[c + 1]) f |= CF_PX;
            if (j + 1 < d.ny && isrow[c + sy]) f |= CF_PY;
            if (k + 1 < d.nz && isrow[c + sz]) f |= CF_PZ;
            if (i > 0 && isrow[c - 1]) f |= CF_MX;
            if (j > 0 && isrow[c - sy]) f |= CF_MY;
            if (k > 0 && isrow[c - sz]) f |= CF_MZ;
        }
        cf[c] = f;
    }
}

void launch_cell_flags(const Dims &d, const uint8_t *isrow, unsigned char *cflags,
                       cudaStream_t st) {
    k_cell_flags<<<nblocks(d.ncells()), kThreads, 0, st>>>(d, isrow, cflags);
}

// Tile shapes compiled in; FLIPB200_WAVE_TILE=<ty>x<tz> selects one (tuning).
struct TileShape {
    int ty, tz;
};
static const TileShape kShapes[] = {{16, 8}, {16, 16}, {32, 8}, {8, 8}, {32, 4}, {32, 16}};

static TileShape wave_shape() {
    static TileShape sh = [] {
        TileShape t{WAVE_TY, WAVE_TZ};
        if (const char *e = getenv("FLIPB200_WAVE_TILE")) {
            int a = 0, b = 0;
            if (sscanf(e, "%dx%d", &a, &b) == 2)
                for (auto &k : kShapes)
                    if (k.ty == a && k.tz == b) t = k;
        }
        return t;
    }();
    return sh;
}

int64_t wave_halo_doubles(int64_t nx, int64_t ny, int64_t nz) {
    TileShape t = wave_shape();
    int64_t tiles = (ny / t.ty + 9) * (nz / t.tz + 9);  // + cluster padding
    // k_wave: [tile][lane][x] (x < nx + 2); k_mic_lane2: [tile][step][lane]
    // with steps = x span + ty + tz - 2
    return tiles * (t.ty + t.tz) * (nx + 2 + t.ty + t.tz) + 64;
}

template <int MODE, int TY, int TZ>
static cudaError_t launch_shape(const WaveArgs &A, cudaStream_t st) {
    int64_t tiles = (int64_t)A.geom.TB * A.geom.TC;
    int64_t nh = tiles * (TY + TZ) * A.geom.ispan_pad;  // halo_y then halo_z, contiguous
    k_wave_prep<<<nblocks(nh), kThreads, 0, st>>>(A.halo_y, nh, A.ticket, A.sc);
    static const bool generic = getenv("FLIPB200_WAVE_GENERIC") != nullptr;
    if (MODE == WV_MIC_FWD && !generic)
        k_mic_sweep<false, TY, TZ><<<(unsigned)tiles, TY * TZ, 0, st>>>(A);
    else if (MODE == WV_MIC_BWD && !generic)
        k_mic_sweep<true, TY, TZ><<<(unsigned)tiles, TY * TZ, 0, st>>>(A);
    else
        k_wave<MODE, TY, TZ><<<(unsigned)tiles, TY * TZ, 0, st>>>(A);
    return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_wave_t(const WaveArgs &A, cudaStream_t st) {
    TileShape t = wave_shape();
    if (t.ty == 16 && t.tz == 16) return launch_shape<MODE, 16, 16>(A, st);
    if (t.ty == 32 && t.tz == 8) return launch_shape<MODE, 32, 8>(A, st);
    if (t.ty == 8 && t.tz == 8) return launch_shape<MODE, 8, 8>(A, st);
    if (t.ty == 32 && t.tz == 4) return launch_shape<MODE, 32, 4>(A, st);
    return launch_shape<MODE, 16, 8>(A, st);
}

cudaError_t launch_wave(int mode, const WaveArgs &A, cudaStream_t st) {
    switch (mode) {
        case WV_MIC_BUILD: return launch_wave_t<WV_MIC_BUILD>(A, st);
        case WV_MIC_FWD: return launch_wave_t<WV_MIC_FWD>(A, st);
        case WV_MIC_BWD: return launch_wave_t<WV_MIC_BWD>(A, st);
        default: return launch_wave_t<WV_GS>(A, st);
    }
}

int64_t lane_entries(const WaveGeom &g) { return (int64_t)g.TB * g.TC * g.nsteps * g.ty * g.tz; }

int64_t lane_entries_max(int64_t nx, int64_t ny, int64_t nz) {
    TileShape t = wave_shape();
    // + cluster padding (wave_geom): at most 7 tiles per axis
    return ((ny + t.ty - 1) / t.ty + 7) * ((nz + t.tz - 1) / t.tz + 7) * (nx + t.ty + t.tz) * t.ty *
           t.tz;
}

void launch_lane_map(const WaveGeom &g, const Dims &d, const uint8_t *isrow, const int *rowscan,
                     int *lrow, int *posL, double *absent1, double *absent2, cudaStream_t st) {
    int64_t nL = lane_entries(g);
    k_lane_map<<<nblocks(nL), kThreads, 0, st>>>(g, d, g.ty, g.tz, isrow, rowscan, lrow, posL,
                                                absent1, absent2, nL);
}

void launch_rows_to_lane(const double *v, const int *posL, int64_t n, double *L,
                         const DevScalars *sc, cudaStream_t st) {
    k_rows_to_lane<<<nblocks(n), kThreads, 0, st>>>(v, posL, n, L, sc);
}

void launch_lane_to_rows(const double *L, const int *posL, int64_t n, double *v,
                         const DevScalars *sc, cudaStream_t st) {
    k_lane_to_rows<<<nblocks(n), kThreads, 0, st>>>(L, posL, n, v, sc);
}

// prefetch depth (steps) of k_mic_lane2's operand and halo rings
static int lane_depth() {
    static const int d = [] {
        const char *e = getenv("FLIPB200_LANE_DEPTH");
        return e ? atoi(e) : 4;
    }();
    return d;
}
// operand staging: 1 = bulk-copy chunks into smem (default), 0 = register ring
static int lane_chunk() {
    static const int d = [] {
        const char *e = getenv("FLIPB200_LANE_BULK");
        return e ? atoi(e) : 1;
    }();
    return d;
}

template <bool REV, int TY, int TZ>
static cudaError_t launch_lane_shape(const LaneArgs &A, cudaStream_t st) {
    int64_t tiles = (int64_t)A.geom.TB * A.geom.TC;
    static const bool v1 = getenv("FLIPB200_LANE_V1") != nullptr;
    const bool lane2 = TY + TZ <= 32 && !v1;  // step-major halo (k_mic_lane2 / k_mic_cl)
    int64_t nh = tiles * (TY + TZ) * (lane2 ? (int64_t)A.geom.nsteps : A.geom.ispan_pad);
    static bool cluster_ok = true;
    int cy = 0, cz = 0;
    const bool try_cluster = lane2 && TY == 16 && TZ == 16 && cluster_ok &&
                             mic_cluster_pad(&cy, &cz) && A.geom.TB % cy == 0 &&
                             A.geom.TC % cz == 0;
    static const bool full_prep = getenv("FLIPB200_FULL_HALO_PREP") != nullptr;
    if (try_cluster && !full_prep) {
        const int64_t nsel = (int64_t)(A.geom.TB / cy) * A.geom.TC * A.geom.nsteps * TZ +
                             (int64_t)A.geom.TB * (A.geom.TC / cz) * A.geom.nsteps * TY;
        launch_pdl(k_wave_prep_cl, nblocks(nsel), kThreads, 0, st, A.halo_y,
                   A.halo_y + tiles * A.geom.nsteps * TZ, A.geom.TB, A.geom.TC, A.geom.nsteps, TY,
                   TZ, cy, cz, REV ? 1 : 0, A.ticket, A.sc);
    } else {
        k_wave_prep<<<nblocks(nh), kThreads, 0, st>>>(A.halo_y, nh, A.ticket, A.sc);
    }
    if constexpr (TY + TZ > 32) {
        k_mic_lane<REV, TY, TZ><<<(unsigned)tiles, TY * TZ, 0, st>>>(A);
    } else {
        if (!lane2) {
            k_mic_lane<REV, TY, TZ><<<(unsigned)tiles, TY * TZ, 0, st>>>(A);
            return cudaPeekAtLastError();
        }
        LaneArgs B = A;
        B.halo_z = A.halo_y + tiles * A.geom.nsteps * TZ;
        // DSMEM cluster kernel when its cluster shape can be scheduled here;
        // otherwise (e.g. no 16-CTA clusters on this device) k_mic_lane2 for
        // the rest of the process: same arithmetic, same padded tile grid
        if (TY == 16 && TZ == 16 && cluster_ok) {
            cudaError_t e = launch_mic_cluster(REV, B, st);
            if (e == cudaSuccess) return e;
            if (e != cudaErrorNotSupported) {
                cudaGetLastError();  // a refused launch is not a sticky error
                cluster_ok = false;
                fprintf(stderr, "flipb200: cluster sweep unavailable (%s); using k_mic_lane2\n",
                        cudaGetErrorString(e));
            }
        }
        // k_mic_lane2 reads every tile's halo: the whole of it after a selective prep
        if (try_cluster && !full_prep)
            k_wave_prep<<<nblocks(nh), kThreads, 0, st>>>(A.halo_y, nh, A.ticket, A.sc);
        if (lane_chunk() > 0) {
            constexpr int KC = 8;
            constexpr int smem = LANE_NB * 2 * KC * TY * TZ * 8;
            static bool attr = [] {
                cudaFuncSetAttribute(k_mic_lane2<REV, TY, TZ, 4, KC>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                cudaFuncSetAttribute(k_mic_lane2<REV, TY, TZ, 8, KC>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                cudaFuncSetAttribute(k_mic_lane2<REV, TY, TZ, 16, KC>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                return true;
            }();
            (void)attr;
            if (lane_depth() == 16)
                k_mic_lane2<REV, TY, TZ, 16, KC><<<(unsigned)tiles, TY * TZ + 32, smem, st>>>(B);
            else if (lane_depth() == 8)
                k_mic_lane2<REV, TY, TZ, 8, KC><<<(unsigned)tiles, TY * TZ + 32, smem, st>>>(B);
            else
                k_mic_lane2<REV, TY, TZ, 4, KC><<<(unsigned)tiles, TY * TZ + 32, smem, st>>>(B);
        } else if (lane_depth() == 16)
            k_mic_lane2<REV, TY, TZ, 16, 0><<<(unsigned)tiles, TY * TZ + 32, 0, st>>>(B);
        else if (lane_depth() == 8)
            k_mic_lane2<REV, TY, TZ, 8, 0><<<(unsigned)tiles, TY * TZ + 32, 0, st>>>(B);
        else
            k_mic_lane2<REV, TY, TZ, 4, 0><<<(unsigned)tiles, TY * TZ + 32, 0, st>>>(B);
    }
    return cudaPeekAtLastError();
}

// MIC(0) build on the quad wavefront (launch_mic_quad_build), after the
// forward direction's halo reset (as launch_mic_lane does for a sweep).
cudaError_t launch_mic_lane_build(const LaneArgs &A, cudaStream_t st) {
    if (!A.geom.quad) return cudaErrorNotSupported;
    const int64_t tiles = (int64_t)A.geom.TB * A.geom.TC;
    int cy = 0, cz = 0;
    quad_cluster_shape(&cy, &cz);
    const int QW = A.geom.ty;
    const int64_t nsel = (int64_t)(A.geom.TB / cy) * A.geom.TC * A.geom.nsteps * QW +
                         (int64_t)A.geom.TB * (A.geom.TC / cz) * A.geom.nsteps * QW;
    LaneArgs B = A;
    B.halo_z = A.halo_y + tiles * A.geom.nsteps * QW;
    launch_pdl(k_wave_prep_cl, nblocks(nsel), kThreads, 0, st, A.halo_y, B.halo_z, A.geom.TB,
               A.geom.TC, A.geom.nsteps, QW, QW, cy, cz, 0, A.ticket, (const DevScalars *)nullptr);
    return launch_mic_quad_build(B, st);
}

cudaError_t launch_mic_lane(bool rev, const LaneArgs &A, cudaStream_t st) {
    if (A.geom.quad) {
        // cross-cluster faces only (as k_wave_prep_cl for k_mic_cl), 32 wide
        const int64_t tiles = (int64_t)A.geom.TB * A.geom.TC;
        int cy = 0, cz = 0;
        quad_cluster_shape(&cy, &cz);
        const int QW = A.geom.ty;  // face width
        const int64_t nsel = (int64_t)(A.geom.TB / cy) * A.geom.TC * A.geom.nsteps * QW +
                             (int64_t)A.geom.TB * (A.geom.TC / cz) * A.geom.nsteps * QW;
        LaneArgs B = A;
        B.halo_z = A.halo_y + tiles * A.geom.nsteps * QW;
        if (!A.prepped) launch_pdl(k_wave_prep_cl, nblocks(nsel), kThreads, 0, st, A.halo_y, B.halo_z,
                   A.geom.TB, A.geom.TC, A.geom.nsteps, QW, QW, cy, cz, rev ? 1 : 0, A.ticket,
                   (const DevScalars *)A.sc);
        return launch_mic_quad(rev, B, st);
    }
    TileShape t = wave_shape();
#define LANE_CASE(a, b)                                                                   \
    if (t.ty == a && t.tz == b)                                                           \
        return rev ? launch_lane_shape<true, a, b>(A, st) : launch_lane_shape<false, a, b>(A, st);
    LANE_CASE(16, 16)
    LANE_CASE(32, 8)
    LANE_CASE(8, 8)
    LANE_CASE(32, 4)
    LANE_CASE(32, 16)
#undef LANE_CASE
    return rev ? launch_lane_shape<true, 16, 8>(A, st) : launch_lane_shape<false, 16, 8>(A, st);
}

WaveGeom wave_geom(const int lo[3], const int hi[3]) {
    TileShape t = wave_shape();
    WaveGeom g{};
    g.ilo = lo[0];
    g.ihi = hi[0];
    g.jlo = lo[1];
    g.jhi = hi[1];
    g.klo = lo[2];
    g.khi = hi[2];
    g.ty = t.ty;
    g.tz = t.tz;
    g.TB = (hi[1] - lo[1] + t.ty) / t.ty;
    g.TC = (hi[2] - lo[2] + t.tz) / t.tz;
    int cy, cz;
    if (t.ty == 16 && t.tz == 16 && mic_cluster_pad(&cy, &cz)) {
        // whole clusters of tiles (the padding tiles hold no rows)
        g.TB = (g.TB + cy - 1) / cy * cy;
        g.TC = (g.TC + cz - 1) / cz * cz;
    }
    g.ispan = hi[0] - lo[0] + 1;
    g.ispan_pad = (g.ispan + 1) & ~1;
    g.nsteps = g.ispan + (t.ty - 1) + (t.tz - 1);
    return g;
}

}  // namespace flip
