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
constexpr unsigned long long WAVE_ABSENT = 0x7FF4DEAD5EED0002ULL;

__device__ __forceinline__ bool present(double v) {
    return (unsigned long long)__double_as_longlong(v) != WAVE_ABSENT;
}

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

// halo <- pending marker, ticket <- 0 (skipped after PCG convergence)
__global__ void k_wave_prep(double *halo, int64_t nh, int *ticket, const DevScalars *sc) {
    if (sc && sc->done) return;
    if (gtid() == 0) *ticket = 0;
    double m = __longlong_as_double((long long)WAVE_PENDING);
    for (int64_t i = gtid(); i < nh; i += gstride()) halo[i] = m;
}

// CF_* flags per cell from the row mask (pressure rows = unpinned FLUID).
__global__ void k_cell_flags(Dims d, const uint8_t *__restrict__ isrow,
                             unsigned char *__restrict__ cf) {
    int64_t nc = d.ncells(), sy = d.nx, sz = (int64_t)d.nx * d.ny;
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        int i = (int)(c % d.nx), j = (int)((c / d.nx) % d.ny), k = (int)(c / sz);
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
static const TileShape kShapes[] = {{16, 8}, {16, 16}, {32, 8}, {8, 8}, {32, 4}};

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
    int64_t tiles = (ny / t.ty + 2) * (nz / t.tz + 2);
    return tiles * (t.ty + t.tz) * (nx + 2) + 64;
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
    g.ispan = hi[0] - lo[0] + 1;
    g.ispan_pad = (g.ispan + 1) & ~1;
    g.nsteps = g.ispan + (t.ty - 1) + (t.tz - 1);
    return g;
}

}  // namespace flip
