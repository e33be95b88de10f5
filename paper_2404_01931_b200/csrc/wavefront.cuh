// wavefront.cuh — per-row arithmetic of the pipelined sweeps (wavefront.cu).
#pragma once
#include "ops.cuh"

namespace flip {

enum WaveMode { WV_MIC_BUILD = 0, WV_MIC_FWD = 1, WV_MIC_BWD = 2, WV_GS = 3 };

#ifndef WAVE_TY
#define WAVE_TY 16
#endif
#ifndef WAVE_TZ
#define WAVE_TZ 16
#endif

// "Not yet written" marker pre-filled into the halo buffers.  A NaN with a
// payload IEEE arithmetic never produces (hardware NaNs are canonical), so a
// consumer reading one 8-byte word sees either the marker or the final value:
// the data is its own ready flag and no fences are needed.
constexpr unsigned long long WAVE_PENDING = 0x7FF4DEAD5EED0001ULL;
// Entry of the lane-major layout that holds no row (k_lane_map).
constexpr unsigned long long WAVE_ABSENT = 0x7FF4DEAD5EED0002ULL;

// Per-cell sweep flags (built once per assembly, k_cell_flags).
constexpr unsigned char CF_ROW = 1;                                      // cell is a row
constexpr unsigned char CF_PX = 2, CF_PY = 4, CF_PZ = 8;                 // +x/+y/+z is a row
constexpr unsigned char CF_MX = 16, CF_MY = 32, CF_MZ = 64;              // -x/-y/-z is a row

struct WaveGeom {
    int ilo, ihi, jlo, jhi, klo, khi;  // bounding box of the rows
    int TB, TC;                         // tiles along y and z
    int ty, tz;                         // tile shape
    int nsteps;                         // x span + ty + tz - 2
    int ispan;                          // ihi - ilo + 1
    int ispan_pad;                      // ispan rounded up to even (halo lane stride)
    int quad = 0;                       // 1: k_mic_quad geometry (2 x 2 pencils per thread)
};

struct WaveArgs {
    Dims d;
    WaveGeom geom;
    const int *rowscan;          // exclusive scan of isrow (ncells + 1)
    const unsigned char *cflags; // per-cell CF_* flags
    int64_t n;                   // rows
    const double *diag, *rhs, *src, *precon;
    double *dst;                 // output row vector
    double *halo_y, *halo_z;     // [tile][lane][ispan] boundary values
    double scale, tau, sigma;
    int *ticket;
    const DevScalars *sc;        // early exit when sc->done (PCG after convergence)
    unsigned long long *trace;   // optional [tile][4]: start ns, end ns, spin cycles, b|c
};

// Spin with exponential backoff: every poll is an L2 round trip that sits in
// the SM's in-order load-completion queue ahead of the other warps' loads,
// so hammering it slows the whole SM.
__device__ __forceinline__ double poll_ready(const double *p) {
    unsigned long long v;
    unsigned ns = 20;
    while (true) {
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
        if (v != WAVE_PENDING) break;
        __nanosleep(ns);
        ns = ns < 320 ? ns * 2 : ns;
    }
    return __longlong_as_double((long long)v);
}

__device__ __forceinline__ double poll_spin(const double *p) {
    unsigned long long v;
    do {
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    } while (v == WAVE_PENDING);
    return __longlong_as_double((long long)v);
}

__device__ __forceinline__ double ld_relaxed(const double *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return __longlong_as_double((long long)v);
}

// Weak (non-.STRONG) variants for timing experiments: the load never
// allocates in L1, so every execution still reads the L2 copy.
__device__ __forceinline__ double ld_na(const double *p) {
    unsigned long long v;
    asm volatile("ld.global.L1::no_allocate.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return __longlong_as_double((long long)v);
}

__device__ __forceinline__ void publish_weak(double *p, double v) {
    asm volatile("st.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v)) : "memory");
}

__device__ __forceinline__ void publish(double *p, double v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v))
                 : "memory");
}

__device__ __forceinline__ bool present(double v) {
    return (unsigned long long)__double_as_longlong(v) != WAVE_ABSENT;
}

__device__ __forceinline__ bool is_pending(double v) {
    return (unsigned long long)__double_as_longlong(v) == WAVE_PENDING;
}

// ---- bulk-copy (TMA engine, non-tensor) + mbarrier helpers -----------------
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// global -> shared bulk copy, completion counted on *bar (bytes % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes,
                                         unsigned long long *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// L2 prefetch of [src, src + bytes) by the bulk-copy engine (bytes % 16 == 0)
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Lane-major MIC(0) substitution arguments (k_mic_lane).
struct LaneArgs {
    WaveGeom geom;
    const double *src;     // L layout; ABSENT at non-row entries
    const double *precon;  // L layout
    double *dst;           // L layout (only row entries written)
    double *halo_y, *halo_z;
    double scale;
    int *ticket;
    const DevScalars *sc;
    unsigned long long *trace;  // optional per-step clock of tile 0 lane 0
    int dbg;                    // traced tile index (FLIPB200_LANE_DBG, with FLIPB200_WAVE_TRACE)
    int prepped = 0;            // quad: halo + ticket already reset (by k_pcg_update)
    int pf = 1;                 // quad: face values loaded ahead by the helper warp
    int hw = 1;                 // quad: helper warps (2: one per face)
    int lag = 0;                // quad: extra start lag behind cross-cluster producers
    int trace_t0 = 0;           // quad trace: first of the 8 tiles with per-step stamps
    // probe (quad): per-launch [first CTA start, last CTA end] %globaltimer
    // stamps, starts at ts[slot], ends at ts[kProbeSlots + slot], slot =
    // 2 * iteration + direction
    unsigned long long *ts = nullptr;
};
constexpr int kProbeSlots = 1024;

// Reset of the quad sweeps' cross-cluster halo slots and tickets, folded
// into the kernel that precedes the forward sweep (k_pcg_update) instead of
// one k_wave_prep_cl launch per sweep.  Buffer 0 serves the forward sweep,
// buffer 1 the backward one (k_wave_prep_cl's slot selection with rev 0/1).
struct HaloReset {
    double *hy[2];
    int *ticket[2];
    int TB, TC, nsteps, W, cy, cz;
    int on;
};
__device__ __forceinline__ void halo_reset(const HaloReset &H, int64_t tid, int64_t stride) {
    if (!H.on) return;
    if (tid == 0) {
        *H.ticket[0] = 0;
        *H.ticket[1] = 0;
    }
    const double m = __longlong_as_double((long long)WAVE_PENDING);
    const int64_t tiles = (int64_t)H.TB * H.TC;
    const int64_t yrow = (int64_t)H.TC * H.nsteps * H.W;
    const int64_t ny = (int64_t)(H.TB / H.cy) * yrow;
    const int64_t ztile = (int64_t)H.nsteps * H.W;
    const int64_t nzs = (int64_t)H.TB * (H.TC / H.cz) * ztile;
    for (int64_t e = tid; e < 2 * (ny + nzs); e += stride) {
        const int rev = e >= ny + nzs;
        const int64_t f0 = rev ? e - (ny + nzs) : e;
        double *hy = rev ? H.hy[1] : H.hy[0];
        double *hz = hy + tiles * H.nsteps * H.W;
        if (f0 < ny) {
            const int64_t q = f0 / yrow;
            const int64_t b = rev ? q * H.cy : q * H.cy + H.cy - 1;
            hy[b * yrow + f0 % yrow] = m;
        } else {
            const int64_t f = f0 - ny, t = f / ztile;
            const int64_t b = t / (H.TC / H.cz), qc = t % (H.TC / H.cz);
            const int64_t c = rev ? qc * H.cz : qc * H.cz + H.cz - 1;
            hz[(b * H.TC + c) * ztile + f % ztile] = m;
        }
    }
}

cudaError_t launch_wave(int mode, const WaveArgs &A, cudaStream_t st);
// wavequad.cu: 2 x 2 pencils per thread (FLIPB200_QUAD=0 disables)
bool mic_quad_enabled();
bool mic_quad_supported(int nsteps);
int quad_cluster_shape(int *cy, int *cz);
WaveGeom quad_geom(const int lo[3], const int hi[3]);
cudaError_t launch_mic_quad(bool rev, const LaneArgs &A, cudaStream_t st);
cudaError_t launch_mic_quad_build(const LaneArgs &A, cudaStream_t st);
__global__ void k_wave_prep_cl(double *halo_y, double *halo_z, int TB, int TC, int nsteps, int ty,
                               int tz, int cy, int cz, int rev, int *ticket, const DevScalars *sc);
__global__ void k_wave_prep(double *halo, int64_t nh, int *ticket, const DevScalars *sc);
cudaError_t launch_mic_lane(bool rev, const LaneArgs &A, cudaStream_t st);
cudaError_t launch_mic_lane_build(const LaneArgs &A, cudaStream_t st);
// wavecl.cu: cluster/DSMEM variant (FLIPB200_CLUSTER=CYxCZ); NotSupported if off
cudaError_t launch_mic_cluster(bool rev, const LaneArgs &A, cudaStream_t st);
int mic_cluster_pad(int *cy, int *cz);
int64_t lane_entries(const WaveGeom &g);
int64_t lane_entries_max(int64_t nx, int64_t ny, int64_t nz);
void launch_lane_map(const WaveGeom &g, const Dims &d, const uint8_t *isrow, const int *rowscan,
                     int *lrow, int *posL, double *absent1, double *absent2, cudaStream_t st);
void launch_rows_to_lane(const double *v, const int *posL, int64_t n, double *L,
                         const DevScalars *sc, cudaStream_t st);
void launch_lane_to_rows(const double *L, const int *posL, int64_t n, double *v,
                         const DevScalars *sc, cudaStream_t st);
WaveGeom wave_geom(const int lo[3], const int hi[3]);
int64_t wave_halo_doubles(int64_t nx, int64_t ny, int64_t nz);
void launch_cell_flags(const Dims &d, const uint8_t *isrow, unsigned char *cflags,
                       cudaStream_t st);

}  // namespace flip
