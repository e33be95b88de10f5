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
// Schedule: a CTA owns a TY x TZ tile of x-pencils (one thread per pencil)
// spanning the rows' full x range.  Thread (jj,kk) handles cell
// i = ilo + s - jj - kk at step s, so inside a tile the -y/-z predecessor
// was produced one step earlier by the neighbouring thread and is passed
// through shared memory; the -x predecessor stays in a register.  Tiles are
// claimed in anti-diagonal order from an atomic ticket, so a tile only ever
// waits for tiles already running (no deadlock for any residency).  A tile
// publishes "steps completed" with a gpu-scope release every PUB steps; its
// +y/+z successors acquire it before reading the boundary values from global
// memory (L2, ld.cg).  The critical path is ~(nx+ny+nz) steps plus a small
// lag per tile hop, instead of one grid-wide barrier per hyperplane.
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "ops.cuh"
#include "wavefront.cuh"

namespace flip {

__device__ __forceinline__ int ld_acquire(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int *p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

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

template <int MODE, int TY, int TZ>
__global__ void __launch_bounds__(TY *TZ) k_wave(WaveArgs A) {
    constexpr bool REV = (MODE == WV_MIC_BWD);  // backward substitution runs high -> low
    __shared__ double sval[2][TZ][TY];
    __shared__ unsigned char sflag[2][TZ][TY];
    __shared__ int s_tile, s_nrows;
    const int jj = threadIdx.x % TY, kk = threadIdx.x / TY;
    if (A.sc && A.sc->done) return;
    const WaveGeom G = A.geom;
    const Dims d = A.d;
    if (threadIdx.x == 0) {
        s_tile = atomicAdd(A.ticket, 1);
        s_nrows = 0;
    }
    __syncthreads();
    // tile (b, c) in the sweep frame; REV mirrors y and z so that the
    // predecessors are always tiles b-1 and c-1
    int b, c;
    ticket_tile(s_tile, G.TB, G.TC, b, c);
    const int tile = b * G.TC + c;
    const int j = REV ? G.jhi - (b * TY + jj) : G.jlo + b * TY + jj;
    const int k = REV ? G.khi - (c * TZ + kk) : G.klo + c * TZ + kk;
    const bool valid = j >= G.jlo && j <= G.jhi && k >= G.klo && k <= G.khi;
    const int64_t sxy = (int64_t)d.nx * d.ny;
    int rbeg = 0, rend = 0;
    if (valid) {  // rows of my pencil are contiguous: all rows of grid row (j, k)
        int64_t c0 = (int64_t)j * d.nx + k * sxy;
        rbeg = A.rowscan[c0];
        rend = A.rowscan[c0 + d.nx];
    }
    if (rend > rbeg) atomicAdd(&s_nrows, rend - rbeg);
    __syncthreads();
    const int nsteps = G.nsteps;
    if (s_nrows == 0) {  // no rows: successors may pass at once
        if (threadIdx.x == 0) st_release(A.progress + tile, nsteps);
        return;
    }
    const bool has_y = b > 0, has_z = c > 0;
    const int tile_y = tile - G.TC, tile_z = tile - 1;
    int seen_y = has_y ? 0 : nsteps, seen_z = has_z ? 0 : nsteps;
    int r = REV ? rend - 1 : rbeg;  // next row of the pencil in sweep order
    // i of the next row; INT_MIN once the pencil is exhausted (the skewed
    // step index i itself runs outside [ilo, ihi], e.g. to -1)
    int ri = (r >= rbeg && r < rend) ? (int)(A.cell_of_row[r] % d.nx) : INT_MIN;
    Nb prev{0, 0.0};
    for (int s = 0; s < nsteps; s++) {
        const int i = REV ? G.ihi - (s - jj - kk) : G.ilo + s - jj - kk;
        if (threadIdx.x == 0) {  // predecessors must have finished steps < s + TY (+TZ)
            int need = min(s + TY, nsteps);
            if (has_y && seen_y < need)
                while ((seen_y = ld_acquire(A.progress + tile_y)) < need) {
                }
            need = min(s + TZ, nsteps);
            if (has_z && seen_z < need)
                while ((seen_z = ld_acquire(A.progress + tile_z)) < need) {
                }
        }
        __syncthreads();  // all threads finished step s-1; remote inputs ready
        if (threadIdx.x == 0 && s > 0 && (s % A.pub) == 0) st_release(A.progress + tile, s);
        const int cur = s & 1, prv = cur ^ 1;
        Nb out{0, 0.0};
        if (valid && ri == i) {
            const int row = r;
            Nb ny, nz;
            if (jj > 0) {
                ny = {sflag[prv][kk][jj - 1], sval[prv][kk][jj - 1]};
            } else {
                int nb = A.nbr[(REV ? 3 : 2) * A.ldn + row];
                ny = nb >= 0 ? wave_remote<MODE>(A, nb) : Nb{0, 0.0};
            }
            if (kk > 0) {
                nz = {sflag[prv][kk - 1][jj], sval[prv][kk - 1][jj]};
            } else {
                int nb = A.nbr[(REV ? 5 : 4) * A.ldn + row];
                nz = nb >= 0 ? wave_remote<MODE>(A, nb) : Nb{0, 0.0};
            }
            out = wave_row<MODE>(A, row, prev, ny, nz);
            r += REV ? -1 : 1;
            ri = (r >= rbeg && r < rend) ? (int)(A.cell_of_row[r] % d.nx) : INT_MIN;
        }
        sval[cur][kk][jj] = out.v;
        sflag[cur][kk][jj] = out.fl;
        prev = out;
    }
    __syncthreads();
    if (threadIdx.x == 0) st_release(A.progress + tile, nsteps);
}

// Tile shapes compiled in; FLIPB200_WAVE_TILE=<ty>x<tz> selects one (tuning).
struct TileShape {
    int ty, tz;
};
static const TileShape kShapes[] = {{16, 8}, {16, 16}, {32, 8}, {32, 16}, {32, 32}, {8, 8}};

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

int wave_pub() {
    static int p = [] {
        const char *e = getenv("FLIPB200_WAVE_PUB");
        int v = e ? atoi(e) : 2;
        return v > 0 ? v : 2;
    }();
    return p;
}

template <int MODE, int TY, int TZ>
static cudaError_t launch_shape(const WaveArgs &A, cudaStream_t st) {
    k_wave<MODE, TY, TZ><<<A.geom.TB * A.geom.TC, TY * TZ, 0, st>>>(A);
    return cudaGetLastError();
}

template <int MODE>
static cudaError_t launch_wave_t(const WaveArgs &A, cudaStream_t st) {
    TileShape t = wave_shape();
    if (t.ty == 16 && t.tz == 16) return launch_shape<MODE, 16, 16>(A, st);
    if (t.ty == 32 && t.tz == 8) return launch_shape<MODE, 32, 8>(A, st);
    if (t.ty == 32 && t.tz == 16) return launch_shape<MODE, 32, 16>(A, st);
    if (t.ty == 32 && t.tz == 32) return launch_shape<MODE, 32, 32>(A, st);
    if (t.ty == 8 && t.tz == 8) return launch_shape<MODE, 8, 8>(A, st);
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
    g.TB = (hi[1] - lo[1] + t.ty) / t.ty;
    g.TC = (hi[2] - lo[2] + t.tz) / t.tz;
    g.nsteps = (hi[0] - lo[0] + 1) + (t.ty - 1) + (t.tz - 1);
    return g;
}

}  // namespace flip
