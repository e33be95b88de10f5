// wavefront.cuh — per-row arithmetic of the pipelined sweeps (wavefront.cu).
#pragma once
#include "ops.cuh"

namespace flip {

enum WaveMode { WV_MIC_BUILD = 0, WV_MIC_FWD = 1, WV_MIC_BWD = 2, WV_GS = 3 };

#ifndef WAVE_TY
#define WAVE_TY 16
#endif
#ifndef WAVE_TZ
#define WAVE_TZ 8
#endif
#ifndef WAVE_PUB
#define WAVE_PUB 2
#endif

struct WaveGeom {
    int ilo, ihi, jlo, jhi, klo, khi;  // bounding box of the rows
    int TB, TC;                         // tiles along y and z
    int nsteps;                         // x span + TY + TZ - 2
};

struct WaveArgs {
    Dims d;
    WaveGeom geom;
    const int *rowscan;      // exclusive scan of isrow (ncells + 1)
    const int *cell_of_row;
    const int *nbr;          // [6][ldn]
    int64_t ldn;
    const double *diag, *rhs, *src, *precon;
    double *dst;
    double scale, tau, sigma;
    int *progress;           // [TB*TC] steps completed per tile
    int *ticket;
    int pub;                 // publish progress every `pub` steps
    const DevScalars *sc;    // early exit when sc->done (PCG after convergence)
};

// flags published with each value: bit0 row, bits1..3 has a +x/+y/+z row
constexpr unsigned char FL_ROW = 1, FL_PX = 2, FL_PY = 4, FL_PZ = 8;

struct Nb {
    unsigned char fl;
    double v;
};

__device__ __forceinline__ unsigned char plus_flags(const WaveArgs &A, int row) {
    return (unsigned char)(FL_ROW | (A.nbr[1 * A.ldn + row] >= 0 ? FL_PX : 0) |
                           (A.nbr[3 * A.ldn + row] >= 0 ? FL_PY : 0) |
                           (A.nbr[5 * A.ldn + row] >= 0 ? FL_PZ : 0));
}

// Value a predecessor row `nb` in another tile published (read through L2).
template <int MODE>
__device__ __forceinline__ Nb wave_remote(const WaveArgs &A, int nb) {
    double v = __ldcg(A.dst + nb);
    if (MODE == WV_MIC_FWD) return {FL_ROW, (A.scale * A.precon[nb]) * v};
    if (MODE == WV_MIC_BUILD) return {plus_flags(A, nb), v};
    return {FL_ROW, v};
}

// One row of the sweep; p/y/z are the sweep-direction predecessors along
// x/y/z.  Returns the value this row publishes to its successors.
template <int MODE>
__device__ __forceinline__ Nb wave_row(const WaveArgs &A, int row, Nb p, Nb y, Nb z) {
    const double sc = A.scale;
    if (MODE == WV_MIC_FWD) {  // _core.pyx:322-332
        double t = A.src[row];
        if (p.fl) t += p.v;
        if (y.fl) t += y.v;
        if (z.fl) t += z.v;
        double pr = A.precon[row];
        double q = t * pr;
        A.dst[row] = q;
        return {FL_ROW, (sc * pr) * q};
    } else if (MODE == WV_MIC_BWD) {  // _core.pyx:333-346
        double t = A.src[row];
        double pr = A.precon[row];
        if (p.fl) t += sc * pr * p.v;
        if (y.fl) t += sc * pr * y.v;
        if (z.fl) t += sc * pr * z.v;
        double zz = t * pr;
        A.dst[row] = zz;
        return {FL_ROW, zz};
    } else if (MODE == WV_GS) {  // _core.pyx:237-252, sum order -x,+x,-y,+y,-z,+z
        double s = 0.0;
        if (p.fl) s += p.v;
        int nb = A.nbr[1 * A.ldn + row];
        if (nb >= 0) s += A.dst[nb];  // +x: not yet updated
        if (y.fl) s += y.v;
        nb = A.nbr[3 * A.ldn + row];
        if (nb >= 0) s += A.dst[nb];
        if (z.fl) s += z.v;
        nb = A.nbr[5 * A.ldn + row];
        if (nb >= 0) s += A.dst[nb];
        double xn = (A.rhs[row] / sc + s) / A.diag[row];
        A.dst[row] = xn;
        return {FL_ROW, xn};
    } else {  // WV_MIC_BUILD, _core.pyx:291-307
        double dg = A.diag[row];
        double e = dg * sc;
        const Nb nbs[3] = {p, y, z};
        const unsigned char o1[3] = {FL_PY, FL_PX, FL_PX}, o2[3] = {FL_PZ, FL_PZ, FL_PY};
#pragma unroll
        for (int q = 0; q < 3; q++) {
            if (!nbs[q].fl) continue;
            double pq = nbs[q].v;
            e -= (sc * pq) * (sc * pq);
            double others = 0.0;
            if (nbs[q].fl & o1[q]) others -= sc;
            if (nbs[q].fl & o2[q]) others -= sc;
            e -= A.tau * (-sc) * others * pq * pq;
        }
        if (e < A.sigma * dg * sc) e = dg * sc;
        double pre = 1.0 / sqrt(e);
        A.dst[row] = pre;
        return {plus_flags(A, row), pre};
    }
}

cudaError_t launch_wave(int mode, const WaveArgs &A, cudaStream_t st);
int wave_pub();
WaveGeom wave_geom(const int lo[3], const int hi[3]);

}  // namespace flip
