// common.cuh — shared device helpers for libflipb200 (sm_100a).
//
// Bit-exactness with the reference (flipsim, CPU float64) rests on three
// rules applied everywhere in this library:
//   1. compiled with --fmad=false: no a*b+c contraction (the reference's
//      x86-64 build has no FMA), and the reference's association order is
//      spelled out with explicit parentheses;
//   2. IEEE division / sqrt (nvcc's default for double);
//   3. reductions whose order matters (dot products) replicate numpy's
//      pairwise tree; order-free ones (max, integer counts) use atomics.
#pragma once
#include <cuda_runtime.h>
#include <cstdio>
#include <stdint.h>

#include "../../include/flipb200.h"

#define SOLID 0
#define FLUID 1
#define AIR 2
#define MIN_PER_CELL 3   // flipsim/particles.py:151
#define MAX_PER_CELL 12  // flipsim/particles.py:152

namespace flip {

// Bounds checks of the checked build (make checked -> libflipb200_checked.so,
// loaded with FLIPB200_CHECKED=1): a failed check prints the site and the
// offending value and traps, which fails the launch (compute-sanitizer is
// not available on the GPU pool).  Compiled out of the production library.
#ifdef FLIP_CHECKED
#define FLIP_CHECK(cond, what, v, lim)                                                       \
    do {                                                                                 \
        if (!(cond)) {                                                                   \
            printf("FLIP_CHECK failed: %s (%lld vs %lld) at %s:%d block %d thread %d\n", \
                   what, (long long)(v), (long long)(lim), __FILE__, __LINE__,          \
                   (int)blockIdx.x, (int)threadIdx.x);                                 \
            __trap();                                                                    \
        }                                                                                \
    } while (0)
#else
#define FLIP_CHECK(cond, what, v, lim) \
    do {                               \
    } while (0)
#endif
#define FLIP_CHECK_RANGE(i, n, what) FLIP_CHECK((i) >= 0 && (i) < (n), what, i, n)

constexpr int kThreads = 256;

struct Dims {
    int nx, ny, nz;
    double dtau, ox, oy, oz;
    double inv_dtau;  // exact reciprocal; only used when pow2 is set
    int pow2;         // dtau is an exact power of two => x/dtau == x*inv_dtau bitwise
    __host__ __device__ int64_t ncells() const { return (int64_t)nx * ny * nz; }
};

// Division by the cell size.  When dtau = 2^-k the quotient x/dtau is the
// exact scaling x*2^k, so the multiply is bit-identical and ~10x cheaper in
// fp64 (matters in the P2G gather, SURVEY §7 hard part 3).
__device__ __forceinline__ double div_dtau(const Dims &d, double x) {
    return d.pow2 ? x * d.inv_dtau : x / d.dtau;
}

// div_dtau with the power-of-two test resolved at compile time (hot loops)
template <int P2>
__device__ __forceinline__ double div_dtau_t(const Dims &d, double x) {
    return P2 ? x * d.inv_dtau : x / d.dtau;
}

// (i, j, k) of cell c with 32-bit unsigned division (cell counts are below
// 2^31, checked by flip_create).
__device__ __forceinline__ void cell_ijk(const Dims &d, int64_t c, int &i, int &j, int &k) {
    const unsigned u = (unsigned)c, q = u / (unsigned)d.nx;
    i = (int)(u - q * (unsigned)d.nx);
    const unsigned r = q / (unsigned)d.ny;
    j = (int)(q - r * (unsigned)d.ny);
    k = (int)r;
}

// flipsim/_kernels/_core.pyx:17-19
__device__ __forceinline__ double hat(double r) {
    r = fabs(r);
    return r < 1.0 ? 1.0 - r : 0.0;
}

// flipsim/_kernels/_core.pyx:22-65 — clamped trilinear sample on an
// (mx, my, mz) lattice, identical arithmetic order.
__device__ __forceinline__ double tri_one(const double *__restrict__ arr, int mx, int my, int mz,
                                          double gx, double gy, double gz) {
    if (gx < 0.0) gx = 0.0;
    if (gx > (double)mx - 1.0) gx = (double)mx - 1.0;
    if (gy < 0.0) gy = 0.0;
    if (gy > (double)my - 1.0) gy = (double)my - 1.0;
    if (gz < 0.0) gz = 0.0;
    if (gz > (double)mz - 1.0) gz = (double)mz - 1.0;
    int i0 = (int)gx, j0 = (int)gy, k0 = (int)gz;
    if (i0 > mx - 2) i0 = mx - 2;
    if (j0 > my - 2) j0 = my - 2;
    if (k0 > mz - 2) k0 = mz - 2;
    if (i0 < 0) i0 = 0;
    if (j0 < 0) j0 = 0;
    if (k0 < 0) k0 = 0;
    double fx = gx - (double)i0, fy = gy - (double)j0, fz = gz - (double)k0;
    int i1 = i0 + 1 < mx ? i0 + 1 : mx - 1;
    int j1 = j0 + 1 < my ? j0 + 1 : my - 1;
    int k1 = k0 + 1 < mz ? k0 + 1 : mz - 1;
    int64_t sy = mx, sz = (int64_t)mx * my;
    double c00 = __ldg(arr + i0 + j0 * sy + k0 * sz) * (1.0 - fx) + __ldg(arr + i1 + j0 * sy + k0 * sz) * fx;
    double c10 = __ldg(arr + i0 + j1 * sy + k0 * sz) * (1.0 - fx) + __ldg(arr + i1 + j1 * sy + k0 * sz) * fx;
    double c01 = __ldg(arr + i0 + j0 * sy + k1 * sz) * (1.0 - fx) + __ldg(arr + i1 + j0 * sy + k1 * sz) * fx;
    double c11 = __ldg(arr + i0 + j1 * sy + k1 * sz) * (1.0 - fx) + __ldg(arr + i1 + j1 * sy + k1 * sz) * fx;
    double c0 = c00 * (1.0 - fy) + c10 * fy;
    double c1 = c01 * (1.0 - fy) + c11 * fy;
    return c0 * (1.0 - fz) + c1 * fz;
}

// tri_one on two arrays of the same lattice at the same point (G2P samples
// grid and grid_old there): the clamping, indices and weights are computed
// once, each value with tri_one's exact arithmetic.
__device__ __forceinline__ void tri_pair(const double *__restrict__ a, const double *__restrict__ b,
                                         int mx, int my, int mz, double gx, double gy, double gz,
                                         double &va, double &vb) {
    if (gx < 0.0) gx = 0.0;
    if (gx > (double)mx - 1.0) gx = (double)mx - 1.0;
    if (gy < 0.0) gy = 0.0;
    if (gy > (double)my - 1.0) gy = (double)my - 1.0;
    if (gz < 0.0) gz = 0.0;
    if (gz > (double)mz - 1.0) gz = (double)mz - 1.0;
    int i0 = (int)gx, j0 = (int)gy, k0 = (int)gz;
    if (i0 > mx - 2) i0 = mx - 2;
    if (j0 > my - 2) j0 = my - 2;
    if (k0 > mz - 2) k0 = mz - 2;
    if (i0 < 0) i0 = 0;
    if (j0 < 0) j0 = 0;
    if (k0 < 0) k0 = 0;
    const double fx = gx - (double)i0, fy = gy - (double)j0, fz = gz - (double)k0;
    const int i1 = i0 + 1 < mx ? i0 + 1 : mx - 1;
    const int j1 = j0 + 1 < my ? j0 + 1 : my - 1;
    const int k1 = k0 + 1 < mz ? k0 + 1 : mz - 1;
    const int64_t sy = mx, sz = (int64_t)mx * my;
    const int64_t o[8] = {i0 + j0 * sy + k0 * sz, i1 + j0 * sy + k0 * sz, i0 + j1 * sy + k0 * sz,
                          i1 + j1 * sy + k0 * sz, i0 + j0 * sy + k1 * sz, i1 + j0 * sy + k1 * sz,
                          i0 + j1 * sy + k1 * sz, i1 + j1 * sy + k1 * sz};
    double A[8], B[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
        A[q] = __ldg(a + o[q]);
        B[q] = __ldg(b + o[q]);
    }
    const double ex = 1.0 - fx, ey = 1.0 - fy, ez = 1.0 - fz;
    {
        const double c00 = A[0] * ex + A[1] * fx, c10 = A[2] * ex + A[3] * fx;
        const double c01 = A[4] * ex + A[5] * fx, c11 = A[6] * ex + A[7] * fx;
        const double c0 = c00 * ey + c10 * fy, c1 = c01 * ey + c11 * fy;
        va = c0 * ez + c1 * fz;
    }
    {
        const double c00 = B[0] * ex + B[1] * fx, c10 = B[2] * ex + B[3] * fx;
        const double c01 = B[4] * ex + B[5] * fx, c11 = B[6] * ex + B[7] * fx;
        const double c0 = c00 * ey + c10 * fy, c1 = c01 * ey + c11 * fy;
        vb = c0 * ez + c1 * fz;
    }
}

// flipsim/_kernels/_core.pyx:84-89 — staggered-lattice velocity at a point.
// (x - origin) / dtau is an exact multiply when dtau = 2^-k (div_dtau).
__device__ __forceinline__ void sample_vel(const Dims &d, const double *u, const double *v,
                                           const double *w, double px, double py, double pz,
                                           double &vx, double &vy, double &vz) {
    double gx = div_dtau(d, px - d.ox);
    double gy = div_dtau(d, py - d.oy);
    double gz = div_dtau(d, pz - d.oz);
    vx = tri_one(u, d.nx + 1, d.ny, d.nz, gx, gy - 0.5, gz - 0.5);
    vy = tri_one(v, d.nx, d.ny + 1, d.nz, gx - 0.5, gy, gz - 0.5);
    vz = tri_one(w, d.nx, d.ny, d.nz + 1, gx - 0.5, gy - 0.5, gz);
}

// sample_vel on the new and old grids at once (G2P, transfer.py:60-82)
__device__ __forceinline__ void sample_vel_pair(const Dims &d, const double *un, const double *vn,
                                                const double *wn, const double *uo,
                                                const double *vo, const double *wo, double px,
                                                double py, double pz, double &ax, double &ay,
                                                double &az, double &bx, double &by, double &bz) {
    const double gx = div_dtau(d, px - d.ox);
    const double gy = div_dtau(d, py - d.oy);
    const double gz = div_dtau(d, pz - d.oz);
    tri_pair(un, uo, d.nx + 1, d.ny, d.nz, gx, gy - 0.5, gz - 0.5, ax, bx);
    tri_pair(vn, vo, d.nx, d.ny + 1, d.nz, gx - 0.5, gy, gz - 0.5, ay, by);
    tri_pair(wn, wo, d.nx, d.ny, d.nz + 1, gx - 0.5, gy - 0.5, gz, az, bz);
}

// flipsim/rng.py:19-33
__device__ __host__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ double uniform01(uint64_t seed, uint64_t stream, uint64_t lane) {
    uint64_t z = seed + ((stream << 20) + lane + 1ULL) * 0x9E3779B97F4A7C15ULL;
    z = mix64(z);
    return (double)(z >> 11) * 0x1.0p-53;
}

// flipsim/particles.py:113-130 for one (cell, subcell).
__device__ __forceinline__ void jitter_pos(const Dims &d, int64_t c, int64_t s, int density,
                                           uint64_t seed, double &px, double &py, double &pz) {
    double sub_len = d.dtau / (double)density;
    int ci, cj, ck;  // cell counts are below 2^31 (flip_create): 32-bit division
    cell_ijk(d, c, ci, cj, ck);
    const int si32 = (int)s;
    int si = si32 % density, sj = (si32 / density) % density, sk = si32 / (density * density);
    double jx = uniform01(seed, (uint64_t)c, (uint64_t)(s * 4 + 0));
    double jy = uniform01(seed, (uint64_t)c, (uint64_t)(s * 4 + 1));
    double jz = uniform01(seed, (uint64_t)c, (uint64_t)(s * 4 + 2));
    px = (d.ox + (double)ci * d.dtau) + (((double)si + jx) * sub_len);
    py = (d.oy + (double)cj * d.dtau) + (((double)sj + jy) * sub_len);
    pz = (d.oz + (double)ck * d.dtau) + (((double)sk + jz) * sub_len);
}

// numpy float64 -> int64 cast of floor() followed by np.clip (binning.py:39-41)
__device__ __forceinline__ int floor_clip(double x, int hi) {
    double f = floor(x);
    if (!(f >= 0.0)) return 0;  // negatives and NaN (numpy: INT64_MIN -> clip 0)
    if (f >= 9.2233720368547758e18) return 0;  // out-of-range cast: INT64_MIN -> clip 0
    if (f >= (double)hi) return hi;
    return (int)f;
}

__device__ __forceinline__ int cell_of(const Dims &d, double px, double py, double pz) {
    int i = floor_clip((px - d.ox) / d.dtau, d.nx - 1);
    int j = floor_clip((py - d.oy) / d.dtau, d.ny - 1);
    int k = floor_clip((pz - d.oz) / d.dtau, d.nz - 1);
    return i + j * d.nx + k * d.nx * d.ny;
}

// Order-free max of non-negative doubles via their IEEE bit patterns.
__device__ __forceinline__ void atomic_max_nonneg(unsigned long long *addr, double v) {
    atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

__device__ __forceinline__ int64_t gtid() { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int64_t gstride() { return (int64_t)gridDim.x * blockDim.x; }

}  // namespace flip
