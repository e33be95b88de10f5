/*
 * flip_oracle.c — CPU restatement of the reference FLIP timestep.
 *
 * TEST INFRASTRUCTURE ONLY (parity checker + bench cpu_baseline arm).  The
 * product never links or calls this file.  Reference = flipsim at
 * /root/reference/pkg/src/flipsim (abbreviated F/ below).  Arithmetic order
 * follows the reference operation by operation; compiled with
 * -ffp-contract=off so no FMA is formed (the reference's gcc -O3 x86-64
 * build has no FMA either).  Parallel loops (OpenMP) are pure gathers or
 * elementwise maps, so results do not depend on the thread count; the
 * reference's serial loops (counting sort, GS, MIC(0)) stay serial.
 */
#include "flip_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SOLID 0
#define FLUID 1
#define AIR 2
#define MIN_PER_CELL 3  /* F/particles.py:151 */
#define MAX_PER_CELL 12 /* F/particles.py:152 */

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ---------------------------------------------------------------- rng -- */
/* F/rng.py:19-33: splitmix64 finaliser over a golden-ratio Weyl counter. */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double orc_uniform01(uint64_t seed, uint64_t stream, uint64_t lane) {
    uint64_t counter = stream * (1ULL << 20) + lane;
    uint64_t z = seed + (counter + 1ULL) * 0x9E3779B97F4A7C15ULL;
    z = mix64(z);
    return (double)(z >> 11) * 0x1.0p-53;
}

/* F/rng.py:36-41 */
uint64_t orc_derive_seed(uint64_t base, uint64_t stream) {
    return mix64(base + (stream + 1ULL) * 0x9E3779B97F4A7C15ULL);
}

/* ------------------------------------------------------------ seeding -- */
/* F/particles.py:103-110 with SeedRegion.contains (F/particles.py:92-100). */
static inline void cell_center(const orc_dims *d, int64_t idx, double *cx, double *cy, double *cz) {
    *cx = d->ox + ((double)(idx % d->nx) + 0.5) * d->dtau;
    *cy = d->oy + ((double)((idx / d->nx) % d->ny) + 0.5) * d->dtau;
    *cz = d->oz + ((double)(idx / (d->nx * d->ny)) + 0.5) * d->dtau;
}

int64_t orc_covered_cells_box(const orc_dims *d, const double lo[3], const double hi[3], int64_t *out) {
    int64_t nc = d->nx * d->ny * d->nz, m = 0;
    for (int64_t idx = 0; idx < nc; idx++) {
        double cx, cy, cz;
        cell_center(d, idx, &cx, &cy, &cz);
        if (cx >= lo[0] && cx <= hi[0] && cy >= lo[1] && cy <= hi[1] && cz >= lo[2] && cz <= hi[2])
            out[m++] = idx;
    }
    return m;
}

int64_t orc_covered_cells_sphere(const orc_dims *d, const double c[3], double r, int64_t *out) {
    int64_t nc = d->nx * d->ny * d->nz, m = 0;
    double r2 = r * r;
    for (int64_t idx = 0; idx < nc; idx++) {
        double cx, cy, cz;
        cell_center(d, idx, &cx, &cy, &cz);
        double dx = cx - c[0], dy = cy - c[1], dz = cz - c[2];
        if (((dx * dx) + (dy * dy)) + (dz * dz) <= r2) out[m++] = idx;
    }
    return m;
}

/* F/particles.py:113-130 */
void orc_jittered_positions(const orc_dims *d, int64_t m, const int64_t *cells, const int64_t *subs,
                            int64_t density, uint64_t seed, double *px, double *py, double *pz) {
    double sub_len = d->dtau / (double)density;
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < m; t++) {
        int64_t c = cells[t], s = subs[t];
        int64_t ci = c % d->nx, cj = (c / d->nx) % d->ny, ck = c / (d->nx * d->ny);
        int64_t si = s % density, sj = (s / density) % density, sk = s / (density * density);
        double jx = orc_uniform01(seed, (uint64_t)c, (uint64_t)(s * 4 + 0));
        double jy = orc_uniform01(seed, (uint64_t)c, (uint64_t)(s * 4 + 1));
        double jz = orc_uniform01(seed, (uint64_t)c, (uint64_t)(s * 4 + 2));
        px[t] = (d->ox + (double)ci * d->dtau) + (((double)si + jx) * sub_len);
        py[t] = (d->oy + (double)cj * d->dtau) + (((double)sj + jy) * sub_len);
        pz[t] = (d->oz + (double)ck * d->dtau) + (((double)sk + jz) * sub_len);
    }
}

/* ------------------------------------------------------ dt and advect -- */
/* F/particles.py:214-224 */
double orc_compute_dt(int64_t n, const double *vx, const double *vy, const double *vz,
                      double dtau, double alpha, double dt_max) {
    if (n == 0) return dt_max;
    double m = -INFINITY;
    #pragma omp parallel for reduction(max : m) schedule(static)
    for (int64_t t = 0; t < n; t++) {
        double s2 = ((vx[t] * vx[t]) + (vy[t] * vy[t])) + (vz[t] * vz[t]);
        if (s2 > m) m = s2;
    }
    double s_max = sqrt(m);
    if (s_max == 0.0) return dt_max;
    double cand = (alpha * dtau) / s_max;
    return cand < dt_max ? cand : dt_max;
}

/* F/grid.py:121-132 */
int orc_interior_box(const orc_dims *d, const uint8_t *label, double lo[3], double hi[3]) {
    int64_t imin = INT64_MAX, jmin = INT64_MAX, kmin = INT64_MAX, imax = -1, jmax = -1, kmax = -1;
    for (int64_t k = 0; k < d->nz; k++)
        for (int64_t j = 0; j < d->ny; j++)
            for (int64_t i = 0; i < d->nx; i++) {
                if (label[i + j * d->nx + k * d->nx * d->ny] == SOLID) continue;
                if (i < imin) imin = i;
                if (i > imax) imax = i;
                if (j < jmin) jmin = j;
                if (j > jmax) jmax = j;
                if (k < kmin) kmin = k;
                if (k > kmax) kmax = k;
            }
    if (imax < 0) return -1;
    lo[0] = d->ox + (double)imin * d->dtau;
    lo[1] = d->oy + (double)jmin * d->dtau;
    lo[2] = d->oz + (double)kmin * d->dtau;
    hi[0] = d->ox + (double)(imax + 1) * d->dtau;
    hi[1] = d->oy + (double)(jmax + 1) * d->dtau;
    hi[2] = d->oz + (double)(kmax + 1) * d->dtau;
    return 0;
}

/* F/particles.py:227-248: forward Euler, then per-axis clamp of escapees. */
void orc_advect(int64_t n, double *px, double *py, double *pz,
                const double *vx, const double *vy, const double *vz,
                double dt, const double lo[3], const double hi[3], double skin) {
    double *pos[3] = {px, py, pz};
    const double *vel[3] = {vx, vy, vz};
    for (int a = 0; a < 3; a++) {
        double *p = pos[a];
        const double *v = vel[a];
        double l = lo[a], h = hi[a], lpos = lo[a] + skin, hpos = hi[a] - skin;
        #pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < n; t++) {
            double q = p[t] + (v[t] * dt);
            if (q <= l) q = lpos;
            else if (q >= h) q = hpos;
            p[t] = q;
        }
    }
}

/* ------------------------------------------------------------ binning -- */
static inline int64_t clampi(int64_t x, int64_t lo, int64_t hi) {
    return x < lo ? lo : (x > hi ? hi : x);
}

static inline int64_t f2i(double x) {
    /* numpy float64 -> int64 cast of floor(); finite inputs only matter */
    if (!(x == x)) return INT64_MIN;
    if (x >= 9.2233720368547758e18 || x < -9.2233720368547758e18) return INT64_MIN;
    return (int64_t)x;
}

/* F/binning.py:37-42 */
void orc_cell_index_many(const orc_dims *d, int64_t n, const double *px, const double *py,
                         const double *pz, int64_t *cells) {
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n; t++) {
        int64_t i = clampi(f2i(floor((px[t] - d->ox) / d->dtau)), 0, d->nx - 1);
        int64_t j = clampi(f2i(floor((py[t] - d->oy) / d->dtau)), 0, d->ny - 1);
        int64_t k = clampi(f2i(floor((pz[t] - d->oz) / d->dtau)), 0, d->nz - 1);
        cells[t] = i + j * d->nx + k * d->nx * d->ny;
    }
}

/* F/binning.py:45-79 (exact integer prefix sum; tree vs sequential is moot) */
void orc_exclusive_scan(int64_t n, const int64_t *in, int64_t *out) {
    int64_t acc = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t v = in[i];
        out[i] = acc;
        acc += v;
    }
}

/* F/_kernels/_core.pyx:179-193: sequential scatter with per-cell cursors. */
void orc_counting_sort_perm(int64_t n, const int64_t *cells, const int64_t *offset,
                            int64_t ncells, int64_t *perm) {
    int64_t *cursor = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncells > 0 ? ncells : 1));
    memcpy(cursor, offset, sizeof(int64_t) * (size_t)ncells);
    for (int64_t t = 0; t < n; t++) perm[cursor[cells[t]]++] = t;
    free(cursor);
}

/* F/binning.py:82-97 + ParticleSet.reorder (F/particles.py:54-64). */
void orc_bin_particles(const orc_dims *d, int64_t n, double *arrs[6], double *scratch,
                       int64_t *count, int64_t *offset, int64_t *cells, int64_t *perm) {
    int64_t nc = d->nx * d->ny * d->nz;
    orc_cell_index_many(d, n, arrs[0], arrs[1], arrs[2], cells);
    memset(count, 0, sizeof(int64_t) * (size_t)nc);
    for (int64_t t = 0; t < n; t++) count[cells[t]]++;
    orc_exclusive_scan(nc, count, offset);
    orc_counting_sort_perm(n, cells, offset, nc, perm);
    for (int a = 0; a < 6; a++) {
        double *src = arrs[a];
        #pragma omp parallel for schedule(static)
        for (int64_t t = 0; t < n; t++) scratch[t] = src[perm[t]];
        memcpy(src, scratch, sizeof(double) * (size_t)n);
    }
}

/* F/grid.py:185-190 */
void orc_classify_cells(int64_t ncells, const int64_t *count, uint8_t *label) {
    #pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < ncells; c++)
        if (label[c] != SOLID) label[c] = count[c] > 0 ? FLUID : AIR;
}

/* ------------------------------------------------------------ sampling -- */
/* F/_kernels/_core.pyx:22-65 */
static inline double tri_one(const double *arr, int64_t mx, int64_t my, int64_t mz,
                             double gx, double gy, double gz) {
    if (gx < 0.0) gx = 0.0;
    if (gx > (double)mx - 1.0) gx = (double)mx - 1.0;
    if (gy < 0.0) gy = 0.0;
    if (gy > (double)my - 1.0) gy = (double)my - 1.0;
    if (gz < 0.0) gz = 0.0;
    if (gz > (double)mz - 1.0) gz = (double)mz - 1.0;
    int64_t i0 = (int64_t)gx, j0 = (int64_t)gy, k0 = (int64_t)gz;
    if (i0 > mx - 2) i0 = mx - 2;
    if (j0 > my - 2) j0 = my - 2;
    if (k0 > mz - 2) k0 = mz - 2;
    if (i0 < 0) i0 = 0;
    if (j0 < 0) j0 = 0;
    if (k0 < 0) k0 = 0;
    double fx = gx - (double)i0, fy = gy - (double)j0, fz = gz - (double)k0;
    int64_t i1 = i0 + 1 < mx ? i0 + 1 : mx - 1;
    int64_t j1 = j0 + 1 < my ? j0 + 1 : my - 1;
    int64_t k1 = k0 + 1 < mz ? k0 + 1 : mz - 1;
    int64_t sy = mx, sz = mx * my;
    double c00 = arr[i0 + j0 * sy + k0 * sz] * (1.0 - fx) + arr[i1 + j0 * sy + k0 * sz] * fx;
    double c10 = arr[i0 + j1 * sy + k0 * sz] * (1.0 - fx) + arr[i1 + j1 * sy + k0 * sz] * fx;
    double c01 = arr[i0 + j0 * sy + k1 * sz] * (1.0 - fx) + arr[i1 + j0 * sy + k1 * sz] * fx;
    double c11 = arr[i0 + j1 * sy + k1 * sz] * (1.0 - fx) + arr[i1 + j1 * sy + k1 * sz] * fx;
    double c0 = c00 * (1.0 - fy) + c10 * fy;
    double c1 = c01 * (1.0 - fy) + c11 * fy;
    return c0 * (1.0 - fz) + c1 * fz;
}

/* F/_kernels/_core.pyx:68-90 */
void orc_sample_velocity_many(const orc_dims *d, const double *u, const double *v, const double *w,
                              int64_t n, const double *px, const double *py, const double *pz,
                              double *vx, double *vy, double *vz) {
    int64_t nx = d->nx, ny = d->ny, nz = d->nz;
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n; t++) {
        double gx = (px[t] - d->ox) / d->dtau;
        double gy = (py[t] - d->oy) / d->dtau;
        double gz = (pz[t] - d->oz) / d->dtau;
        vx[t] = tri_one(u, nx + 1, ny, nz, gx, gy - 0.5, gz - 0.5);
        vy[t] = tri_one(v, nx, ny + 1, nz, gx - 0.5, gy, gz - 0.5);
        vz[t] = tri_one(w, nx, ny, nz + 1, gx - 0.5, gy - 0.5, gz);
    }
}

/* Extension, opt-in (SceneSpec.advection = "rk2"): explicit-midpoint RK2
 * through the grid velocity field the previous step left (the north star
 * names "RK2 particle advection"; the reference itself is forward Euler on
 * the particle velocities, F/particles.py:227-248, and SPEC.md:211 lists
 * RK2 as a non-goal, so this restatement is the only definition):
 *   k1 = sample(grid, p)            (F/_kernels/_core.pyx:68-90 sampling)
 *   m  = p + (k1 * (0.5 * dt))
 *   k2 = sample(grid, m)
 *   p' = p + (k2 * dt), then the reference's per-axis clamp
 *        (<= lo -> lo + skin, >= hi -> hi - skin, F/particles.py:237-247).
 * Particle velocities are not touched (as in the Euler advect). */
static inline void sample3(const orc_dims *d, const double *u, const double *v, const double *w,
                           double x, double y, double z, double out[3]) {
    int64_t nx = d->nx, ny = d->ny, nz = d->nz;
    double gx = (x - d->ox) / d->dtau;
    double gy = (y - d->oy) / d->dtau;
    double gz = (z - d->oz) / d->dtau;
    out[0] = tri_one(u, nx + 1, ny, nz, gx, gy - 0.5, gz - 0.5);
    out[1] = tri_one(v, nx, ny + 1, nz, gx - 0.5, gy, gz - 0.5);
    out[2] = tri_one(w, nx, ny, nz + 1, gx - 0.5, gy - 0.5, gz);
}

void orc_advect_rk2(const orc_dims *d, const double *u, const double *v, const double *w,
                    int64_t n, double *px, double *py, double *pz, double dt,
                    const double lo[3], const double hi[3], double skin) {
    const double h = 0.5 * dt;
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n; t++) {
        double p[3] = {px[t], py[t], pz[t]}, k1[3], k2[3], m[3];
        sample3(d, u, v, w, p[0], p[1], p[2], k1);
        for (int a = 0; a < 3; a++) m[a] = p[a] + (k1[a] * h);
        sample3(d, u, v, w, m[0], m[1], m[2], k2);
        for (int a = 0; a < 3; a++) {
            double q = p[a] + (k2[a] * dt);
            if (q <= lo[a]) q = lo[a] + skin;
            else if (q >= hi[a]) q = hi[a] - skin;
            p[a] = q;
        }
        px[t] = p[0];
        py[t] = p[1];
        pz[t] = p[2];
    }
}

/* ---------------------------------------------------------------- P2G -- */
static inline double hat(double r) {  /* F/_kernels/_core.pyx:17-19 */
    r = fabs(r);
    return r < 1.0 ? 1.0 - r : 0.0;
}

/* F/_kernels/_core.pyx:93-176: per-face Kahan gather over candidate cells
 * (z outer, y, x inner) and each cell's particle segment in hash order. */
void orc_p2g_component(const orc_dims *d, int comp, const double *vel_p, const double *px,
                       const double *py, const double *pz, const int64_t *offset,
                       const int64_t *count, double *out, double *den) {
    int64_t nx = d->nx, ny = d->ny, nz = d->nz, fnx, fny, fnz;
    double offx, offy, offz, dtau = d->dtau;
    if (comp == 0) { fnx = nx + 1; fny = ny; fnz = nz; offx = 0.0; offy = 0.5; offz = 0.5; }
    else if (comp == 1) { fnx = nx; fny = ny + 1; fnz = nz; offx = 0.5; offy = 0.0; offz = 0.5; }
    else { fnx = nx; fny = ny; fnz = nz + 1; offx = 0.5; offy = 0.5; offz = 0.0; }
    int64_t nfaces = fnx * fny * fnz;
    #pragma omp parallel for schedule(static)
    for (int64_t f = 0; f < nfaces; f++) {
        int64_t fi = f % fnx, fj = (f / fnx) % fny, fk = f / (fnx * fny);
        double fpx = d->ox + ((double)fi + offx) * dtau;
        double fpy = d->oy + ((double)fj + offy) * dtau;
        double fpz = d->oz + ((double)fk + offz) * dtau;
        int64_t cxlo = fi - 1, cxhi = comp == 0 ? fi : fi + 1;
        int64_t cylo = fj - 1, cyhi = comp == 1 ? fj : fj + 1;
        int64_t czlo = fk - 1, czhi = comp == 2 ? fk : fk + 1;
        if (cxlo < 0) cxlo = 0;
        if (cylo < 0) cylo = 0;
        if (czlo < 0) czlo = 0;
        if (cxhi > nx - 1) cxhi = nx - 1;
        if (cyhi > ny - 1) cyhi = ny - 1;
        if (czhi > nz - 1) czhi = nz - 1;
        double num = 0.0, dsum = 0.0, cn = 0.0, cd = 0.0;
        for (int64_t cz = czlo; cz <= czhi; cz++)
            for (int64_t cy = cylo; cy <= cyhi; cy++)
                for (int64_t cx = cxlo; cx <= cxhi; cx++) {
                    int64_t cell = cx + cy * nx + cz * nx * ny;
                    int64_t t0 = offset[cell], t1 = t0 + count[cell];
                    for (int64_t t = t0; t < t1; t++) {
                        double wgt = (hat((px[t] - fpx) / dtau) * hat((py[t] - fpy) / dtau)) *
                                     hat((pz[t] - fpz) / dtau);
                        if (wgt > 0.0) {
                            double yk = wgt * vel_p[t] - cn;
                            double tk = num + yk;
                            cn = (tk - num) - yk;
                            num = tk;
                            yk = wgt - cd;
                            tk = dsum + yk;
                            cd = (tk - dsum) - yk;
                            dsum = tk;
                        }
                    }
                }
        den[f] = dsum;
        out[f] = dsum > 0.0 ? num / dsum : 0.0;
    }
}

/* ----------------------------------------------------- forces, walls -- */
/* F/grid.py:193-202 */
void orc_add_body_force(const orc_dims *d, double *u, double *v, double *w,
                        const double g[3], double dt) {
    int64_t nu = (d->nx + 1) * d->ny * d->nz, nv = d->nx * (d->ny + 1) * d->nz,
            nw = d->nx * d->ny * (d->nz + 1);
    double *arr[3] = {u, v, w};
    int64_t len[3] = {nu, nv, nw};
    for (int a = 0; a < 3; a++) {
        if (g[a] == 0.0) continue;
        double inc = g[a] * dt;
        double *p = arr[a];
        #pragma omp parallel for schedule(static)
        for (int64_t f = 0; f < len[a]; f++) p[f] = p[f] + inc;
    }
}

/* F/grid.py:205-228: faces touching SOLID or on the domain boundary -> 0. */
void orc_enforce_solid_boundaries(const orc_dims *d, const uint8_t *label,
                                  double *u, double *v, double *w) {
    int64_t nx = d->nx, ny = d->ny, nz = d->nz;
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nz; k++)
        for (int64_t j = 0; j < ny; j++)
            for (int64_t i = 0; i <= nx; i++) {
                int z = (i == 0 || i == nx) ||
                        label[(i - 1) + j * nx + k * nx * ny] == SOLID ||
                        label[i + j * nx + k * nx * ny] == SOLID;
                if (z) u[i + j * (nx + 1) + k * (nx + 1) * ny] = 0.0;
            }
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nz; k++)
        for (int64_t j = 0; j <= ny; j++)
            for (int64_t i = 0; i < nx; i++) {
                int z = (j == 0 || j == ny) ||
                        label[i + (j - 1) * nx + k * nx * ny] == SOLID ||
                        label[i + j * nx + k * nx * ny] == SOLID;
                if (z) v[i + j * nx + k * nx * (ny + 1)] = 0.0;
            }
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k <= nz; k++)
        for (int64_t j = 0; j < ny; j++)
            for (int64_t i = 0; i < nx; i++) {
                int z = (k == 0 || k == nz) ||
                        label[i + j * nx + (k - 1) * nx * ny] == SOLID ||
                        label[i + j * nx + k * nx * ny] == SOLID;
                if (z) w[i + j * nx + k * nx * ny] = 0.0;
            }
}

/* F/grid.py:231-263.  Synchronous layers; accumulation order
 * 0 + v(k+1) + v(k-1) + v(j+1) + v(j-1) + v(i+1) + v(i-1). */
void orc_extrapolate_component(int64_t mx, int64_t my, int64_t mz, double *arr,
                               uint8_t *known, int layers, double *acc,
                               int64_t *cnt, uint8_t *kold) {
    int64_t n = mx * my * mz, sy = mx, sz = mx * my;
    for (int layer = 0; layer < layers; layer++) {
        memcpy(kold, known, (size_t)n);
        int64_t filled = 0;
        #pragma omp parallel for schedule(static) reduction(+ : filled)
        for (int64_t k = 0; k < mz; k++)
            for (int64_t j = 0; j < my; j++)
                for (int64_t i = 0; i < mx; i++) {
                    int64_t f = i + j * sy + k * sz;
                    if (kold[f]) continue;
                    double a = 0.0;
                    int64_t c = 0;
                    if (k + 1 < mz) { c += kold[f + sz]; a = a + (kold[f + sz] ? arr[f + sz] : 0.0); }
                    else a = a + 0.0;
                    if (k - 1 >= 0) { c += kold[f - sz]; a = a + (kold[f - sz] ? arr[f - sz] : 0.0); }
                    else a = a + 0.0;
                    if (j + 1 < my) { c += kold[f + sy]; a = a + (kold[f + sy] ? arr[f + sy] : 0.0); }
                    else a = a + 0.0;
                    if (j - 1 >= 0) { c += kold[f - sy]; a = a + (kold[f - sy] ? arr[f - sy] : 0.0); }
                    else a = a + 0.0;
                    if (i + 1 < mx) { c += kold[f + 1]; a = a + (kold[f + 1] ? arr[f + 1] : 0.0); }
                    else a = a + 0.0;
                    if (i - 1 >= 0) { c += kold[f - 1]; a = a + (kold[f - 1] ? arr[f - 1] : 0.0); }
                    else a = a + 0.0;
                    acc[f] = a;
                    cnt[f] = c;
                    if (c > 0) filled++;
                }
        /* apply after the whole layer was read (synchronous) */
        #pragma omp parallel for schedule(static)
        for (int64_t f = 0; f < n; f++) {
            if (!kold[f] && cnt[f] > 0) {
                arr[f] = acc[f] / (double)cnt[f];
                known[f] = 1;
            }
        }
        #pragma omp parallel for schedule(static)
        for (int64_t f = 0; f < n; f++) cnt[f] = 0;
        if (filled == 0) break;
    }
}

/* ----------------------------------------------------------- assembly -- */
static int64_t uf_find(int64_t *par, int64_t x) {
    while (par[x] != x) {
        par[x] = par[par[x]];
        x = par[x];
    }
    return x;
}

static inline uint8_t lab_at(const orc_dims *d, const uint8_t *label, int64_t i, int64_t j, int64_t k) {
    if (i < 0 || j < 0 || k < 0 || i >= d->nx || j >= d->ny || k >= d->nz) return SOLID;
    return label[i + j * d->nx + k * d->nx * d->ny];
}

/* F/pressure.py:76-166.  Sealed components (scipy.ndimage.label with the
 * 6-connected structure, F/pressure.py:112-113) are found by union-find with
 * the minimum raw index as root, which is exactly the pinned cell
 * (np.minimum.at(first, comp, fluid), F/pressure.py:119-121). */
int64_t orc_assemble(const orc_dims *d, const uint8_t *label, const double *u, const double *v,
                     const double *w, int64_t *row_of, int64_t *cells_out, double *diag,
                     int64_t *nbr_rows, double *rhs, int64_t *pinned_out, int64_t *npinned) {
    int64_t nx = d->nx, ny = d->ny, nz = d->nz, nc = nx * ny * nz, sxy = nx * ny;
    static const int DI[6] = {-1, 1, 0, 0, 0, 0}, DJ[6] = {0, 0, -1, 1, 0, 0}, DK[6] = {0, 0, 0, 0, -1, 1};
    int64_t *par = (int64_t *)malloc(sizeof(int64_t) * (size_t)nc);
    uint8_t *has_air = (uint8_t *)calloc((size_t)nc, 1);
    for (int64_t c = 0; c < nc; c++) par[c] = c;
    for (int64_t k = 0; k < nz; k++)
        for (int64_t j = 0; j < ny; j++)
            for (int64_t i = 0; i < nx; i++) {
                int64_t c = i + j * nx + k * sxy;
                if (label[c] != FLUID) continue;
                int64_t nb[3] = {i > 0 ? c - 1 : -1, j > 0 ? c - nx : -1, k > 0 ? c - sxy : -1};
                for (int q = 0; q < 3; q++) {
                    if (nb[q] < 0 || label[nb[q]] != FLUID) continue;
                    int64_t ra = uf_find(par, c), rb = uf_find(par, nb[q]);
                    if (ra == rb) continue;
                    if (ra < rb) par[rb] = ra; else par[ra] = rb;
                }
            }
    for (int64_t k = 0; k < nz; k++)
        for (int64_t j = 0; j < ny; j++)
            for (int64_t i = 0; i < nx; i++) {
                int64_t c = i + j * nx + k * sxy;
                if (label[c] != FLUID) continue;
                int air = 0;
                for (int q = 0; q < 6; q++) air |= lab_at(d, label, i + DI[q], j + DJ[q], k + DK[q]) == AIR;
                if (air) has_air[uf_find(par, c)] = 1;
            }
    /* rows: FLUID cells ascending minus pinned roots (sealed components) */
    int64_t n = 0, np_ = 0;
    for (int64_t c = 0; c < nc; c++) {
        row_of[c] = -1;
        if (label[c] != FLUID) continue;
        int64_t r = uf_find(par, c);
        if (r == c && !has_air[c]) {
            pinned_out[np_++] = c;
            continue;
        }
        row_of[c] = n;
        cells_out[n++] = c;
    }
    *npinned = np_;
    #pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; r++) {
        int64_t c = cells_out[r];
        int64_t i = c % nx, j = (c / nx) % ny, k = c / sxy;
        int64_t ns = 0;
        for (int q = 0; q < 6; q++) {
            int64_t ii = i + DI[q], jj = j + DJ[q], kk = k + DK[q];
            uint8_t l = lab_at(d, label, ii, jj, kk);
            ns += l != SOLID;
            int64_t nbr = -1;
            if (l == FLUID) nbr = row_of[ii + jj * nx + kk * sxy];
            nbr_rows[r * 6 + q] = nbr;
        }
        diag[r] = (double)ns;
        /* rhs = -div with solid-face velocities zeroed (F/pressure.py:144-151) */
        int64_t fu0 = i + j * (nx + 1) + k * (nx + 1) * ny, fu1 = fu0 + 1;
        int64_t fv0 = i + j * nx + k * nx * (ny + 1), fv1 = fv0 + nx;
        int64_t fw0 = i + j * nx + k * sxy, fw1 = fw0 + sxy;
        uint8_t sl = lab_at(d, label, i, j, k) == SOLID;
        double u0 = (i == 0 || sl || lab_at(d, label, i - 1, j, k) == SOLID) ? 0.0 : u[fu0];
        double u1 = (i + 1 == nx || sl || lab_at(d, label, i + 1, j, k) == SOLID) ? 0.0 : u[fu1];
        double v0 = (j == 0 || sl || lab_at(d, label, i, j - 1, k) == SOLID) ? 0.0 : v[fv0];
        double v1 = (j + 1 == ny || sl || lab_at(d, label, i, j + 1, k) == SOLID) ? 0.0 : v[fv1];
        double w0 = (k == 0 || sl || lab_at(d, label, i, j, k - 1) == SOLID) ? 0.0 : w[fw0];
        double w1 = (k + 1 == nz || sl || lab_at(d, label, i, j, k + 1) == SOLID) ? 0.0 : w[fw1];
        double div = (((((u1 - u0) + v1) - v0) + w1) - w0) / d->dtau;
        rhs[r] = -div;
    }
    free(par);
    free(has_air);
    return n;
}

/* ------------------------------------------------------------ solvers -- */
/* F/_kernels/_core.pyx:196-213 */
void orc_laplacian_matvec(int64_t n, const double *diag, const int64_t *nbr, const double *x,
                          double scale, double *y) {
    #pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; r++) {
        double s = 0.0;
        for (int q = 0; q < 6; q++) {
            int64_t c = nbr[r * 6 + q];
            if (c >= 0) s = s + x[c];
        }
        y[r] = scale * (diag[r] * x[r] - s);
    }
}

/* F/_kernels/_core.pyx:216-234 */
void orc_jacobi_iter(int64_t n, const double *diag, const int64_t *nbr, const double *rhs,
                     const double *x, double scale, double *out) {
    #pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; r++) {
        double s = 0.0;
        for (int q = 0; q < 6; q++) {
            int64_t c = nbr[r * 6 + q];
            if (c >= 0) s = s + x[c];
        }
        out[r] = (rhs[r] / scale + s) / diag[r];
    }
}

/* F/_kernels/_core.pyx:237-252 */
void orc_gs_sweep(int64_t n, const double *diag, const int64_t *nbr, const double *rhs,
                  double *x, double scale) {
    for (int64_t r = 0; r < n; r++) {
        double s = 0.0;
        for (int q = 0; q < 6; q++) {
            int64_t c = nbr[r * 6 + q];
            if (c >= 0) s += x[c];
        }
        x[r] = (rhs[r] / scale + s) / diag[r];
    }
}

/* F/_kernels/_core.pyx:255-272 */
void orc_gs_sweep_rows(int64_t m, const int64_t *rows, const double *diag, const int64_t *nbr,
                       const double *rhs, double *x, double scale) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; i++) {
        int64_t r = rows[i];
        double s = 0.0;
        for (int q = 0; q < 6; q++) {
            int64_t c = nbr[r * 6 + q];
            if (c >= 0) s = s + x[c];
        }
        x[r] = (rhs[r] / scale + s) / diag[r];
    }
}

/* F/_kernels/_core.pyx:275-308 */
void orc_mic0_build(int64_t n, const double *diag, const int64_t *nbr, double scale,
                    double tau, double sigma, double *precon) {
    static const int dprev[3] = {0, 2, 4}, o1[3] = {3, 1, 1}, o2[3] = {5, 5, 3};
    for (int64_t r = 0; r < n; r++) precon[r] = 0.0;
    for (int64_t r = 0; r < n; r++) {
        double e = diag[r] * scale;
        for (int p = 0; p < 3; p++) {
            int64_t q = nbr[r * 6 + dprev[p]];
            if (q >= 0) {
                double pq = precon[q];
                e -= (scale * pq) * (scale * pq);
                double others = 0.0;
                if (nbr[q * 6 + o1[p]] >= 0) others -= scale;
                if (nbr[q * 6 + o2[p]] >= 0) others -= scale;
                e -= tau * (-scale) * others * pq * pq;
            }
        }
        if (e < sigma * diag[r] * scale) e = diag[r] * scale;
        precon[r] = 1.0 / sqrt(e);
    }
}

/* F/_kernels/_core.pyx:311-347 */
void orc_mic0_apply(int64_t n, const double *precon, const int64_t *nbr, const double *r,
                    double scale, double *q, double *z) {
    for (int64_t i = 0; i < n; i++) {
        double t = r[i];
        int64_t nb = nbr[i * 6 + 0];
        if (nb >= 0) t += scale * precon[nb] * q[nb];
        nb = nbr[i * 6 + 2];
        if (nb >= 0) t += scale * precon[nb] * q[nb];
        nb = nbr[i * 6 + 4];
        if (nb >= 0) t += scale * precon[nb] * q[nb];
        q[i] = t * precon[i];
    }
    for (int64_t i = n - 1; i >= 0; i--) {
        double t = q[i];
        int64_t nb = nbr[i * 6 + 1];
        if (nb >= 0) t += scale * precon[i] * z[nb];
        nb = nbr[i * 6 + 3];
        if (nb >= 0) t += scale * precon[i] * z[nb];
        nb = nbr[i * 6 + 5];
        if (nb >= 0) t += scale * precon[i] * z[nb];
        z[i] = t * precon[i];
    }
}

/* numpy DOUBLE_pairwise_sum (numpy/_core/src/umath/loops_utils.h.src), which
 * np.add.reduce uses on a contiguous float64 array (verified bit-exact
 * against numpy 2.3 in tests/test_oracle_pins.py). */
static double pw_sum(const double *a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[j];
        int64_t i;
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
    }
}

double orc_pairwise_sum(int64_t n, const double *a) { return pw_sum(a, n); }

double orc_pairwise_dot(int64_t n, const double *a, const double *b) {
    double *tmp = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) tmp[i] = a[i] * b[i];
    double s = pw_sum(tmp, n);
    free(tmp);
    return s;
}

static double max_abs(int64_t n, const double *a) {
    double m = -INFINITY;
    #pragma omp parallel for reduction(max : m) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double v = fabs(a[i]);
        if (v > m) m = v;
    }
    return m;
}

/* F/pressure.py:185-193 */
static double solve_target(int64_t n, const double *rhs, double tol) {
    double rhs_max = n ? max_abs(n, rhs) : 0.0;
    return tol * (rhs_max > 1.0 ? rhs_max : 1.0);
}

/* F/pressure.py:200-332 */
int orc_solve(int kind, int precond, int64_t n, const int64_t *cells, const double *diag,
              const int64_t *nbr, const double *rhs, double scale, int64_t max_iters,
              double tol, const int64_t *red_rows, int64_t nred, const int64_t *black_rows,
              int64_t nblack, double *x, double *history, orc_solve_result *res) {
    memset(res, 0, sizeof(*res));
    res->err_cell = -1;
    for (int64_t r = 0; r < n; r++)
        if (!(diag[r] > 0)) {  /* _check_diagonal F/pressure.py:185-188 */
            res->err_cell = cells[r];
            return 1;
        }
    if (n == 0) {
        res->iterations = 0;
        res->residual = 0.0;
        res->converged = 1;
        return 0;
    }
    double target = solve_target(n, rhs, tol);
    size_t bytes = sizeof(double) * (size_t)n;
    for (int64_t i = 0; i < n; i++) x[i] = 0.0;
    if (kind != 3) {  /* _relaxation_solve F/pressure.py:200-220 */
        double *tmp = (double *)malloc(bytes), *y = (double *)malloc(bytes);
        double rr = INFINITY;
        int64_t it = 0;
        for (it = 1; it <= max_iters; it++) {
            if (kind == 0) {
                orc_jacobi_iter(n, diag, nbr, rhs, x, scale, tmp);
                memcpy(x, tmp, bytes);
            } else if (kind == 1) {
                orc_gs_sweep(n, diag, nbr, rhs, x, scale);
            } else {  /* red rows (parity 0) then black rows (F/pressure.py:259-263) */
                orc_gs_sweep_rows(nred, red_rows, diag, nbr, rhs, x, scale);
                orc_gs_sweep_rows(nblack, black_rows, diag, nbr, rhs, x, scale);
            }
            orc_laplacian_matvec(n, diag, nbr, x, scale, y);
            double m = -INFINITY;
            for (int64_t r = 0; r < n; r++) {
                double e = fabs(rhs[r] - y[r]);
                if (e > m) m = e;
            }
            rr = m;
            if (history) history[it - 1] = rr;
            if (rr <= target) break;
        }
        if (it > max_iters) it = max_iters;
        res->iterations = it;
        res->residual = rr;
        res->converged = rr <= target;
        free(tmp);
        free(y);
        return 0;
    }
    /* solve_pcg F/pressure.py:274-332 */
    double *r = (double *)malloc(bytes), *z = (double *)malloc(bytes), *s = (double *)malloc(bytes),
           *q = (double *)malloc(bytes), *pc = (double *)malloc(bytes), *tq = (double *)malloc(bytes);
    if (precond == 0) orc_mic0_build(n, diag, nbr, scale, 0.97, 0.25, pc);
    else if (precond == 1)
        for (int64_t i = 0; i < n; i++) pc[i] = 1.0 / (scale * diag[i]);
    memcpy(r, rhs, bytes);
    double rr = max_abs(n, r);
    int rc = 0;
    res->converged = 0;
    if (rr <= target) {
        res->iterations = 0;
        res->residual = rr;
        res->converged = 1;
        goto done;
    }
#define APPLY_PC(dst, src)                                                      \
    do {                                                                       \
        if (precond == 0) orc_mic0_apply(n, pc, nbr, src, scale, tq, dst);     \
        else if (precond == 1) {                                               \
            for (int64_t i_ = 0; i_ < n; i_++) dst[i_] = src[i_] * pc[i_];     \
        } else memcpy(dst, src, bytes);                                        \
    } while (0)
    APPLY_PC(z, r);
    memcpy(s, z, bytes);
    double sigma = orc_pairwise_dot(n, z, r);
    int64_t it;
    for (it = 1; it <= max_iters; it++) {
        orc_laplacian_matvec(n, diag, nbr, s, scale, q);
        double curv = orc_pairwise_dot(n, s, q);
        if (curv <= 0.0) {
            res->err_it = it;
            res->err_value = curv;
            rc = 2;
            goto done;
        }
        double alpha = sigma / curv;
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) {
            x[i] = x[i] + alpha * s[i];
            r[i] = r[i] - alpha * q[i];
        }
        rr = max_abs(n, r);
        if (history) history[it - 1] = rr;
        if (rr <= target) {
            res->iterations = it;
            res->residual = rr;
            res->converged = 1;
            goto done;
        }
        APPLY_PC(z, r);
        double sigma_new = orc_pairwise_dot(n, z, r);
        double beta = sigma_new / sigma;
        #pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < n; i++) s[i] = z[i] + beta * s[i];
        sigma = sigma_new;
    }
#undef APPLY_PC
    res->iterations = max_iters;
    res->residual = rr;
    res->converged = 0;
done:
    free(r); free(z); free(s); free(q); free(pc); free(tq);
    return rc;
}

/* -------------------------------------------------- gradient, G2P ------ */
/* F/pressure.py:343-380 */
void orc_apply_pressure_gradient(const orc_dims *d, const uint8_t *label, const double *p,
                                 double dt, double rho, double *u, double *v, double *w) {
    int64_t nx = d->nx, ny = d->ny, nz = d->nz, sxy = nx * ny;
    double scale = dt / (rho * d->dtau);
    /* u: axis x */
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nz; k++)
        for (int64_t j = 0; j < ny; j++)
            for (int64_t i = 0; i <= nx; i++) {
                int64_t f = i + j * (nx + 1) + k * (nx + 1) * ny;
                if (i == 0 || i == nx) { u[f] = 0.0; continue; }
                int64_t lo = (i - 1) + j * nx + k * sxy, hi = lo + 1;
                uint8_t a = label[lo], b = label[hi];
                if (a == SOLID || b == SOLID) u[f] = 0.0;
                else if (a == FLUID || b == FLUID) u[f] = u[f] - scale * (p[hi] - p[lo]);
            }
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nz; k++)
        for (int64_t j = 0; j <= ny; j++)
            for (int64_t i = 0; i < nx; i++) {
                int64_t f = i + j * nx + k * nx * (ny + 1);
                if (j == 0 || j == ny) { v[f] = 0.0; continue; }
                int64_t lo = i + (j - 1) * nx + k * sxy, hi = lo + nx;
                uint8_t a = label[lo], b = label[hi];
                if (a == SOLID || b == SOLID) v[f] = 0.0;
                else if (a == FLUID || b == FLUID) v[f] = v[f] - scale * (p[hi] - p[lo]);
            }
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k <= nz; k++)
        for (int64_t j = 0; j < ny; j++)
            for (int64_t i = 0; i < nx; i++) {
                int64_t f = i + j * nx + k * sxy;
                if (k == 0 || k == nz) { w[f] = 0.0; continue; }
                int64_t lo = i + j * nx + (k - 1) * sxy, hi = lo + sxy;
                uint8_t a = label[lo], b = label[hi];
                if (a == SOLID || b == SOLID) w[f] = 0.0;
                else if (a == FLUID || b == FLUID) w[f] = w[f] - scale * (p[hi] - p[lo]);
            }
}

/* F/transfer.py:60-82 */
void orc_g2p(const orc_dims *d, const double *un, const double *vn, const double *wn,
             const double *uo, const double *vo, const double *wo, int64_t n,
             const double *px, const double *py, const double *pz,
             double *vx, double *vy, double *vz, double f) {
    int64_t nx = d->nx, ny = d->ny, nz = d->nz;
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n; t++) {
        double gx = (px[t] - d->ox) / d->dtau;
        double gy = (py[t] - d->oy) / d->dtau;
        double gz = (pz[t] - d->oz) / d->dtau;
        double ax = tri_one(un, nx + 1, ny, nz, gx, gy - 0.5, gz - 0.5);
        double ay = tri_one(vn, nx, ny + 1, nz, gx - 0.5, gy, gz - 0.5);
        double az = tri_one(wn, nx, ny, nz + 1, gx - 0.5, gy - 0.5, gz);
        if (f == 0.0) {
            vx[t] = ax; vy[t] = ay; vz[t] = az;
            continue;
        }
        double bx = tri_one(uo, nx + 1, ny, nz, gx, gy - 0.5, gz - 0.5);
        double by = tri_one(vo, nx, ny + 1, nz, gx - 0.5, gy, gz - 0.5);
        double bz = tri_one(wo, nx, ny, nz + 1, gx - 0.5, gy - 0.5, gz);
        vx[t] = (1.0 - f) * ax + f * ((vx[t] + ax) - bx);
        vy[t] = (1.0 - f) * ay + f * ((vy[t] + ay) - by);
        vz[t] = (1.0 - f) * az + f * ((vz[t] + az) - bz);
    }
}

/* ------------------------------------------------------------- reseed -- */
/* F/particles.py:157-178 */
int64_t orc_reseed_counts(int64_t ncells, const int64_t *count, const uint8_t *label,
                          int64_t density, int64_t *n_add, int64_t *new_count,
                          int64_t *new_offset) {
    int64_t target = density * density * density;
    if (target > MAX_PER_CELL) target = MAX_PER_CELL;
    #pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < ncells; c++) {
        int64_t cnt = count[c];
        int64_t add = 0;
        if (label[c] == FLUID && cnt < MIN_PER_CELL) add = target - cnt > 0 ? target - cnt : 0;
        n_add[c] = add;
        new_count[c] = (cnt < MAX_PER_CELL ? cnt : MAX_PER_CELL) + add;
    }
    orc_exclusive_scan(ncells, new_count, new_offset);
    return ncells ? new_offset[ncells - 1] + new_count[ncells - 1] : 0;
}

/* F/particles.py:180-211 */
void orc_reseed_fill(const orc_dims *d, int64_t ncells, const int64_t *count,
                     const int64_t *offset, const int64_t *n_add, const int64_t *new_offset,
                     int64_t density, uint64_t seed, const double *in[6], double *out[6],
                     const double *u, const double *v, const double *w) {
    #pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t c = 0; c < ncells; c++) {
        int64_t cnt = count[c], keep = cnt < MAX_PER_CELL ? cnt : MAX_PER_CELL;
        int64_t src = offset[c], dst = new_offset[c];
        for (int64_t t = 0; t < keep; t++)
            for (int a = 0; a < 6; a++) out[a][dst + t] = in[a][src + t];
        int64_t add = n_add[c];
        for (int64_t j = 0; j < add; j++) {
            int64_t sub = cnt + j, at = dst + keep + j;
            double px, py, pz, vx, vy, vz;
            orc_jittered_positions(d, 1, &c, &sub, density, seed, &px, &py, &pz);
            orc_sample_velocity_many(d, u, v, w, 1, &px, &py, &pz, &vx, &vy, &vz);
            out[0][at] = px; out[1][at] = py; out[2][at] = pz;
            out[3][at] = vx; out[4][at] = vy; out[5][at] = vz;
        }
    }
}

/* F/grid.py:147-156 */
void orc_divergence_field(const orc_dims *d, const double *u, const double *v, const double *w,
                          double *div) {
    int64_t nx = d->nx, ny = d->ny, nz = d->nz, sxy = nx * ny;
    #pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nz; k++)
        for (int64_t j = 0; j < ny; j++)
            for (int64_t i = 0; i < nx; i++) {
                int64_t fu0 = i + j * (nx + 1) + k * (nx + 1) * ny;
                int64_t fv0 = i + j * nx + k * nx * (ny + 1);
                int64_t fw0 = i + j * nx + k * sxy;
                div[i + j * nx + k * sxy] =
                    (((((u[fu0 + 1] - u[fu0]) + v[fv0 + nx]) - v[fv0]) + w[fw0 + sxy]) - w[fw0]) / d->dtau;
            }
}
