// mg.cu — geometric multigrid preconditioner for the pressure PCG
// (opt-in with precond = FLIP_PRECOND_MG).
//
// Not in the reference (which hard-wires MIC(0), pressure.py:274): results
// differ from it and are validated to the solver tolerance instead of bit
// for bit.  Everything here is data-parallel, which
// is the point: MIC(0) is a sequential recurrence whose sweeps dominate the
// step, and at 256^3 it stops at the 100-iteration cap unconverged.
//
// Cell-centred levels, coarsened by 2 down to 4 cells per axis.  A cell is a
// ROW (an unknown), DIRICHLET (air or a pinned cell: pressure 0) or SOLID.
// Level 0 follows the assembled system: ROW = a pressure row, diag = number
// of non-SOLID neighbours (outside the grid is SOLID), off-diagonals -1 to
// ROW neighbours, all times `scale` (pressure.py:134-166).  A coarse cell is
// ROW if any child is, SOLID if every child is, DIRICHLET otherwise; its
// operator is the same stencil rediscretised with scale / 4.  The V-cycle
// (damped Jacobi, w = 2/3, same count before and after; restriction = mean
// of the 8 children, prolongation = injection, so R = P^T / 8; a fixed
// Jacobi solve on the coarsest level) is a symmetric positive definite
// linear operator, as CG requires.
#include <cstdio>
#include <vector>

#include "ops.cuh"

namespace flip {

constexpr uint8_t MG_SOLID = 0, MG_DIR = 1, MG_ROW = 2;
constexpr int MG_MAXL = 12;

struct MgLevel {
    int nx = 0, ny = 0, nz = 0;     // this solve's extent (level 0: rows' box + 1-cell border)
    int64_t nc = 0;
    uint8_t *type = nullptr, *diag = nullptr;
    double *x = nullptr, *x2 = nullptr, *b = nullptr, *r = nullptr;
    double s = 0.0;  // operator scale at this level
    uint8_t open = 0;  // bit a (0..5: -x,+x,-y,+y,-z,+z): beyond the region on that side
                       // is interior (air-like, Dirichlet) rather than the domain wall
};

struct MgCtx {
    int L = 0;        // levels allocated (full-grid capacity)
    int Lrun = 0;     // levels used by the current solve
    int ox = 0, oy = 0, oz = 0;  // level-0 region origin in grid cells
    Dims d{};
    MgLevel lv[MG_MAXL];
    int pre = 2, post = 2, coarse = 24;
    double omega = 2.0 / 3.0;
};

static MgCtx *mg_ctx(Ctx &c) { return reinterpret_cast<MgCtx *>(c.mg); }

// level-0 types over the region [o, o + n) of the grid
__global__ void k_mg_type0(const uint8_t *__restrict__ label, const uint8_t *__restrict__ isrow,
                           Dims d, int ox, int oy, int oz, int nx, int ny, int nz,
                           uint8_t *__restrict__ type) {
    const int64_t nc = (int64_t)nx * ny * nz;
    for (int64_t q = gtid(); q < nc; q += gstride()) {
        const int i = (int)(q % nx) + ox, j = (int)((q / nx) % ny) + oy,
                  k = (int)(q / ((int64_t)nx * ny)) + oz;
        const int64_t c = i + (int64_t)j * d.nx + (int64_t)k * d.nx * d.ny;
        type[q] = isrow[c] ? MG_ROW : (label[c] == SOLID ? MG_SOLID : MG_DIR);
    }
}

__global__ void k_mg_coarsen(const uint8_t *__restrict__ tf, int fx, int fy, int fz,
                             uint8_t *__restrict__ tc, int cx, int cy, int cz) {
    const int64_t nc = (int64_t)cx * cy * cz;
    for (int64_t q = gtid(); q < nc; q += gstride()) {
        const int I = (int)(q % cx), J = (int)((q / cx) % cy), K = (int)(q / ((int64_t)cx * cy));
        bool row = false, all_solid = true;
        for (int k = 2 * K; k < min(2 * K + 2, fz); k++)
            for (int j = 2 * J; j < min(2 * J + 2, fy); j++)
                for (int i = 2 * I; i < min(2 * I + 2, fx); i++) {
                    const uint8_t t = tf[i + (int64_t)j * fx + (int64_t)k * fx * fy];
                    row |= t == MG_ROW;
                    all_solid &= t == MG_SOLID;
                }
        tc[q] = row ? MG_ROW : (all_solid ? MG_SOLID : MG_DIR);
    }
}

__device__ __forceinline__ uint8_t mg_t(const uint8_t *t, int nx, int ny, int nz, uint8_t open,
                                        int i, int j, int k) {
    if (i < 0) return (open & 1) ? MG_DIR : MG_SOLID;
    if (i >= nx) return (open & 2) ? MG_DIR : MG_SOLID;
    if (j < 0) return (open & 4) ? MG_DIR : MG_SOLID;
    if (j >= ny) return (open & 8) ? MG_DIR : MG_SOLID;
    if (k < 0) return (open & 16) ? MG_DIR : MG_SOLID;
    if (k >= nz) return (open & 32) ? MG_DIR : MG_SOLID;
    return t[i + (int64_t)j * nx + (int64_t)k * nx * ny];
}

__global__ void k_mg_diag(const uint8_t *__restrict__ t, int nx, int ny, int nz, uint8_t open,
                          uint8_t *__restrict__ diag) {
    const int64_t nc = (int64_t)nx * ny * nz;
    for (int64_t q = gtid(); q < nc; q += gstride()) {
        const int i = (int)(q % nx), j = (int)((q / nx) % ny), k = (int)(q / ((int64_t)nx * ny));
        int d = 0;
        d += mg_t(t, nx, ny, nz, open, i - 1, j, k) != MG_SOLID;
        d += mg_t(t, nx, ny, nz, open, i + 1, j, k) != MG_SOLID;
        d += mg_t(t, nx, ny, nz, open, i, j - 1, k) != MG_SOLID;
        d += mg_t(t, nx, ny, nz, open, i, j + 1, k) != MG_SOLID;
        d += mg_t(t, nx, ny, nz, open, i, j, k - 1) != MG_SOLID;
        d += mg_t(t, nx, ny, nz, open, i, j, k + 1) != MG_SOLID;
        diag[q] = (uint8_t)d;
    }
}

// (A x)_c for a ROW cell
__device__ __forceinline__ double mg_ax(const MgLevel &L, const double *__restrict__ x, int64_t q) {
    const int nx = L.nx, ny = L.ny, nz = L.nz;
    const int i = (int)(q % nx), j = (int)((q / nx) % ny), k = (int)(q / ((int64_t)nx * ny));
    const int64_t sy = nx, sz = (int64_t)nx * ny;
    double s = 0.0;
    if (i > 0 && L.type[q - 1] == MG_ROW) s += x[q - 1];
    if (i + 1 < nx && L.type[q + 1] == MG_ROW) s += x[q + 1];
    if (j > 0 && L.type[q - sy] == MG_ROW) s += x[q - sy];
    if (j + 1 < ny && L.type[q + sy] == MG_ROW) s += x[q + sy];
    if (k > 0 && L.type[q - sz] == MG_ROW) s += x[q - sz];
    if (k + 1 < nz && L.type[q + sz] == MG_ROW) s += x[q + sz];
    return L.s * ((double)L.diag[q] * x[q] - s);
}

// x_out = x + w D^-1 (b - A x) on ROW cells (x_in == nullptr: x = 0)
__global__ void k_mg_jacobi(MgLevel L, const double *__restrict__ xin, double *__restrict__ xout,
                            double w, const DevScalars *sc) {
    if (sc && sc->done) return;
    for (int64_t q = gtid(); q < L.nc; q += gstride()) {
        // an isolated coarse ROW cell (every neighbour SOLID, diag 0) has
        // no equation to relax: leave it at 0 instead of dividing by 0
        if (L.type[q] != MG_ROW || L.diag[q] == 0) {
            xout[q] = 0.0;
            continue;
        }
        const double dd = L.s * (double)L.diag[q];
        if (!xin) {
            xout[q] = w * L.b[q] / dd;
            continue;
        }
        xout[q] = xin[q] + w * (L.b[q] - mg_ax(L, xin, q)) / dd;
    }
}

__global__ void k_mg_residual(MgLevel L, const double *__restrict__ x, const DevScalars *sc) {
    if (sc && sc->done) return;
    for (int64_t q = gtid(); q < L.nc; q += gstride())
        L.r[q] = L.type[q] == MG_ROW ? L.b[q] - mg_ax(L, x, q) : 0.0;
}

__global__ void k_mg_restrict(MgLevel F, MgLevel Cl, const DevScalars *sc) {
    if (sc && sc->done) return;
    for (int64_t q = gtid(); q < Cl.nc; q += gstride()) {
        if (Cl.type[q] != MG_ROW) {
            Cl.b[q] = 0.0;
            continue;
        }
        const int I = (int)(q % Cl.nx), J = (int)((q / Cl.nx) % Cl.ny),
                  K = (int)(q / ((int64_t)Cl.nx * Cl.ny));
        double s = 0.0;
        for (int k = 2 * K; k < min(2 * K + 2, F.nz); k++)
            for (int j = 2 * J; j < min(2 * J + 2, F.ny); j++)
                for (int i = 2 * I; i < min(2 * I + 2, F.nx); i++)
                    s += F.r[i + (int64_t)j * F.nx + (int64_t)k * F.nx * F.ny];
        Cl.b[q] = 0.125 * s;
    }
}

__global__ void k_mg_prolong_add(MgLevel F, const double *__restrict__ xc, MgLevel Cl,
                                 double *__restrict__ x, const DevScalars *sc) {
    if (sc && sc->done) return;
    for (int64_t q = gtid(); q < F.nc; q += gstride()) {
        if (F.type[q] != MG_ROW) continue;
        const int i = (int)(q % F.nx), j = (int)((q / F.nx) % F.ny),
                  k = (int)(q / ((int64_t)F.nx * F.ny));
        x[q] += xc[(i >> 1) + (int64_t)(j >> 1) * Cl.nx + (int64_t)(k >> 1) * Cl.nx * Cl.ny];
    }
}

__device__ __forceinline__ int64_t mg_region(const Dims &d, int ox, int oy, int oz, int nx, int ny,
                                             int64_t c) {
    const int i = (int)(c % d.nx) - ox, j = (int)((c / d.nx) % d.ny) - oy,
              k = (int)(c / ((int64_t)d.nx * d.ny)) - oz;
    return i + (int64_t)j * nx + (int64_t)k * nx * ny;
}

__global__ void k_mg_scatter(const double *__restrict__ rrows, const int *__restrict__ cell_of_row,
                             int64_t n, Dims d, int ox, int oy, int oz, int nx, int ny,
                             double *__restrict__ b0, const DevScalars *sc) {
    if (sc && sc->done) return;
    for (int64_t r = gtid(); r < n; r += gstride())
        b0[mg_region(d, ox, oy, oz, nx, ny, cell_of_row[r])] = rrows[r];
}

__global__ void k_mg_gather(const double *__restrict__ x0, const int *__restrict__ cell_of_row,
                            int64_t n, Dims d, int ox, int oy, int oz, int nx, int ny,
                            double *__restrict__ zrows, const DevScalars *sc) {
    if (sc && sc->done) return;
    for (int64_t r = gtid(); r < n; r += gstride())
        zrows[r] = x0[mg_region(d, ox, oy, oz, nx, ny, cell_of_row[r])];
}

// Coarsest level in one CTA: all `sweeps` damped-Jacobi sweeps from x = 0
// in shared memory (same arithmetic and order as k_mg_jacobi, one launch).
constexpr int MG_COARSE_MAX = 2048;  // cells

__global__ void __launch_bounds__(1024) k_mg_coarse(MgLevel L, int sweeps, double w,
                                                    const DevScalars *sc) {
    if (sc && sc->done) return;
    __shared__ double xa[MG_COARSE_MAX], xb[MG_COARSE_MAX];
    const int nc = (int)L.nc;
    for (int q = threadIdx.x; q < nc; q += blockDim.x) xa[q] = 0.0;
    __syncthreads();
    double *cur = xa, *nxt = xb;
    for (int it = 0; it < sweeps; it++) {
        for (int q = threadIdx.x; q < nc; q += blockDim.x) {
            if (L.type[q] != MG_ROW || L.diag[q] == 0) {  // isolated: see k_mg_jacobi
                nxt[q] = 0.0;
                continue;
            }
            const double dd = L.s * (double)L.diag[q];
            if (it == 0) {
                nxt[q] = w * L.b[q] / dd;
                continue;
            }
            nxt[q] = cur[q] + w * (L.b[q] - mg_ax(L, cur, q)) / dd;
        }
        __syncthreads();
        double *t = cur;
        cur = nxt;
        nxt = t;
    }
    for (int q = threadIdx.x; q < nc; q += blockDim.x) L.x[q] = cur[q];
}

// ------------------------------------------------------------------ host --
void mg_free(Ctx &c) {
    MgCtx *m = mg_ctx(c);
    if (!m) return;
    for (int l = 0; l < m->L; l++) {
        MgLevel &L = m->lv[l];
        cudaFree(L.type);
        cudaFree(L.diag);
        cudaFree(L.x);
        cudaFree(L.x2);
        cudaFree(L.b);
        cudaFree(L.r);
    }
    delete m;
    c.mg = nullptr;
}

static int mg_alloc(Ctx &c) {
    if (c.mg) return 0;
    MgCtx *m = new MgCtx();
    int nx = c.d.nx, ny = c.d.ny, nz = c.d.nz;
    while (m->L < MG_MAXL) {
        MgLevel &L = m->lv[m->L];
        L.nx = nx;
        L.ny = ny;
        L.nz = nz;
        L.nc = (int64_t)nx * ny * nz;
        // capacity: the full grid at this level; the extent is set per solve
        if (cudaMalloc(&L.type, L.nc) || cudaMalloc(&L.diag, L.nc) ||
            cudaMalloc(&L.x, 8 * L.nc) || cudaMalloc(&L.x2, 8 * L.nc) ||
            cudaMalloc(&L.b, 8 * L.nc) || cudaMalloc(&L.r, 8 * L.nc)) {
            m->L++;
            c.mg = m;
            mg_free(c);
            set_error("multigrid allocation failed");
            return FLIP_E_CUDA;
        }
        m->L++;
        if (nx <= 4 || ny <= 4 || nz <= 4) break;
        nx = (nx + 1) / 2;
        ny = (ny + 1) / 2;
        nz = (nz + 1) / 2;
    }
    c.mg = m;
    return 0;
}

// Level types and diagonals from the current labels / rows (once per solve).
int mg_setup(Ctx &c, double scale, const int lo[3], const int hi[3], cudaStream_t st) {
    if (int rc = mg_alloc(c)) return rc;
    MgCtx *m = mg_ctx(c);
    m->d = c.d;
    // level 0: the rows' bounding box plus a one-cell border (every row's
    // neighbours inside, so its diagonal and stencil are exact); beyond it
    // the coarse levels see SOLID, which only shapes the preconditioner
    const int n3[3] = {c.d.nx, c.d.ny, c.d.nz};
    int o[3], e[3];
    for (int a = 0; a < 3; a++) {
        o[a] = lo[a] - 1 < 0 ? 0 : lo[a] - 1;
        const int h = hi[a] + 1 > n3[a] - 1 ? n3[a] - 1 : hi[a] + 1;
        e[a] = h - o[a] + 1;
    }
    m->ox = o[0];
    m->oy = o[1];
    m->oz = o[2];
    int nx = e[0], ny = e[1], nz = e[2];
    // sides where the region stops short of the domain (level 0 never looks
    // past its border; coarse levels treat beyond-the-region as Dirichlet)
    uint8_t open = 0;
    for (int a = 0; a < 3; a++) {
        if (o[a] > 0) open |= (uint8_t)(1 << (2 * a));
        if (o[a] + e[a] < n3[a]) open |= (uint8_t)(2 << (2 * a));
    }
    m->Lrun = 0;
    for (int l = 0; l < m->L; l++) {
        MgLevel &L = m->lv[l];
        L.nx = nx;
        L.ny = ny;
        L.nz = nz;
        L.nc = (int64_t)nx * ny * nz;
        L.open = l == 0 ? 0 : open;
        m->Lrun++;
        if (nx <= 4 || ny <= 4 || nz <= 4) break;
        nx = (nx + 1) / 2;
        ny = (ny + 1) / 2;
        nz = (nz + 1) / 2;
    }
    MgLevel &L0 = m->lv[0];
    k_mg_type0<<<nblocks(L0.nc), kThreads, 0, st>>>(c.label, c.isrow, c.d, m->ox, m->oy, m->oz,
                                                    L0.nx, L0.ny, L0.nz, L0.type);
    c.launches++;
    for (int l = 0; l < m->Lrun; l++) {
        MgLevel &L = m->lv[l];
        L.s = l == 0 ? scale : m->lv[l - 1].s * 0.25;
        if (l > 0) {
            MgLevel &F = m->lv[l - 1];
            k_mg_coarsen<<<nblocks(L.nc), kThreads, 0, st>>>(F.type, F.nx, F.ny, F.nz, L.type,
                                                             L.nx, L.ny, L.nz);
            c.launches++;
        }
        k_mg_diag<<<nblocks(L.nc), kThreads, 0, st>>>(L.type, L.nx, L.ny, L.nz, L.open, L.diag);
        c.launches++;
    }
    return 0;
}

// x_l = V-cycle(b_l); result in lv[l].x
static void vcycle(const MgCtx &m, int l, const DevScalars *sc, cudaStream_t st, int64_t *launches) {
    MgLevel L = m.lv[l];
    const bool last = l == m.Lrun - 1;
    if (last && L.nc <= MG_COARSE_MAX) {
        k_mg_coarse<<<1, 1024, 0, st>>>(L, m.coarse, m.omega, sc);
        (*launches)++;
        return;
    }
    const int pre = last ? m.coarse : m.pre;
    // damped Jacobi from x = 0, ping-pong between x and x2, ending in x
    double *cur = (pre % 2) ? L.x : L.x2, *nxt = (pre % 2) ? L.x2 : L.x;
    k_mg_jacobi<<<nblocks(L.nc), kThreads, 0, st>>>(L, nullptr, cur, m.omega, sc);
    for (int k = 1; k < pre; k++) {
        k_mg_jacobi<<<nblocks(L.nc), kThreads, 0, st>>>(L, cur, nxt, m.omega, sc);
        std::swap(cur, nxt);
    }
    *launches += pre;
    if (last) return;  // cur == L.x
    MgLevel C = m.lv[l + 1];
    k_mg_residual<<<nblocks(L.nc), kThreads, 0, st>>>(L, L.x, sc);
    k_mg_restrict<<<nblocks(C.nc), kThreads, 0, st>>>(L, C, sc);
    *launches += 2;
    vcycle(m, l + 1, sc, st, launches);
    k_mg_prolong_add<<<nblocks(L.nc), kThreads, 0, st>>>(L, C.x, C, L.x, sc);
    (*launches)++;
    cur = L.x;
    nxt = L.x2;
    for (int k = 0; k < m.post; k++) {
        k_mg_jacobi<<<nblocks(L.nc), kThreads, 0, st>>>(L, cur, nxt, m.omega, sc);
        std::swap(cur, nxt);
    }
    *launches += m.post;
    if (cur != L.x) {
        cudaMemcpyAsync(L.x, cur, 8 * L.nc, cudaMemcpyDeviceToDevice, st);
    }
}

// z = M^-1 r on the assembled rows
void mg_apply(Ctx &c, const double *r, double *z, int64_t n, const DevScalars *sc,
              cudaStream_t st, int64_t *launches) {
    MgCtx *m = mg_ctx(c);
    MgLevel &L0 = m->lv[0];
    cudaMemsetAsync(L0.b, 0, 8 * L0.nc, st);
    k_mg_scatter<<<nblocks(n), kThreads, 0, st>>>(r, c.cell_of_row, n, m->d, m->ox, m->oy, m->oz,
                                                  L0.nx, L0.ny, L0.b, sc);
    vcycle(*m, 0, sc, st, launches);
    k_mg_gather<<<nblocks(n), kThreads, 0, st>>>(L0.x, c.cell_of_row, n, m->d, m->ox, m->oy,
                                                 m->oz, L0.nx, L0.ny, z, sc);
    *launches += 2;
}

}  // namespace flip
