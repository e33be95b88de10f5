// grid.cu — face-lattice stages: body force + wall enforcement, pressure
// gradient subtract, layered velocity extrapolation, divergence.
#include <cstdlib>

#include "ops.cuh"

namespace flip {

struct Lat {
    int mx, my, mz;
};

__host__ __device__ inline Lat lat(const Dims &d, int comp) {
    if (comp == 0) return {d.nx + 1, d.ny, d.nz};
    if (comp == 1) return {d.nx, d.ny + 1, d.nz};
    return {d.nx, d.ny, d.nz + 1};
}

// (i, j, k) of face f with 32-bit unsigned division (face counts are below
// 2^31, checked by flip_create): two divides instead of three 64-bit ones.
__device__ __forceinline__ void lat_ijk(const Lat &L, unsigned f, int &i, int &j, int &k) {
    const unsigned q = f / (unsigned)L.mx;
    i = (int)(f - q * (unsigned)L.mx);
    const unsigned r = q / (unsigned)L.my;
    j = (int)(q - r * (unsigned)L.my);
    k = (int)r;
}
__device__ __forceinline__ unsigned ugtid() { return blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ unsigned ugstride() { return gridDim.x * blockDim.x; }

// Low/high cell of an interior face along its component axis; false on the
// domain boundary.
__device__ __forceinline__ bool face_cells(const Dims &d, int comp, int i, int j, int k,
                                           int64_t &lo, int64_t &hi) {
    int64_t sxy = (int64_t)d.nx * d.ny;
    hi = i + (int64_t)j * d.nx + k * sxy;
    if (comp == 0) {
        if (i == 0 || i == d.nx) return false;
        lo = hi - 1;
    } else if (comp == 1) {
        if (j == 0 || j == d.ny) return false;
        lo = hi - d.nx;
    } else {
        if (k == 0 || k == d.nz) return false;
        lo = hi - sxy;
    }
    return true;
}

// add_body_force (grid.py:193-202) then enforce_solid_boundaries (grid.py:219-228)
// over one component; force skipped when g == 0 or apply_force == 0.
__global__ void k_force_enforce(double *__restrict__ a, Dims d, int comp, double g,
                                const DevScalars *__restrict__ sc, int apply_force,
                                const uint8_t *__restrict__ label, unsigned f_lo, unsigned f_hi) {
    Lat L = lat(d, comp);
    const unsigned n = f_hi;
    double inc = (apply_force && g != 0.0) ? g * sc->dt : 0.0;
    for (unsigned f = f_lo + ugtid(); f < n; f += ugstride()) {
        int i, j, k;
        lat_ijk(L, f, i, j, k);
        int64_t lo, hi;
        bool solid = !face_cells(d, comp, i, j, k, lo, hi) || label[lo] == SOLID || label[hi] == SOLID;
        if (solid) a[f] = 0.0;
        else if (apply_force && g != 0.0) a[f] = a[f] + inc;
    }
}

void stage_force(Ctx &c, const flip_step_params &prm) {
    double *arr[3] = {c.u, c.v, c.w};
    int64_t nf[3] = {c.nfu, c.nfv, c.nfw};
    (void)nf;
    for (int comp = 0; comp < 3; comp++) {
        int64_t lo, hi;
        slab_face_range(c, comp, &lo, &hi);
        k_force_enforce<<<nblocks(hi - lo), kThreads, 0, c.st>>>(arr[comp], c.d, comp,
                                                                 prm.gravity[comp], c.sc, 1,
                                                                 c.label, (unsigned)lo,
                                                                 (unsigned)hi);
        c.launches++;
    }
}

// Faces that enforce_solid_boundaries zeroes (domain boundary or next to a
// SOLID cell): static while no label setter runs, so they are listed once
// (order irrelevant) and the per-step enforcement is a scatter of zeros.
__global__ void k_solid_faces(Dims d, int comp, const uint8_t *__restrict__ label,
                              int *__restrict__ list, unsigned long long *cnt) {
    Lat L = lat(d, comp);
    const unsigned n = (unsigned)L.mx * L.my * L.mz;
    for (unsigned f = ugtid(); f < n; f += ugstride()) {
        int i, j, k;
        lat_ijk(L, f, i, j, k);
        int64_t lo, hi;
        if (!face_cells(d, comp, i, j, k, lo, hi) || label[lo] == SOLID || label[hi] == SOLID) {
            const unsigned long long q = atomicAdd(cnt, 1ull);
            if (list) list[q] = (int)f;
        }
    }
}

__global__ void k_zero_list(double *__restrict__ a, const int *__restrict__ list, int64_t n) {
    for (int64_t t = gtid(); t < n; t += gstride()) a[list[t]] = 0.0;
}

static int build_solid_lists(Ctx &c) {
    unsigned long long cnt[3];
    FLIP_CUDA_OK(cudaMemsetAsync(c.u64_scratch, 0, 3 * sizeof(unsigned long long), c.st));
    for (int comp = 0; comp < 3; comp++) {
        Lat L = lat(c.d, comp);
        k_solid_faces<<<nblocks((int64_t)L.mx * L.my * L.mz), kThreads, 0, c.st>>>(
            c.d, comp, c.label, nullptr, c.u64_scratch + comp);
    }
    FLIP_CUDA_OK(cudaMemcpyAsync(cnt, c.u64_scratch, sizeof(cnt), cudaMemcpyDeviceToHost, c.st));
    FLIP_CUDA_OK(cudaStreamSynchronize(c.st));
    const int64_t total = (int64_t)(cnt[0] + cnt[1] + cnt[2]);
    if (total > c.solid_cap) {
        cudaFree(c.solid_list);
        c.solid_list = nullptr;
        c.solid_cap = 0;
        FLIP_CUDA_OK(cudaMalloc(&c.solid_list, sizeof(int) * (size_t)(total > 0 ? total : 1)));
        c.solid_cap = total;
    }
    FLIP_CUDA_OK(cudaMemsetAsync(c.u64_scratch, 0, 3 * sizeof(unsigned long long), c.st));
    int64_t off = 0;
    for (int comp = 0; comp < 3; comp++) {
        Lat L = lat(c.d, comp);
        k_solid_faces<<<nblocks((int64_t)L.mx * L.my * L.mz), kThreads, 0, c.st>>>(
            c.d, comp, c.label, c.solid_list + off, c.u64_scratch + comp);
        c.solid_off[comp] = off;
        c.solid_cnt[comp] = (int64_t)cnt[comp];
        off += (int64_t)cnt[comp];
    }
    c.launches += 6;
    c.faces_valid = 1;
    return 0;
}

void launch_enforce(Ctx &c, double *u, double *v, double *w) {
    if (!c.faces_valid && build_solid_lists(c) != 0) cudaGetLastError();  // else: full pass
    if (c.faces_valid) {
        double *arr[3] = {u, v, w};
        for (int comp = 0; comp < 3; comp++) {
            if (c.solid_cnt[comp] == 0) continue;
            k_zero_list<<<nblocks(c.solid_cnt[comp]), kThreads, 0, c.st>>>(
                arr[comp], c.solid_list + c.solid_off[comp], c.solid_cnt[comp]);
            c.launches++;
        }
        return;
    }
    double *arr[3] = {u, v, w};
    int64_t nf[3] = {c.nfu, c.nfv, c.nfw};
    for (int comp = 0; comp < 3; comp++) {
        k_force_enforce<<<nblocks(nf[comp]), kThreads, 0, c.st>>>(arr[comp], c.d, comp, 0.0, c.sc,
                                                                  0, c.label, 0u,
                                                                  (unsigned)nf[comp]);
        c.launches++;
    }
}

// apply_pressure_gradient (pressure.py:343-380): scale = dt / (rho*dtau).
__global__ void k_gradient(double *__restrict__ a, Dims d, int comp, const double *__restrict__ p,
                           const uint8_t *__restrict__ label, const DevScalars *__restrict__ sc,
                           double rho_dtau, unsigned f_lo, unsigned f_hi) {
    Lat L = lat(d, comp);
    const unsigned n = f_hi;
    double scale = sc->dt / rho_dtau;
    for (unsigned f = f_lo + ugtid(); f < n; f += ugstride()) {
        int i, j, k;
        lat_ijk(L, f, i, j, k);
        int64_t lo, hi;
        if (!face_cells(d, comp, i, j, k, lo, hi)) {
            a[f] = 0.0;
            continue;
        }
        uint8_t la = label[lo], lb = label[hi];
        if (la == SOLID || lb == SOLID) a[f] = 0.0;
        else if (la == FLUID || lb == FLUID) a[f] = a[f] - scale * (p[hi] - p[lo]);
    }
}

// One synchronous extrapolation layer (grid.py:231-263) on two arrays that
// share masks (grid and grid_old, sim.py:276-279).  Reads values only where
// kin is set and writes only where it is not, so the update is in place.
// Accumulation order: 0 + v(k+1) + v(k-1) + v(j+1) + v(j-1) + v(i+1) + v(i-1).
__global__ void k_extrap_layer(double *__restrict__ A, double *__restrict__ B, Lat L,
                               const uint8_t *__restrict__ kin, uint8_t *__restrict__ kout,
                               unsigned f_lo, unsigned f_hi) {
    const unsigned n = f_hi;
    const int64_t sy = L.mx, sz = (int64_t)L.mx * L.my;
    for (unsigned f = f_lo + ugtid(); f < n; f += ugstride()) {
        if (kin[f]) {
            kout[f] = 1;
            continue;
        }
        int i, j, k;
        lat_ijk(L, f, i, j, k);
        int64_t nb[6] = {f + sz, f - sz, f + sy, f - sy, f + 1, f - 1};
        bool ok[6] = {k + 1 < L.mz, k >= 1, j + 1 < L.my, j >= 1, i + 1 < L.mx, i >= 1};
        double a = 0.0, b = 0.0;
        int cnt = 0;
#pragma unroll
        for (int q = 0; q < 6; q++) {
            bool kn = ok[q] && kin[nb[q]];
            cnt += kn;
            a = a + (kn ? A[nb[q]] : 0.0);
            if (B) b = b + (kn ? B[nb[q]] : 0.0);
        }
        if (cnt > 0) {
            A[f] = a / (double)cnt;
            if (B) B[f] = b / (double)cnt;
            kout[f] = 1;
        } else {
            kout[f] = 0;
        }
    }
}

// k_extrap_layer over the faces that can change (one GPU, P2G known masks):
// every known face lies within the particle cell box grown by one face
// (a particle in cell c weights faces c, c+1 along the lattice's own axis and
// c-1..c+1 across it), so after layer l-1 the known faces lie within that box
// grown by l faces (V_l) and layer l fills faces within V_l grown by one
// (B_l).  Layer l visits B_l only, reads its input mask inside V_l only
// (outside it the face is unknown: for l >= 1 the scratch mask there is
// stale), and writes its output mask over B_l, which is V_{l+1}.  Faces
// outside B_l keep their values, as in the full-lattice kernel.  Same
// neighbour order and arithmetic.
__global__ void k_extrap_layer_box(double *__restrict__ A, double *__restrict__ B, Lat L,
                                   const uint8_t *__restrict__ kin, uint8_t *__restrict__ kout,
                                   const DevScalars *__restrict__ sc, int layer) {
    if (sc->pbox_max[0] < 0) return;  // no particles: nothing is known
    const int m[3] = {L.mx, L.my, L.mz};
    int lo[3], hi[3], vlo[3], vhi[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
        lo[a] = max(sc->pbox_min[a] - 2 - layer, 0);
        hi[a] = min(sc->pbox_max[a] + 2 + layer, m[a] - 1);
        vlo[a] = layer ? max(sc->pbox_min[a] - 1 - layer, 0) : 0;
        vhi[a] = layer ? min(sc->pbox_max[a] + 1 + layer, m[a] - 1) : m[a] - 1;
    }
    const unsigned bx = hi[0] - lo[0] + 1, by = hi[1] - lo[1] + 1, bz = hi[2] - lo[2] + 1;
    const unsigned V = bx * by * bz;
    const int64_t sy = L.mx, sz = (int64_t)L.mx * L.my;
    for (unsigned t = ugtid(); t < V; t += ugstride()) {
        const unsigned q = t / bx, r = q / by;
        const int i = lo[0] + (int)(t - q * bx), j = lo[1] + (int)(q - r * by), k = lo[2] + (int)r;
        const int64_t f = i + j * sy + k * sz;
        const bool in_v = i >= vlo[0] && i <= vhi[0] && j >= vlo[1] && j <= vhi[1] && k >= vlo[2] &&
                          k <= vhi[2];
        if (in_v && kin[f]) {
            kout[f] = 1;
            continue;
        }
        const int64_t nb[6] = {f + sz, f - sz, f + sy, f - sy, f + 1, f - 1};
        // the neighbour is inside V (hence inside the lattice) and known
        const bool ok[6] = {k + 1 <= vhi[2] && i >= vlo[0] && i <= vhi[0] && j >= vlo[1] && j <= vhi[1],
                            k - 1 >= vlo[2] && i >= vlo[0] && i <= vhi[0] && j >= vlo[1] && j <= vhi[1],
                            j + 1 <= vhi[1] && i >= vlo[0] && i <= vhi[0] && k >= vlo[2] && k <= vhi[2],
                            j - 1 >= vlo[1] && i >= vlo[0] && i <= vhi[0] && k >= vlo[2] && k <= vhi[2],
                            i + 1 <= vhi[0] && j >= vlo[1] && j <= vhi[1] && k >= vlo[2] && k <= vhi[2],
                            i - 1 >= vlo[0] && j >= vlo[1] && j <= vhi[1] && k >= vlo[2] && k <= vhi[2]};
        double a = 0.0, b = 0.0;
        int cnt = 0;
#pragma unroll
        for (int qn = 0; qn < 6; qn++) {
            const bool kn = ok[qn] && kin[nb[qn]];
            cnt += kn;
            a = a + (kn ? A[nb[qn]] : 0.0);
            if (B) b = b + (kn ? B[nb[qn]] : 0.0);
        }
        if (cnt > 0) {
            A[f] = a / (double)cnt;
            if (B) B[f] = b / (double)cnt;
            kout[f] = 1;
        } else {
            kout[f] = 0;
        }
    }
}

// pressure_field (pressure.py:49-53) is written by stage_project.
// Slab mode: every kernel covers the own face planes, and the face planes
// next to the slab are refreshed from the neighbours between the passes that
// read them (gradient -> layer 0 -> layer 1 -> ... -> enforce -> G2P).
int stage_apply_gradient(Ctx &c, const flip_step_params &prm) {
    double *g[3] = {c.u, c.v, c.w}, *o[3] = {c.uo, c.vo, c.wo};
    uint8_t *k0[3] = {c.ku, c.kv, c.kw};
    // scratch mask pairs: layer l reads (l == 0 ? P2G mask : s[(l-1)&1]), writes s[l&1]
    uint8_t *s0[3] = {c.ku1, c.kv1, c.kw1};
    uint8_t *s1[3] = {c.ku1 + c.nfu, c.kv1 + c.nfv, c.kw1 + c.nfw};
    int64_t lo[3], hi[3];
    for (int comp = 0; comp < 3; comp++) slab_face_range(c, comp, &lo[comp], &hi[comp]);
    for (int comp = 0; comp < 3; comp++) {
        k_gradient<<<nblocks(hi[comp] - lo[comp]), kThreads, 0, c.st>>>(
            g[comp], c.d, comp, c.p, c.label, c.sc, prm.rho_dtau_h, (unsigned)lo[comp],
            (unsigned)hi[comp]);
        c.launches++;
    }
    const int layers = prm.extrapolation_layers;
    // the layers visit the particle box only (FLIPB200_EXTRAP_BOX=0: every face)
    static const bool box_env = !getenv("FLIPB200_EXTRAP_BOX") || atoi(getenv("FLIPB200_EXTRAP_BOX"));
    const bool use_box = c.known_box && !c.slab.on && box_env;
    if (c.slab.on && layers > 0)
        if (int rc = slab_face_halo(c, SLAB_H_GRID)) return rc;
    for (int l = 0; l < layers; l++) {
        for (int comp = 0; comp < 3; comp++) {
            Lat L = lat(c.d, comp);
            const uint8_t *kin = l == 0 ? k0[comp] : ((l - 1) & 1 ? s1[comp] : s0[comp]);
            uint8_t *kout = (l & 1) ? s1[comp] : s0[comp];
            if (use_box)
                k_extrap_layer_box<<<nblocks(hi[comp] - lo[comp]), kThreads, 0, c.st>>>(
                    g[comp], o[comp], L, kin, kout, c.sc, l);
            else
                k_extrap_layer<<<nblocks(hi[comp] - lo[comp]), kThreads, 0, c.st>>>(
                    g[comp], o[comp], L, kin, kout, (unsigned)lo[comp], (unsigned)hi[comp]);
            c.launches++;
        }
        if (c.slab.on && l + 1 < layers)
            if (int rc = slab_face_halo(c, SLAB_H_GRID | SLAB_H_OLD |
                                               ((l & 1) ? SLAB_H_SCRATCH1 : SLAB_H_SCRATCH0)))
                return rc;
    }
    launch_enforce(c, c.u, c.v, c.w);
    // G2P and reseed sample both grids one plane beyond the slab
    if (c.slab.on)
        if (int rc = slab_face_halo(c, SLAB_H_GRID | SLAB_H_OLD)) return rc;
    return 0;
}

// divergence_field (grid.py:147-156)
__global__ void k_divergence(Dims d, const double *__restrict__ u, const double *__restrict__ v,
                             const double *__restrict__ w, double *__restrict__ div) {
    int64_t nc = d.ncells(), sxy = (int64_t)d.nx * d.ny;
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        int i, j, k;
        cell_ijk(d, c, i, j, k);
        int64_t fu = i + (int64_t)j * (d.nx + 1) + k * (int64_t)(d.nx + 1) * d.ny;
        int64_t fv = i + (int64_t)j * d.nx + k * (int64_t)d.nx * (d.ny + 1);
        int64_t fw = c;
        div[c] = (((((u[fu + 1] - u[fu]) + v[fv + d.nx]) - v[fv]) + w[fw + sxy]) - w[fw]) / d.dtau;
    }
}

void launch_divergence(Ctx &c, double *div_dev) {
    k_divergence<<<nblocks(c.ncells), kThreads, 0, c.st>>>(c.d, c.u, c.v, c.w, div_dev);
    c.launches++;
}

}  // namespace flip
