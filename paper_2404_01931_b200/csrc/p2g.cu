// p2g.cu — particle-to-grid transfer as a deterministic per-face gather
// (flipsim/transfer.py:35-57 -> _kernels/_core.pyx:93-176), no atomics.
//
// Each thread owns one face of one component lattice and accumulates, with
// Kahan compensation, w*v and w over the particles of its candidate cells in
// the reference's order (cells z-outer, y, x-inner; particles in hash order).
// Because particles are cell-sorted, the candidate cells of one (y,z) row are
// one contiguous particle range [offset[first], offset[last+1]), so a face
// walks at most 9 contiguous ranges.  The epilogue fuses
// grid_old.copy_velocities_from (grid.py:104-107), the known mask
// (weights > 0, transfer.py:53), add_body_force (grid.py:193-202) and
// enforce_solid_boundaries (grid.py:219-228).
#include <climits>
#include <cstdlib>

#include "ops.cuh"

namespace flip {

struct FaceLattice {
    int fnx, fny, fnz;
    double offx, offy, offz;
};

__host__ __device__ inline FaceLattice lattice(const Dims &d, int comp) {
    if (comp == 0) return {d.nx + 1, d.ny, d.nz, 0.0, 0.5, 0.5};
    if (comp == 1) return {d.nx, d.ny + 1, d.nz, 0.5, 0.0, 0.5};
    return {d.nx, d.ny, d.nz + 1, 0.5, 0.5, 0.0};
}

// Face touches SOLID or lies on the domain boundary (grid.py:205-216).
__device__ __forceinline__ bool face_solid(const Dims &d, const uint8_t *__restrict__ label,
                                           int comp, int fi, int fj, int fk) {
    int64_t sxy = (int64_t)d.nx * d.ny;
    if (comp == 0) {
        if (fi == 0 || fi == d.nx) return true;
        int64_t hi = fi + (int64_t)fj * d.nx + fk * sxy;
        return label[hi - 1] == SOLID || label[hi] == SOLID;
    }
    if (comp == 1) {
        if (fj == 0 || fj == d.ny) return true;
        int64_t hi = fi + (int64_t)fj * d.nx + fk * sxy;
        return label[hi - d.nx] == SOLID || label[hi] == SOLID;
    }
    if (fk == 0 || fk == d.nz) return true;
    int64_t hi = fi + (int64_t)fj * d.nx + fk * sxy;
    return label[hi - sxy] == SOLID || label[hi] == SOLID;
}

struct P2GOut {
    double *grid;     // value (+ force, walls zeroed when fuse_force)
    double *old;      // raw value (grid_old), may be null
    uint8_t *known;   // weights > 0, may be null
    double *den;      // raw weights, may be null
};

// CONTIG: offset has ncells+1 entries and segments are back to back (a hash
// from bin_particles).  !CONTIG: generic (offset, count) pairs per cell like
// the Cython signature, used by the plugin API.
// MINB 5 (48 registers, no spill since the power-of-two test left the
// loop): P2G 6.44 -> 6.12 ms/step; 6 (40 registers): 6.29, 8: 7.38
__device__ __forceinline__ void ld_rec(const double *p, double &x, double &y, double &z, double &v) {
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(x), "=d"(y), "=d"(z), "=d"(v)
                 : "l"(p));
}

// REC: candidates read from the bin gather's records {x, y, z, v_comp} (one
// 256-bit load instead of four 8-byte loads: the walk is bound by L1
// wavefronts, ~16 per scattered 8-byte warp load); rec = px (+ 4 t).
template <bool CONTIG, int P2 = 0, int MINB = 5, bool REC = false>
__global__ void __launch_bounds__(kThreads, MINB)
k_p2g(Dims d, int comp, const double *__restrict__ px, const double *__restrict__ py,
      const double *__restrict__ pz, const double *__restrict__ vel,
      const int *__restrict__ offset, const int *__restrict__ count, P2GOut out,
      const uint8_t *__restrict__ label, const DevScalars *__restrict__ sc, double g,
      int fuse_force, unsigned f_lo, unsigned f_hi, int use_box) {
    FaceLattice L = lattice(d, comp);
    // 32-bit index math: flip_create rejects grids with >= 2^31 faces;
    // [f_lo, f_hi): all faces, or the own planes of a slab
    const unsigned nf = f_hi;
    int nx = d.nx, ny = d.ny, nz = d.nz;
    const int sxy = nx * ny;
    double gdt = 0.0;
    if (fuse_force && g != 0.0) gdt = g * sc->dt;
    // faces whose candidate cells all lie outside the box of the cells
    // holding particles (k_classify) gather nothing: num = dsum = 0, as the
    // loop over their empty ranges would give
    int blo[3] = {INT_MIN, INT_MIN, INT_MIN}, bhi[3] = {INT_MAX, INT_MAX, INT_MAX};
    if (use_box) {
#pragma unroll
        for (int a = 0; a < 3; a++) {
            blo[a] = sc->pbox_min[a] - 1;
            bhi[a] = sc->pbox_max[a] + 1;
        }
    }
    for (unsigned f = f_lo + blockIdx.x * blockDim.x + threadIdx.x; f < nf;
         f += gridDim.x * blockDim.x) {
        const unsigned fq = f / (unsigned)L.fnx;
        int fi = (int)(f - fq * (unsigned)L.fnx);
        int fj = (int)(fq % (unsigned)L.fny);
        int fk = (int)(fq / (unsigned)L.fny);
        double fpx = d.ox + ((double)fi + L.offx) * d.dtau;
        double fpy = d.oy + ((double)fj + L.offy) * d.dtau;
        double fpz = d.oz + ((double)fk + L.offz) * d.dtau;
        int cxlo = max(fi - 1, 0), cxhi = min(comp == 0 ? fi : fi + 1, nx - 1);
        int cylo = max(fj - 1, 0), cyhi = min(comp == 1 ? fj : fj + 1, ny - 1);
        int czlo = max(fk - 1, 0), czhi = min(comp == 2 ? fk : fk + 1, nz - 1);
        double num = 0.0, dsum = 0.0, cn = 0.0, cd = 0.0;
        const bool empty = fi < blo[0] || fi > bhi[0] || fj < blo[1] || fj > bhi[1] || fk < blo[2] ||
                           fk > bhi[2];
        if (empty) czhi = czlo - 1;  // no candidate rows
        for (int cz = czlo; cz <= czhi; cz++) {
            for (int cy = cylo; cy <= cyhi; cy++) {
                const int row = cy * nx + cz * sxy;
                int nseg = CONTIG ? 1 : cxhi - cxlo + 1;
                for (int sgi = 0; sgi < nseg; sgi++) {
                    int t0, t1;
                    if (CONTIG) {
                        t0 = __ldg(offset + row + cxlo);
                        t1 = __ldg(offset + row + cxhi + 1);
                    } else {
                        const int cell = row + cxlo + sgi;
                        t0 = __ldg(offset + cell);
                        t1 = t0 + __ldg(count + cell);
                    }
                    // two particles per trip with all eight loads issued up
                    // front (the loop is load-latency bound); the Kahan
                    // updates still run in particle order
                    auto kahan = [&](double wgt, double v) {
                        if (wgt > 0.0) {
                            double yk = wgt * v - cn;
                            double tk = num + yk;
                            cn = (tk - num) - yk;
                            num = tk;
                            yk = wgt - cd;
                            tk = dsum + yk;
                            cd = (tk - dsum) - yk;
                            dsum = tk;
                        }
                    };
                    auto weight = [&](double x, double y, double z) {
                        double hx = hat(div_dtau_t<P2>(d, x - fpx));
                        double hy = hat(div_dtau_t<P2>(d, y - fpy));
                        double hz = hat(div_dtau_t<P2>(d, z - fpz));
                        return (hx * hy) * hz;  // 0 whenever one factor is 0
                    };
                    int t = t0;
                    if (REC) {
                        for (; t + 1 < t1; t += 2) {
                            double x0, y0, z0, v0, x1, y1, z1, v1;
                            ld_rec(px + 4 * (int64_t)t, x0, y0, z0, v0);
                            ld_rec(px + 4 * (int64_t)(t + 1), x1, y1, z1, v1);
                            const double w0 = weight(x0, y0, z0), w1 = weight(x1, y1, z1);
                            kahan(w0, v0);
                            kahan(w1, v1);
                        }
                        if (t < t1) {
                            double x0, y0, z0, v0;
                            ld_rec(px + 4 * (int64_t)t, x0, y0, z0, v0);
                            kahan(weight(x0, y0, z0), v0);
                        }
                        continue;
                    }
                    for (; t + 1 < t1; t += 2) {
                        const double x0 = __ldg(px + t), x1 = __ldg(px + t + 1);
                        const double y0 = __ldg(py + t), y1 = __ldg(py + t + 1);
                        const double z0 = __ldg(pz + t), z1 = __ldg(pz + t + 1);
                        const double v0 = __ldg(vel + t), v1 = __ldg(vel + t + 1);
                        const double w0 = weight(x0, y0, z0), w1 = weight(x1, y1, z1);
                        kahan(w0, v0);
                        kahan(w1, v1);
                    }
                    if (t < t1) kahan(weight(__ldg(px + t), __ldg(py + t), __ldg(pz + t)), __ldg(vel + t));
                }
            }
        }
        double val = dsum > 0.0 ? num / dsum : 0.0;
        if (out.den) out.den[f] = dsum;
        if (out.old) out.old[f] = val;
        if (out.known) out.known[f] = dsum > 0.0;
        double gv = val;
        if (fuse_force) {
            if (g != 0.0) gv = val + gdt;
            if (face_solid(d, label, comp, fi, fj, fk)) gv = 0.0;
        }
        out.grid[f] = gv;
    }
}

void stage_p2g_impl(Ctx &c, const flip_step_params *prm, int fuse_force) {
    double *grid[3] = {c.u, c.v, c.w}, *old[3] = {c.uo, c.vo, c.wo};
    uint8_t *known[3] = {c.ku, c.kv, c.kw};
    int64_t nf[3] = {c.nfu, c.nfv, c.nfw};
    (void)nf;
    static const bool box_env = !getenv("FLIPB200_P2G_BOX") || atoi(getenv("FLIPB200_P2G_BOX"));
    const bool use_box = c.pbox_valid && !c.slab.on && box_env;
    for (int comp = 0; comp < 3; comp++) {
        P2GOut o{grid[comp], old[comp], known[comp], nullptr};
        double g = prm ? prm->gravity[comp] : 0.0;
        int64_t f_lo, f_hi;
        slab_face_range(c, comp, &f_lo, &f_hi);
        // the power-of-two test of div_dtau resolved at compile time: one
        // uniform branch and constant load less per hat (7.45 -> 6.50 ms/step)
        const bool rec = c.prec_valid && c.prec && !c.slab.on;
        static const int rec_minb = getenv("FLIPB200_P2G_REC_MINB") ? atoi(getenv("FLIPB200_P2G_REC_MINB")) : 5;
        auto kp = rec ? (rec_minb == 4 ? (c.d.pow2 ? k_p2g<true, 1, 4, true> : k_p2g<true, 0, 4, true>)
                                       : (c.d.pow2 ? k_p2g<true, 1, 5, true> : k_p2g<true, 0, 5, true>))
                      : (c.d.pow2 ? k_p2g<true, 1> : k_p2g<true, 0>);
        const double *rx = rec ? c.prec + (int64_t)comp * c.prec_cap * 4 : c.P.a[0];
        kp<<<nblocks(f_hi - f_lo, kThreads, (int64_t)1 << 30), kThreads, 0, c.st>>>(
            c.d, comp, rx, c.P.a[1], c.P.a[2], c.P.a[3 + comp], c.offset, nullptr, o,
            c.label, c.sc, g, fuse_force, (unsigned)f_lo, (unsigned)f_hi, use_box ? 1 : 0);
        c.launches++;
    }
    c.known_valid = 1;
    c.known_box = c.pbox_valid && !c.slab.on;  // known faces lie within the particle box + 1
}

void stage_p2g(Ctx &c, const flip_step_params &prm) { stage_p2g_impl(c, &prm, 0); }

void launch_p2g_component(const Dims &d, int comp, const double *vel, const double *px,
                          const double *py, const double *pz, const int *offset,
                          const int *count, double *out, double *den, cudaStream_t st) {
    FaceLattice L = lattice(d, comp);
    int64_t nf = (int64_t)L.fnx * L.fny * L.fnz;
    P2GOut o{out, nullptr, nullptr, den};
    k_p2g<false><<<nblocks(nf, kThreads, (int64_t)1 << 30), kThreads, 0, st>>>(
        d, comp, px, py, pz, vel, offset, count, o, nullptr, nullptr, 0.0, 0, 0u, (unsigned)nf, 0);
}

}  // namespace flip
