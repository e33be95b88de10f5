// particles.cu — particle-side stages: CFL dt, advection fused with the cell
// key + histogram, binning, classification, G2P, reseeding and scene seeding.
// Each kernel cites the reference function it re-implements; arithmetic is
// written in the reference's association order (see common.cuh).
#include <climits>
#include <cstdlib>

#include "ops.cuh"

namespace flip {

// ------------------------------------------------------------ compute_dt --
// flipsim/particles.py:214-224.  max is order-free -> atomicMax on bits.
__global__ void k_maxv2(ParticlePtrs P, int64_t n, unsigned long long *out) {
    double m = 0.0;
    for (int64_t t = gtid(); t < n; t += gstride()) {
        double vx = P.a[3][t], vy = P.a[4][t], vz = P.a[5][t];
        double s2 = ((vx * vx) + (vy * vy)) + (vz * vz);
        m = fmax(m, s2);
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomic_max_nonneg(out, m);
}

__global__ void k_dt_final(DevScalars *sc, double alpha_dtau, double dt_max) {
    double s_max = sqrt(__longlong_as_double((long long)sc->s2max_bits));
    double dt = dt_max;
    if (s_max != 0.0) {
        double cand = alpha_dtau / s_max;
        dt = cand < dt_max ? cand : dt_max;
    }
    sc->dt = dt;
}

int stage_dt(Ctx &c, const flip_step_params &prm) {
    cudaMemsetAsync(&c.sc->s2max_bits, 0, sizeof(unsigned long long), c.st);
    if (c.n > 0) {
        k_maxv2<<<nblocks(c.n), kThreads, 0, c.st>>>(c.P, c.n, &c.sc->s2max_bits);
        c.launches++;
    }
    // slab mode: max |v|^2 over every rank (a non-negative double: its bits
    // order like the value), so dt is the 1-GPU dt bit for bit
    if (c.slab.on)
        if (int rc = slab_allreduce(c, (int64_t *)&c.sc->s2max_bits, 1, FLIP_OP_MAX)) return rc;
    k_dt_final<<<1, 1, 0, c.st>>>(c.sc, prm.alpha_dtau_h, prm.dt_max);
    c.launches++;
    return 0;
}

// ---------------------------------------------------------------- advect --
// interior_box (flipsim/grid.py:121-132): bounding box of non-SOLID cells.
__global__ void k_box_reset(DevScalars *sc) {
    for (int a = 0; a < 3; a++) {
        sc->box_min[a] = 0x7fffffff;
        sc->box_max[a] = -1;
    }
}

__global__ void k_box_reduce(const uint8_t *__restrict__ label, Dims d, DevScalars *sc) {
    int64_t nc = d.ncells();
    int mn[3] = {0x7fffffff, 0x7fffffff, 0x7fffffff}, mx[3] = {-1, -1, -1};
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        if (label[c] == SOLID) continue;
        int i, j, k;
        cell_ijk(d, c, i, j, k);
        mn[0] = min(mn[0], i); mx[0] = max(mx[0], i);
        mn[1] = min(mn[1], j); mx[1] = max(mx[1], j);
        mn[2] = min(mn[2], k); mx[2] = max(mx[2], k);
    }
    for (int a = 0; a < 3; a++) {
        for (int o = 16; o; o >>= 1) {
            mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
        if ((threadIdx.x & 31) == 0 && mx[a] >= 0) {
            atomicMin(&sc->box_min[a], mn[a]);
            atomicMax(&sc->box_max[a], mx[a]);
        }
    }
}

__global__ void k_box_final(Dims d, DevScalars *sc) {
    double o[3] = {d.ox, d.oy, d.oz};
    for (int a = 0; a < 3; a++) {
        sc->lo[a] = o[a] + (double)sc->box_min[a] * d.dtau;
        sc->hi[a] = o[a] + (double)(sc->box_max[a] + 1) * d.dtau;
    }
}

// flipsim/particles.py:227-248 (forward Euler + per-axis clamp), fused with
// cell_index_many (binning.py:37-42) and the per-cell count (binning.py:90).
template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
k_advect_key(ParticlePtrs P, int64_t n, const DevScalars *__restrict__ sc,
                             double skin, Dims d, int *__restrict__ keys, int *__restrict__ count) {
    double dt = sc->dt;
    double lo[3] = {sc->lo[0], sc->lo[1], sc->lo[2]}, hi[3] = {sc->hi[0], sc->hi[1], sc->hi[2]};
    for (int64_t t = gtid(); t < n; t += gstride()) {
        double pos[3];
#pragma unroll
        for (int a = 0; a < 3; a++) {
            double q = P.a[a][t] + (P.a[3 + a][t] * dt);
            if (q <= lo[a]) q = lo[a] + skin;
            else if (q >= hi[a]) q = hi[a] - skin;
            P.a[a][t] = q;
            pos[a] = q;
        }
        int cell = cell_of(d, pos[0], pos[1], pos[2]);
        keys[t] = cell;
        atomicAdd(&count[cell], 1);
    }
}

// Extension (SceneSpec.advection = "rk2"): explicit-midpoint RK2 through
// the grid velocity field left by the previous step, then the reference's
// per-axis clamp; restated in oracle/flip_oracle.c (orc_advect_rk2).  The
// reference advects by forward Euler only (particles.py:227-248).
__global__ void k_advect_rk2_key(ParticlePtrs P, int64_t n, const DevScalars *__restrict__ sc,
                                 double skin, Dims d, const double *__restrict__ u,
                                 const double *__restrict__ v, const double *__restrict__ w,
                                 int *__restrict__ keys, int *__restrict__ count) {
    const double dt = sc->dt, h = 0.5 * dt;
    double lo[3] = {sc->lo[0], sc->lo[1], sc->lo[2]}, hi[3] = {sc->hi[0], sc->hi[1], sc->hi[2]};
    for (int64_t t = gtid(); t < n; t += gstride()) {
        double p[3] = {P.a[0][t], P.a[1][t], P.a[2][t]}, k1[3], k2[3], m[3];
        sample_vel(d, u, v, w, p[0], p[1], p[2], k1[0], k1[1], k1[2]);
#pragma unroll
        for (int a = 0; a < 3; a++) m[a] = p[a] + (k1[a] * h);
        sample_vel(d, u, v, w, m[0], m[1], m[2], k2[0], k2[1], k2[2]);
#pragma unroll
        for (int a = 0; a < 3; a++) {
            double q = p[a] + (k2[a] * dt);
            if (q <= lo[a]) q = lo[a] + skin;
            else if (q >= hi[a]) q = hi[a] - skin;
            P.a[a][t] = q;
            p[a] = q;
        }
        int cell = cell_of(d, p[0], p[1], p[2]);
        keys[t] = cell;
        atomicAdd(&count[cell], 1);
    }
}

void stage_advect(Ctx &c, const flip_step_params &prm) {
    // interior_box (grid.py:121-132) depends only on the SOLID cells, which no
    // stage changes: recomputed after a label setter invalidated it
    if (!c.box_valid) {
        k_box_reset<<<1, 1, 0, c.st>>>(c.sc);
        k_box_reduce<<<nblocks(c.ncells), kThreads, 0, c.st>>>(c.label, c.d, c.sc);
        k_box_final<<<1, 1, 0, c.st>>>(c.d, c.sc);
        c.launches += 3;
        c.box_valid = 1;
    }
    cudaMemsetAsync(c.count, 0, sizeof(int) * c.ncells, c.st);
    if (c.n > 0 && prm.advection == FLIP_ADVECT_RK2) {
        k_advect_rk2_key<<<nblocks(c.n), kThreads, 0, c.st>>>(c.P, c.n, c.sc, prm.skin_h, c.d, c.u,
                                                              c.v, c.w, c.keys0, c.count);
        c.launches++;
    } else if (c.n > 0) {
        // 8 CTAs/SM (32 registers): ADVECT 0.588 -> 0.351 ms (4: 0.475, 6: 0.413)
        static const int minb = getenv("FLIPB200_ADVECT_MINB") ? atoi(getenv("FLIPB200_ADVECT_MINB")) : 8;
        auto k = minb == 4 ? k_advect_key<4> : minb == 6 ? k_advect_key<6> : minb == 8 ? k_advect_key<8> : k_advect_key<3>;
        k<<<nblocks(c.n), kThreads, 0, c.st>>>(c.P, c.n, c.sc, prm.skin_h, c.d, c.keys0, c.count);
        c.launches++;
    }
}

// ------------------------------------------------------------------- bin --
// cell_index_many + bincount (binning.py:88-90) when advect did not run.
__global__ void k_keys_count(ParticlePtrs P, int64_t n, Dims d, int *__restrict__ keys,
                             int *__restrict__ count) {
    for (int64_t t = gtid(); t < n; t += gstride()) {
        int cell = cell_of(d, P.a[0][t], P.a[1][t], P.a[2][t]);
        keys[t] = cell;
        atomicAdd(&count[cell], 1);
    }
}

void stage_bin_from_keys(Ctx &c) {
    c.pbox_valid = 0;  // the counts change: k_classify recomputes the box
    c.prec_valid = 0;
    // offset = exclusive_scan(count) (binning.py:91); offset[ncells] = N
    exclusive_scan(ArrayIn{c.count}, c.ncells, c.offset, c.offset + c.ncells, c.scan_tmp, c.st);
    c.launches += 3;
    int *perm = nullptr;
    radix_sort_cells(c.keys0, c.keys1, c.vals0, c.vals1, c.n, c.ncells, c.hist, c.scan_tmp,
                     &c.sc->total, c.st, &c.keys_sorted, &perm, &c.launches);
    if (c.n > 0) {
        // P2G records alongside (one GPU, opt-in FLIPB200_P2G_REC=1): P2G 6.10 -> 5.40 ms
        // at 256^3, but the 2.5 GB of record stores cost BIN +0.46 ms and the step
        // comes out +0.1 ms, so the SoA walk stays the default
        static const bool rec_env = getenv("FLIPB200_P2G_REC") && atoi(getenv("FLIPB200_P2G_REC"));
        bool rec = rec_env && !c.slab.on;
        if (rec && c.n > c.prec_cap) {
            if (c.prec) cudaFree(c.prec);
            c.prec = nullptr;
            c.prec_cap = 0;
            const int64_t want = c.n + c.n / 4 + 4096;
            if (cudaMalloc(&c.prec, sizeof(double) * 12 * (size_t)want) == cudaSuccess) c.prec_cap = want;
            else cudaGetLastError();
        }
        rec = rec && c.prec;
        if (rec)
            k_gather6_rec<<<nblocks(c.n), kThreads, 0, c.st>>>(c.P, c.Q, perm, c.n, c.prec, c.prec_cap);
        else
            k_gather6<<<nblocks(c.n), kThreads, 0, c.st>>>(c.P, c.Q, perm, c.n);
        c.prec_valid = rec ? 1 : 0;
        c.launches++;
        std::swap(c.P, c.Q);
    }
    c.keys_valid = 1;
}

void stage_bin(Ctx &c) {
    cudaMemsetAsync(c.count, 0, sizeof(int) * c.ncells, c.st);
    if (c.n > 0) {
        k_keys_count<<<nblocks(c.n), kThreads, 0, c.st>>>(c.P, c.n, c.d, c.keys0, c.count);
        c.launches++;
    }
    stage_bin_from_keys(c);
}

// -------------------------------------------------------------- classify --
// flipsim/grid.py:185-190
// Also the box of the cells that hold particles (sc->pbox_*, BOX), which
// bounds the P2G known masks for the extrapolation (grid.cu).
template <bool BOX>
__global__ void k_classify(uint8_t *__restrict__ label, const int *__restrict__ count, int64_t nc,
                           Dims d, DevScalars *sc) {
    int mn[3] = {INT_MAX, INT_MAX, INT_MAX}, mx[3] = {-1, -1, -1};
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        uint8_t l = label[c];
        const int cnt = count[c];
        if (l != SOLID) label[c] = cnt > 0 ? FLUID : AIR;
        if (BOX && cnt > 0) {
            int ijk[3];
            cell_ijk(d, c, ijk[0], ijk[1], ijk[2]);
#pragma unroll
            for (int a = 0; a < 3; a++) {
                mn[a] = min(mn[a], ijk[a]);
                mx[a] = max(mx[a], ijk[a]);
            }
        }
    }
    if (!BOX) return;
    __shared__ int smn[3], smx[3];
    if (threadIdx.x < 3) {
        smn[threadIdx.x] = INT_MAX;
        smx[threadIdx.x] = -1;
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 3; a++) {
        for (int o = 16; o; o >>= 1) {
            mn[a] = min(mn[a], __shfl_xor_sync(0xffffffffu, mn[a], o));
            mx[a] = max(mx[a], __shfl_xor_sync(0xffffffffu, mx[a], o));
        }
        if ((threadIdx.x & 31) == 0 && mx[a] >= 0) {
            atomicMin(&smn[a], mn[a]);
            atomicMax(&smx[a], mx[a]);
        }
    }
    __syncthreads();
    if (threadIdx.x < 3 && smx[threadIdx.x] >= 0) {
        atomicMin(&sc->pbox_min[threadIdx.x], smn[threadIdx.x]);
        atomicMax(&sc->pbox_max[threadIdx.x], smx[threadIdx.x]);
    }
}

__global__ void k_pbox_reset(DevScalars *sc) {
    for (int a = 0; a < 3; a++) {
        sc->pbox_min[a] = INT_MAX;
        sc->pbox_max[a] = -1;
    }
}

void stage_classify(Ctx &c) {
    // slab mode: the own cells only (the other planes arrive by slab_labels)
    const int64_t c0 = c.slab.on ? c.slab_c0 : 0, c1 = c.slab.on ? c.slab_c1 : c.ncells;
    if (c.slab.on) {
        k_classify<false><<<nblocks(c1 - c0), kThreads, 0, c.st>>>(c.label + c0, c.count + c0,
                                                                   c1 - c0, c.d, c.sc);
        c.launches++;
        c.pbox_valid = 0;
        return;
    }
    k_pbox_reset<<<1, 1, 0, c.st>>>(c.sc);
    k_classify<true><<<nblocks(c.ncells), kThreads, 0, c.st>>>(c.label, c.count, c.ncells, c.d, c.sc);
    c.launches += 2;
    c.pbox_valid = 1;
}

// ------------------------------------------------------------------- G2P --
// flipsim/transfer.py:60-82 with sample_velocity_many (_core.pyx:68-90).
template <int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
k_g2p(ParticlePtrs P, int64_t n, Dims d, const double *__restrict__ un,
                      const double *__restrict__ vn, const double *__restrict__ wn,
                      const double *__restrict__ uo, const double *__restrict__ vo,
                      const double *__restrict__ wo, double f) {
    for (int64_t t = gtid(); t < n; t += gstride()) {
        double px = P.a[0][t], py = P.a[1][t], pz = P.a[2][t];
        double ax, ay, az;
        if (f == 0.0) {
            sample_vel(d, un, vn, wn, px, py, pz, ax, ay, az);
            P.a[3][t] = ax;
            P.a[4][t] = ay;
            P.a[5][t] = az;
            continue;
        }
        double bx, by, bz;
        sample_vel_pair(d, un, vn, wn, uo, vo, wo, px, py, pz, ax, ay, az, bx, by, bz);
        double g = 1.0 - f;
        P.a[3][t] = g * ax + f * ((P.a[3][t] + ax) - bx);
        P.a[4][t] = g * ay + f * ((P.a[4][t] + ay) - by);
        P.a[5][t] = g * az + f * ((P.a[5][t] + az) - bz);
    }
}

void stage_g2p(Ctx &c, const flip_step_params &prm) {
    if (c.n == 0) return;
    // 3 CTAs/SM (80 registers): 1.14 -> 0.93 ms/step at 256^3 (4: 0.98, 5 spills: 1.41,
    // unbounded 126 registers: 1.14)
    static const int minb = getenv("FLIPB200_G2P_MINB") ? atoi(getenv("FLIPB200_G2P_MINB")) : 3;
    auto k = minb == 4 ? k_g2p<4> : minb == 5 ? k_g2p<5> : minb == 3 ? k_g2p<3> : k_g2p<1>;
    k<<<nblocks(c.n), kThreads, 0, c.st>>>(c.P, c.n, c.d, c.u, c.v, c.w, c.uo, c.vo, c.wo,
                                           prm.flip_fraction);
    c.launches++;
}

__global__ void k_sample_many(Dims d, const double *__restrict__ u, const double *__restrict__ v,
                              const double *__restrict__ w, int64_t n, const double *px,
                              const double *py, const double *pz, double *vx, double *vy,
                              double *vz) {
    for (int64_t t = gtid(); t < n; t += gstride())
        sample_vel(d, u, v, w, px[t], py[t], pz[t], vx[t], vy[t], vz[t]);
}

void launch_sample_many(const Dims &d, const double *u, const double *v, const double *w,
                        int64_t n, const double *px, const double *py, const double *pz,
                        double *vx, double *vy, double *vz, cudaStream_t st) {
    if (n <= 0) return;
    k_sample_many<<<nblocks(n), kThreads, 0, st>>>(d, u, v, w, n, px, py, pz, vx, vy, vz);
}

// FLIP v1 snapshot payload (io.py:23-55): f64 SoA <-> f32 SoA
__global__ void k_to_f32(ParticlePtrs P, int64_t n, float *__restrict__ out) {
    for (int64_t t = gtid(); t < n; t += gstride())
#pragma unroll
        for (int a = 0; a < 6; a++) out[a * n + t] = __double2float_rn(P.a[a][t]);
}
__global__ void k_from_f32(ParticlePtrs P, int64_t n, const float *__restrict__ in) {
    for (int64_t t = gtid(); t < n; t += gstride())
#pragma unroll
        for (int a = 0; a < 6; a++) P.a[a][t] = (double)in[a * n + t];
}
void launch_particles_f32(Ctx &c, float *buf, bool to_f32) {
    if (c.n <= 0) return;
    if (to_f32) k_to_f32<<<nblocks(c.n), kThreads, 0, c.st>>>(c.P, c.n, buf);
    else k_from_f32<<<nblocks(c.n), kThreads, 0, c.st>>>(c.P, c.n, buf);
    c.launches++;
}

// cell_index_many of the current particles (flip_particle_cells)
__global__ void k_particle_cells(ParticlePtrs P, int64_t n, Dims d, int *__restrict__ out) {
    for (int64_t t = gtid(); t < n; t += gstride()) out[t] = cell_of(d, P.a[0][t], P.a[1][t], P.a[2][t]);
}

void launch_particle_cells(Ctx &c, int *out) {
    if (c.n <= 0) return;
    k_particle_cells<<<nblocks(c.n), kThreads, 0, c.st>>>(c.P, c.n, c.d, out);
    c.launches++;
}

// ---------------------------------------------------------------- reseed --
// flipsim/particles.py:157-178: per-cell refill/cull counts.
// Cells outside [c0, c1) (another rank's slab) are left alone.
__global__ void k_reseed_count(const int *__restrict__ count, const uint8_t *__restrict__ label,
                               int64_t nc, int density, int *__restrict__ nadd,
                               int *__restrict__ new_count, DevScalars *sc, int64_t c0, int64_t c1,
                               int *__restrict__ emit_cells) {
    int target = density * density * density;
    if (target > MAX_PER_CELL) target = MAX_PER_CELL;
    int changed = 0;
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        int cnt = count[c];
        int add = 0;
        if (label[c] == FLUID && cnt < MIN_PER_CELL && c >= c0 && c < c1)
            add = target - cnt > 0 ? target - cnt : 0;
        nadd[c] = add;
        new_count[c] = (cnt < MAX_PER_CELL ? cnt : MAX_PER_CELL) + add;
        if (add > 0 && emit_cells) {  // the refill list (warp-aggregated append)
            const unsigned am = __activemask();
            const int lane = threadIdx.x & 31, leader = __ffs(am) - 1;
            int base = 0;
            if (lane == leader) base = atomicAdd(&sc->emit_n, __popc(am));
            base = __shfl_sync(am, base, leader);
            emit_cells[base + __popc(am & ((1u << lane) - 1u))] = (int)c;
        }
        changed |= (add > 0) | (cnt > MAX_PER_CELL);
    }
    changed = __any_sync(0xffffffffu, changed);
    if (changed && (threadIdx.x & 31) == 0) sc->reseed_changed = 1;
}

// cells_of = np.repeat(arange(ncells), count) (particles.py:183)
__global__ void k_cells_from_hash(const int *__restrict__ offset, int64_t nc, int *__restrict__ cellp) {
    for (int64_t c = gtid(); c < nc; c += gstride())
        for (int t = offset[c]; t < offset[c + 1]; t++) cellp[t] = (int)c;
}

// Survivors keep their within-cell index (particles.py:180-189).
__global__ void k_reseed_copy(ParticlePtrs P, ParticlePtrs Q, int64_t n,
                              const int *__restrict__ cell_of_p, const int *__restrict__ offset,
                              const int *__restrict__ new_offset, const DevScalars *sc) {
    if (!sc->reseed_changed) return;
    for (int64_t t = gtid(); t < n; t += gstride()) {
        int c = cell_of_p[t];
        int within = (int)t - offset[c];
        if (within >= MAX_PER_CELL) continue;
        int64_t dst = (int64_t)new_offset[c] + within;
#pragma unroll
        for (int a = 0; a < 6; a++) Q.a[a][dst] = P.a[a][t];
    }
}

// New particles in the first free subcells, velocity sampled from the grid
// (particles.py:190-206).
__global__ void k_reseed_emit(ParticlePtrs Q, Dims d, const int *__restrict__ count,
                              const int *__restrict__ nadd, const int *__restrict__ new_offset,
                              int density, uint64_t seed, const double *__restrict__ u,
                              const double *__restrict__ v, const double *__restrict__ w,
                              const DevScalars *sc) {
    if (!sc->reseed_changed) return;
    // few cells refill: a block gathers the (cell, particle) jobs of a chunk
    // of kEmitChunk cells in shared memory and runs them densely (a warp per
    // refilled cell with one active lane was 273 us per step at 256^3)
    constexpr int kEmitChunk = 512;
    __shared__ int jobs[kEmitChunk * MAX_PER_CELL];
    __shared__ int njobs;
    const int64_t nc = d.ncells();
    for (int64_t c0 = (int64_t)blockIdx.x * kEmitChunk; c0 < nc; c0 += (int64_t)gridDim.x * kEmitChunk) {
        if (threadIdx.x == 0) njobs = 0;
        __syncthreads();
        for (int k = threadIdx.x; k < kEmitChunk && c0 + k < nc; k += blockDim.x) {
            const int add = nadd[c0 + k];
            if (add) {
                const int p = atomicAdd(&njobs, add);
                for (int j = 0; j < add; j++) jobs[p + j] = k << 4 | j;
            }
        }
        __syncthreads();
        for (int q = threadIdx.x; q < njobs; q += blockDim.x) {
            const int64_t c = c0 + (jobs[q] >> 4);
            const int j = jobs[q] & 15;
            const int cnt = count[c];
            double px, py, pz, vx, vy, vz;
            jitter_pos(d, c, cnt + j, density, seed, px, py, pz);
            sample_vel(d, u, v, w, px, py, pz, vx, vy, vz);
            const int64_t at = (int64_t)new_offset[c] + cnt + j;  // cnt < 3 <= MAX_PER_CELL
            Q.a[0][at] = px;
            Q.a[1][at] = py;
            Q.a[2][at] = pz;
            Q.a[3][at] = vx;
            Q.a[4][at] = vy;
            Q.a[5][at] = vz;
        }
        __syncthreads();
    }
}

// k_reseed_emit over k_reseed_count's list of refilled cells: one thread per
// cell, every thread busy (the per-cell scan left most lanes idle).  Output
// slots are fixed by new_offset, so the list order does not matter.
__global__ void k_reseed_emit_list(ParticlePtrs Q, Dims d, const int *__restrict__ count,
                                   const int *__restrict__ nadd, const int *__restrict__ new_offset,
                                   int density, uint64_t seed, const double *__restrict__ u,
                                   const double *__restrict__ v, const double *__restrict__ w,
                                   const DevScalars *sc, const int *__restrict__ cells) {
    if (!sc->reseed_changed) return;
    const int m = sc->emit_n;
    for (int q = (int)gtid(); q < m; q += (int)gstride()) {
        const int64_t c = cells[q];
        const int add = nadd[c], cnt = count[c];
        const int64_t base = (int64_t)new_offset[c] + cnt;  // cnt < 3 <= MAX_PER_CELL
        for (int j = 0; j < add; j++) {
            double px, py, pz, vx, vy, vz;
            jitter_pos(d, c, cnt + j, density, seed, px, py, pz);
            sample_vel(d, u, v, w, px, py, pz, vx, vy, vz);
            const int64_t at = base + j;
            Q.a[0][at] = px;
            Q.a[1][at] = py;
            Q.a[2][at] = pz;
            Q.a[3][at] = vx;
            Q.a[4][at] = vy;
            Q.a[5][at] = vz;
        }
    }
}

int stage_reseed(Ctx &c, const flip_step_params &prm) {
    c.pbox_valid = 0;
    int *new_count = c.count2, *new_offset = c.offset2, *nadd = c.nadd;
    cudaMemsetAsync(&c.sc->reseed_changed, 0, sizeof(int), c.st);
    static const bool list_env = !getenv("FLIPB200_RESEED_LIST") || atoi(getenv("FLIPB200_RESEED_LIST"));
    int *list = list_env ? c.emit_cells : nullptr;
    if (list) cudaMemsetAsync(&c.sc->emit_n, 0, sizeof(int), c.st);
    const int64_t c1 = c.slab_c1 < 0 ? c.ncells : c.slab_c1;
    k_reseed_count<<<nblocks(c.ncells), kThreads, 0, c.st>>>(c.count, c.label, c.ncells,
                                                             prm.density, nadd, new_count, c.sc,
                                                             c.slab_c0, c1, list);
    exclusive_scan(ArrayIn{new_count}, c.ncells, new_offset, new_offset + c.ncells, c.scan_tmp,
                   c.st);
    c.launches += 4;
    // Below the MAX_PER_CELL-per-cell bound a caller-chosen capacity can be
    // exceeded: read the new total and grow the particle buffers first
    // (growing drops the cell keys, rebuilt from the hash below).
    if (c.cap < (int64_t)MAX_PER_CELL * c.ncells) {
        int total = 0;
        FLIP_CUDA_OK(cudaMemcpyAsync(&total, new_offset + c.ncells, sizeof(int),
                                     cudaMemcpyDeviceToHost, c.st));
        FLIP_CUDA_OK(cudaStreamSynchronize(c.st));
        if (total > c.cap)
            if (int rc = reserve_particles(c, total)) return rc;
    }
    if (!c.keys_valid && c.n > 0) {  // cell of each binned particle from the hash
        k_cells_from_hash<<<nblocks(c.ncells), kThreads, 0, c.st>>>(c.offset, c.ncells, c.keys0);
        c.keys_sorted = c.keys0;
        c.keys_valid = 1;
        c.launches++;
    }
    if (c.n > 0) {
        k_reseed_copy<<<nblocks(c.n), kThreads, 0, c.st>>>(c.P, c.Q, c.n, c.keys_sorted, c.offset,
                                                           new_offset, c.sc);
        c.launches++;
    }
    if (list)
        k_reseed_emit_list<<<nblocks(c.ncells / 64 + 1, kThreads, 8), kThreads, 0, c.st>>>(
            c.Q, c.d, c.count, nadd, new_offset, prm.density, prm.reseed_seed, c.u, c.v, c.w, c.sc,
            list);
    else
        k_reseed_emit<<<nblocks((c.ncells + 1) / 2), kThreads, 0, c.st>>>(c.Q, c.d, c.count, nadd,
                                                                new_offset, prm.density,
                                                                prm.reseed_seed, c.u, c.v, c.w, c.sc);
    c.launches++;
    // the host swaps P<->Q and the hash buffers after reading reseed_changed
    return 0;
}

// --------------------------------------------------------------- seeding --
// set_solid_shell (flipsim/grid.py:110-118)
__global__ void k_solid_shell(uint8_t *label, Dims d) {
    int64_t nc = d.ncells();
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        int i, j, k;
        cell_ijk(d, c, i, j, k);
        if (i == 0 || j == 0 || k == 0 || i == d.nx - 1 || j == d.ny - 1 || k == d.nz - 1)
            label[c] = SOLID;
    }
}

__global__ void k_solid_box(uint8_t *label, Dims d, int i0, int i1, int j0, int j1, int k0, int k1) {
    int64_t nc = d.ncells();
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        int i, j, k;
        cell_ijk(d, c, i, j, k);
        if (i >= i0 && i <= i1 && j >= j0 && j <= j1 && k >= k0 && k <= k1) label[c] = SOLID;
    }
}

void launch_set_solid_box(Ctx &c, const int b[6]) {
    k_solid_box<<<nblocks(c.ncells), kThreads, 0, c.st>>>(c.label, c.d, b[0], b[1], b[2], b[3],
                                                           b[4], b[5]);
    c.launches++;
}

void launch_set_solid_shell(Ctx &c) {
    k_solid_shell<<<nblocks(c.ncells), kThreads, 0, c.st>>>(c.label, c.d);
    c.launches++;
}

// covered_cells (particles.py:103-110) with SeedRegion.contains (:92-100)
struct CoveredIn {
    Dims d;
    flip_region r;
    __device__ int operator()(int64_t idx) const {
        double cx = d.ox + ((double)(idx % d.nx) + 0.5) * d.dtau;
        double cy = d.oy + ((double)((idx / d.nx) % d.ny) + 0.5) * d.dtau;
        double cz = d.oz + ((double)(idx / ((int64_t)d.nx * d.ny)) + 0.5) * d.dtau;
        if (r.kind == 0)
            return cx >= r.a[0] && cx <= r.b[0] && cy >= r.a[1] && cy <= r.b[1] && cz >= r.a[2] &&
                   cz <= r.b[2];
        double dx = cx - r.a[0], dy = cy - r.a[1], dz = cz - r.a[2];
        return ((dx * dx) + (dy * dy)) + (dz * dz) <= r.radius * r.radius;
    }
};

__global__ void k_compact_covered(CoveredIn in, int64_t nc, const int *__restrict__ pos,
                                  int *__restrict__ cells) {
    for (int64_t c = gtid(); c < nc; c += gstride())
        if (in(c)) cells[pos[c]] = (int)c;
}

// seed (particles.py:133-149): region particles are cells x subcells, zero velocity.
__global__ void k_seed_emit(ParticlePtrs P, int64_t base, const int *__restrict__ cells, int64_t m,
                            int density, uint64_t seed, Dims d) {
    int nsub = density * density * density;
    int64_t total = m * nsub;
    for (int64_t t = gtid(); t < total; t += gstride()) {
        int64_t ci = t / nsub;
        int s = (int)(t - ci * nsub);
        double px, py, pz;
        jitter_pos(d, cells[ci], s, density, seed, px, py, pz);
        int64_t at = base + t;
        P.a[0][at] = px;
        P.a[1][at] = py;
        P.a[2][at] = pz;
        P.a[3][at] = 0.0;
        P.a[4][at] = 0.0;
        P.a[5][at] = 0.0;
    }
}

int seed_regions(Ctx &c, int nreg, const flip_region *regs, uint64_t seed) {
    int *pos = c.lvl, *cells = c.lvl_rows;
    for (int k = 0; k < nreg; k++) {
        const flip_region &r = regs[k];
        if (r.density < 1) {
            set_error("seed density must be >= 1");
            return FLIP_E_ARG;
        }
        CoveredIn in{c.d, r};
        exclusive_scan(in, c.ncells, pos, &c.sc->total, c.scan_tmp, c.st);
        k_compact_covered<<<nblocks(c.ncells), kThreads, 0, c.st>>>(in, c.ncells, pos, cells);
        c.launches += 4;
        int m = 0;
        FLIP_CUDA_OK(cudaMemcpyAsync(&m, &c.sc->total, sizeof(int), cudaMemcpyDeviceToHost, c.st));
        FLIP_CUDA_OK(cudaStreamSynchronize(c.st));
        int64_t add = (int64_t)m * r.density * r.density * r.density;
        if (int rc = reserve_particles(c, c.n + add)) return rc;
        if (add > 0) {
            k_seed_emit<<<nblocks(add), kThreads, 0, c.st>>>(c.P, c.n, cells, m, r.density, seed, c.d);
            c.launches++;
        }
        c.n += add;
    }
    return 0;
}

}  // namespace flip
