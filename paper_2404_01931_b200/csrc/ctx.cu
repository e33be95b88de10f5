// ctx.cu — the C ABI (include/flipb200.h): device context lifecycle, state
// transfer, the step orchestrator and the particle-side plugin kernels.
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "ops.cuh"
#include "wavefront.cuh"

namespace flip {

static thread_local std::string g_err;
static thread_local int64_t g_err_cell = -1;
void set_error(const std::string &msg) {
    g_err = msg;
    g_err_cell = -1;
}
void set_error_cell(int64_t cell) { g_err_cell = cell; }

int num_sms() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1)
            n = 148;
        cache[dev] = n;
    }
    return cache[dev];
}

int occupancy_per_sm(const void *fn, int threads) {
    // (kernel, device, threads) -> resident CTAs per SM; a handful of entries
    struct Ent { const void *fn; int dev, threads, per_sm; };
    static std::vector<Ent> cache;
    static std::mutex mu;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    for (const Ent &e : cache)
        if (e.fn == fn && e.dev == dev && e.threads == threads) return e.per_sm;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
    if (per_sm < 1) per_sm = 1;
    cache.push_back({fn, dev, threads, per_sm});
    return per_sm;
}

Dims make_dims(int64_t nx, int64_t ny, int64_t nz, double dtau, const double origin[3]) {
    Dims d{};
    d.nx = (int)nx;
    d.ny = (int)ny;
    d.nz = (int)nz;
    d.dtau = dtau;
    d.ox = origin ? origin[0] : 0.0;
    d.oy = origin ? origin[1] : 0.0;
    d.oz = origin ? origin[2] : 0.0;
    int e = 0;
    double m = std::frexp(dtau, &e);
    d.pow2 = (m == 0.5);
    d.inv_dtau = d.pow2 ? std::ldexp(1.0, 1 - e) : 1.0 / dtau;
    return d;
}

__global__ void k_fill_u8(uint8_t *a, int64_t n, uint8_t v) {
    for (int64_t i = gtid(); i < n; i += gstride()) a[i] = v;
}

__global__ void k_hash_from64(const long long *__restrict__ off, const long long *__restrict__ cnt,
                              int64_t nc, int *__restrict__ o32, int *__restrict__ c32) {
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        o32[c] = (int)off[c];
        c32[c] = (int)cnt[c];
        if (c == nc - 1) o32[nc] = (int)(off[c] + cnt[c]);
    }
}

__global__ void k_u8_from_any(const uint8_t *__restrict__ a, uint8_t *__restrict__ b, int64_t n) {
    for (int64_t i = gtid(); i < n; i += gstride()) b[i] = a[i] != 0;
}

struct PosIn {
    const int *count;
    __device__ int operator()(int64_t c) const { return count[c] > 0; }
};

__global__ void k_compact_pos(const int *__restrict__ count, int64_t nc, const int *__restrict__ pos,
                              long long *__restrict__ out) {
    for (int64_t c = gtid(); c < nc; c += gstride())
        if (count[c] > 0) out[pos[c]] = c;
}

__global__ void k_energy_terms(ParticlePtrs P, int64_t n, double floor_y, double *ke, double *pe) {
    for (int64_t t = gtid(); t < n; t += gstride()) {
        double vx = P.a[3][t], vy = P.a[4][t], vz = P.a[5][t];
        ke[t] = ((vx * vx) + (vy * vy)) + (vz * vz);  // sim.py:311-312
        pe[t] = P.a[1][t] - floor_y;                   // sim.py:314
    }
}

}  // namespace flip

using namespace flip;

struct flip_ctx : public Ctx {};

extern "C" const char *flip_last_error(void) { return g_err.c_str(); }
extern "C" int64_t flip_last_error_cell(void) { return g_err_cell; }

extern "C" int flip_device_count(int *count) {
    FLIP_CUDA_OK(cudaGetDeviceCount(count));
    return 0;
}

template <class T>
static int dalloc(T **p, int64_t n) {
    FLIP_CUDA_OK(cudaMalloc((void **)p, sizeof(T) * (size_t)(n > 0 ? n : 1)));
    return 0;
}

// Reallocate every particle-sized buffer for `cap` particles plus `front`
// entries before index 0 (the slab ghost plane below, slab.cu).  The live
// particles [0, n) are kept; the scratch buffers (Q, radix keys/values,
// histograms) are simply reallocated.
int flip::realloc_particles(Ctx &c, int64_t cap, int64_t front) {
    const int64_t lim = ((int64_t)1 << 31) - 1;
    if (cap + front > lim) {
        set_error("particle count exceeds the int32 indexing limit of one device");
        return FLIP_E_CAPACITY;
    }
    FLIP_CUDA_OK(cudaStreamSynchronize(c.st));
    for (int a = 0; a < 6; a++) {
        double *np_ = nullptr;
        if (int rc = dalloc(&np_, cap + front)) return rc;
        if (c.n > 0)
            FLIP_CUDA_OK(cudaMemcpyAsync(np_ + front, c.P.a[a], sizeof(double) * c.n,
                                         cudaMemcpyDeviceToDevice, c.st));
        FLIP_CUDA_OK(cudaStreamSynchronize(c.st));
        if (c.P.a[a]) cudaFree(c.P.a[a] - c.pfront);
        c.P.a[a] = np_ + front;
        if (c.Q.a[a]) cudaFree(c.Q.a[a] - c.pfront);
        c.Q.a[a] = nullptr;
        if (int rc = dalloc(&np_, cap + front)) return rc;
        c.Q.a[a] = np_ + front;
    }
    if (cap != c.cap) {
        int **ints[4] = {&c.keys0, &c.keys1, &c.vals0, &c.vals1};
        for (int **q : ints) {
            cudaFree(*q);
            *q = nullptr;
            if (int rc = dalloc(q, cap)) return rc;
        }
        cudaFree(c.hist);
        c.hist = nullptr;
        if (int rc = dalloc(&c.hist, radix_hist_ints(cap, c.ncells))) return rc;
        cudaFree(c.scan_tmp);
        c.scan_tmp = nullptr;
        const int64_t scan_n = std::max<int64_t>(radix_hist_ints(cap, c.ncells), c.ncells + 2);
        if (int rc = dalloc(&c.scan_tmp, scan_tmp_ints(scan_n) + 64)) return rc;
        c.keys_valid = 0;
        c.pbox_valid = 0;
        c.prec_valid = 0;
    }
    c.cap = cap;
    c.pfront = front;
    return 0;
}

// Grow every particle-sized buffer to hold at least n particles (the
// reference's ParticleSet has no fixed capacity).  Called before any launch
// that would exceed the capacity.
int flip::reserve_particles(Ctx &c, int64_t n) {
    if (n <= c.cap) return 0;
    const int64_t lim = ((int64_t)1 << 31) - 1;
    if (n > lim) {
        set_error("particle count exceeds the int32 indexing limit of one device");
        return FLIP_E_CAPACITY;
    }
    const int64_t cap = std::min(lim - c.pfront, std::max(n, c.cap + c.cap / 2));
    return realloc_particles(c, cap, c.pfront);
}

#define ALLOC(ptr, n)                                \
    do {                                             \
        if (int rc_ = dalloc(&(ptr), (int64_t)(n))) { \
            flip_destroy(c);                         \
            return rc_;                              \
        }                                            \
    } while (0)

extern "C" void flip_destroy(flip_ctx *c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->st) cudaStreamSynchronize(c->st);
    mg_free(*c);
    slab_free(*c);
    for (int a = 0; a < 6; a++) {
        if (c->P.a[a]) cudaFree(c->P.a[a] - c->pfront);
        if (c->Q.a[a]) cudaFree(c->Q.a[a] - c->pfront);
    }
    void *ptrs[] = {c->u, c->v, c->w, c->p,
                    c->label, c->uo, c->vo, c->wo, c->ku, c->kv, c->kw, c->ku1, c->kv1, c->kw1,
                    c->count, c->offset, c->count2, c->offset2, c->nadd, c->emit_cells, c->keys0, c->keys1,
                    c->vals0, c->vals1, c->hist, c->scan_tmp, c->rowscan, c->isrow, c->parent,
                    c->has_air, c->cell_of_row, c->nbr, c->diagd, c->rhs, c->x, c->r, c->z, c->s,
                    c->q, c->tq, c->precon, c->xtmp, c->u64_scratch, c->lvl, c->lvl_rows,
                    c->lvl_off, c->lvl_cnt, c->dot_part, c->wave_prog, c->wave_halo, c->cflags, c->wave_trace, c->lrow, c->posL, c->laneA, c->laneB, c->laneC, c->laneD, c->sc, c->f32_buf, c->nb_meta, c->nb_dy, c->nb_dz, c->solid_list};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (c->sch) cudaFreeHost(c->sch);
    if (c->prec) cudaFree(c->prec);
    if (c->probe.ts) cudaFree(c->probe.ts);
    if (c->probe.ts_host) cudaFreeHost(c->probe.ts_host);
    for (auto &e : c->ev)
        if (e) cudaEventDestroy(e);
    for (auto &e : c->probe.ev)
        if (e) cudaEventDestroy(e);
    if (c->st) cudaStreamDestroy(c->st);
    if (c->st2) {
        cudaStreamSynchronize(c->st2);
        cudaStreamDestroy(c->st2);
    }
    if (c->ev_fork) cudaEventDestroy(c->ev_fork);
    if (c->ev_side) cudaEventDestroy(c->ev_side);
    delete c;
}

extern "C" int flip_create(int device, int64_t nx, int64_t ny, int64_t nz, double dtau,
                           const double origin[3], int64_t capacity, flip_ctx **out) {
    *out = nullptr;
    if (nx < 1 || ny < 1 || nz < 1) {
        set_error("grid needs at least one cell per axis");
        return FLIP_E_ARG;
    }
    if (!(dtau > 0)) {
        set_error("cell size must be positive");
        return FLIP_E_ARG;
    }
    int64_t nc = nx * ny * nz;
    if (nc >= (int64_t)1 << 31 || (nx + 1) * ny * nz >= (int64_t)1 << 31) {
        set_error("grid too large for int32 indexing on one device (use slabs)");
        return FLIP_E_ARG;
    }
    FLIP_CUDA_OK(cudaSetDevice(device));
    flip_ctx *c = new flip_ctx();
    c->device = device;
    if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->st2, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming) != cudaSuccess) {
        set_error("cudaStreamCreate failed");
        flip_destroy(c);
        return FLIP_E_CUDA;
    }
    c->d = make_dims(nx, ny, nz, dtau, origin);
    c->ncells = nc;
    c->nfu = (nx + 1) * ny * nz;
    c->nfv = nx * (ny + 1) * nz;
    c->nfw = nx * ny * (nz + 1);
    if (capacity <= 0) capacity = 12 * nc;  // reseed bound: <= MAX_PER_CELL per cell
    if (capacity >= (int64_t)1 << 31) capacity = ((int64_t)1 << 31) - 1;
    c->cap = capacity;
    for (int a = 0; a < 6; a++) {
        ALLOC(c->P.a[a], capacity);
        ALLOC(c->Q.a[a], capacity);
    }
    ALLOC(c->u, c->nfu);
    ALLOC(c->v, c->nfv);
    ALLOC(c->w, c->nfw);
    ALLOC(c->p, nc);
    ALLOC(c->label, nc);
    ALLOC(c->uo, c->nfu);
    ALLOC(c->vo, c->nfv);
    ALLOC(c->wo, c->nfw);
    ALLOC(c->ku, c->nfu);
    ALLOC(c->kv, c->nfv);
    ALLOC(c->kw, c->nfw);
    ALLOC(c->ku1, 2 * c->nfu);
    ALLOC(c->kv1, 2 * c->nfv);
    ALLOC(c->kw1, 2 * c->nfw);
    ALLOC(c->count, nc + 1);
    ALLOC(c->offset, nc + 1);
    ALLOC(c->count2, nc + 1);
    ALLOC(c->offset2, nc + 1);
    ALLOC(c->nadd, nc + 1);
    ALLOC(c->emit_cells, nc + 1);
    ALLOC(c->keys0, capacity);
    ALLOC(c->keys1, capacity);
    ALLOC(c->vals0, capacity);
    ALLOC(c->vals1, capacity);
    ALLOC(c->hist, radix_hist_ints(capacity, nc));
    int64_t scan_n = std::max<int64_t>(radix_hist_ints(capacity, nc), nc + 2);
    ALLOC(c->scan_tmp, scan_tmp_ints(scan_n) + 64);
    ALLOC(c->rowscan, nc + 1);
    ALLOC(c->isrow, nc);
    ALLOC(c->parent, nc);
    ALLOC(c->has_air, nc);
    ALLOC(c->cell_of_row, nc);
    ALLOC(c->nbr, 6 * nc);
    ALLOC(c->nb_meta, nc);
    ALLOC(c->nb_dy, nc);
    ALLOC(c->nb_dz, nc);
    ALLOC(c->diagd, nc);
    ALLOC(c->rhs, nc);
    ALLOC(c->x, nc);
    ALLOC(c->r, nc);
    ALLOC(c->z, nc);
    ALLOC(c->s, nc);
    ALLOC(c->q, nc);
    ALLOC(c->tq, nc);
    ALLOC(c->precon, nc);
    ALLOC(c->xtmp, nc);
    ALLOC(c->u64_scratch, 4);
    int64_t nlev = nx + ny + nz + 2;
    ALLOC(c->lvl, nc);
    ALLOC(c->lvl_rows, nc);
    ALLOC(c->lvl_off, nlev + 1);
    ALLOC(c->lvl_cnt, nlev + 1);
    ALLOC(c->dot_part, dot_tmp_doubles(nc));
    // the fused pairwise dot keeps a ticket word in this scratch: start at 0
    FLIP_CUDA_OK(cudaMemsetAsync(c->dot_part, 0, sizeof(double) * dot_tmp_doubles(nc), c->st));
    ALLOC(c->wave_prog, 8);
    ALLOC(c->wave_halo, wave_halo_doubles(nx, ny, nz));
    ALLOC(c->cflags, nc);
    c->lane_cap = lane_entries_max(nx, ny, nz);
    ALLOC(c->lrow, c->lane_cap);
    ALLOC(c->posL, nc);
    ALLOC(c->laneA, c->lane_cap);
    ALLOC(c->laneB, c->lane_cap);
    ALLOC(c->laneC, c->lane_cap);
    ALLOC(c->laneD, c->lane_cap);
    ALLOC(c->wave_trace, 32768);
    ALLOC(c->sc, 1);
    if (cudaMallocHost((void **)&c->sch, sizeof(DevScalars)) != cudaSuccess) {
        set_error("cudaMallocHost failed");
        flip_destroy(c);
        return FLIP_E_CUDA;
    }
    for (auto &e : c->ev) cudaEventCreate(&e);
    // MacGrid(dims): zero velocities/pressure, every label AIR (grid.py:65-72)
    cudaMemsetAsync(c->u, 0, sizeof(double) * c->nfu, c->st);
    cudaMemsetAsync(c->v, 0, sizeof(double) * c->nfv, c->st);
    cudaMemsetAsync(c->w, 0, sizeof(double) * c->nfw, c->st);
    cudaMemsetAsync(c->uo, 0, sizeof(double) * c->nfu, c->st);
    cudaMemsetAsync(c->vo, 0, sizeof(double) * c->nfv, c->st);
    cudaMemsetAsync(c->wo, 0, sizeof(double) * c->nfw, c->st);
    cudaMemsetAsync(c->p, 0, sizeof(double) * nc, c->st);
    k_fill_u8<<<nblocks(nc), kThreads, 0, c->st>>>(c->label, nc, AIR);
    cudaMemsetAsync(c->count, 0, sizeof(int) * (nc + 1), c->st);
    cudaMemsetAsync(c->offset, 0, sizeof(int) * (nc + 1), c->st);
    cudaMemsetAsync(c->sc, 0, sizeof(DevScalars), c->st);
    if (cudaStreamSynchronize(c->st) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        set_error("device initialisation failed");
        flip_destroy(c);
        return FLIP_E_CUDA;
    }
    *out = c;
    return 0;
}

extern "C" int flip_synchronize(flip_ctx *c) {
    FLIP_CUDA_OK(cudaStreamSynchronize(c->st));
    FLIP_CUDA_OK(cudaGetLastError());
    return 0;
}

extern "C" int flip_get_stream(flip_ctx *c, void **stream) {
    *stream = (void *)c->st;
    return 0;
}

static int h2d(void *dst, const void *src, size_t bytes, cudaStream_t st) {
    if (!src || !bytes) return 0;
    FLIP_CUDA_OK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return 0;
}

static int d2h(void *dst, const void *src, size_t bytes, cudaStream_t st) {
    if (!dst || !bytes) return 0;
    FLIP_CUDA_OK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    return 0;
}

#define TRY(expr)                  \
    do {                           \
        if (int rc_ = (expr)) return rc_; \
    } while (0)

extern "C" int flip_set_grid(flip_ctx *c, const double *u, const double *v, const double *w,
                             const double *p, const uint8_t *label) {
    cudaSetDevice(c->device);
    TRY(h2d(c->u, u, sizeof(double) * c->nfu, c->st));
    TRY(h2d(c->v, v, sizeof(double) * c->nfv, c->st));
    TRY(h2d(c->w, w, sizeof(double) * c->nfw, c->st));
    TRY(h2d(c->p, p, sizeof(double) * c->ncells, c->st));
    TRY(h2d(c->label, label, c->ncells, c->st));
    c->box_valid = 0;
    c->faces_valid = 0;
    return flip_synchronize(c);
}

extern "C" int flip_get_grid(flip_ctx *c, double *u, double *v, double *w, double *p,
                             uint8_t *label) {
    cudaSetDevice(c->device);
    TRY(d2h(u, c->u, sizeof(double) * c->nfu, c->st));
    TRY(d2h(v, c->v, sizeof(double) * c->nfv, c->st));
    TRY(d2h(w, c->w, sizeof(double) * c->nfw, c->st));
    TRY(d2h(p, c->p, sizeof(double) * c->ncells, c->st));
    TRY(d2h(label, c->label, c->ncells, c->st));
    return flip_synchronize(c);
}

extern "C" int flip_set_grid_old(flip_ctx *c, const double *u, const double *v, const double *w) {
    cudaSetDevice(c->device);
    TRY(h2d(c->uo, u, sizeof(double) * c->nfu, c->st));
    TRY(h2d(c->vo, v, sizeof(double) * c->nfv, c->st));
    TRY(h2d(c->wo, w, sizeof(double) * c->nfw, c->st));
    return flip_synchronize(c);
}

extern "C" int flip_get_grid_old(flip_ctx *c, double *u, double *v, double *w) {
    cudaSetDevice(c->device);
    TRY(d2h(u, c->uo, sizeof(double) * c->nfu, c->st));
    TRY(d2h(v, c->vo, sizeof(double) * c->nfv, c->st));
    TRY(d2h(w, c->wo, sizeof(double) * c->nfw, c->st));
    return flip_synchronize(c);
}

extern "C" int flip_set_particles(flip_ctx *c, int64_t n, const double *px, const double *py,
                                  const double *pz, const double *vx, const double *vy,
                                  const double *vz) {
    cudaSetDevice(c->device);
    if (n < 0) {
        set_error("negative particle count");
        return FLIP_E_ARG;
    }
    TRY(reserve_particles(*c, n));
    const double *src[6] = {px, py, pz, vx, vy, vz};
    for (int a = 0; a < 6; a++) TRY(h2d(c->P.a[a], src[a], sizeof(double) * n, c->st));
    c->n = n;
    c->keys_valid = 0;
    c->pbox_valid = 0;
    c->prec_valid = 0;
    return flip_synchronize(c);
}

extern "C" int flip_get_particles(flip_ctx *c, double *px, double *py, double *pz, double *vx,
                                  double *vy, double *vz) {
    cudaSetDevice(c->device);
    double *dst[6] = {px, py, pz, vx, vy, vz};
    for (int a = 0; a < 6; a++) TRY(d2h(dst[a], c->P.a[a], sizeof(double) * c->n, c->st));
    return flip_synchronize(c);
}

extern "C" int flip_get_dev_ptrs(flip_ctx *c, flip_dev_ptrs *o) {
    for (int a = 0; a < 3; a++) {
        o->pos[a] = c->P.a[a];
        o->vel[a] = c->P.a[3 + a];
    }
    o->count = c->count;
    o->offset = c->offset;
    o->label = c->label;
    o->u = c->u;
    o->v = c->v;
    o->w = c->w;
    o->p = c->p;
    o->uo = c->uo;
    o->vo = c->vo;
    o->wo = c->wo;
    o->ku = c->ku;
    o->kv = c->kv;
    o->kw = c->kw;
    o->capacity = c->cap;
    o->n = c->n;
    return 0;
}

extern "C" int flip_reserve_particles(flip_ctx *c, int64_t n) {
    if (n < 0) {
        set_error("negative particle count");
        return FLIP_E_ARG;
    }
    cudaSetDevice(c->device);
    return reserve_particles(*c, n);
}

extern "C" int flip_set_particle_count(flip_ctx *c, int64_t n) {
    if (n < 0 || n > c->cap) {
        set_error("particle count exceeds capacity");
        return FLIP_E_CAPACITY;
    }
    c->n = n;
    c->keys_valid = 0;
    c->pbox_valid = 0;
    c->prec_valid = 0;
    return 0;
}

extern "C" int flip_set_slab(flip_ctx *c, int64_t k0, int64_t k1) {
    if (k0 < 0 || k1 > c->d.nz || k0 > k1) {
        set_error("slab planes out of range");
        return FLIP_E_ARG;
    }
    const int64_t plane = (int64_t)c->d.nx * c->d.ny;
    c->slab_c0 = k0 * plane;
    c->slab_c1 = k1 * plane;
    return 0;
}

extern "C" int flip_particle_cells(flip_ctx *c, int32_t *cells_dev) {
    cudaSetDevice(c->device);
    launch_particle_cells(*c, cells_dev);
    FLIP_CUDA_OK(cudaGetLastError());
    return 0;
}

// f32 staging for snapshots: allocated on first use, grown on demand, freed
// by flip_destroy.
static int f32_stage(flip_ctx *c, int64_t n, float **buf) {
    const size_t need = sizeof(float) * 6 * (size_t)(n > 0 ? n : 1);
    if (c->f32_cap < need) {
        if (c->f32_buf) cudaFree(c->f32_buf);
        c->f32_buf = nullptr;
        c->f32_cap = 0;
        FLIP_CUDA_OK(cudaMalloc(&c->f32_buf, need));
        c->f32_cap = need;
    }
    *buf = (float *)c->f32_buf;
    return 0;
}

extern "C" int flip_get_particles_f32(flip_ctx *c, float *out) {
    cudaSetDevice(c->device);
    float *buf;
    TRY(f32_stage(c, c->n, &buf));
    launch_particles_f32(*c, buf, true);
    TRY(d2h(out, buf, sizeof(float) * 6 * c->n, c->st));
    return flip_synchronize(c);
}

extern "C" int flip_set_particles_f32(flip_ctx *c, int64_t n, const float *in) {
    cudaSetDevice(c->device);
    if (n < 0) {
        set_error("negative particle count");
        return FLIP_E_ARG;
    }
    TRY(reserve_particles(*c, n));
    float *buf;
    TRY(f32_stage(c, n, &buf));
    TRY(h2d(buf, in, sizeof(float) * 6 * n, c->st));
    c->n = n;
    c->keys_valid = 0;
    c->pbox_valid = 0;
    c->prec_valid = 0;
    launch_particles_f32(*c, buf, false);
    return flip_synchronize(c);
}

extern "C" int flip_particle_count(flip_ctx *c, int64_t *n) {
    *n = c->n;
    return 0;
}

extern "C" int flip_set_hash(flip_ctx *c, const int64_t *offset, const int64_t *count) {
    cudaSetDevice(c->device);
    long long *o64 = nullptr, *c64 = nullptr;
    FLIP_CUDA_OK(cudaMalloc(&o64, sizeof(long long) * c->ncells));
    FLIP_CUDA_OK(cudaMalloc(&c64, sizeof(long long) * c->ncells));
    int rc = h2d(o64, offset, sizeof(int64_t) * c->ncells, c->st);
    if (!rc) rc = h2d(c64, count, sizeof(int64_t) * c->ncells, c->st);
    if (!rc) k_hash_from64<<<nblocks(c->ncells), kThreads, 0, c->st>>>(o64, c64, c->ncells, c->offset, c->count);
    if (!rc) rc = flip_synchronize(c);
    cudaFree(o64);
    cudaFree(c64);
    c->keys_valid = 0;
    c->pbox_valid = 0;
    c->prec_valid = 0;
    return rc;
}

extern "C" int flip_get_hash(flip_ctx *c, int64_t *offset, int64_t *count) {
    cudaSetDevice(c->device);
    std::vector<int> o(c->ncells), n(c->ncells);
    TRY(d2h(o.data(), c->offset, sizeof(int) * c->ncells, c->st));
    TRY(d2h(n.data(), c->count, sizeof(int) * c->ncells, c->st));
    TRY(flip_synchronize(c));
    for (int64_t i = 0; i < c->ncells; i++) {
        if (offset) offset[i] = o[i];
        if (count) count[i] = n[i];
    }
    return 0;
}

extern "C" int flip_get_fluid_cells(flip_ctx *c, int64_t *out, int64_t *nfluid) {
    cudaSetDevice(c->device);
    long long *d = nullptr;
    FLIP_CUDA_OK(cudaMalloc(&d, sizeof(long long) * c->ncells));
    PosIn in{c->count};
    exclusive_scan(in, c->ncells, c->lvl, &c->sc->total, c->scan_tmp, c->st);
    k_compact_pos<<<nblocks(c->ncells), kThreads, 0, c->st>>>(c->count, c->ncells, c->lvl, d);
    int m = 0;
    int rc = d2h(&m, &c->sc->total, sizeof(int), c->st);
    if (!rc) rc = flip_synchronize(c);
    if (!rc) rc = d2h(out, d, sizeof(long long) * m, c->st);
    if (!rc) rc = flip_synchronize(c);
    cudaFree(d);
    *nfluid = m;
    return rc;
}

extern "C" int flip_set_dt(flip_ctx *c, double dt) {
    cudaSetDevice(c->device);
    TRY(h2d(&c->sc->dt, &dt, sizeof(double), c->st));
    return flip_synchronize(c);
}

extern "C" int flip_get_dt(flip_ctx *c, double *dt) {
    cudaSetDevice(c->device);
    TRY(d2h(dt, &c->sc->dt, sizeof(double), c->st));
    return flip_synchronize(c);
}

extern "C" int flip_set_known(flip_ctx *c, const uint8_t *ku, const uint8_t *kv, const uint8_t *kw) {
    cudaSetDevice(c->device);
    TRY(h2d(c->ku, ku, c->nfu, c->st));
    TRY(h2d(c->kv, kv, c->nfv, c->st));
    TRY(h2d(c->kw, kw, c->nfw, c->st));
    c->known_valid = 1;
    c->known_box = 0;
    return flip_synchronize(c);
}

extern "C" int flip_get_known(flip_ctx *c, uint8_t *ku, uint8_t *kv, uint8_t *kw) {
    cudaSetDevice(c->device);
    TRY(d2h(ku, c->ku, c->nfu, c->st));
    TRY(d2h(kv, c->kv, c->nfv, c->st));
    TRY(d2h(kw, c->kw, c->nfw, c->st));
    return flip_synchronize(c);
}

extern "C" int flip_set_solid_shell(flip_ctx *c) {
    cudaSetDevice(c->device);
    launch_set_solid_shell(*c);
    c->box_valid = 0;
    c->faces_valid = 0;
    return flip_synchronize(c);
}

extern "C" int flip_set_solid_box(flip_ctx *c, int64_t i0, int64_t i1, int64_t j0, int64_t j1,
                                  int64_t k0, int64_t k1) {
    cudaSetDevice(c->device);
    const int64_t n[3] = {c->d.nx, c->d.ny, c->d.nz};
    int64_t lo[3] = {i0, j0, k0}, hi[3] = {i1, j1, k1};
    int b[6];
    for (int a = 0; a < 3; a++) {
        lo[a] = lo[a] < 0 ? 0 : lo[a];
        hi[a] = hi[a] > n[a] - 1 ? n[a] - 1 : hi[a];
        if (lo[a] > hi[a]) return 0;  // empty after clipping
        b[2 * a] = (int)lo[a];
        b[2 * a + 1] = (int)hi[a];
    }
    launch_set_solid_box(*c, b);
    c->box_valid = 0;
    c->faces_valid = 0;
    return flip_synchronize(c);
}

extern "C" int flip_seed_regions(flip_ctx *c, int32_t nregions, const flip_region *regions,
                                 uint64_t rng_seed) {
    cudaSetDevice(c->device);
    TRY(seed_regions(*c, nregions, regions, rng_seed));
    c->keys_valid = 0;
    c->pbox_valid = 0;
    c->prec_valid = 0;
    return flip_synchronize(c);
}

// Runs stages [first, last] in reference order (sim.py:233-292).
extern "C" int flip_run_stages(flip_ctx *c, const flip_step_params *prm, int32_t first, int32_t last,
                               flip_step_report *rep) {
    cudaSetDevice(c->device);
    flip_step_report local{};
    if (!rep) rep = &local;
    std::memset(rep, 0, sizeof(*rep));
    if (first < 0 || last >= FLIP_NSTAGES || first > last) {
        set_error("bad stage range");
        return FLIP_E_ARG;
    }
    if (prm->solver < 0 || prm->solver > 3 || prm->precond < 0 || prm->precond > FLIP_PRECOND_MG) {
        set_error("unknown solver or preconditioner");
        return FLIP_E_CONFIG;
    }
    if (c->slab.on && prm->advection == FLIP_ADVECT_RK2) {
        // the RK2 midpoint samples the grid up to 1.5 cells beyond the slab:
        // the 1-plane halos do not cover it
        set_error("RK2 advection is not supported with a slab decomposition");
        return FLIP_E_CONFIG;
    }
    int64_t launches0 = c->launches;
    bool keys_from_advect = false, force_fused = false, reseed_ran = false;
    int status = 0;
    c->proj_pre = 0;
    // a prefetched pressure structure (project_prefetch, side stream) that
    // stage_project did not consume (an error between P2G and PROJECT): the
    // main stream waits for it, so no later call races with the side stream
    struct SideJoin {
        flip_ctx *c;
        ~SideJoin() {
            if (c->proj_pre) {
                cudaStreamWaitEvent(c->st, c->ev_side, 0);
                c->proj_pre = 0;
            }
        }
    } side_join{c};
    // NVTX: one range per stage (StageTimings keys, sim.py:24-46), visible
    // to nsys / ncu --nvtx; a no-op without an attached tool
    static const char *kStageNames[FLIP_NSTAGES] = {
        "flip/dt_compute", "flip/advect", "flip/bin", "flip/classify", "flip/p2g",
        "flip/force", "flip/project", "flip/apply_gradient", "flip/g2p", "flip/reseed"};
    struct NvtxRange {
        bool on = false;
        void push(const char *n) { nvtxRangePushA(n); on = true; }
        ~NvtxRange() { if (on) nvtxRangePop(); }
    };
    for (int s = first; s <= last && !status; s++) {
        NvtxRange nv;
        nv.push(kStageNames[s]);
        cudaEventRecord(c->ev[s], c->st);
        switch (s) {
            case FLIP_STAGE_DT:
                if (int rc = stage_dt(*c, *prm)) return rc;
                break;
            case FLIP_STAGE_ADVECT:
                stage_advect(*c, *prm);
                if (c->slab.on) {  // particles to the rank owning their new cell
                    if (int rc = slab_migrate(*c)) return rc;
                } else {
                    keys_from_advect = true;
                }
                break;
            case FLIP_STAGE_BIN:
                if (keys_from_advect) stage_bin_from_keys(*c);
                else stage_bin(*c);
                break;
            case FLIP_STAGE_CLASSIFY:
                stage_classify(*c);
                if (c->slab.on)
                    if (int rc = slab_labels(*c)) return rc;
                break;
            case FLIP_STAGE_P2G:
                force_fused = last >= FLIP_STAGE_FORCE;
                if (c->slab.on)
                    if (int rc = slab_ghosts(*c)) return rc;
                // the pressure system's structure depends on the labels only:
                // built on the side stream while P2G runs
                if (last >= FLIP_STAGE_PROJECT) project_prefetch(*c);
                stage_p2g_impl(*c, prm, force_fused ? 1 : 0);
                if (c->slab.on) {
                    slab_ghosts_clear(*c);
                    if (int rc = slab_face_halo(*c, SLAB_H_GRID | SLAB_H_OLD | SLAB_H_KNOWN))
                        return rc;
                }
                break;
            case FLIP_STAGE_FORCE:
                if (!force_fused) {
                    stage_force(*c, *prm);
                    if (c->slab.on)
                        if (int rc = slab_face_halo(*c, SLAB_H_GRID)) return rc;
                }
                break;
            case FLIP_STAGE_PROJECT: {
                int rc = stage_project(*c, *prm, rep);
                if (rc) return rc;
                status = rep->status;
                break;
            }
            case FLIP_STAGE_APPLY_GRADIENT:
                if (!c->known_valid) {
                    set_error("apply_gradient needs the P2G known masks (run P2G or flip_set_known)");
                    return FLIP_E_ARG;
                }
                if (int rc = stage_apply_gradient(*c, *prm)) return rc;
                break;
            case FLIP_STAGE_G2P:
                stage_g2p(*c, *prm);
                break;
            case FLIP_STAGE_RESEED:
                if (int rc = stage_reseed(*c, *prm)) return rc;
                reseed_ran = true;
                break;
        }
        cudaEventRecord(c->ev[s + 1], c->st);
    }
    if (reseed_ran)
        cudaMemcpyAsync(&c->sc->new_total, c->offset2 + c->ncells, sizeof(int),
                        cudaMemcpyDeviceToDevice, c->st);
    cudaMemcpyAsync(c->sch, c->sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, c->st);
    FLIP_CUDA_OK(cudaStreamSynchronize(c->st));
    FLIP_CUDA_OK(cudaGetLastError());
    if (reseed_ran && c->sch->reseed_changed) {
        std::swap(c->P, c->Q);
        std::swap(c->count, c->count2);
        std::swap(c->offset, c->offset2);
        c->n = c->sch->new_total;
        c->keys_valid = 0;
        c->pbox_valid = 0;
        c->prec_valid = 0;
    }
    int stop = status ? FLIP_STAGE_PROJECT : last;
    for (int s = first; s <= stop; s++) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, c->ev[s], c->ev[s + 1]);
        rep->stage_ms[s] = ms;
    }
    rep->dt = c->sch->dt;
    rep->particle_count = c->n;
    rep->gpu_launches = c->launches - launches0;
    if (status) {
        set_error(status == FLIP_E_SINGULAR ? "singular pressure system" : "conjugate-gradient breakdown");
        if (status == FLIP_E_SINGULAR) set_error_cell(rep->err_cell);
        return status;
    }
    return 0;
}

extern "C" int flip_step(flip_ctx *c, const flip_step_params *prm, flip_step_report *rep) {
    return flip_run_stages(c, prm, 0, FLIP_NSTAGES - 1, rep);
}

// Debug/test access to internal device buffers by name (bytes clipped to the
// buffer size); used by the parity tests to localise mismatches.
extern "C" int flip_debug_copy(flip_ctx *c, const char *name, void *host, int64_t bytes) {
    cudaSetDevice(c->device);
    struct E {
        const char *n;
        const void *p;
        int64_t sz;
    } tab[] = {{"precon", c->precon, 8 * c->ncells}, {"x", c->x, 8 * c->ncells},
               {"rhs", c->rhs, 8 * c->ncells},       {"diag", c->diagd, 8 * c->ncells},
               {"cell_of_row", c->cell_of_row, 4 * c->ncells}, {"rowscan", c->rowscan, 4 * c->ncells},
               {"nbr", c->nbr, 24 * c->ncells},      {"z", c->z, 8 * c->ncells},
               {"tq", c->tq, 8 * c->ncells},         {"r", c->r, 8 * c->ncells},
               {"wave_trace", c->wave_trace, 8 * 32768}};
    for (auto &e : tab)
        if (!strcmp(e.n, name)) {
            TRY(d2h(host, e.p, (size_t)std::min(bytes, e.sz), c->st));
            return flip_synchronize(c);
        }
    set_error(std::string("unknown buffer ") + name);
    return FLIP_E_ARG;
}

extern "C" int flip_set_probe(flip_ctx *c, int32_t kind) {
    cudaSetDevice(c->device);
    if (kind && !c->probe.ev[0])
        for (auto &e : c->probe.ev) FLIP_CUDA_OK(cudaEventCreate(&e));
    if (kind && !c->probe.ts) {
        FLIP_CUDA_OK(cudaMalloc(&c->probe.ts, sizeof(unsigned long long) * 2 * kProbeSlots));
        FLIP_CUDA_OK(cudaMallocHost(&c->probe.ts_host, sizeof(unsigned long long) * 2 * kProbeSlots));
    }
    if (c->probe.ts) {
        FLIP_CUDA_OK(cudaMemsetAsync(c->probe.ts, 0xff, sizeof(unsigned long long) * kProbeSlots, c->st));
        FLIP_CUDA_OK(cudaMemsetAsync(c->probe.ts + kProbeSlots, 0,
                                     sizeof(unsigned long long) * kProbeSlots, c->st));
    }
    c->probe.kind = kind;
    c->probe.used = 0;
    c->probe.bytes = 0.0;
    c->probe.launches = 0;
    c->probe.stamp_ms = 0.0;
    c->probe.stamp_bytes = 0.0;
    c->probe.stamp_launches = 0;
    return 0;
}

extern "C" int flip_get_probe(flip_ctx *c, double *total_ms, int64_t *launches, double *bytes) {
    cudaSetDevice(c->device);
    TRY(flip_synchronize(c));
    double tot = 0.0;
    for (int k = 0; k < c->probe.used; k++) {
        float ms = 0.f;
        FLIP_CUDA_OK(cudaEventElapsedTime(&ms, c->probe.ev[2 * k], c->probe.ev[2 * k + 1]));
        tot += ms;
    }
    *total_ms = tot + c->probe.stamp_ms;
    *launches = c->probe.used + c->probe.stamp_launches;
    *bytes = (c->probe.used == c->probe.launches
                  ? c->probe.bytes
                  : c->probe.bytes * c->probe.used / c->probe.launches) +
             c->probe.stamp_bytes;
    return 0;
}

extern "C" int flip_divergence_field(flip_ctx *c, double *div) {
    cudaSetDevice(c->device);
    launch_divergence(*c, c->xtmp);
    TRY(d2h(div, c->xtmp, sizeof(double) * c->ncells, c->st));
    return flip_synchronize(c);
}

extern "C" int flip_energy_sums(flip_ctx *c, double floor_y, double *ke2, double *pe) {
    cudaSetDevice(c->device);
    *ke2 = 0.0;
    *pe = 0.0;
    if (c->n == 0) return 0;
    // reuse the back particle buffer as scratch (n <= cap)
    double *ke = c->Q.a[0], *pp = c->Q.a[1], *res = c->Q.a[2];
    k_energy_terms<<<nblocks(c->n), kThreads, 0, c->st>>>(c->P, c->n, floor_y, ke, pp);
    double *tmp = nullptr;
    FLIP_CUDA_OK(cudaMalloc(&tmp, sizeof(double) * dot_tmp_doubles(c->n)));
    FLIP_CUDA_OK(cudaMemsetAsync(tmp, 0, sizeof(double) * dot_tmp_doubles(c->n), c->st));
    int64_t l = 0;
    launch_pairwise_dot(ke, nullptr, c->n, tmp, res, c->st, &l);
    launch_pairwise_dot(pp, nullptr, c->n, tmp, res + 1, c->st, &l);
    int rc = d2h(ke2, res, sizeof(double), c->st);
    if (!rc) rc = d2h(pe, res + 1, sizeof(double), c->st);
    if (!rc) rc = flip_synchronize(c);
    cudaFree(tmp);
    return rc;
}

// ------------------------------------------------------- plugin kernels ----
namespace {
struct Scratch {
    std::vector<void *> p;
    ~Scratch() {
        for (void *q : p) cudaFree(q);
    }
    template <class T>
    T *get(int64_t n) {
        void *q = nullptr;
        if (cudaMalloc(&q, sizeof(T) * (size_t)(n > 0 ? n : 1)) != cudaSuccess) return nullptr;
        p.push_back(q);
        return (T *)q;
    }
};
struct Stream {
    cudaStream_t st = nullptr;
    Stream() { cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking); }
    ~Stream() { cudaStreamDestroy(st); }
};
}  // namespace

__global__ void k_widen(const int *__restrict__ a, long long *__restrict__ b, int64_t n) {
    for (int64_t i = gtid(); i < n; i += gstride()) b[i] = a[i];
}

__global__ void k_narrow(const long long *__restrict__ a, int *__restrict__ b, int64_t n) {
    for (int64_t i = gtid(); i < n; i += gstride()) b[i] = (int)a[i];
}

extern "C" int flip_k_sample_velocity_many(const double *u, const double *v, const double *w,
                                           int64_t nx, int64_t ny, int64_t nz, double dtau,
                                           double ox, double oy, double oz, int64_t n,
                                           const double *px, const double *py, const double *pz,
                                           double *vx, double *vy, double *vz) {
    double o[3] = {ox, oy, oz};
    Dims d = make_dims(nx, ny, nz, dtau, o);
    Stream S;
    Scratch sc;
    int64_t nu = (nx + 1) * ny * nz, nv = nx * (ny + 1) * nz, nw = nx * ny * (nz + 1);
    double *du = sc.get<double>(nu), *dv = sc.get<double>(nv), *dw = sc.get<double>(nw);
    double *dp[3] = {sc.get<double>(n), sc.get<double>(n), sc.get<double>(n)};
    double *dvv[3] = {sc.get<double>(n), sc.get<double>(n), sc.get<double>(n)};
    TRY(h2d(du, u, sizeof(double) * nu, S.st));
    TRY(h2d(dv, v, sizeof(double) * nv, S.st));
    TRY(h2d(dw, w, sizeof(double) * nw, S.st));
    const double *hp[3] = {px, py, pz};
    for (int a = 0; a < 3; a++) TRY(h2d(dp[a], hp[a], sizeof(double) * n, S.st));
    launch_sample_many(d, du, dv, dw, n, dp[0], dp[1], dp[2], dvv[0], dvv[1], dvv[2], S.st);
    double *hv[3] = {vx, vy, vz};
    for (int a = 0; a < 3; a++) TRY(d2h(hv[a], dvv[a], sizeof(double) * n, S.st));
    FLIP_CUDA_OK(cudaStreamSynchronize(S.st));
    FLIP_CUDA_OK(cudaGetLastError());
    return 0;
}

extern "C" int flip_k_p2g_component(int32_t comp, int64_t n, const double *vel_p, const double *px,
                                    const double *py, const double *pz, const int64_t *offset,
                                    const int64_t *count, int64_t nx, int64_t ny, int64_t nz,
                                    double dtau, double ox, double oy, double oz, double *values,
                                    double *weights) {
    double o[3] = {ox, oy, oz};
    Dims d = make_dims(nx, ny, nz, dtau, o);
    Stream S;
    Scratch sc;
    int64_t nc = nx * ny * nz;
    int64_t nf = comp == 0 ? (nx + 1) * ny * nz : comp == 1 ? nx * (ny + 1) * nz : nx * ny * (nz + 1);
    double *dvel = sc.get<double>(n), *dp[3] = {sc.get<double>(n), sc.get<double>(n), sc.get<double>(n)};
    long long *o64 = sc.get<long long>(nc), *c64 = sc.get<long long>(nc);
    int *o32 = sc.get<int>(nc), *c32 = sc.get<int>(nc);
    double *dout = sc.get<double>(nf), *dden = sc.get<double>(nf);
    TRY(h2d(dvel, vel_p, sizeof(double) * n, S.st));
    const double *hp[3] = {px, py, pz};
    for (int a = 0; a < 3; a++) TRY(h2d(dp[a], hp[a], sizeof(double) * n, S.st));
    TRY(h2d(o64, offset, sizeof(int64_t) * nc, S.st));
    TRY(h2d(c64, count, sizeof(int64_t) * nc, S.st));
    k_narrow<<<nblocks(nc), kThreads, 0, S.st>>>(o64, o32, nc);
    k_narrow<<<nblocks(nc), kThreads, 0, S.st>>>(c64, c32, nc);
    launch_p2g_component(d, comp, dvel, dp[0], dp[1], dp[2], o32, c32, dout, dden, S.st);
    TRY(d2h(values, dout, sizeof(double) * nf, S.st));
    TRY(d2h(weights, dden, sizeof(double) * nf, S.st));
    FLIP_CUDA_OK(cudaStreamSynchronize(S.st));
    FLIP_CUDA_OK(cudaGetLastError());
    return 0;
}

extern "C" int flip_k_counting_sort_perm(int64_t n, const int64_t *cells, int64_t ncells,
                                         const int64_t *offset, int64_t *perm) {
    (void)offset;  // the stable permutation is unique given the keys
    Stream S;
    Scratch sc;
    long long *c64 = sc.get<long long>(n), *p64 = sc.get<long long>(n);
    int *k0 = sc.get<int>(n), *k1 = sc.get<int>(n), *v0 = sc.get<int>(n), *v1 = sc.get<int>(n);
    int *hist = sc.get<int>(radix_hist_ints(n, ncells));
    int *tmp = sc.get<int>(scan_tmp_ints(radix_hist_ints(n, ncells)) + 64);
    int *tot = sc.get<int>(1);
    TRY(h2d(c64, cells, sizeof(int64_t) * n, S.st));
    if (n > 0) k_narrow<<<nblocks(n), kThreads, 0, S.st>>>(c64, k0, n);
    int *ks = nullptr, *pm = nullptr;
    int64_t l = 0;
    radix_sort_cells(k0, k1, v0, v1, n, ncells, hist, tmp, tot, S.st, &ks, &pm, &l);
    if (n > 0) k_widen<<<nblocks(n), kThreads, 0, S.st>>>(pm, p64, n);
    TRY(d2h(perm, p64, sizeof(int64_t) * n, S.st));
    FLIP_CUDA_OK(cudaStreamSynchronize(S.st));
    FLIP_CUDA_OK(cudaGetLastError());
    return 0;
}
