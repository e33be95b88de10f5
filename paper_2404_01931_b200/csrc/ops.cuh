// ops.cuh — device context and kernel launcher declarations for libflipb200.
#pragma once
#include <string>
#include <vector>

#include "common.cuh"
#include "scan.cuh"

namespace flip {

struct ParticlePtrs {
    double *a[6];  // pos_x, pos_y, pos_z, vel_x, vel_y, vel_z (particles.py:23-28)
};

// Device-resident scalars of one step (one struct, read back once per step).
struct DevScalars {
    double dt;
    unsigned long long s2max_bits;      // compute_dt max |v|^2
    int box_min[3], box_max[3];         // interior_box (grid.py:121-132)
    double lo[3], hi[3];
    int n_particles;                    // count entering the stage
    int nrows, npinned;
    int total;                          // scratch total for scans
    unsigned long long rhsmax_bits;     // max |rhs|
    unsigned long long res_bits;        // max |r| or max residual
    double target, res, sigma, sigma_new, curv, alpha, beta;
    int iter, done, converged, status;  // solver loop state
    long long err_cell, err_it;
    double err_value;
    int reseed_changed, new_total;
    int nlevels;
    int row_lo[3], row_hi[3];           // bounding box of the pressure rows
    int pad;
    unsigned upd_ticket;                // k_pcg_update's last-block ticket (re-armed to 0)
    int x_it;                           // last iteration whose x += alpha s k_pcg_dir applied
    unsigned dir_ticket;                // k_pcg_dir's last-block ticket (re-armed to 0)
    int pbox_min[3], pbox_max[3];       // cells holding particles (k_classify), inclusive
    int emit_n;                         // cells reseed refills (k_reseed_count's list)
};

// CUDA-event bracketing of one kernel class (bench roofline evidence).
struct Probe {
    int kind = 0;              // 0 off, 1 MIC(0) substitution sweeps
    int used = 0;
    static constexpr int kMax = 4096;
    cudaEvent_t ev[2 * kMax]{};
    double bytes = 0.0;        // algorithmic bytes of the bracketed launches
    int64_t launches = 0;
    // quad sweeps: device stamps instead of events (no event record between
    // the kernels, so the probed step is the unprobed one; also works inside
    // the solver graph).  ts: [kProbeSlots starts | kProbeSlots ends].
    unsigned long long *ts = nullptr, *ts_host = nullptr;
    double stamp_ms = 0.0, stamp_bytes = 0.0;
    int64_t stamp_launches = 0;
};

// z-slab decomposition state (flip_set_slab_comm, slab.cu).  All arrays
// keep their full-grid size and global indexing; a rank only computes its
// own planes / rows / particles and exchanges the boundary planes.
struct Slab {
    bool on = false;
    int rank = 0, world = 1;
    std::vector<int64_t> kstart;   // world + 1 plane starts
    int *kstart_dev = nullptr;     // same, on the device (int)
    flip_comm comm{};
    int64_t k0 = 0, k1 = 0;        // own cell planes [k0, k1)
    int64_t g_lo = 0, g_hi = 0;    // ghost particles placed for the current P2G
    // pressure rows (global numbering; set by stage_project)
    std::vector<int64_t> rstart;   // world + 1: first global row of each rank
    int64_t R0 = 0, R1 = 0;        // own rows
    int64_t Rlo = 0, Rhi = 0;      // own rows plus the rows of planes k0-1 and k1
    int64_t R0f = 0, R1l = 0;      // end of the rows of plane k0 / start of plane k1-1
    // exchange staging and migration scratch (grown on demand)
    char *xbuf = nullptr;
    size_t xcap = 0;
    int *mig = nullptr;            // 5 int arrays of mig_cap + histogram
    int64_t mig_cap = 0;
    int64_t *cnt_dev = nullptr;    // world x world counts / small scalars
    double *dotbuf = nullptr;      // distributed dot scratch (pressure.cu)
    int *gscan = nullptr;          // ghost planes' count prefix sums (2 x nx*ny + 16)
    size_t dotcap = 0;
    int64_t bytes = 0, calls = 0;  // exchange accounting (flip_slab_bytes)
};

struct Ctx {
    int device = 0;
    cudaStream_t st = nullptr;
    // side stream: the pressure system's structure (union-find, row numbering,
    // neighbours) runs there while P2G runs on st (project_prefetch)
    cudaStream_t st2 = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_side = nullptr;
    int proj_pre = 0;  // project_prefetch issued the structure phase for this step
    Dims d{};
    int64_t ncells = 0, nfu = 0, nfv = 0, nfw = 0;
    int64_t cap = 0;        // particle capacity (entries from P.a[a][0])
    // P2G particle records: rec[comp][i] = {x, y, z, v_comp} (32 B, one 256-bit
    // load per candidate), written by the bin gather; prec_valid while they
    // match the binned particles
    double *prec = nullptr;
    int64_t prec_cap = 0;
    int prec_valid = 0;
    int64_t pfront = 0;     // extra entries before P.a[a][0] (slab ghost plane below)
    int64_t n = 0;          // particle count (host mirror)
    int64_t slab_c0 = 0, slab_c1 = -1;  // reseed cell range (flip_set_slab); -1: all
    void *f32_buf = nullptr;           // snapshot staging (flip_*_particles_f32)
    void *mg = nullptr;                // multigrid levels (mg.cu), allocated on first use
    int box_valid = 0;                 // sc->lo/hi hold interior_box of the current SOLID cells
    int faces_valid = 0;               // solid_list holds the faces enforce_solid_boundaries zeroes
    int *solid_list = nullptr;
    int64_t solid_cap = 0, solid_off[3] = {0, 0, 0}, solid_cnt[3] = {0, 0, 0};
    unsigned short *nb_meta = nullptr; // compact PCG stencil (k_compact_nbr), nc entries
    unsigned *nb_dy = nullptr;
    int2 *nb_dz = nullptr;
    size_t f32_cap = 0;
    ParticlePtrs P{}, Q{};  // current and back particle buffers
    double *u = nullptr, *v = nullptr, *w = nullptr, *p = nullptr;
    uint8_t *label = nullptr;
    double *uo = nullptr, *vo = nullptr, *wo = nullptr;
    uint8_t *ku = nullptr, *kv = nullptr, *kw = nullptr, *ku1 = nullptr, *kv1 = nullptr,
            *kw1 = nullptr;
    int *count = nullptr, *offset = nullptr;  // offset has ncells + 1 entries
    int *count2 = nullptr, *offset2 = nullptr, *nadd = nullptr;  // reseed output hash
    int *emit_cells = nullptr;         // cells reseed refills, in no particular order
    int *keys0 = nullptr, *keys1 = nullptr, *vals0 = nullptr, *vals1 = nullptr;
    int *keys_sorted = nullptr;  // cell of each binned particle (valid after BIN)
    int *hist = nullptr;
    int *scan_tmp = nullptr;
    // pressure system (rows = unpinned FLUID cells ascending, pressure.py:76-166)
    int *rowscan = nullptr;      // exclusive scan of isrow over cells
    uint8_t *isrow = nullptr;
    int *parent = nullptr;       // union-find over FLUID cells
    uint8_t *has_air = nullptr;
    int *cell_of_row = nullptr;
    int *nbr = nullptr;          // [6][ncells] neighbour rows, -1 = none
    double *diagd = nullptr;     // non-SOLID neighbour count (float64 like the reference)
    double *rhs = nullptr, *x = nullptr, *r = nullptr, *z = nullptr, *s = nullptr, *q = nullptr,
           *tq = nullptr, *precon = nullptr, *xtmp = nullptr;
    unsigned long long *u64_scratch = nullptr;
    int *lvl = nullptr, *lvl_rows = nullptr, *lvl_off = nullptr, *lvl_cnt = nullptr;
    double *dot_part = nullptr;
    int *wave_prog = nullptr;    // wavefront tile ticket
    double *wave_halo = nullptr; // wavefront tile-face halo buffers
    unsigned long long *wave_trace = nullptr;  // optional per-tile timing
    unsigned char *cflags = nullptr;  // per-cell sweep flags
    // lane-major MIC(0) operand layout (wavefront.cu, k_mic_lane)
    int64_t lane_cap = 0;
    int *lrow = nullptr, *posL = nullptr;
    double *laneA = nullptr, *laneB = nullptr, *laneC = nullptr, *laneD = nullptr;
    DevScalars *sc = nullptr;    // device
    DevScalars *sch = nullptr;   // pinned host mirror
    cudaEvent_t ev[FLIP_NSTAGES + 1]{};
    int64_t launches = 0;
    Probe probe;
    int known_valid = 0;
    int keys_valid = 0;   // keys_sorted matches the current binned particles
    int pbox_valid = 0;   // sc->pbox_* is the cell box of the current binned particles
    int known_box = 0;    // the known masks vanish outside sc->pbox_* grown by one face
    Slab slab;
};

// ---- sort / scan ----
__global__ void k_iota(int *a, int64_t n);
__global__ void k_gather6(ParticlePtrs src, ParticlePtrs dst, const int *__restrict__ perm,
                          int64_t n);
__global__ void k_gather6_rec(ParticlePtrs src, ParticlePtrs dst, const int *__restrict__ perm,
                              int64_t n, double *__restrict__ rec, int64_t ld);
int64_t radix_hist_ints(int64_t cap, int64_t ncells);
int radix_sort_cells(int *k0, int *k1, int *v0, int *v1, int64_t n, int64_t ncells, int *hist,
                     int *scan_tmp, int *scan_total, cudaStream_t st, int **keys_sorted,
                     int **perm_out, int64_t *launches);

// ---- stage launchers (ctx-based, stream-ordered, no host sync) ----
int stage_dt(Ctx &c, const flip_step_params &prm);
void stage_advect(Ctx &c, const flip_step_params &prm);
void stage_bin(Ctx &c);                                // keys + count + scan + sort + gather
void stage_bin_from_keys(Ctx &c);                      // same, keys/count already computed
void stage_classify(Ctx &c);
void stage_p2g(Ctx &c, const flip_step_params &prm);   // + grid_old copy, known masks
void stage_p2g_impl(Ctx &c, const flip_step_params *prm, int fuse_force);
void stage_force(Ctx &c, const flip_step_params &prm); // body force + enforce
int stage_project(Ctx &c, const flip_step_params &prm, flip_step_report *rep);  // syncs
void project_prefetch(Ctx &c);  // structure phase of stage_project on c.st2 (one GPU)
int stage_apply_gradient(Ctx &c, const flip_step_params &prm);
void stage_g2p(Ctx &c, const flip_step_params &prm);
int stage_reseed(Ctx &c, const flip_step_params &prm);
void launch_particle_cells(Ctx &c, int *out);
void launch_set_solid_box(Ctx &c, const int b[6]);
void launch_particles_f32(Ctx &c, float *buf, bool to_f32);
// mg.cu: multigrid preconditioner (precond = FLIP_PRECOND_MG)
int mg_setup(Ctx &c, double scale, const int lo[3], const int hi[3], cudaStream_t st);
void mg_apply(Ctx &c, const double *r, double *z, int64_t n, const DevScalars *sc,
              cudaStream_t st, int64_t *launches);
void mg_free(Ctx &c);

void launch_set_solid_shell(Ctx &c);
int seed_regions(Ctx &c, int nreg, const flip_region *regs, uint64_t seed);
int reserve_particles(Ctx &c, int64_t n);
void launch_divergence(Ctx &c, double *div_dev);
void launch_enforce(Ctx &c, double *u, double *v, double *w);

// ---- slab decomposition (slab.cu) ----
int slab_neighbors(Ctx &c, const void *slo, int64_t nslo, const void *shi, int64_t nshi,
                   void *rlo, int64_t nrlo, void *rhi, int64_t nrhi);
int slab_allreduce(Ctx &c, int64_t *buf, int64_t n, int op);
int slab_allgatherv(Ctx &c, void *buf, const int64_t *offsets);
char *slab_xbuf(Ctx &c, size_t bytes);
int slab_migrate(Ctx &c);                   // after ADVECT: particles to their owners
int slab_labels(Ctx &c);                    // after CLASSIFY: full label array
int slab_ghosts(Ctx &c);                    // before P2G: neighbour particle planes
void slab_ghosts_clear(Ctx &c);             // after P2G
int slab_face_halo(Ctx &c, int what);       // 1-plane face halos (SLAB_H_* bits)
int slab_row_halo(Ctx &c, double *vec);     // 1-plane row halo of a row vector
int slab_rows(Ctx &c);                      // global row ranges (after the row scan)
int slab_free(Ctx &c);
// own face range of lattice comp: [lo, hi) flat indices
void slab_face_range(const Ctx &c, int comp, int64_t *lo, int64_t *hi);
enum { SLAB_H_GRID = 1, SLAB_H_OLD = 2, SLAB_H_KNOWN = 4, SLAB_H_SCRATCH0 = 8, SLAB_H_SCRATCH1 = 16 };
// distributed numpy-pairwise dot over the own rows (pressure.cu)
int realloc_particles(Ctx &c, int64_t cap, int64_t front);

// ---- kernel-level helpers shared with the plugin API ----
void launch_sample_many(const Dims &d, const double *u, const double *v, const double *w,
                        int64_t n, const double *px, const double *py, const double *pz,
                        double *vx, double *vy, double *vz, cudaStream_t st);
void launch_p2g_component(const Dims &d, int comp, const double *vel, const double *px,
                          const double *py, const double *pz, const int *offset,
                          const int *count, double *out, double *den, cudaStream_t st);

// pairwise (numpy) dot: result written to *out_dev; tmp holds >= dot_tmp_doubles(n)
int64_t dot_tmp_doubles(int64_t n);
void launch_pairwise_dot(const double *a, const double *b, int64_t n, double *tmp,
                         double *out_dev, cudaStream_t st, int64_t *launches);

// Programmatic dependent launch: kernels launched with launch_pdl may be
// scheduled while their predecessor on the stream drains; they execute
// pdl_wait() before touching anything it wrote (a no-op without the launch
// attribute, so the same kernels stay safe from any other call site).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), unsigned grid, unsigned block, size_t smem,
                       cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

// Streaming-multiprocessor count of the current device (queried once per
// device; 148 on B200, fewer on MIG slices or other parts).
int num_sms();
// Resident CTAs per SM of kernel fn at `threads` threads (cached per kernel
// and device).
int occupancy_per_sm(const void *fn, int threads);

// One resident wave of k (grid-stride kernels), from the occupancy calculator.
template <typename K>
inline unsigned wave_blocks(K k, int64_t n, int threads = kThreads) {
    const int per_sm = occupancy_per_sm((const void *)k, threads);
    int64_t b = (n + threads - 1) / threads, cap = (int64_t)num_sms() * per_sm;
    return (unsigned)(b < 1 ? 1 : b > cap ? cap : b);
}

// Grid-stride grid: enough CTAs for n, at most `per_sm` per SM.
inline unsigned nblocks(int64_t n, int threads = kThreads, int64_t per_sm = 32) {
    int64_t b = (n + threads - 1) / threads, cap = (int64_t)num_sms() * per_sm;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (unsigned)b;
}

// Dims from grid size; pow2 flags dtau == 2^-k exactly.
Dims make_dims(int64_t nx, int64_t ny, int64_t nz, double dtau, const double origin[3]);

void set_error(const std::string &msg);
// SingularSystemError.cell of the last FLIP_E_SINGULAR (after set_error).
void set_error_cell(int64_t cell);

#define FLIP_CUDA_OK(expr)                                                                 \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            ::flip::set_error(std::string(#expr) + ": " + cudaGetErrorString(e_));         \
            return FLIP_E_CUDA;                                                            \
        }                                                                                  \
    } while (0)

}  // namespace flip
