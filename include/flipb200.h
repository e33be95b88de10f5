/*
 * flipb200.h — C ABI of libflipb200.so, the B200-native (sm_100a) PIC/FLIP
 * timestep that drops in for the reference's `flipsim.sim.step()` path.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src):
 *   flip_create / flip_destroy / flip_set_* / flip_get_*
 *       -> the state containers MacGrid (flipsim/grid.py:62-107),
 *          ParticleSet (flipsim/particles.py:13-64), SpaceHash
 *          (flipsim/binning.py:15-24) and SimState (flipsim/sim.py:76-83);
 *          the ctx owns all device buffers, host buffers are borrowed for the
 *          duration of one copy.
 *   flip_seed_regions + flip_run_stages(BIN..CLASSIFY)
 *       -> make_scene (flipsim/sim.py:204-223): seed (particles.py:133-149),
 *          bin_particles (binning.py:82-97), classify_cells (grid.py:185-190).
 *   flip_step          -> step (flipsim/sim.py:226-300), all ten stages.
 *   flip_run_stages    -> the same stages one at a time (StageTimings keys,
 *                         sim.py:24-46), for per-stage parity tests.
 *   flip_k_*           -> the kernel-backend plugin API flipsim._kernels
 *                         (_kernels/__init__.py:22-72) whose modules export
 *                         _kernels/_core.pyx:68-347 signatures.  HOST
 *                         pointers in and out, like the Cython memoryviews.
 *   flip_solve_system  -> SOLVERS[name](system, max_iters, tol)
 *                         (flipsim/pressure.py:200-340) on an assembled system.
 *
 * Conventions: every function returns 0 on success or a FLIP_E_* code, with
 * a message in flip_last_error() (thread-local).  No call is re-entrant on one
 * ctx.  Arrays are C-contiguous; floating point is IEEE binary64 throughout
 * (the reference stores all state as float64, grid.py:68-71); labels are
 * uint8 SOLID=0 FLUID=1 AIR=2 (grid.py:17-19); index arrays are int64 at the
 * boundary like the reference's.
 */
#ifndef FLIPB200_H
#define FLIPB200_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to flipsim.errors in the Python layer) ---- */
#define FLIP_OK 0
#define FLIP_E_CONFIG 1      /* ConfigError (errors.py:8-9) */
#define FLIP_E_SINGULAR 2    /* SingularSystemError(cell) (errors.py:16-22) */
#define FLIP_E_BREAKDOWN 3   /* SolverBreakdownError (errors.py:25-26) */
#define FLIP_E_CUDA 4        /* CUDA runtime failure */
#define FLIP_E_ARG 5         /* bad argument / ValueError */
#define FLIP_E_CAPACITY 6    /* particle count beyond int32 indexing / flip_set_particle_count > capacity */

/* ---- step stages, in reference order (sim.py:233-292) ---- */
#define FLIP_STAGE_DT 0
#define FLIP_STAGE_ADVECT 1
#define FLIP_STAGE_BIN 2
#define FLIP_STAGE_CLASSIFY 3
#define FLIP_STAGE_P2G 4
#define FLIP_STAGE_FORCE 5
#define FLIP_STAGE_PROJECT 6
#define FLIP_STAGE_APPLY_GRADIENT 7
#define FLIP_STAGE_G2P 8
#define FLIP_STAGE_RESEED 9
#define FLIP_NSTAGES 10

/* ---- solver selectors (pressure.py:335-340; precond pressure.py:274) ---- */
#define FLIP_SOLVER_JACOBI 0
#define FLIP_SOLVER_GS 1
#define FLIP_SOLVER_RBGS 2
#define FLIP_SOLVER_PCG 3
#define FLIP_PRECOND_MIC0 0
#define FLIP_PRECOND_JACOBI 1
#define FLIP_PRECOND_NONE 2
/* extension: geometric multigrid V-cycle; results differ from
 * the reference (which has only MIC(0)) and are validated to tolerance */
#define FLIP_PRECOND_MG 3

/* ---- advection schemes (extension; the reference is forward Euler) ---- */
#define FLIP_ADVECT_EULER 0
#define FLIP_ADVECT_RK2 1

typedef struct flip_ctx flip_ctx;

/* SceneSpec (sim.py:50-72) as the step consumes it.  The *_h fields are the
 * host-side products the reference evaluates in Python floats before they
 * meet device data (alpha*dtau, rho*dtau**2, rho*dtau, skin_fraction*dtau),
 * computed by the caller exactly as the reference spells them. */
typedef struct {
    double gravity[3];
    double dt_max;
    double flip_fraction;
    double tol;
    double alpha_dtau_h;   /* alpha * dtau               (particles.py:224) */
    double rho_dtau2_h;    /* rho * dtau ** 2            (pressure.py:164) */
    double rho_dtau_h;     /* rho * dtau                 (pressure.py:354) */
    double skin_h;         /* skin_fraction * dtau       (sim.py:243) */
    int64_t max_iters;     /* resolved_max_iters()       (sim.py:69-72) */
    int32_t solver;        /* FLIP_SOLVER_* */
    int32_t precond;       /* FLIP_PRECOND_* (pcg only) */
    int32_t extrapolation_layers;
    int32_t density;
    uint64_t reseed_seed;  /* rng.derive_seed(rng_seed, step_count + 1) (sim.py:291) */
    int32_t solver_check_every; /* PCG/relaxation convergence poll period (perf knob; 0 = auto) */
    int32_t advection;     /* FLIP_ADVECT_EULER (the reference, particles.py:227-248) or
                              FLIP_ADVECT_RK2 (extension: midpoint through the grid) */
} flip_step_params;

/* StepReport (sim.py:87-93) plus diagnostics. */
typedef struct {
    double dt;
    int64_t particle_count;
    int64_t solver_iterations;
    double solver_residual;
    int32_t solver_converged;
    int32_t status;        /* FLIP_OK or FLIP_E_SINGULAR / FLIP_E_BREAKDOWN */
    int64_t err_cell;      /* SingularSystemError.cell */
    int64_t err_iteration; /* breakdown iteration */
    double err_value;      /* breakdown curvature */
    int64_t nrows;         /* pressure unknowns (LaplacianSystem.nrows) */
    int64_t npinned;       /* sealed regions pinned (pressure.py:109-130) */
    double stage_ms[FLIP_NSTAGES]; /* CUDA-event time per stage */
    int64_t gpu_launches;  /* kernels launched by this call */
} flip_step_report;

/* Seed region (particles.py:67-100): kind 0 = box [a, b], 1 = sphere (a, r). */
typedef struct {
    int32_t kind;
    int32_t density;
    double a[3];
    double b[3];
    double radius;
} flip_region;

const char *flip_last_error(void);
/* SingularSystemError.cell of the last FLIP_E_SINGULAR on this thread, else -1. */
int64_t flip_last_error_cell(void);
int flip_device_count(int *count);

/* ctx lifecycle.  capacity is the initial particle-buffer size; <= 0 picks
 * 12 * ncells (the reseed bound, particles.py:152-177).  The buffers grow on
 * demand (flip_set_particles*, flip_seed_regions, the reseed stage), as the
 * reference's ParticleSet has no capacity; FLIP_E_CAPACITY only reports the
 * int32 indexing limit (2^31 particles per device).  Grid starts as
 * MacGrid(dims): zero velocities and pressure, every label AIR
 * (grid.py:65-72), no particles. */
int flip_create(int device, int64_t nx, int64_t ny, int64_t nz, double dtau,
                const double origin[3], int64_t capacity, flip_ctx **out);
void flip_destroy(flip_ctx *ctx);
int flip_synchronize(flip_ctx *ctx);
/* The cudaStream_t every kernel of this ctx is launched on (for timing). */
int flip_get_stream(flip_ctx *ctx, void **stream);

/* State transfer (host pointers; NULL entries are skipped). */
int flip_set_grid(flip_ctx *ctx, const double *u, const double *v, const double *w,
                  const double *p, const uint8_t *label);
int flip_get_grid(flip_ctx *ctx, double *u, double *v, double *w, double *p, uint8_t *label);
int flip_set_grid_old(flip_ctx *ctx, const double *u, const double *v, const double *w);
int flip_get_grid_old(flip_ctx *ctx, double *u, double *v, double *w);
/* Uploads particles in the given order (not binned; run FLIP_STAGE_BIN). */
int flip_set_particles(flip_ctx *ctx, int64_t n, const double *px, const double *py,
                       const double *pz, const double *vx, const double *vy, const double *vz);
int flip_get_particles(flip_ctx *ctx, double *px, double *py, double *pz, double *vx,
                       double *vy, double *vz);
int flip_particle_count(flip_ctx *ctx, int64_t *n);
/* FLIP v1 snapshot payload (io.py:23-55): the six particle arrays as
 * float32 SoA (out[6 * n], host), converted on the device with
 * round-to-nearest (numpy astype('<f4')); and the reverse, widening exactly
 * (the set is unbinned afterwards, as with flip_set_particles). */
int flip_get_particles_f32(flip_ctx *ctx, float *out_soa);
int flip_set_particles_f32(flip_ctx *ctx, int64_t n, const float *in_soa);
/* SpaceHash: offset/count int64[ncells]; uploading sets the binned hash. */
int flip_set_hash(flip_ctx *ctx, const int64_t *offset, const int64_t *count);
int flip_get_hash(flip_ctx *ctx, int64_t *offset, int64_t *count);
/* fluid_cells = flatnonzero(count > 0) (binning.py:95); out sized ncells */
int flip_get_fluid_cells(flip_ctx *ctx, int64_t *out, int64_t *nfluid);
/* Inter-stage data: dt (stage DT output) and the P2G known masks. */
int flip_set_dt(flip_ctx *ctx, double dt);
int flip_get_dt(flip_ctx *ctx, double *dt);
int flip_set_known(flip_ctx *ctx, const uint8_t *ku, const uint8_t *kv, const uint8_t *kw);
int flip_get_known(flip_ctx *ctx, uint8_t *ku, uint8_t *kv, uint8_t *kw);

/* make_scene seeding on the device: appends each region's jittered particles
 * (region order, covered cells ascending, subcells ascending) to the
 * particle set.  Mark the shell with flip_set_solid_shell first. */
int flip_set_solid_shell(flip_ctx *ctx);
/* Scene extension (BASELINE config 4): mark the cells
 * [i0,i1] x [j0,j1] x [k0,k1] (inclusive, clipped to the grid) SOLID.  The
 * reference has only the wall shell; every stage already honours arbitrary
 * SOLID labels, so obstacles are labels injected after the shell. */
int flip_set_solid_box(flip_ctx *ctx, int64_t i0, int64_t i1, int64_t j0, int64_t j1,
                       int64_t k0, int64_t k1);
int flip_seed_regions(flip_ctx *ctx, int32_t nregions, const flip_region *regions,
                      uint64_t rng_seed);

/* One full timestep (stages 0..9) on the device. */
int flip_step(flip_ctx *ctx, const flip_step_params *params, flip_step_report *report);
/* Stages [first, last] only (inclusive). */
int flip_run_stages(flip_ctx *ctx, const flip_step_params *params, int32_t first,
                    int32_t last, flip_step_report *report);

/* Slab decomposition support (multi-GPU, one ctx per GPU; the exchanges run
 * in the host layer over NCCL, paper_2404_01931_b200/dist.py).  Device
 * pointers stay valid until the next stage or particle setter call (binning
 * and reseed swap the particle buffers; growth reallocates them). */
typedef struct {
    double *pos[3], *vel[3];   /* particle SoA, `capacity` entries */
    int32_t *count, *offset;   /* hash: count[ncells], offset[ncells + 1] */
    uint8_t *label;            /* ncells */
    double *u, *v, *w, *p;     /* grid */
    double *uo, *vo, *wo;      /* grid_old */
    uint8_t *ku, *kv, *kw;     /* P2G known masks */
    int64_t capacity, n;
} flip_dev_ptrs;
int flip_get_dev_ptrs(flip_ctx *ctx, flip_dev_ptrs *out);
/* Grow the particle buffers (keeping the live particles) so that at least n
 * fit; device pointers from flip_get_dev_ptrs are invalidated if they move.
 * Call before writing more than `capacity` rows into the device views. */
int flip_reserve_particles(flip_ctx *ctx, int64_t n);
/* The particle arrays were rewritten in place (device) with n particles, in
 * any order: the next FLIP_STAGE_BIN recomputes the keys. */
int flip_set_particle_count(flip_ctx *ctx, int64_t n);
/* Reseed (particles.py:157-211) only refills/culls cells in z-planes
 * [k0, k1) (the rank's slab); default the whole grid. */
int flip_set_slab(flip_ctx *ctx, int64_t k0, int64_t k1);
/* cell_index_many (binning.py:37-42) of the current particles into a device
 * int32 buffer of n entries. */
int flip_particle_cells(flip_ctx *ctx, int32_t *cells_dev);

/* ---- z-slab decomposition driven from inside the step ----
 * Rank r of `world` owns the cell planes [plane_start[r], plane_start[r+1])
 * and the particles in them.  Every stage then runs on the rank's share
 * (particles: its own; faces/cells/rows: its planes), and the step calls
 * back into the host transport for each exchange (one NCCL/gloo collective
 * per call; device pointers; `stream` is the ctx stream the data is ordered
 * on).  Exchanges per step: dt MAX allreduce, particle migration
 * (all-to-all), the label planes (all-gather; the sealed-region labelling
 * is global), one ghost particle plane per neighbour, 1-plane face halos
 * (after P2G, gradient, each extrapolation layer and the final enforce),
 * per solver iteration a 1-plane row halo, MAX allreduces and the pairwise
 * dot's boundary/partial all-gathers (bit-exact numpy tree), plus an
 * all-gather of r per MIC(0) application (the substitution is a global
 * recurrence: replicated on every rank).  The results are bit-identical
 * to one GPU.  Callbacks return 0 on success. */
#define FLIP_OP_MAX 0   /* int64 max (also non-negative doubles as bits) */
#define FLIP_OP_MIN 1   /* int64 min */
#define FLIP_OP_SUM 2   /* int64 sum */
typedef struct {
    void *user;
    /* bytes to rank-1 / rank+1 and from rank-1 / rank+1 (sizes agree
     * pairwise; 0 at the ends) */
    int (*neighbors)(void *user, void *stream, const void *send_lo, int64_t nsend_lo,
                     const void *send_hi, int64_t nsend_hi, void *recv_lo, int64_t nrecv_lo,
                     void *recv_hi, int64_t nrecv_hi);
    /* in place over n int64 on the device */
    int (*allreduce)(void *user, void *stream, int64_t *buf, int64_t n, int32_t op);
    /* in place: rank q's bytes are buf[offsets[q], offsets[q+1]); on return
     * every rank holds all of them (offsets: host array of world+1) */
    int (*allgatherv)(void *user, void *stream, void *buf, const int64_t *offsets);
    /* send[sum send_bytes[<q]...] goes to rank q; recv grouped by source
     * rank in rank order (host arrays of world byte counts) */
    int (*alltoallv)(void *user, void *stream, const void *send, const int64_t *send_bytes,
                     void *recv, const int64_t *recv_bytes);
} flip_comm;
/* Enter slab mode (comm copied; NULL comm or world 1 leaves it).  The
 * particles must already be restricted to the rank's planes. */
int flip_set_slab_comm(flip_ctx *ctx, int32_t rank, int32_t world, const int64_t *plane_start,
                       const flip_comm *comm);
/* Bytes exchanged by this ctx since the last call (then reset). */
int flip_slab_bytes(flip_ctx *ctx, int64_t *sent, int64_t *calls);

/* Diagnostics: divergence_field (grid.py:147-156) of the current grid into
 * host div[ncells]; total_energy sums (sim.py:303-315) with numpy pairwise
 * order: ke2 = sum(vx^2+vy^2+vz^2), pe = sum(py - floor_y). */
int flip_divergence_field(flip_ctx *ctx, double *div);
/* Timing probe (bench roofline evidence): kind 1 brackets every MIC(0)
 * substitution sweep launch with CUDA events on the ctx stream; get returns
 * the summed duration, the number of bracketed launches (<= 1024 per
 * flip_set_probe) and their algorithmic bytes (3 x 8 B per row). */
int flip_set_probe(flip_ctx *ctx, int32_t kind);
int flip_get_probe(flip_ctx *ctx, double *total_ms, int64_t *launches, double *alg_bytes);
/* Test hook: copy an internal device buffer ("precon", "x", "rhs", "diag",
 * "cell_of_row", "rowscan", "nbr", "z", "tq", "r") to host. */
int flip_debug_copy(flip_ctx *ctx, const char *name, void *host, int64_t bytes);
int flip_energy_sums(flip_ctx *ctx, double floor_y, double *ke2, double *pe);

/* ---- kernel-backend plugin API (flipsim._kernels module functions) ---- */
/* _core.pyx:68-90 */
int flip_k_sample_velocity_many(const double *u, const double *v, const double *w,
                                int64_t nx, int64_t ny, int64_t nz, double dtau, double ox,
                                double oy, double oz, int64_t n, const double *px,
                                const double *py, const double *pz, double *vx, double *vy,
                                double *vz);
/* _core.pyx:93-176 */
int flip_k_p2g_component(int32_t comp, int64_t n, const double *vel_p, const double *px,
                         const double *py, const double *pz, const int64_t *offset,
                         const int64_t *count, int64_t nx, int64_t ny, int64_t nz, double dtau,
                         double ox, double oy, double oz, double *values, double *weights);
/* _core.pyx:179-193 */
int flip_k_counting_sort_perm(int64_t n, const int64_t *cells, int64_t ncells,
                              const int64_t *offset, int64_t *perm);
/* _core.pyx:196-213 */
int flip_k_laplacian_matvec(int64_t n, const double *diag, const int64_t *nbr_rows,
                            const double *x, double scale, double *y);
/* _core.pyx:216-234 */
int flip_k_jacobi_iter(int64_t n, const double *diag, const int64_t *nbr_rows,
                       const double *rhs, const double *x, double scale, double *out);
/* _core.pyx:237-252 (x updated in place) */
int flip_k_gs_sweep(int64_t n, const double *diag, const int64_t *nbr_rows, const double *rhs,
                    double *x, double scale);
/* _core.pyx:255-272 (x updated in place) */
int flip_k_gs_sweep_rows(int64_t m, const int64_t *rows, int64_t n, const double *diag,
                         const int64_t *nbr_rows, const double *rhs, double *x, double scale);
/* _core.pyx:275-308 */
int flip_k_mic0_build(int64_t n, const double *diag, const int64_t *nbr_rows, double scale,
                      double tau, double sigma, double *precon);
/* _core.pyx:311-347 */
int flip_k_mic0_apply(int64_t n, const double *precon, const int64_t *nbr_rows,
                      const double *r, double scale, double *z);
/* numpy np.add.reduce(a * b) in pairwise order (pressure.py:269-271) */
int flip_k_pairwise_dot(int64_t n, const double *a, const double *b, double *out);

/* Whole solve on an assembled system (pressure.py:200-332).
 * history may be NULL (else max_iters doubles). */
int flip_solve_system(int32_t solver, int32_t precond, int64_t n, const int64_t *cells,
                      const double *diag, const int64_t *nbr_rows, const double *rhs,
                      double scale, int64_t max_iters, double tol, const int64_t *red_rows,
                      int64_t nred, const int64_t *black_rows, int64_t nblack, double *x,
                      int64_t *iterations, double *residual, int32_t *converged,
                      int64_t *err_cell, int64_t *err_iteration, double *err_value);

#ifdef __cplusplus
}
#endif
#endif
