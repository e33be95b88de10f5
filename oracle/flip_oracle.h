/*
 * flip_oracle.h — CPU restatement of the reference FLIP timestep
 * (flipsim.sim.step, /root/reference/pkg/src/flipsim/sim.py:226-300).
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker (and the bench's
 * cpu_baseline / --impl reference arm).  The product (libflipb200.so) never
 * links, loads or calls it.  Every function cites the reference file:line it
 * restates; arithmetic order follows the reference exactly (no FMA: build
 * with -ffp-contract=off) so results are bit-identical to the reference's
 * Cython backend.  Pinned against the real reference by
 * tests/test_oracle_vs_reference.py (build container) and the committed
 * fixtures in tests/golden/ (anywhere).
 *
 * Conventions: all arrays caller-owned, C-contiguous; indices/counts int64
 * like the reference; labels uint8 SOLID=0 FLUID=1 AIR=2 (grid.py:17-19).
 */
#ifndef FLIP_ORACLE_H
#define FLIP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t nx, ny, nz;
    double dtau, ox, oy, oz;
} orc_dims;

/* rng.py:19-41 */
double orc_uniform01(uint64_t seed, uint64_t stream, uint64_t lane);
uint64_t orc_derive_seed(uint64_t base, uint64_t stream);

/* particles.py:103-130 (covered_cells + _jittered_positions) */
int64_t orc_covered_cells_box(const orc_dims *d, const double lo[3], const double hi[3], int64_t *out);
int64_t orc_covered_cells_sphere(const orc_dims *d, const double c[3], double r, int64_t *out);
void orc_jittered_positions(const orc_dims *d, int64_t m, const int64_t *cells, const int64_t *subs,
                            int64_t density, uint64_t seed, double *px, double *py, double *pz);

/* particles.py:214-224 */
double orc_compute_dt(int64_t n, const double *vx, const double *vy, const double *vz,
                      double dtau, double alpha, double dt_max);
/* grid.py:121-132; returns 0 on success, -1 if no non-solid cell */
int orc_interior_box(const orc_dims *d, const uint8_t *label, double lo[3], double hi[3]);
/* particles.py:227-248 */
void orc_advect(int64_t n, double *px, double *py, double *pz,
                const double *vx, const double *vy, const double *vz,
                double dt, const double lo[3], const double hi[3], double skin);

/* binning.py:37-42, 82-97 and _core.pyx:179-193, particles.py:54-64 */
void orc_cell_index_many(const orc_dims *d, int64_t n, const double *px, const double *py,
                         const double *pz, int64_t *cells);
void orc_exclusive_scan(int64_t n, const int64_t *in, int64_t *out);
void orc_counting_sort_perm(int64_t n, const int64_t *cells, const int64_t *offset,
                            int64_t ncells, int64_t *perm);
/* bin_particles: sorts the six arrays in place (via scratch) and fills count/offset */
void orc_bin_particles(const orc_dims *d, int64_t n, double *arrs[6], double *scratch,
                       int64_t *count, int64_t *offset, int64_t *cells_scratch, int64_t *perm_scratch);

/* grid.py:185-190 */
void orc_classify_cells(int64_t ncells, const int64_t *count, uint8_t *label);

/* _core.pyx:68-90 */
void orc_advect_rk2(const orc_dims *d, const double *u, const double *v, const double *w,
                    int64_t n, double *px, double *py, double *pz, double dt,
                    const double lo[3], const double hi[3], double skin);
void orc_sample_velocity_many(const orc_dims *d, const double *u, const double *v, const double *w,
                              int64_t n, const double *px, const double *py, const double *pz,
                              double *vx, double *vy, double *vz);
/* _core.pyx:93-176 */
void orc_p2g_component(const orc_dims *d, int comp, const double *vel_p, const double *px,
                       const double *py, const double *pz, const int64_t *offset,
                       const int64_t *count, double *out, double *den);

/* grid.py:193-228 */
void orc_add_body_force(const orc_dims *d, double *u, double *v, double *w,
                        const double g[3], double dt);
void orc_enforce_solid_boundaries(const orc_dims *d, const uint8_t *label,
                                  double *u, double *v, double *w);
/* grid.py:231-263 for one component lattice (mx,my,mz); known is updated */
void orc_extrapolate_component(int64_t mx, int64_t my, int64_t mz, double *arr,
                               uint8_t *known, int layers, double *acc_scratch,
                               int64_t *cnt_scratch, uint8_t *known_scratch);

/* pressure.py:76-166.  Outputs sized by ncells (row_of, cells_out, pinned_out)
 * or by nrows (diag, nbr_rows[n*6], rhs).  Returns nrows; *npinned set. */
int64_t orc_assemble(const orc_dims *d, const uint8_t *label, const double *u, const double *v,
                     const double *w, int64_t *row_of, int64_t *cells_out, double *diag,
                     int64_t *nbr_rows, double *rhs, int64_t *pinned_out, int64_t *npinned);

/* _core.pyx:196-347 (kernel-level API) */
void orc_laplacian_matvec(int64_t n, const double *diag, const int64_t *nbr, const double *x,
                          double scale, double *y);
void orc_jacobi_iter(int64_t n, const double *diag, const int64_t *nbr, const double *rhs,
                     const double *x, double scale, double *out);
void orc_gs_sweep(int64_t n, const double *diag, const int64_t *nbr, const double *rhs,
                  double *x, double scale);
void orc_gs_sweep_rows(int64_t m, const int64_t *rows, const double *diag, const int64_t *nbr,
                       const double *rhs, double *x, double scale);
void orc_mic0_build(int64_t n, const double *diag, const int64_t *nbr, double scale,
                    double tau, double sigma, double *precon);
void orc_mic0_apply(int64_t n, const double *precon, const int64_t *nbr, const double *r,
                    double scale, double *q_scratch, double *z);
/* numpy np.add.reduce(a*b) (pressure.py:269-271) — recursive pairwise sum */
double orc_pairwise_dot(int64_t n, const double *a, const double *b);
double orc_pairwise_sum(int64_t n, const double *a);

/* pressure.py:200-332.  kind: 0 jacobi, 1 gs, 2 rbgs, 3 pcg.
 * precond (pcg only): 0 mic0, 1 jacobi, 2 none.
 * Returns 0 ok, 1 singular (err_cell set), 2 breakdown (err_it set, curvature in *residual). */
typedef struct {
    int64_t iterations;
    double residual;
    int converged;
    int64_t err_cell;
    int64_t err_it;
    double err_value;
} orc_solve_result;
int orc_solve(int kind, int precond, int64_t n, const int64_t *cells, const double *diag,
              const int64_t *nbr, const double *rhs, double scale, int64_t max_iters,
              double tol, const int64_t *red_rows, int64_t nred, const int64_t *black_rows,
              int64_t nblack, double *x, double *history, orc_solve_result *res);

/* pressure.py:343-380 (p dense, zero off rows) */
void orc_apply_pressure_gradient(const orc_dims *d, const uint8_t *label, const double *p,
                                 double dt, double rho, double *u, double *v, double *w);

/* transfer.py:60-82 */
void orc_g2p(const orc_dims *d, const double *un, const double *vn, const double *wn,
             const double *uo, const double *vo, const double *wo, int64_t n,
             const double *px, const double *py, const double *pz,
             double *vx, double *vy, double *vz, double flip);

/* particles.py:157-211: pass 1 computes new_count/new_offset and returns the total */
int64_t orc_reseed_counts(int64_t ncells, const int64_t *count, const uint8_t *label,
                          int64_t density, int64_t *n_add, int64_t *new_count,
                          int64_t *new_offset);
/* pass 2 fills the six output arrays (size total) */
void orc_reseed_fill(const orc_dims *d, int64_t ncells, const int64_t *count,
                     const int64_t *offset, const int64_t *n_add, const int64_t *new_offset,
                     int64_t density, uint64_t seed, const double *in[6], double *out[6],
                     const double *u, const double *v, const double *w);

/* divergence_field (grid.py:147-156) */
void orc_divergence_field(const orc_dims *d, const double *u, const double *v, const double *w,
                          double *div);

int orc_num_threads(void);
void orc_set_num_threads(int n);

#ifdef __cplusplus
}
#endif
#endif
