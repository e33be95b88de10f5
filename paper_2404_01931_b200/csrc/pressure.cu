// pressure.cu — pressure projection: assembly (flipsim/pressure.py:76-166),
// solvers (pressure.py:200-340, _kernels/_core.pyx:196-347) and the
// pressure field scatter (pressure.py:49-53).
//
// Unknowns are the unpinned FLUID cells in ascending raw order, stored as
// compact row vectors exactly like the reference, so every per-row formula
// and numpy's pairwise dot order carry over unchanged:
//   * matvec / Jacobi / RBGS rows are independent gathers;
//   * lexicographic GS and MIC(0) substitutions are wavefronts: a row only
//     reads -x/-y/-z rows (forward) or +x/+y/+z rows (backward), so rows on one
//     hyperplane i+j+k are independent and the sequential result is
//     reproduced exactly, row by row;
//   * s.q and z.r follow numpy's recursive pairwise summation tree
//     (np.add.reduce, pressure.py:269-271), evaluated in parallel;
//   * max-norms are order-free (atomicMax on IEEE bits).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "ops.cuh"
#include "wavefront.cuh"

namespace cg = cooperative_groups;

namespace flip {

// ================================================================ assembly
// Union-find over 6-connected FLUID cells with the minimum raw index as the
// root (hooks always point larger roots at smaller ones), equivalent to
// scipy.ndimage.label + np.minimum.at (pressure.py:110-121) for the pinning.
__device__ __forceinline__ int uf_rep(volatile int *par, int x) {
    int cur = par[x];
    if (cur != x) {
        int nxt, prev = x;
        while (cur > (nxt = par[cur])) {
            par[prev] = nxt;
            prev = cur;
            cur = nxt;
        }
    }
    return cur;
}

__global__ void k_uf_init(const uint8_t *__restrict__ label, int64_t nc, int *par, uint8_t *has_air) {
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        par[c] = label[c] == FLUID ? (int)c : -1;
        has_air[c] = 0;
    }
}

__device__ __forceinline__ void uf_unite(int *par, int a, int b) {
    volatile int *vp = par;
    int va = uf_rep(vp, a), vb = uf_rep(vp, b);
    bool repeat;
    do {
        repeat = false;
        if (va != vb) {
            int ret;
            if (va < vb) {
                if ((ret = atomicCAS(&par[vb], vb, va)) != vb) {
                    vb = ret;
                    repeat = true;
                }
            } else {
                if ((ret = atomicCAS(&par[va], va, vb)) != va) {
                    va = ret;
                    repeat = true;
                }
            }
        }
    } while (repeat);
}

// Parent of each FLUID cell = the first cell of its x-run (one warp per
// x-row, ballots with a carry across 32-cell chunks): the x links of the
// union-find come for free, no atomics.  The run start is the run's lowest
// cell, consistent with union by smaller root.
__global__ void k_uf_runs(const uint8_t *__restrict__ label, Dims d, int *par,
                          uint8_t *has_air) {
    const int lane = threadIdx.x & 31;
    const int64_t nrow = (int64_t)d.ny * d.nz;
    const int64_t w0 = (int64_t)(blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = w0; row < nrow; row += nw) {
        const int64_t base = row * d.nx;
        int carry = -1;  // start of the run reaching the chunk's first cell
        for (int x0 = 0; x0 < d.nx; x0 += 32) {
            const int x = x0 + lane;
            const bool in = x < d.nx;
            const bool fl = in && label[base + x] == FLUID;
            const unsigned notfl = __ballot_sync(0xffffffffu, !fl);
            const unsigned upto = notfl & (0xffffffffu >> (31 - lane));  // lanes <= me
            int start;
            if (upto) start = x0 + (31 - __clz(upto)) + 1;  // after the last non-fluid
            else start = carry >= 0 ? carry : x0;
            if (in) {
                par[base + x] = fl ? (int)(base + start) : -1;
                has_air[base + x] = 0;
            }
            // carry into the next chunk: lane 31's run start if it is fluid
            const int s31 = __shfl_sync(0xffffffffu, start, 31);
            const bool f31 = __shfl_sync(0xffffffffu, fl ? 1 : 0, 31);
            carry = f31 ? s31 : -1;
        }
    }
}

// y/z links between x-runs: only the first cell of each overlap segment
// (where the -x neighbour pair is not already linked) unites.
__global__ void k_uf_link_runs(const uint8_t *__restrict__ label, Dims d, int *par) {
    int64_t nc = d.ncells(), sxy = (int64_t)d.nx * d.ny;
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        if (label[c] != FLUID) continue;
        int i, j, k;
        cell_ijk(d, c, i, j, k);
        const bool wfl = i > 0 && label[c - 1] == FLUID;
        if (j > 0 && label[c - d.nx] == FLUID && !(wfl && label[c - 1 - d.nx] == FLUID))
            uf_unite(par, (int)c, (int)(c - d.nx));
        if (k > 0 && label[c - sxy] == FLUID && !(wfl && label[c - 1 - sxy] == FLUID))
            uf_unite(par, (int)c, (int)(c - sxy));
    }
}

__global__ void k_uf_link(const uint8_t *__restrict__ label, Dims d, int *par) {
    int64_t nc = d.ncells(), sxy = (int64_t)d.nx * d.ny;
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        if (label[c] != FLUID) continue;
        int i, j, k;
        cell_ijk(d, c, i, j, k);
        if (i > 0 && label[c - 1] == FLUID) uf_unite(par, (int)c, (int)(c - 1));
        if (j > 0 && label[c - d.nx] == FLUID) uf_unite(par, (int)c, (int)(c - d.nx));
        if (k > 0 && label[c - sxy] == FLUID) uf_unite(par, (int)c, (int)(c - sxy));
    }
}

__device__ __forceinline__ uint8_t lab_at(const uint8_t *label, const Dims &d, int i, int j, int k) {
    if (i < 0 || j < 0 || k < 0 || i >= d.nx || j >= d.ny || k >= d.nz) return SOLID;
    return label[i + (int64_t)j * d.nx + (int64_t)k * d.nx * d.ny];
}

__global__ void k_uf_finish(const uint8_t *__restrict__ label, Dims d, int *par, uint8_t *has_air) {
    int64_t nc = d.ncells(), sxy = (int64_t)d.nx * d.ny;
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        if (label[c] != FLUID) continue;
        int root = uf_rep((volatile int *)par, (int)c);
        par[c] = root;
        int i, j, k;
        cell_ijk(d, c, i, j, k);
        bool air = lab_at(label, d, i - 1, j, k) == AIR || lab_at(label, d, i + 1, j, k) == AIR ||
                   lab_at(label, d, i, j - 1, k) == AIR || lab_at(label, d, i, j + 1, k) == AIR ||
                   lab_at(label, d, i, j, k - 1) == AIR || lab_at(label, d, i, j, k + 1) == AIR;
        if (air) has_air[root] = 1;
    }
}

// A FLUID cell is a row unless it is the root (lowest cell) of a component
// with no AIR neighbour anywhere (pressure.py:114-130).
struct IsRowIn {
    const uint8_t *label;
    const int *par;
    const uint8_t *has_air;
    __device__ int operator()(int64_t c) const {
        if (label[c] != FLUID) return 0;
        return !(par[c] == (int)c && !has_air[c]);
    }
};

__global__ void k_rows_compact(IsRowIn in, int64_t nc, const int *__restrict__ rowscan,
                               uint8_t *__restrict__ isrow, int *__restrict__ cell_of_row,
                               DevScalars *sc) {
    int pinned = 0;
    for (int64_t c = gtid(); c < nc; c += gstride()) {
        int r = in(c);
        isrow[c] = (uint8_t)r;
        if (r) cell_of_row[rowscan[c]] = (int)c;
        else if (in.label[c] == FLUID) pinned++;
    }
    if (pinned) atomicAdd(&sc->npinned, pinned);
}

// Per-row diag, neighbour rows (order -x,+x,-y,+y,-z,+z, pressure.py:25) and
// rhs = -div with solid faces zeroed (pressure.py:144-151).
template <bool STRUCT, bool RHS>
__global__ void k_assemble_rows(Dims d, const uint8_t *__restrict__ label,
                                const uint8_t *__restrict__ isrow, const int *__restrict__ rowscan,
                                const int *__restrict__ cell_of_row, const DevScalars *sc,
                                const double *__restrict__ u, const double *__restrict__ v,
                                const double *__restrict__ w, int *__restrict__ nbr, int64_t ldn,
                                double *__restrict__ diag, double *__restrict__ rhs,
                                unsigned long long *rhsmax, DevScalars *scw, int64_t a_lo,
                                int64_t a_hi, int64_t rhs_lo, int64_t rhs_hi) {
    // rows [a_lo, a_hi) get their structure (a_hi < 0: all rows); rhs only
    // on [rhs_lo, rhs_hi) (a slab's own rows; rhs_hi < 0: all), 0 elsewhere
    const int64_t n = a_hi < 0 ? (int64_t)sc->nrows : a_hi;
    if (rhs_hi < 0) rhs_hi = n;
    int64_t sxy = (int64_t)d.nx * d.ny;
    double m = 0.0;
    int lo[3] = {0x7fffffff, 0x7fffffff, 0x7fffffff}, hi[3] = {-1, -1, -1};
    for (int64_t r = a_lo + gtid(); r < n; r += gstride()) {
        int64_t c = cell_of_row[r];
        int i, j, k;
        cell_ijk(d, c, i, j, k);
        const int di[6] = {-1, 1, 0, 0, 0, 0}, dj[6] = {0, 0, -1, 1, 0, 0}, dk[6] = {0, 0, 0, 0, -1, 1};
        int ns = 0;
        uint8_t nl[6];
#pragma unroll
        for (int q = 0; q < 6; q++) {
            int ii = i + di[q], jj = j + dj[q], kk = k + dk[q];
            uint8_t l = lab_at(label, d, ii, jj, kk);
            nl[q] = l;
            ns += l != SOLID;
            if (STRUCT) {
                int nb = -1;
                if (l == FLUID) {
                    int64_t cc = ii + (int64_t)jj * d.nx + kk * sxy;
                    if (isrow[cc]) nb = rowscan[cc];
                }
                nbr[q * ldn + r] = nb;
            }
        }
        if (STRUCT) diag[r] = (double)ns;
        if (!RHS) {
        } else if (r >= rhs_lo && r < rhs_hi) {
            int64_t fu0 = i + (int64_t)j * (d.nx + 1) + (int64_t)k * (d.nx + 1) * d.ny;
            int64_t fv0 = i + (int64_t)j * d.nx + (int64_t)k * d.nx * (d.ny + 1);
            int64_t fw0 = c;
            double u0 = nl[0] == SOLID ? 0.0 : u[fu0];
            double u1 = nl[1] == SOLID ? 0.0 : u[fu0 + 1];
            double v0 = nl[2] == SOLID ? 0.0 : v[fv0];
            double v1 = nl[3] == SOLID ? 0.0 : v[fv0 + d.nx];
            double w0 = nl[4] == SOLID ? 0.0 : w[fw0];
            double w1 = nl[5] == SOLID ? 0.0 : w[fw0 + sxy];
            double div = (((((u1 - u0) + v1) - v0) + w1) - w0) / d.dtau;
            double rh = -div;
            rhs[r] = rh;
            m = fmax(m, fabs(rh));
        } else {
            rhs[r] = 0.0;
        }
        lo[0] = min(lo[0], i); hi[0] = max(hi[0], i);
        lo[1] = min(lo[1], j); hi[1] = max(hi[1], j);
        lo[2] = min(lo[2], k); hi[2] = max(hi[2], k);
    }
    if (RHS) {
        for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0 && m > 0.0) atomic_max_nonneg(rhsmax, m);
    }
    if (!STRUCT) return;
    // bounding box of the rows (wavefront geometry)
    for (int a = 0; a < 3; a++) {
        for (int o = 16; o; o >>= 1) {
            lo[a] = min(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
            hi[a] = max(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
        }
        if ((threadIdx.x & 31) == 0 && hi[a] >= 0) {
            atomicMin(&scw->row_lo[a], lo[a]);
            atomicMax(&scw->row_hi[a], hi[a]);
        }
    }
}

__global__ void k_bbox_reset(DevScalars *sc) {
    for (int a = 0; a < 3; a++) {
        sc->row_lo[a] = 0x7fffffff;
        sc->row_hi[a] = -1;
    }
}

// pressure_field (pressure.py:49-53): dense p, solution on rows, 0 elsewhere.
__global__ void k_pressure_field(double *__restrict__ p, int64_t nc, const uint8_t *__restrict__ isrow,
                                 const int *__restrict__ rowscan, const double *__restrict__ x) {
    for (int64_t c = gtid(); c < nc; c += gstride()) p[c] = isrow[c] ? x[rowscan[c]] : 0.0;
}

// ======================================================= pairwise dot (numpy)
// numpy DOUBLE_pairwise_sum (loops_utils.h.src): n < 8 sequential from 0;
// n <= 128: 8 strided accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
// then the tail sequentially; else split at n2 = n/2 - (n/2)%8 and add halves.
__device__ __forceinline__ int64_t pw_split(int64_t n) {
    int64_t n2 = n / 2;
    return n2 - n2 % 8;
}

constexpr int kDotBlocksPerSM = 5;  // 48 registers: the batched leaf loads do not spill

// Element loaders for the pairwise dot: ld(i) returns the i-th summand and
// is called exactly once per element, so a loader may also produce a vector
// (the fused matvec and lane-gather variants below).
struct LdProd {
    const double *a, *b;
    __device__ __forceinline__ double operator()(int64_t i) const { return b ? a[i] * b[i] : a[i]; }
};

// 8 lanes (aligned group) evaluate one leaf; result valid in group lane 0.
template <class LD>
__device__ __forceinline__ double pw_leaf8(const LD &ld, int64_t s, int64_t len, int g) {
    unsigned mask = 0xffu << (threadIdx.x & 24);
    double res = 0.0;
    if (len < 8) {
        if (g == 0)
            for (int64_t i = 0; i < len; i++) res += ld(s + i);
        return res;
    }
    // len <= 128: a lane owns at most 16 summands.  Two batches of 8 loads (register count low enough for the dot's
    // occupancy); the accumulation order is unchanged.  The loads are
    // unconditional, at a clamped (always valid) index, and the unused
    // values are dropped afterwards: a guarded load compiles to a branch per
    // element and serialises the round trips.  A loader with a side effect
    // (z[i] = ...) repeats the same store for the clamped index.
    const int cntv = (int)(len / 8);
    double r;
    {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = ld(s + g + 8 * min(k, cntv - 1));
        r = v[0];
#pragma unroll
        for (int k = 1; k < 8; k++) r = k < cntv ? r + v[k] : r;
    }
    if (cntv > 8) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = ld(s + g + 8 * min(k + 8, cntv - 1));
#pragma unroll
        for (int k = 0; k < 8; k++) r = k + 8 < cntv ? r + v[k] : r;
    }
    const int64_t m = (int64_t)cntv * 8;
    r = r + __shfl_xor_sync(mask, r, 1, 8);
    r = r + __shfl_xor_sync(mask, r, 2, 8);
    r = r + __shfl_xor_sync(mask, r, 4, 8);
    if (g == 0 && m < len) {
        // the len % 8 tail in order; its loads issued together at a clamped
        // (valid) index instead of one round trip per element
        const int rem = (int)(len - m);
        double tv[7];
#pragma unroll
        for (int k = 0; k < 7; k++) tv[k] = ld(s + min(m + k, len - 1));
#pragma unroll
        for (int k = 0; k < 7; k++)
            if (k < rem) r += tv[k];
    }
    return r;
}

// Exact evaluation of a (small) subtree by one 8-lane group.  Nodes at the
// cut level differ in length by a few multiples of 8 and one of them is
// <= 128, so two more splits always reach the leaves; the depth is a
// template parameter so everything inlines (no call stack).
template <int DEPTH, class LD>
__device__ __forceinline__ double pw_node8(const LD &ld, int64_t s, int64_t len, int g) {
    if constexpr (DEPTH == 0) {
        return pw_leaf8(ld, s, len, g);
    } else {
        if (len <= 128) return pw_leaf8(ld, s, len, g);
        int64_t n2 = pw_split(len);
        double l = pw_node8<DEPTH - 1>(ld, s, n2, g);
        double r = pw_node8<DEPTH - 1>(ld, s + n2, len - n2, g);
        return l + r;
    }
}

// Phase 1: the 2^cut nodes at the deepest complete level, 32 per block, then
// a perfect-tree reduction of the block's 32 node sums (pairs 2i, 2i+1 first).
// Skipped once sc->done (the epilogue then ignores the sum).
template <class LD>
__global__ void k_dot_nodes(LD ld, int64_t n, int cut, double *__restrict__ out,
                            const DevScalars *sc) {
    if (sc && sc->done) return;
    __shared__ double sv[32];
    int64_t nodes = (int64_t)1 << cut;
    int64_t node = (int64_t)blockIdx.x * 32 + (threadIdx.x >> 3);
    int g = threadIdx.x & 7;
    double val = 0.0;
    if (node < nodes) {
        int64_t s = 0, len = n;
        for (int lvl = cut - 1; lvl >= 0; lvl--) {
            int64_t n2 = pw_split(len);
            if ((node >> lvl) & 1) {
                s += n2;
                len -= n2;
            } else {
                len = n2;
            }
        }
        val = pw_node8<2>(ld, s, len, g);
    }
    if (g == 0) sv[threadIdx.x >> 3] = val;
    __syncthreads();
    int cnt = nodes < 32 ? (int)nodes : 32;
    if (threadIdx.x == 0) {
        for (int st = 1; st < cnt; st <<= 1)
            for (int i = 0; i + st < cnt; i += 2 * st) sv[i] = sv[i] + sv[i + st];
        out[blockIdx.x] = sv[0];
    }
}

enum DotEpi { EPI_STORE = 0, EPI_CURV = 1, EPI_SIGMA_NEW = 2, EPI_SIGMA0 = 3 };

__device__ void dot_epilogue(double v, int epi, double *out, DevScalars *sc) {
    if (epi == EPI_STORE) {
        *out = v;
    } else if (epi == EPI_SIGMA0) {
        sc->sigma = v;
    } else if (sc->done) {
        return;  // iteration skipped after convergence / breakdown
    } else if (epi == EPI_CURV) {  // pressure.py:316-320
        sc->curv = v;
        if (v <= 0.0) {
            sc->status = FLIP_E_BREAKDOWN;
            sc->err_it = sc->iter + 1;
            sc->err_value = v;
            sc->done = 1;
        } else {
            sc->alpha = sc->sigma / v;
        }
    } else {  // EPI_SIGMA_NEW: pressure.py:328-330
        sc->beta = v / sc->sigma;
        sc->sigma = v;
    }
}

// Perfect-tree reduction of cnt (power of two) values, up to 1024 per block.
__global__ void k_dot_tree(const double *__restrict__ in, int64_t cnt, double *__restrict__ out,
                           int epi, DevScalars *sc, double *final_out) {
    __shared__ double sv[1024];
    int64_t base = (int64_t)blockIdx.x * 1024;
    int m = cnt - base < 1024 ? (int)(cnt - base) : 1024;
    for (int i = threadIdx.x; i < m; i += blockDim.x) sv[i] = in[base + i];
    __syncthreads();
    for (int st = 1; st < m; st <<= 1) {
        for (int i = threadIdx.x * 2 * st; i + st < m; i += blockDim.x * 2 * st) sv[i] = sv[i] + sv[i + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (gridDim.x == 1) dot_epilogue(sv[0], epi, final_out, sc);
        else out[blockIdx.x] = sv[0];
    }
}

// k_dot_nodes + k_dot_tree in one launch when the node partials fit one tree
// block (<= 1024): every block publishes its partial, the last block to
// finish (threadfence + ticket) runs k_dot_tree's perfect-tree reduction and
// the epilogue, then re-arms the ticket.  Same summation order.
template <class LD, int MINB = kDotBlocksPerSM>
__global__ void __launch_bounds__(256, MINB)
k_dot_fused(LD ld, int64_t n, int cut, double *__restrict__ part, unsigned *ticket, int epi,
            DevScalars *sc, double *final_out, int skip_when_done) {
    pdl_wait();
    if (skip_when_done && sc->done) return;
    __shared__ double sv[8];
    __shared__ double sv2[1024];
    __shared__ bool last;
    const int64_t nodes = (int64_t)1 << cut;
    const int64_t nparts = (nodes + 31) / 32;  // one partial per 32 nodes
    const int g = threadIdx.x & 7;
    // the grid is sized to the resident block slots; each block walks node
    // blocks of 32 (no wave quantisation, one ticket per block at the end)
    for (int64_t pb = blockIdx.x; pb < nparts; pb += gridDim.x) {
        const int64_t node = pb * 32 + (threadIdx.x >> 3);
        double val = 0.0;
        if (node < nodes) {
            int64_t s0 = 0, len = n;
            for (int lvl = cut - 1; lvl >= 0; lvl--) {
                int64_t n2 = pw_split(len);
                if ((node >> lvl) & 1) {
                    s0 += n2;
                    len -= n2;
                } else {
                    len = n2;
                }
            }
            val = pw_node8<2>(ld, s0, len, g);
        }
        // the perfect tree over these 32 nodes (pairs 2i, 2i+1 first):
        // levels 1-2 inside the warp (node sums sit in lanes 0, 8, 16, 24;
        // a + b == b + a exactly, so lane 0 holds the left+right bits),
        // levels 3-5 over the 8 warp sums; levels that do not exist
        // (nodes < 32) are skipped
        if (nodes >= 2) val = val + __shfl_xor_sync(0xffffffffu, val, 8);
        if (nodes >= 4) val = val + __shfl_xor_sync(0xffffffffu, val, 16);
        if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = val;
        __syncthreads();
        if (threadIdx.x == 0) {
            const int cw = nodes >= 32 ? 8 : (nodes >= 4 ? (int)(nodes / 4) : 1);
            for (int st = 1; st < cw; st <<= 1)
                for (int i = 0; i + st < cw; i += 2 * st) sv[i] = sv[i] + sv[i + st];
            part[pb] = sv[0];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    // perfect tree over the nparts (<= 1024, a power of two) partials
    const int m = (int)nparts;
    for (int i = threadIdx.x; i < m; i += blockDim.x) sv2[i] = __ldcg(part + i);
    __syncthreads();
    for (int st = 1; st < m; st <<= 1) {
        for (int i = threadIdx.x * 2 * st; i + st < m; i += blockDim.x * 2 * st) sv2[i] = sv2[i] + sv2[i + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        dot_epilogue(sv2[0], epi, final_out, sc);
        *ticket = 0u;  // re-armed for the next dot
    }
}

static int pw_cut(int64_t n) {
    // deepest depth at which all nodes exist (all shallower nodes split)
    std::vector<int64_t> sizes{n};
    int cut = 0;
    while (true) {
        bool all_split = !sizes.empty();
        for (int64_t s : sizes) all_split &= s > 128;
        if (!all_split) break;
        std::vector<int64_t> nxt;
        for (int64_t s : sizes) {
            int64_t n2 = s / 2 - (s / 2) % 8;
            nxt.push_back(n2);
            nxt.push_back(s - n2);
        }
        std::sort(nxt.begin(), nxt.end());
        nxt.erase(std::unique(nxt.begin(), nxt.end()), nxt.end());
        sizes.swap(nxt);
        cut++;
    }
    return cut;
}

int64_t dot_tmp_doubles(int64_t n) {
    int cut = pw_cut(n > 0 ? n : 1);
    int64_t nodes = (int64_t)1 << cut;
    // k_dot_fused/k_dot_nodes partials, or k_dot_staged's units (nodes / 8 at most)
    return std::max<int64_t>(2 * ((nodes + 31) / 32), nodes / 8 + 1) + 64;
}

// epi/sc select a fused scalar update; for EPI_STORE the sum goes to *out_dev.
template <class LD>
static void launch_dot_f(const LD &ld, int64_t n, double *tmp, double *out_dev, int epi,
                         DevScalars *sc, cudaStream_t st, int64_t *launches) {
    int cut = pw_cut(n > 0 ? n : 1);
    int64_t nodes = (int64_t)1 << cut;
    int64_t nb1 = (nodes + 31) / 32;
    // tmp[0..1]: the fused dot's ticket word, at a fixed slot so a later
    // call with another n never finds a stale partial there; partials follow
    double *p0 = tmp + 2, *p1 = p0 + nb1;
    // only the solver's in-loop dots may skip their work after convergence
    const bool skip = epi == EPI_CURV || epi == EPI_SIGMA_NEW;
    if (nb1 <= 1024) {
        // ticket zeroed at allocation and re-armed to 0 by the last block
        unsigned *ticket = reinterpret_cast<unsigned *>(tmp);
        static const int dminb = getenv("FLIPB200_DOT_MINB") ? atoi(getenv("FLIPB200_DOT_MINB")) : kDotBlocksPerSM;
        const int per_sm = dminb == 6 ? 6 : dminb == 8 ? 8 : kDotBlocksPerSM;
        const unsigned grid = (unsigned)std::min<int64_t>(nb1, (int64_t)num_sms() * per_sm);
        auto kd = per_sm == 6 ? k_dot_fused<LD, 6> : per_sm == 8 ? k_dot_fused<LD, 8> : k_dot_fused<LD>;
        launch_pdl(kd, grid, 256, 0, st, ld, n, cut, p0, ticket, epi, sc, out_dev, skip ? 1 : 0);
        (*launches)++;
        return;
    }
    k_dot_nodes<LD><<<(unsigned)nb1, 256, 0, st>>>(ld, n, cut, p0, skip ? sc : nullptr);
    (*launches)++;
    int64_t cnt = nb1;
    double *in = p0, *outp = p1;
    while (true) {
        int64_t blocks = (cnt + 1023) / 1024;
        k_dot_tree<<<(unsigned)blocks, 256, 0, st>>>(in, cnt, outp, epi, sc, out_dev);
        (*launches)++;
        if (blocks == 1) break;
        cnt = blocks;
        std::swap(in, outp);
    }
}

void launch_dot(const double *a, const double *b, int64_t n, double *tmp, double *out_dev, int epi,
                DevScalars *sc, cudaStream_t st, int64_t *launches) {
    launch_dot_f(LdProd{a, b}, n, tmp, out_dev, epi, sc, st, launches);
}

void launch_pairwise_dot(const double *a, const double *b, int64_t n, double *tmp, double *out_dev,
                         cudaStream_t st, int64_t *launches) {
    launch_dot(a, b, n, tmp, out_dev, EPI_STORE, nullptr, st, launches);
}

// ============================================ distributed pairwise dot (slab)
// The same numpy tree over the GLOBAL row vector (length n), with rank r
// holding rows [R0, R1).  Rank r evaluates the cut-level nodes that START in
// its rows (a node reaching past R1 reads the next ranks' leading products,
// all-gathered), reduces them to the maximal aligned blocks of the perfect
// tree above the cut, and every rank merges all ranks' blocks in index
// order: each internal node is still left + right, so the sum is bit-
// identical to the one-GPU dot (and to np.add.reduce).
struct DotPlan {
    int64_t n = -1;      // global rows the plan was built for
    int cut = 0;
    int64_t na = 0, nb = 0;  // my nodes
    int64_t X = 0;       // longest cut-level node
    int64_t pre_len = 0; // my leading products published (min(X, own rows))
    std::vector<int64_t> pre_off;  // bytes, world + 1
    int64_t ext_off = 0; // element offset of rank r+1's prefix in the gather buffer
};

static void node_span(int64_t n, int cut, int64_t node, int64_t *s, int64_t *len) {
    int64_t s0 = 0, l = n;
    for (int lvl = cut - 1; lvl >= 0; lvl--) {
        int64_t n2 = l / 2;
        n2 -= n2 % 8;
        if ((node >> lvl) & 1) {
            s0 += n2;
            l -= n2;
        } else {
            l = n2;
        }
    }
    *s = s0;
    *len = l;
}

static int64_t first_node_at_or_after(int64_t n, int cut, int64_t row) {
    int64_t lo = 0, hi = (int64_t)1 << cut;  // first node with start >= row
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2, s, l;
        node_span(n, cut, mid, &s, &l);
        if (s >= row) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

template <class LD>
struct LdExt {  // rows >= R1 come from the gathered leading products
    LD ld;
    int64_t R1;
    const double *ext;
    __device__ __forceinline__ double operator()(int64_t i) const {
        return i < R1 ? ld(i) : ext[i - R1];
    }
};

template <class LD>
__global__ void k_dotd_prefix(LD ld, int64_t R0, int64_t m, double *__restrict__ out,
                              const DevScalars *sc, int skip) {
    if (skip && sc->done) return;
    for (int64_t i = gtid(); i < m; i += gstride()) out[i] = ld(R0 + i);
}

template <class LD>
__global__ void k_dotd_nodes(LD ld, int64_t n, int cut, int64_t na, int64_t nb,
                             double *__restrict__ out, const DevScalars *sc, int skip) {
    if (skip && sc->done) return;
    const int g = threadIdx.x & 7;
    const int64_t groups = ((int64_t)gridDim.x * blockDim.x) >> 3;
    for (int64_t node = na + (gtid() >> 3); node < nb; node += groups) {
        int64_t s0 = 0, len = n;
        for (int lvl = cut - 1; lvl >= 0; lvl--) {
            int64_t n2 = pw_split(len);
            if ((node >> lvl) & 1) {
                s0 += n2;
                len -= n2;
            } else {
                len = n2;
            }
        }
        const double v = pw_node8<2>(ld, s0, len, g);
        if (g == 0) out[node - na] = v;
    }
}

// In place: the perfect tree inside every aligned block [g, g + 2^k) that
// lies within [na, nb); then the maximal blocks, in order, as (level, index,
// value) entries (entry 0 holds the count).
__global__ void __launch_bounds__(1024) k_dotd_canon(double *__restrict__ v, int64_t na, int64_t nb,
                                                     double *__restrict__ ent, const DevScalars *sc,
                                                     int skip) {
    if (skip && sc->done) return;
    const int64_t cnt = nb - na;
    for (int64_t st = 1; st < cnt; st <<= 1) {
        for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
            const int64_t g = na + i;
            if (g % (2 * st) == 0 && g + 2 * st <= nb) v[i] = v[i] + v[i + st];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        int k = 0;
        int64_t g = na;
        while (g < nb) {
            int lvl = 0;
            while (((g >> lvl) & 1) == 0 && g + ((int64_t)2 << lvl) <= nb && lvl < 62) lvl++;
            // largest aligned block at g inside [g, nb)
            while (g + ((int64_t)1 << lvl) > nb) lvl--;
            const long long key = ((long long)lvl << 56) | (long long)(g >> lvl);
            ent[2 + 2 * k] = __longlong_as_double(key);
            ent[3 + 2 * k] = v[g - na];
            k++;
            g += (int64_t)1 << lvl;
        }
        ent[0] = (double)k;
    }
}

constexpr int kDotEnt = 2 + 2 * 64;  // doubles per rank slot: header + up to 64 blocks

__global__ void k_dotd_merge(const double *__restrict__ ent, int world, int epi, double *out,
                             DevScalars *sc, int skip) {
    if (skip && sc->done) return;
    long long lv[128], ix[128];
    double val[128];
    int sp = 0;
    for (int q = 0; q < world; q++) {
        const double *e = ent + (int64_t)q * kDotEnt;
        const int k = (int)e[0];
        for (int t = 0; t < k; t++) {
            const long long key = __double_as_longlong(e[2 + 2 * t]);
            lv[sp] = key >> 56;
            ix[sp] = key & ((1ll << 56) - 1);
            val[sp] = e[3 + 2 * t];
            sp++;
            while (sp >= 2 && lv[sp - 1] == lv[sp - 2] && (ix[sp - 2] & 1) == 0 &&
                   ix[sp - 1] == ix[sp - 2] + 1) {
                val[sp - 2] = val[sp - 2] + val[sp - 1];
                lv[sp - 2] += 1;
                ix[sp - 2] >>= 1;
                sp--;
            }
        }
    }
    dot_epilogue(sp == 1 ? val[0] : __longlong_as_double(0x7ff8000000000001ll), epi, out, sc);
}

struct SlabDot {
    Ctx *c;
    DotPlan plan;
    double *nodes = nullptr;   // node sums (device)
    double *pre = nullptr;     // gathered leading products
    double *ent = nullptr;     // gathered canonical blocks
};

static int slabdot_plan(SlabDot &D, int64_t n) {
    Ctx &c = *D.c;
    Slab &S = c.slab;
    DotPlan &P = D.plan;
    if (P.n == n) return 0;
    P.n = n;
    P.cut = pw_cut(n > 0 ? n : 1);
    // longest node at the cut level
    {
        std::vector<int64_t> sizes{n};
        for (int l = 0; l < P.cut; l++) {
            std::vector<int64_t> nx;
            for (int64_t sz : sizes) {
                int64_t n2 = sz / 2 - (sz / 2) % 8;
                nx.push_back(n2);
                nx.push_back(sz - n2);
            }
            std::sort(nx.begin(), nx.end());
            nx.erase(std::unique(nx.begin(), nx.end()), nx.end());
            sizes.swap(nx);
        }
        P.X = sizes.empty() ? 0 : sizes.back();
    }
    P.na = first_node_at_or_after(n, P.cut, S.R0);
    P.nb = first_node_at_or_after(n, P.cut, S.R1);
    if (S.R1 >= n) P.nb = (int64_t)1 << P.cut;  // the last rank owns the tail
    if (S.R0 >= n) P.na = P.nb;
    P.pre_off.assign(S.world + 1, 0);
    for (int q = 0; q < S.world; q++) {
        const int64_t rows = S.rstart[q + 1] - S.rstart[q];
        P.pre_off[q + 1] = P.pre_off[q] + 8 * std::min(P.X, rows);
    }
    P.pre_len = (P.pre_off[S.rank + 1] - P.pre_off[S.rank]) / 8;
    P.ext_off = P.pre_off[std::min(S.rank + 1, S.world)] / 8;
    size_t need = 8 * ((size_t)(P.nb - P.na) + (size_t)(P.pre_off[S.world] / 8) +
                       (size_t)S.world * kDotEnt + 64);
    if (need > S.dotcap) {
        cudaStreamSynchronize(c.st);
        cudaFree(S.dotbuf);
        S.dotbuf = nullptr;
        S.dotcap = 0;
        FLIP_CUDA_OK(cudaMalloc(&S.dotbuf, need));
        S.dotcap = need;
    }
    D.nodes = S.dotbuf;
    D.pre = D.nodes + (P.nb - P.na) + 8;
    D.ent = D.pre + P.pre_off[S.world] / 8 + 8;
    return 0;
}

template <class LD>
static int launch_dot_slab(SlabDot &D, const LD &ld, int64_t n, double *out_dev, int epi,
                           DevScalars *sc, cudaStream_t st, int64_t *launches) {
    Ctx &c = *D.c;
    Slab &S = c.slab;
    if (int rc = slabdot_plan(D, n)) return rc;
    const DotPlan &P = D.plan;
    const int skip = (epi == EPI_CURV || epi == EPI_SIGMA_NEW) ? 1 : 0;
    // (1) leading products of every rank
    if (P.pre_len > 0) {
        k_dotd_prefix<<<nblocks(P.pre_len), kThreads, 0, st>>>(
            ld, S.R0, P.pre_len, D.pre + P.pre_off[S.rank] / 8, sc, skip);
        (*launches)++;
    }
    if (int rc = slab_allgatherv(c, D.pre, P.pre_off.data())) return rc;
    // (2) my nodes, (3) my maximal blocks
    const int64_t m = P.nb - P.na;
    double *ent = D.ent + (int64_t)S.rank * kDotEnt;
    if (m > 0) {
        LdExt<LD> le{ld, S.R1, D.pre + P.ext_off};
        k_dotd_nodes<<<nblocks(8 * m), kThreads, 0, st>>>(le, n, P.cut, P.na, P.nb, D.nodes, sc, skip);
        k_dotd_canon<<<1, 1024, 0, st>>>(D.nodes, P.na, P.nb, ent, sc, skip);
        *launches += 2;
    } else {
        FLIP_CUDA_OK(cudaMemsetAsync(ent, 0, sizeof(double) * kDotEnt, st));
    }
    // (4) everyone's blocks, merged in index order
    std::vector<int64_t> off(S.world + 1);
    for (int q = 0; q <= S.world; q++) off[q] = (int64_t)q * kDotEnt * 8;
    if (int rc = slab_allgatherv(c, D.ent, off.data())) return rc;
    k_dotd_merge<<<1, 1, 0, st>>>(D.ent, S.world, epi, out_dev, sc, skip);
    (*launches)++;
    return 0;
}

// ================================================================ solvers
struct SysView {
    int64_t n;
    const int *cell;       // raw cell per row (SingularSystemError cell)
    const int *nbr;        // [6][ldn]
    int64_t ldn;
    const double *diag;
    const double *rhs;
    double scale;          // host value, or taken from sc->... when from_dt
    // optional compact stencil of a grid-assembled system (k_compact_nbr):
    // meta = 6 presence bits (nbr order -x,+x,-y,+y,-z,+z) | diag count << 8;
    // -x/+x are rows r-1/r+1, dy = (r - row(-y)) | (row(+y) - r) << 16,
    // dz = (r - row(-z), row(+z) - r).  14 bytes per row instead of 32.
    const unsigned short *meta = nullptr;
    const unsigned *dy = nullptr;
    const int2 *dz = nullptr;
    // rows [r0, r0 + n) are computed (global row numbering); a slab rank's
    // own rows, 0 otherwise
    int64_t r0 = 0;
};

__device__ __forceinline__ double nbr_sum(const int *__restrict__ nbr, int64_t ldn, int64_t r,
                                          const double *__restrict__ x) {
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 6; q++) {
        int nb = nbr[q * ldn + r];
        if (nb >= 0) s = s + x[nb];
    }
    return s;
}

// _core.pyx:196-213; optionally residual max |rhs - y| (pressure.py:59-62)
// and copy-back of a Jacobi iterate (x <- xnew).
__global__ void k_matvec(SysView S, const double *__restrict__ x, double *__restrict__ y,
                         const double *__restrict__ rhs, unsigned long long *resmax,
                         double *__restrict__ copy_to, const DevScalars *sc, int check_done) {
    if (check_done && sc->done) return;
    double m = 0.0;
    for (int64_t r = S.r0 + gtid(); r < S.r0 + S.n; r += gstride()) {
        double s = nbr_sum(S.nbr, S.ldn, r, x);
        double xr = x[r];
        double yr = S.scale * (S.diag[r] * xr - s);
        if (y) y[r] = yr;
        if (resmax) m = fmax(m, fabs(rhs[r] - yr));
        if (copy_to) copy_to[r] = xr;
    }
    if (resmax) {
        for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if ((threadIdx.x & 31) == 0 && m > 0.0) atomic_max_nonneg(resmax, m);
    }
}

// Compact stencil of a system assembled on the grid (k_assemble_rows): rows
// are numbered in cell order, so an x-neighbour row is r -/+ 1 and a
// y-neighbour lies at most nx rows away.  Exact: diag holds a small integer.
__global__ void k_compact_nbr(SysView S, unsigned short *__restrict__ meta,
                              unsigned *__restrict__ dy, int2 *__restrict__ dz) {
    for (int64_t r = S.r0 + gtid(); r < S.r0 + S.n; r += gstride()) {
        unsigned m = (unsigned)S.diag[r] << 8;
        int nb[6];
#pragma unroll
        for (int q = 0; q < 6; q++) {
            nb[q] = S.nbr[q * S.ldn + r];
            if (nb[q] >= 0) m |= 1u << q;
        }
        meta[r] = (unsigned short)m;
        const unsigned ym = nb[2] >= 0 ? (unsigned)(r - nb[2]) : 0u;
        const unsigned yp = nb[3] >= 0 ? (unsigned)(nb[3] - r) : 0u;
        dy[r] = ym | yp << 16;
        dz[r] = make_int2(nb[4] >= 0 ? (int)(r - nb[4]) : 0, nb[5] >= 0 ? (int)(nb[5] - r) : 0);
    }
}

// k_matvec (y = A x) over the compact stencil; same additions in the same
// order as nbr_sum, so the result is bit-identical.
__global__ void __launch_bounds__(256)
k_matvec_c(SysView S, const double *__restrict__ x, double *__restrict__ y, const DevScalars *sc) {
    pdl_wait();
    if (sc->done) return;
    for (int64_t r = S.r0 + gtid(); r < S.r0 + S.n; r += gstride()) {
        const unsigned m = S.meta[r];
        const unsigned d = S.dy[r];
        const int2 z = S.dz[r];
        double s = 0.0;
        if (m & 1u) s = s + x[r - 1];
        if (m & 2u) s = s + x[r + 1];
        if (m & 4u) s = s + x[r - (int64_t)(d & 0xffffu)];
        if (m & 8u) s = s + x[r + (int64_t)(d >> 16)];
        if (m & 16u) s = s + x[r - (int64_t)z.x];
        if (m & 32u) s = s + x[r + (int64_t)z.y];
        y[r] = S.scale * ((double)(m >> 8) * x[r] - s);
    }
}

// q = A s fused into the s.q dot (pressure.py:315-316): k_matvec's
// arithmetic for row r, q[r] written, s[r]*q[r] returned.
struct LdMatvecDot {
    SysView S;
    const double *x;
    double *y;
    __device__ __forceinline__ double operator()(int64_t r) const {
        double s = nbr_sum(S.nbr, S.ldn, r, x);
        double xr = x[r];
        double yr = S.scale * (S.diag[r] * xr - s);
        y[r] = yr;
        return xr * yr;
    }
};

// z taken from the lane-major layout of the MIC(0) sweep (k_lane_to_rows
// fused into the z.r dot): z[r] written, z[r]*r[r] returned.
struct LdLaneDot {
    const double *zL;
    const int *posL;
    double *z;
    const double *r;
    int64_t nL = INT64_MAX;  // lane-layout entries (checked build)
    __device__ __forceinline__ double operator()(int64_t i) const {
        FLIP_CHECK_RANGE((int64_t)posL[i], nL, "z.r dot lane gather");
        double zi = zL[posL[i]];
        z[i] = zi;
        return zi * r[i];
    }
};

// _core.pyx:216-234 (out of place)
__global__ void k_jacobi(SysView S, const double *__restrict__ x, double *__restrict__ out,
                         const DevScalars *sc, int check_done) {
    if (check_done && sc->done) return;
    for (int64_t r = S.r0 + gtid(); r < S.r0 + S.n; r += gstride()) {
        double s = nbr_sum(S.nbr, S.ldn, r, x);
        out[r] = (S.rhs[r] / S.scale + s) / S.diag[r];
    }
}

// _core.pyx:255-272 over an explicit row list, or over all rows of one
// colour (parity of i+j+k of the row's cell, pressure.py:166-170).
__global__ void k_gs_rows(SysView S, const int *__restrict__ rows, int64_t m, int color, Dims d,
                          double *x, const DevScalars *sc, int check_done) {
    if (check_done && sc->done) return;
    int64_t cnt = rows ? m : S.n;
    for (int64_t t = gtid(); t < cnt; t += gstride()) {
        int64_t r = rows ? t : S.r0 + t;
        if (rows) {
            r = rows[t];
        } else {
            int64_t c = S.cell[r];
            int par = (int)((c % d.nx) + (c / d.nx) % d.ny + c / ((int64_t)d.nx * d.ny)) & 1;
            if (par != color) continue;
        }
        double s = nbr_sum(S.nbr, S.ldn, r, x);
        x[r] = (S.rhs[r] / S.scale + s) / S.diag[r];
    }
}

// ---- wavefront sweeps (level-scheduled, cooperative) ----
enum SweepMode { SW_MIC_BUILD = 0, SW_MIC_FWD = 1, SW_MIC_BWD = 2, SW_GS = 3 };

struct SweepArgs {
    SysView S;
    const int *lvl_rows;
    const int *lvl_off;
    const int *nlevels;  // device
    int reverse;  // iterate levels in descending order
    double tau, sigma;
    const double *src;   // r (fwd) / q (bwd)
    double *dst;         // q (fwd) / z (bwd) / precon (build) / x (gs)
    const double *precon;
    const DevScalars *sc;
    int check_done;
};

template <int MODE>
__device__ __forceinline__ void sweep_row(const SweepArgs &A, int r) {
    const SysView &S = A.S;
    const int *nb = S.nbr;
    int64_t ld = S.ldn;
    double sc_ = S.scale;
    if (MODE == SW_MIC_BUILD) {  // _core.pyx:291-307
        const int dprev[3] = {0, 2, 4}, o1[3] = {3, 1, 1}, o2[3] = {5, 5, 3};
        double e = S.diag[r] * sc_;
#pragma unroll
        for (int p = 0; p < 3; p++) {
            int q = nb[dprev[p] * ld + r];
            if (q >= 0) {
                double pq = q < r ? A.dst[q] : 0.0;  // precon zero-initialised
                e -= (sc_ * pq) * (sc_ * pq);
                double others = 0.0;
                if (nb[o1[p] * ld + q] >= 0) others -= sc_;
                if (nb[o2[p] * ld + q] >= 0) others -= sc_;
                e -= A.tau * (-sc_) * others * pq * pq;
            }
        }
        if (e < A.sigma * S.diag[r] * sc_) e = S.diag[r] * sc_;
        A.dst[r] = 1.0 / sqrt(e);
    } else if (MODE == SW_MIC_FWD) {  // _core.pyx:322-332
        double t = A.src[r];
#pragma unroll
        for (int q = 0; q < 6; q += 2) {
            int k = nb[q * ld + r];
            if (k >= 0) t += sc_ * A.precon[k] * (k < r ? A.dst[k] : 0.0);
        }
        A.dst[r] = t * A.precon[r];
    } else if (MODE == SW_MIC_BWD) {  // _core.pyx:333-346
        double t = A.src[r];
        double pr = A.precon[r];
#pragma unroll
        for (int q = 1; q < 6; q += 2) {
            int k = nb[q * ld + r];
            if (k >= 0) t += sc_ * pr * (k > r ? A.dst[k] : 0.0);
        }
        A.dst[r] = t * pr;
    } else {  // SW_GS, _core.pyx:237-252 (dst is x, in place)
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 6; q++) {
            int k = nb[q * ld + r];
            if (k >= 0) s += A.dst[k];
        }
        A.dst[r] = (S.rhs[r] / sc_ + s) / S.diag[r];
    }
}

template <int MODE>
__global__ void k_sweep_coop(SweepArgs A) {
    if (A.check_done && A.sc->done) return;
    cg::grid_group grid = cg::this_grid();
    int nl = *A.nlevels;
    for (int li = 0; li < nl; li++) {
        int L = A.reverse ? nl - 1 - li : li;
        int b = A.lvl_off[L], e = A.lvl_off[L + 1];
        for (int64_t i = b + gtid(); i < e; i += gstride()) sweep_row<MODE>(A, A.lvl_rows[i]);
        grid.sync();
    }
}

// MIC(0) backward reads z of rows processed earlier; MIC forward-apply
// needs zero-initialised q for generic (non-assembled) neighbour tables.

// ---- levels ----
// Geometric levels for assembled systems: i+j+k of the row's cell.
__global__ void k_lvl_geom(const int *__restrict__ cell, int64_t n, Dims d, int *lvl,
                           int *lvl_cnt) {
    for (int64_t r = gtid(); r < n; r += gstride()) {
        int64_t c = cell[r];
        int L = (int)((c % d.nx) + (c / d.nx) % d.ny + c / ((int64_t)d.nx * d.ny));
        lvl[r] = L;
        atomicAdd(&lvl_cnt[L], 1);
    }
}

// Generic levels by relaxation (plugin API with arbitrary nbr tables):
//   mode 0 forward (deps: d in {0,2,4}, nb < r), 1 backward (d in {1,3,5}, nb > r,
//   level counted from the end), 2 GS (all nb < r, plus anti-deps q < r reading r).
__global__ void k_lvl_relax(SysView S, int mode, int *lvl, int *changed) {
    for (int64_t r = gtid(); r < S.n; r += gstride()) {
        int L = lvl[r];
        int best = L;
        for (int q = 0; q < 6; q++) {
            int nb = S.nbr[q * S.ldn + r];
            if (nb < 0) continue;
            if (mode == 0 && (q & 1) == 0 && nb < r) best = max(best, lvl[nb] + 1);
            if (mode == 1 && (q & 1) == 1 && nb > r) best = max(best, lvl[nb] + 1);
            if (mode == 2) {
                if (nb < r) best = max(best, lvl[nb] + 1);
                else if (nb > r) {  // r reads old x[nb]: nb must run after r
                    int want = L + 1;
                    if (lvl[nb] < want) {
                        atomicMax(&lvl[nb], want);
                        *changed = 1;
                    }
                }
            }
        }
        if (best > L) {
            atomicMax(&lvl[r], best);
            *changed = 1;
        }
    }
}

__global__ void k_lvl_count(const int *lvl, int64_t n, int *lvl_cnt, int *maxlvl) {
    int m = -1;
    for (int64_t r = gtid(); r < n; r += gstride()) {
        atomicAdd(&lvl_cnt[lvl[r]], 1);
        m = max(m, lvl[r]);
    }
    atomicMax(maxlvl, m);
}

__global__ void k_lvl_scatter(const int *lvl, int64_t n, int *cursor, int *lvl_rows) {
    for (int64_t r = gtid(); r < n; r += gstride()) lvl_rows[atomicAdd(&cursor[lvl[r]], 1)] = (int)r;
}

__global__ void k_copy_int(int *dst, const int *src, int64_t n) {
    for (int64_t i = gtid(); i < n; i += gstride()) dst[i] = src[i];
}

__global__ void k_set_nlevels(DevScalars *sc, int nl) { sc->nlevels = nl; }
__global__ void k_nlev_from_max(int *nlev) { nlev[0] = nlev[1] + 1; }

// Rows bucketed by wavefront level: rows[off[L]..off[L+1]) are independent.
struct Levels {
    int *lvl;    // [n] level per row
    int *cnt;    // [cap] counts, then cursors
    int *off;    // [cap + 1]
    int *rows;   // [n]
    int *nlev;   // device: number of levels
    int reverse; // sweep levels in descending order
};

// cnt must hold the per-level counts for levels [0, nlevels_max).
static void bucket_levels(Levels &Lv, int64_t n, int nlevels_max, int *scan_tmp, cudaStream_t st,
                          int64_t *launches) {
    exclusive_scan(ArrayIn{Lv.cnt}, nlevels_max, Lv.off, Lv.off + nlevels_max, scan_tmp, st);
    k_copy_int<<<nblocks(nlevels_max), kThreads, 0, st>>>(Lv.cnt, Lv.off, nlevels_max);
    if (n > 0) k_lvl_scatter<<<nblocks(n), kThreads, 0, st>>>(Lv.lvl, n, Lv.cnt, Lv.rows);
    *launches += 5;
}

static int coop_blocks(const void *fn) {
    static int dev_sms = 0;
    if (!dev_sms) {
        int dev;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kThreads, 0);
    if (per < 1) per = 1;
    if (per > 4) per = 4;
    return dev_sms * per;
}

template <int MODE>
static cudaError_t launch_sweep(SweepArgs A, cudaStream_t st) {
    static int blocks = 0;
    if (!blocks) blocks = coop_blocks((const void *)k_sweep_coop<MODE>);
    void *args[] = {&A};
    return cudaLaunchCooperativeKernel((const void *)k_sweep_coop<MODE>, blocks, kThreads, args, 0, st);
}

// ---- PCG / relaxation scalar kernels ----
__global__ void k_solve_init(DevScalars *sc, double tol, int64_t n, int relax) {
    double rhsmax = __longlong_as_double((long long)sc->rhsmax_bits);
    sc->target = tol * (rhsmax > 1.0 ? rhsmax : 1.0);  // pressure.py:191-193
    sc->iter = 0;
    sc->x_it = 0;
    sc->done = 0;
    sc->converged = 0;
    sc->status = 0;
    sc->err_cell = -1;
    sc->res_bits = 0;
    if (relax) {
        sc->res = INFINITY;
    } else {
        sc->res = rhsmax;  // r = rhs -> res = max|r| (pressure.py:306)
        if (sc->res <= sc->target) {
            sc->done = 1;
            sc->converged = 1;
        }
    }
    if (n == 0) {
        sc->done = 1;
        sc->converged = 1;
        sc->res = 0.0;
    }
}

__global__ void k_check_diag(SysView S, DevScalars *sc, unsigned long long *first_bad) {
    for (int64_t r = S.r0 + gtid(); r < S.r0 + S.n; r += gstride())
        if (!(S.diag[r] > 0.0)) atomicMin(first_bad, (unsigned long long)r);
}

constexpr unsigned long long kNoRow = 0x7f7f7f7f7f7f7f7fULL;  // memset 0x7f: no bad row

__global__ void k_check_diag_final(SysView S, DevScalars *sc, const unsigned long long *first_bad) {
    if (*first_bad != kNoRow) {
        sc->status = FLIP_E_SINGULAR;
        sc->err_cell = S.cell ? S.cell[*first_bad] : (long long)*first_bad;
        sc->done = 1;
    }
}

// x += alpha s; r -= alpha q; res = max|r|  (pressure.py:321-323)
// (rL, posL): also scatter r into the MIC(0) sweep's lane layout
// (k_rows_to_lane fused).
__device__ __forceinline__ void iter_check_body(DevScalars *sc, int64_t max_iters,
                                                double *history, double res) {
    int it = sc->iter + 1;
    sc->iter = it;
    sc->res = res;
    sc->res_bits = 0;
    if (history) history[it - 1] = res;
    if (res <= sc->target) {
        sc->done = 1;
        sc->converged = 1;
    } else if (it >= max_iters) {
        sc->done = 1;
        sc->converged = 0;
    }
}

// r -= alpha q; max|r| (pressure.py:323-326), four rows in flight per
// thread; one max per block, and the block that finishes last runs the
// convergence test (k_iter_check's body), so the PCG loop needs no separate
// check launch.  x += alpha s (pressure.py:322) is applied by k_pcg_dir,
// which reads s anyway (one pass over s per iteration instead of two).
template <int MINB>
__global__ void __launch_bounds__(256, MINB)
k_pcg_update(int64_t n, double *__restrict__ r, const double *__restrict__ q, DevScalars *sc,
             double *__restrict__ rL, const int *__restrict__ posL, int64_t max_iters,
             double *history, int check, HaloReset H) {
    pdl_wait();
    if (sc->done) return;
    halo_reset(H, gtid(), gstride());  // the next two MIC(0) sweeps' halo slots
    __shared__ double wm[8];
    __shared__ bool last;
    const double alpha = sc->alpha;
    const int64_t stride = gstride();
    double m = 0.0;
    int64_t i = gtid();
    for (; i + 3 * stride < n; i += 4 * stride) {
        double rs[4], qs[4];
        int ps[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int64_t j = i + u * stride;
            rs[u] = r[j];
            qs[u] = q[j];
            ps[u] = rL ? posL[j] : 0;
            if (rL && H.on) FLIP_CHECK_RANGE(ps[u], (int64_t)H.TB * H.TC * H.nsteps * H.W * H.W, "update r scatter");
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int64_t j = i + u * stride;
            const double ri = rs[u] - alpha * qs[u];
            r[j] = ri;
            if (rL) rL[ps[u]] = ri;
            m = fmax(m, fabs(ri));
        }
    }
    for (; i < n; i += stride) {
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        if (rL) rL[posL[i]] = ri;
        m = fmax(m, fabs(ri));
    }
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) m = fmax(m, wm[w]);
        if (m > 0.0) atomic_max_nonneg(&sc->res_bits, m);
        __threadfence();
        last = atomicAdd(&sc->upd_ticket, 1u) == gridDim.x - 1;
        if (last) {
            sc->upd_ticket = 0u;
            const double res = __longlong_as_double(
                (long long)atomicAdd(&sc->res_bits, 0ull));
            // slab mode (check 0): the test runs after the MAX allreduce
            if (check) iter_check_body(sc, max_iters, history, res);
        }
    }
}

// convergence test after an iteration (pressure.py:324-326 / 211-213)
__global__ void k_iter_check(DevScalars *sc, int64_t max_iters, double *history) {
    if (sc->done) return;
    iter_check_body(sc, max_iters, history, __longlong_as_double((long long)sc->res_bits));
}

// Jacobi on the compact stencil (_core.pyx:216-234): the neighbour sum in
// nbr order, (rhs / scale + s) / diag with diag the exact neighbour count.
__device__ __forceinline__ double compact_sum(const SysView &S, const double *__restrict__ x,
                                              int64_t r, unsigned m) {
    const unsigned d = S.dy[r];
    const int2 z = S.dz[r];
    double s = 0.0;
    if (m & 1u) s = s + x[r - 1];
    if (m & 2u) s = s + x[r + 1];
    if (m & 4u) s = s + x[r - (int64_t)(d & 0xffffu)];
    if (m & 8u) s = s + x[r + (int64_t)(d >> 16)];
    if (m & 16u) s = s + x[r - (int64_t)z.x];
    if (m & 32u) s = s + x[r + (int64_t)z.y];
    return s;
}

__global__ void __launch_bounds__(256)
k_jacobi_c(SysView S, const double *__restrict__ x, double *__restrict__ out, const DevScalars *sc) {
    pdl_wait();
    if (sc->done) return;
    for (int64_t r = S.r0 + gtid(); r < S.r0 + S.n; r += gstride()) {
        const unsigned m = S.meta[r];
        out[r] = (S.rhs[r] / S.scale + compact_sum(S, x, r, m)) / (double)(m >> 8);
    }
}

// max |rhs - A x| of the new Jacobi iterate (pressure.py:59-62, k_matvec's
// arithmetic); the block that finishes last runs the convergence test
// (k_iter_check's body), so an iteration is two launches.
__global__ void __launch_bounds__(256)
k_resid_c(SysView S, const double *__restrict__ x, DevScalars *sc, int64_t max_iters,
          double *history) {
    pdl_wait();
    if (sc->done) return;
    __shared__ double wm[8];
    __shared__ bool last;
    double mx = 0.0;
    for (int64_t r = S.r0 + gtid(); r < S.r0 + S.n; r += gstride()) {
        const unsigned m = S.meta[r];
        const double yr = S.scale * ((double)(m >> 8) * x[r] - compact_sum(S, x, r, m));
        mx = fmax(mx, fabs(S.rhs[r] - yr));
    }
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); w++) mx = fmax(mx, wm[w]);
        if (mx > 0.0) atomic_max_nonneg(&sc->res_bits, mx);
        __threadfence();
        last = atomicAdd(&sc->upd_ticket, 1u) == gridDim.x - 1;
        if (last) {
            sc->upd_ticket = 0u;
            const double res = __longlong_as_double((long long)atomicAdd(&sc->res_bits, 0ull));
            iter_check_body(sc, max_iters, history, res);
        }
    }
}

// z = r * inv_diag (Jacobi preconditioner, pressure.py:289-293) or z = r
__global__ void k_precond_diag(int64_t n, const double *__restrict__ r, const double *__restrict__ pc,
                               double *__restrict__ z, const DevScalars *sc, int check_done) {
    if (check_done && sc->done) return;
    for (int64_t i = gtid(); i < n; i += gstride()) z[i] = pc ? r[i] * pc[i] : r[i];
}

__global__ void k_inv_diag(int64_t n, const double *__restrict__ diag, double scale,
                           double *__restrict__ pc) {
    for (int64_t i = gtid(); i < n; i += gstride()) pc[i] = 1.0 / (scale * diag[i]);
}

// x += alpha s (pressure.py:322) for the iteration whose update ran, and,
// unless that update ended the solve, s = z + beta s (pressure.py:329).
// The x step belongs to the iteration k_pcg_update last advanced (sc->iter);
// sc->x_it records the last one applied, so launches past the end of the
// solve (or after a breakdown, whose update never ran) change nothing.  Every
// block reads the flags before the last block (ticket) advances x_it.
__global__ void __launch_bounds__(256)
k_pcg_dir(int64_t n, double *__restrict__ s, const double *__restrict__ z,
          double *__restrict__ x, DevScalars *sc) {
    pdl_wait();
    const int it = sc->iter;
    if (it <= sc->x_it) return;  // this iteration's update did not run
    const bool dir = !sc->done;
    const double alpha = sc->alpha, beta = sc->beta;
    for (int64_t i = gtid(); i < n; i += gstride()) {
        const double si = s[i];
        x[i] = x[i] + alpha * si;
        if (dir) s[i] = z[i] + beta * si;
    }
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&sc->dir_ticket, 1u) == gridDim.x - 1;
        if (last) {
            sc->dir_ticket = 0u;
            sc->x_it = it;
        }
    }
}

// Pairwise dot with its summands produced row-coalesced (a row per thread,
// RB rows per thread in flight) into shared memory, then summed there in
// numpy's order (one GPU).  A unit is npu consecutive cut-level nodes of the
// tree (k_dot_fused's nodes); its rows [start, end) are produced by the whole
// block, then each node is summed by an 8-lane group (pw_node8 on the shared
// copy), the unit's nodes by the perfect tree, and the last block reduces the
// unit partials (perfect tree) and runs the epilogue.  Units are handed out by
// an atomic counter.  Same additions in the same order as k_dot_fused, so
// the same bits; what changes is the access pattern of the producer: a row
// functor F gets three phases (independent loads, dependent loads, compute +
// stores) so a thread's RB rows have their loads in flight together.
struct StagedPlan {
    int64_t n = -1;
    int cut = 0, npu = 0;
    int64_t units = 0, smem = 0;
    bool ok = false;
};
constexpr int kStagedMaxUnits = 4096;  // 16 partials per thread in the last block (2^17 nodes)

__device__ __forceinline__ void pw_node_span(int64_t n, int cut, int64_t node, int64_t *s,
                                             int64_t *len) {
    int64_t s0 = 0, l = n;
    for (int lvl = cut - 1; lvl >= 0; lvl--) {
        const int64_t n2 = pw_split(l);
        if ((node >> lvl) & 1) {
            s0 += n2;
            l -= n2;
        } else {
            l = n2;
        }
    }
    *s = s0;
    *len = l;
}

struct LdSmem {
    const double *p;  // p[i - base] = summand i (base = the unit's first row)
    int64_t base;
    __device__ __forceinline__ double operator()(int64_t i) const { return p[(int)(i - base)]; }
};

// z from the lane-major layout of the MIC(0) sweep (LdLaneDot): z[r] written,
// summand z[r] * r[r]: pressure.py:328-329.
struct RowLaneDot {
    const double *__restrict__ zL;
    const int *__restrict__ posL;
    double *__restrict__ z;
    const double *__restrict__ r;
    int64_t nL;
    struct A { int p; double rr; };
    struct B { double zi; };
    __device__ __forceinline__ A pre(int64_t i) const { return {posL[i], r[i]}; }
    __device__ __forceinline__ B mid(int64_t, const A &a) const {
        FLIP_CHECK_RANGE((int64_t)a.p, nL, "z.r dot lane gather");
        return {zL[a.p]};
    }
    __device__ __forceinline__ double post(int64_t i, const A &a, const B &b) const {
        z[i] = b.zi;
        return b.zi * a.rr;
    }
};

template <class F, int RB, int MINB = 1>
__global__ void __launch_bounds__(256, MINB)
k_dot_staged(F f, int64_t n, int cut, int npu, int64_t units, double *__restrict__ part,
             unsigned *ctr, int epi, DevScalars *sc) {
    extern __shared__ double prod[];
    __shared__ double sv[256];
    __shared__ int64_t span[2];
    __shared__ long long unit_s;
    __shared__ bool last;
    pdl_wait();
    if (sc->done) return;  // uniform: the flag changes only in the last block
    const int tid = threadIdx.x;
    const int grp = tid >> 3, g = tid & 7;
    while (true) {
        if (tid == 0) unit_s = (long long)atomicAdd(&ctr[1], 1u);
        __syncthreads();
        const int64_t u = unit_s;
        if (u >= units) break;
        int64_t ns = 0, nl = 0;
        if (grp < npu) {
            pw_node_span(n, cut, u * npu + grp, &ns, &nl);
            if (tid == 0) span[0] = ns;
            if (grp == npu - 1 && g == 0) span[1] = ns + nl;
        }
        __syncthreads();
        const int64_t a0 = span[0], b0 = span[1];
        for (int64_t rb = a0 + tid; rb < b0; rb += RB * 256) {
            typename F::A pa[RB];
            typename F::B pb[RB];
#pragma unroll
            for (int k = 0; k < RB; k++)
                if (rb + k * 256 < b0) pa[k] = f.pre(rb + k * 256);
#pragma unroll
            for (int k = 0; k < RB; k++)
                if (rb + k * 256 < b0) pb[k] = f.mid(rb + k * 256, pa[k]);
#pragma unroll
            for (int k = 0; k < RB; k++)
                if (rb + k * 256 < b0) prod[rb + k * 256 - a0] = f.post(rb + k * 256, pa[k], pb[k]);
        }
        __syncthreads();
        double val = 0.0;
        if (grp < npu) val = pw_node8<2>(LdSmem{prod, a0}, ns, nl, g);
        // the unit's perfect tree (pairs first): 4 nodes per warp, then warps
        if (npu >= 2) val = val + __shfl_xor_sync(0xffffffffu, val, 8);
        if (npu >= 4) val = val + __shfl_xor_sync(0xffffffffu, val, 16);
        if ((tid & 31) == 0) sv[tid >> 5] = val;
        __syncthreads();
        if (tid == 0) {
            const int cw = npu >= 4 ? npu / 4 : 1;
            for (int st = 1; st < cw; st <<= 1)
                for (int i = 0; i + st < cw; i += 2 * st) sv[i] = sv[i] + sv[i + st];
            part[u] = sv[0];
        }
    }
    if (tid == 0) {
        __threadfence();
        last = atomicAdd(&ctr[0], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    // perfect tree over the unit partials: up to 16 consecutive per thread in
    // registers (the tree's lowest levels), then over the thread sums
    const int m = (int)units;
    const int per = m > 256 ? m / 256 : 1, cnt = m / per;
    if (tid < cnt) {
        double v[16];
#pragma unroll
        for (int k = 0; k < 16; k++) v[k] = k < per ? __ldcg(part + (int64_t)tid * per + k) : 0.0;
#pragma unroll
        for (int st = 1; st < 16; st <<= 1)
#pragma unroll
            for (int i = 0; i + st < 16; i += 2 * st)
                if (i + st < per) v[i] = v[i] + v[i + st];
        sv[tid] = v[0];
    }
    __syncthreads();
    for (int st = 1; st < cnt; st <<= 1) {
        for (int i = tid * 2 * st; i + st < cnt; i += blockDim.x * 2 * st) sv[i] = sv[i] + sv[i + st];
        __syncthreads();
    }
    if (tid == 0) {
        dot_epilogue(sv[0], epi, nullptr, sc);
        ctr[0] = 0u;
        ctr[1] = 0u;
    }
}

static int pw_cut_maxlen(int64_t n, int64_t *maxlen) {
    std::vector<int64_t> sizes{n};
    int cut = 0;
    while (true) {
        bool all_split = true;
        for (int64_t s : sizes) all_split &= s > 128;
        if (!all_split) break;
        std::vector<int64_t> nxt;
        for (int64_t s : sizes) {
            const int64_t n2 = s / 2 - (s / 2) % 8;
            nxt.push_back(n2);
            nxt.push_back(s - n2);
        }
        std::sort(nxt.begin(), nxt.end());
        nxt.erase(std::unique(nxt.begin(), nxt.end()), nxt.end());
        sizes.swap(nxt);
        cut++;
    }
    *maxlen = *std::max_element(sizes.begin(), sizes.end());
    return cut;
}

// Plan of k_dot_staged for n rows; !ok when the shape is out of its range
// (k_dot_fused then runs).
static const StagedPlan &staged_plan(int64_t n) {
    static thread_local StagedPlan P;
    if (P.n == n) return P;
    P = StagedPlan{};
    P.n = n;
    if (n <= 0) return P;
    int64_t maxlen = 0;
    P.cut = pw_cut_maxlen(n, &maxlen);
    const int64_t nodes = (int64_t)1 << P.cut;
    // 32 nodes per unit (every 8-lane group of the block sums one): 8 -> 49.7,
    // 16 -> 49.25, 32 -> 48.98 ms/step at 256^3 (fewer barriers per row)
    const int64_t npu = std::min<int64_t>(nodes, 32);
    if (nodes / npu > kStagedMaxUnits) return P;
    P.npu = (int)npu;
    P.units = nodes / npu;
    P.smem = maxlen * npu * (int64_t)sizeof(double);
    if (P.smem > 48 * 1024) return P;
    P.ok = true;
    return P;
}

template <class F, int RB, int MINB = 1>
static void launch_dot_staged(const F &f, int64_t n, double *tmp, int epi, DevScalars *sc,
                              cudaStream_t st, int64_t *launches) {
    const StagedPlan &P = staged_plan(n);
    static thread_local int64_t occ_smem = -1;
    static thread_local int per_sm = 1;
    if (occ_smem != P.smem) {
        occ_smem = P.smem;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dot_staged<F, RB, MINB>, 256,
                                                          (size_t)P.smem) != cudaSuccess ||
            per_sm < 1) {
            cudaGetLastError();
            per_sm = 1;
        }
    }
    const unsigned grid = (unsigned)std::min<int64_t>(P.units, (int64_t)num_sms() * per_sm);
    // tmp[1]: finish ticket + unit counter (zeroed at allocation, re-armed
    // by the last block); unit partials from tmp + 2
    launch_pdl(k_dot_staged<F, RB, MINB>, grid, 256, (size_t)P.smem, st, f, n, P.cut, P.npu, P.units,
               tmp + 2, reinterpret_cast<unsigned *>(tmp + 1), epi, sc);
    (*launches)++;
}

__global__ void k_fill(double *a, int64_t n, double v) {
    for (int64_t i = gtid(); i < n; i += gstride()) a[i] = v;
}

// ---- solver driver ----
struct SolveBufs {
    double *x, *r, *z, *s, *q, *tq, *precon, *xtmp, *dot_tmp;
    int *scan_tmp;
    unsigned long long *u64_scratch;  // >= 1
};

struct SolveCfg {
    int solver, precond;
    int64_t max_iters;
    double tol;
    int check_every;
    double *history;  // device, may be null
    // RBGS colours: explicit row lists (plugin API) or parity of the row's
    // cell (assembled systems, pressure.py:166-170)
    const int *red, *black;
    int64_t nred, nblack;
    Dims d;
    // slab mode (null otherwise): S covers the rank's own rows; `full` is
    // the whole system for the replicated MIC(0) / GS / multigrid sweeps
    SlabDot *slab = nullptr;
    const SysView *full = nullptr;
};

struct SolveOut {
    int64_t iterations;
    double residual;
    int converged;
    int status;
    int64_t err_cell, err_it;
    double err_value;
};

template <int MODE>
static void sweep(const SysView &S, const Levels &L, int reverse, const double *src, double *dst,
                  const double *precon, DevScalars *sc, int check_done, cudaStream_t st,
                  int64_t *launches) {
    SweepArgs A{S, L.rows, L.off, L.nlev, reverse, 0.97, 0.25, src, dst, precon, sc, check_done};
    launch_sweep<MODE>(A, st);
    (*launches)++;
}

// How the sequential sweeps are scheduled: for assembled systems the
// pipelined tile wavefront (wavefront.cu); for arbitrary neighbour tables
// (plugin API) level-scheduled cooperative sweeps over relaxed levels.
// Lane-major layout of the MIC(0) substitution operands (assembled systems).
struct LaneBufs {
    LaneArgs args;       // geometry, halos, ticket, scale
    const int *posL;     // row -> L entry
    double *rL, *tqL, *zL, *preL;
    HaloReset hr{};      // quad: per-direction halo buffers, reset by k_pcg_update
};

struct SweepLevels {
    const Levels *fwd, *bwd, *gs;
    int bwd_reverse;
    const WaveArgs *wave;  // non-null: use the pipelined wavefront
    Probe *probe;          // optional event bracketing of the MIC substitutions
    const LaneBufs *lane;  // non-null: MIC(0) apply through the lane-major kernels
    Ctx *mg = nullptr;     // multigrid preconditioner state (FLIP_PRECOND_MG)
};

// First sweep-launch failure of the current solve (configuration errors
// such as a shared-memory request are not sticky CUDA errors, and
// cudaGetLastError in the launchers clears them).  Per host thread, like
// the error message, so contexts driven from different threads (one per
// GPU) never see each other's failures.
static thread_local cudaError_t g_sweep_launch_err = cudaSuccess;

template <int MODE>
static void do_sweep(const SysView &S, const SweepLevels &LV, const double *src, double *dst,
                     const double *precon, DevScalars *sc, cudaStream_t st, int64_t *launches) {
    if (LV.wave) {
        WaveArgs A = *LV.wave;
        A.src = src;
        A.dst = dst;
        A.precon = precon;
        A.sc = sc;
        Probe *pb = LV.probe;
        bool probed = pb && pb->kind == 1 && (MODE == SW_MIC_FWD || MODE == SW_MIC_BWD) &&
                      pb->used < Probe::kMax;
        if (probed) cudaEventRecord(pb->ev[2 * pb->used], st);
        cudaError_t e = launch_wave(MODE, A, st);
        if (probed) {
            cudaEventRecord(pb->ev[2 * pb->used + 1], st);
            pb->used++;
            pb->launches++;
            pb->bytes += 24.0 * (double)A.n;  // src + precon read, dst written: 3 x 8 B per row
        }
        if (e != cudaSuccess) {
            set_error(std::string("wavefront launch: ") + cudaGetErrorString(e));
            if (g_sweep_launch_err == cudaSuccess) g_sweep_launch_err = e;  // fails the solve
        }
        *launches += 2;
        return;
    }
    const Levels &L = MODE == SW_GS ? *LV.gs : (MODE == SW_MIC_BWD ? *LV.bwd : *LV.fwd);
    sweep<MODE>(S, L, MODE == SW_MIC_BWD ? LV.bwd_reverse : 0, src, dst, precon, sc, 1, st,
                launches);
}

// z = M^-1 r for the selected preconditioner (pressure.py:284-300).

// fused: the lane path's r -> L and L -> z conversions are done by the
// caller's k_pcg_update and z.r dot (r already in Lb.rL, z left in Lb.zL).
// (Scattering z into row order from inside the backward sweep instead was
// measured slower: +36 us per sweep for -21 us in the dot at 256^3.)
// Pinned read-back slots of the solver's done flag (one ring per host
// thread and device; see run_solve).
constexpr int kPollDepth = 3;
struct PollRing {
    DevScalars *h = nullptr;
    cudaEvent_t ev[kPollDepth] = {};
};
static PollRing &poll_ring() {
    static thread_local PollRing rings[64];
    int dev = 0;
    cudaGetDevice(&dev);
    PollRing &r = rings[dev & 63];
    if (!r.h) {
        cudaMallocHost((void **)&r.h, sizeof(DevScalars) * kPollDepth);
        for (auto &e : r.ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    }
    return r;
}

// Comm failure inside the solve loop (slab mode): the first one fails it.
static thread_local int g_slab_err = 0;

// r (own rows) -> every rank: the MIC(0) / multigrid preconditioners are
// global recurrences, replicated on each rank of a slab decomposition.
static void slab_gather_rows(const SolveCfg &cfg, double *v) {
    Ctx &c = *cfg.slab->c;
    std::vector<int64_t> off(c.slab.world + 1);
    for (int q = 0; q <= c.slab.world; q++) off[q] = 8 * c.slab.rstart[q];
    if (int rc = slab_allgatherv(c, v, off.data()))
        if (!g_slab_err) g_slab_err = rc;
}

static void slab_halo(const SolveCfg &cfg, double *v) {
    if (int rc = slab_row_halo(*cfg.slab->c, v))
        if (!g_slab_err) g_slab_err = rc;
}

static void slab_max(const SolveCfg &cfg, unsigned long long *bits) {
    if (int rc = slab_allreduce(*cfg.slab->c, (int64_t *)bits, 1, FLIP_OP_MAX))
        if (!g_slab_err) g_slab_err = rc;
}

template <class LD>
static void solver_dot(const SolveCfg &cfg, const LD &ld, int64_t n_full, double *tmp, int epi,
                       DevScalars *sc, cudaStream_t st, int64_t *launches) {
    if (cfg.slab) {
        if (int rc = launch_dot_slab(*cfg.slab, ld, n_full, nullptr, epi, sc, st, launches))
            if (!g_slab_err) g_slab_err = rc;
        return;
    }
    launch_dot_f(ld, n_full, tmp, nullptr, epi, sc, st, launches);
}

static void apply_pc(const SysView &S, const SolveCfg &cfg, const SolveBufs &B,
                     const SweepLevels &LV, const double *r, double *z, DevScalars *sc,
                     cudaStream_t st, int64_t *launches, bool fused = false) {
    const bool replicated = cfg.precond == FLIP_PRECOND_MG || cfg.precond == FLIP_PRECOND_MIC0;
    const SysView &F = (cfg.slab && replicated) ? *cfg.full : S;  // rows the sweep covers
    if (cfg.slab && replicated) slab_gather_rows(cfg, const_cast<double *>(r));
    if (cfg.precond == FLIP_PRECOND_MG) {
        mg_apply(*LV.mg, r, z, F.n, sc, st, launches);
        return;
    }
    if (cfg.precond == FLIP_PRECOND_MIC0 && LV.lane) {
        // r -> L layout, forward (L), backward (L), back to rows
        const LaneBufs &Lb = *LV.lane;
        if (!fused || cfg.slab) launch_rows_to_lane(r, Lb.posL, F.n, Lb.rL, sc, st);
        Probe *pb = LV.probe;
        for (int rev = 0; rev < 2; rev++) {
            LaneArgs A = Lb.args;
            A.src = rev ? Lb.tqL : Lb.rL;
            A.dst = rev ? Lb.zL : Lb.tqL;
            A.precon = Lb.preL;
            A.sc = sc;
            if (Lb.hr.on) {  // quad: own halo buffer and ticket per direction
                A.halo_y = Lb.hr.hy[rev];
                A.ticket = Lb.hr.ticket[rev];
                A.prepped = fused ? 1 : 0;  // in the loop k_pcg_update reset them
            }
            const bool stamped = pb && pb->kind == 1 && Lb.hr.on && pb->ts;  // quad: device stamps
            if (stamped) A.ts = pb->ts;
            bool probed = !stamped && pb && pb->kind == 1 && pb->used < Probe::kMax;
            if (probed) cudaEventRecord(pb->ev[2 * pb->used], st);
            cudaError_t e = launch_mic_lane(rev != 0, A, st);
            if (e != cudaSuccess) {
                set_error(std::string("lane sweep launch: ") + cudaGetErrorString(e));
                if (g_sweep_launch_err == cudaSuccess) g_sweep_launch_err = e;  // fails the solve
            }
            if (probed) {
                cudaEventRecord(pb->ev[2 * pb->used + 1], st);
                pb->used++;
                pb->launches++;
                pb->bytes += 24.0 * (double)F.n;  // src + precon read, dst written per row
            }
        }
        if (!fused) launch_lane_to_rows(Lb.zL, Lb.posL, F.n, z, sc, st);
        *launches += 2 * 2 + (fused ? 0 : 2) + (cfg.slab && fused ? 1 : 0);
    } else if (cfg.precond == FLIP_PRECOND_MIC0) {
        // forward substitution into tq, then backward into z
        do_sweep<SW_MIC_FWD>(F, LV, r, B.tq, B.precon, sc, st, launches);
        do_sweep<SW_MIC_BWD>(F, LV, B.tq, z, B.precon, sc, st, launches);
    } else {
        const int64_t o = S.r0;  // own rows (slab) or all rows
        k_precond_diag<<<nblocks(S.n), kThreads, 0, st>>>(
            S.n, r + o, cfg.precond == FLIP_PRECOND_JACOBI ? B.precon + o : nullptr, z + o, sc, 1);
        (*launches)++;
    }
}

// Inputs of the quad MIC(0) build in the lane layout: diag, and per row the
// code k_x + 3 k_y + 9 k_z, k_p = how many of the pair-p lower neighbour's
// o1 / o2 neighbours are rows (_core.pyx:285-303).  Only row entries are
// written (the others keep the ABSENT marker k_lane_map put there).
__global__ void k_build_inputs(SysView S, const int *__restrict__ posL, double *__restrict__ diagL,
                               double *__restrict__ codeL) {
    const int dprev[3] = {0, 2, 4}, o1[3] = {3, 1, 1}, o2[3] = {5, 5, 3};
    const int *nb = S.nbr;
    const int64_t ld = S.ldn;
    for (int64_t r = gtid(); r < S.n; r += gstride()) {
        int code = 0, mul = 1;
#pragma unroll
        for (int p = 0; p < 3; p++) {
            const int q = nb[dprev[p] * ld + r];
            int k = 0;
            if (q >= 0) k = (nb[o1[p] * ld + q] >= 0) + (nb[o2[p] * ld + q] >= 0);
            code += k * mul;
            mul *= 3;
        }
        const int e = posL[r];
        diagL[e] = S.diag[r];
        codeL[e] = (double)code;
    }
}

// Device-driven solver loop: a graph holding one WHILE conditional node
// whose body (captured from the stream) is one solver iteration followed by
// k_loop_cond, which keeps the loop running while the done flag is clear.
__global__ void k_loop_cond(cudaGraphConditionalHandle h, const DevScalars *sc) {
    pdl_wait();
    cudaGraphSetConditional(h, sc->done ? 0u : 1u);
}

template <class F>
static cudaError_t loop_graph(cudaStream_t st, const DevScalars *sc, int unroll, F &&body) {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t x = nullptr;
    cudaGraphConditionalHandle h = 0;
    cudaError_t e = cudaGraphCreate(&g, 0);
    if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams np = {};
    if (e == cudaSuccess) {
        np.type = cudaGraphNodeTypeConditional;
        np.conditional.handle = h;
        np.conditional.type = cudaGraphCondTypeWhile;
        np.conditional.size = 1;
        cudaGraphNode_t node;
        e = cudaGraphAddNode(&node, g, nullptr, 0, &np);
    }
    if (e == cudaSuccess) {
        e = cudaStreamBeginCaptureToGraph(st, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                          cudaStreamCaptureModeRelaxed);
        if (e == cudaSuccess) {
            for (int u = 0; u < unroll; u++) body();  // iterations past `done` exit at once
            launch_pdl(k_loop_cond, 1, 1, 0, st, h, sc);
            cudaGraph_t out = nullptr;
            const cudaError_t e1 = cudaGetLastError();
            const cudaError_t e2 = cudaStreamEndCapture(st, &out);
            e = e1 != cudaSuccess ? e1 : e2;
        }
    }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&x, g, 0);
    if (e == cudaSuccess) e = cudaGraphLaunch(x, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the exec is destroyed below
    if (x) cudaGraphExecDestroy(x);
    if (g) cudaGraphDestroy(g);
    return e;
}

// Runs SOLVERS[solver](sys, max_iters, tol) (pressure.py:200-332) on the
// device.  sc->rhsmax_bits must hold max|rhs|.  Host syncs once per
// check_every iterations to poll the done flag.
//
// Slab mode (cfg.slab): S covers the rank's own rows [S.r0, S.r0 + S.n) of
// the global row vectors; before every stencil pass the rows of the
// neighbouring planes are refreshed (slab_row_halo), max-norms are MAX-
// allreduced, the dots run the distributed numpy tree, and the MIC(0) / GS /
// multigrid sweeps run replicated on the gathered vector.  Every rank makes
// the same sequence of exchanges, and every decision (done, converged) is
// taken on globally reduced values, so all ranks stop together.
static int run_solve(const SysView &S, const SolveCfg &cfg, const SolveBufs &B,
                     const SweepLevels &LV, DevScalars *sc, DevScalars *sch, cudaStream_t st,
                     int64_t *launches, SolveOut *out) {
    const bool sl = cfg.slab != nullptr;
    const int64_t n = S.n;                       // rows computed here
    const int64_t o = S.r0;                      // first of them (global numbering)
    const int64_t nf = sl ? cfg.full->n : n;     // rows of the whole system
    Slab *SL = sl ? &cfg.slab->c->slab : nullptr;
    g_slab_err = 0;
    bool relax = cfg.solver != FLIP_SOLVER_PCG;
    k_solve_init<<<1, 1, 0, st>>>(sc, cfg.tol, nf, relax ? 1 : 0);
    cudaMemsetAsync(B.u64_scratch, 0x7f, sizeof(unsigned long long), st);
    (*launches)++;
    if (nf > 0) {
        k_check_diag<<<nblocks(n), kThreads, 0, st>>>(S, sc, B.u64_scratch);
        if (sl)
            if (int rc = slab_allreduce(*cfg.slab->c, (int64_t *)B.u64_scratch, 1, FLIP_OP_MIN))
                return rc;
        k_check_diag_final<<<1, 1, 0, st>>>(S, sc, B.u64_scratch);
        *launches += 2;
        k_fill<<<nblocks(nf), kThreads, 0, st>>>(B.x, nf, 0.0);
        (*launches)++;
    }
    static const int every_env = getenv("FLIPB200_CHECK_EVERY") ? atoi(getenv("FLIPB200_CHECK_EVERY")) : 0;
    int every = cfg.check_every > 0 ? cfg.check_every : every_env > 0 ? every_env : (relax ? 64 : 8);
    const bool lane = cfg.precond == FLIP_PRECOND_MIC0 && LV.lane;
    if (nf > 0 && !relax) {
        if (cfg.precond == FLIP_PRECOND_MIC0) {
            // quad lane path: the build runs on the quad wavefront too
            // (inputs in the lane layout, precon straight into it); 0.56 ms
            // on the row-layout wavefront at 256^3
            static const bool qbuild = !getenv("FLIPB200_QUAD_BUILD") || atoi(getenv("FLIPB200_QUAD_BUILD"));
            bool built = false;
            if (LV.lane && LV.lane->hr.on && qbuild) {
                const SysView &F = sl ? *cfg.full : S;
                const LaneBufs &Lb = *LV.lane;
                k_build_inputs<<<nblocks(F.n), kThreads, 0, st>>>(F, Lb.posL, Lb.rL, Lb.tqL);
                LaneArgs A = Lb.args;
                A.src = Lb.rL;
                A.precon = Lb.tqL;
                A.dst = Lb.preL;
                A.sc = nullptr;
                A.halo_y = Lb.hr.hy[0];
                A.ticket = Lb.hr.ticket[0];
                const cudaError_t e = launch_mic_lane_build(A, st);
                if (e == cudaSuccess) {
                    // the row-order copy (slab gathers, debug reads)
                    launch_lane_to_rows(Lb.preL, Lb.posL, nf, B.precon, nullptr, st);
                    *launches += 4;
                    built = true;
                } else {
                    cudaGetLastError();
                }
            }
            if (!built) {
                do_sweep<SW_MIC_BUILD>(sl ? *cfg.full : S, LV, nullptr, B.precon, nullptr, sc, st,
                                       launches);
                if (LV.lane) {
                    launch_rows_to_lane(B.precon, LV.lane->posL, nf, LV.lane->preL, sc, st);
                    (*launches)++;
                }
            }
        }
        else if (cfg.precond == FLIP_PRECOND_JACOBI) {
            k_inv_diag<<<nblocks(n), kThreads, 0, st>>>(n, S.diag + o, S.scale, B.precon + o);
            (*launches)++;
        }
        cudaMemcpyAsync(B.r + o, S.rhs + o, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
        apply_pc(S, cfg, B, LV, B.r, B.z, sc, st, launches);
        cudaMemcpyAsync(B.s + o, B.z + o, sizeof(double) * n, cudaMemcpyDeviceToDevice, st);
        if (sl) slab_halo(cfg, B.s);
        solver_dot(cfg, LdProd{B.z, B.r}, nf, B.dot_tmp, EPI_SIGMA0, sc, st, launches);
    }
    if (nf > 0 && relax && cfg.solver == FLIP_SOLVER_GS && sl) {
        // lexicographic GS is one global recurrence: replicated on the
        // gathered rhs (every rank then holds the same full iterate)
        slab_gather_rows(cfg, const_cast<double *>(S.rhs));
    }
    // Jacobi on the compact stencil with ping-pong iterates and the test in
    // the residual kernel (one GPU): two PDL launches per iteration
    static const bool jfast_env = !getenv("FLIPB200_JACOBI_PLAIN");
    const bool jfast = cfg.solver == FLIP_SOLVER_JACOBI && !sl && S.meta && jfast_env;
    int64_t jit = 0;  // Jacobi iterations issued (buffer parity)
    // PCG on one GPU: the z.r dot with the lane gather produces its summands
    // row-coalesced (k_dot_staged: 35.6 -> ~26 us per iteration at 256^3);
    // FLIPB200_STAGED_ZR=0 keeps k_dot_fused<LdLaneDot>
    static const bool st_zr_env = !getenv("FLIPB200_STAGED_ZR") || atoi(getenv("FLIPB200_STAGED_ZR"));
    const bool st_zr = !relax && !sl && nf > 0 && S.r0 == 0 && st_zr_env && staged_plan(n).ok;
    // one iteration of SOLVERS[cfg.solver] (pressure.py:209-213 / 314-331)
    auto one_iter = [&]() {
        if (!relax) {  // pressure.py:314-331
            // r also lands in the lane layout and z comes back through the
            // z.r dot (pressure.py:314-331); q = A s can be fused into the
            // s.q dot too (FLIPB200_FUSE_MATVEC, slower: 8-lane groups
            // coalesce the stencil gathers worse than k_matvec)
            static const bool fuse_mv = getenv("FLIPB200_FUSE_MATVEC") != nullptr;
            if (fuse_mv && !sl) {
                launch_dot_f(LdMatvecDot{S, B.s, B.q}, n, B.dot_tmp, nullptr, EPI_CURV, sc,
                             st, launches);
            } else {
                if (S.meta)
                    launch_pdl(k_matvec_c, wave_blocks(k_matvec_c, n), kThreads, 0, st, S, B.s, B.q, sc);
                else
                    k_matvec<<<nblocks(n), kThreads, 0, st>>>(S, B.s, B.q, nullptr, nullptr,
                                                              nullptr, sc, 1);
                solver_dot(cfg, LdProd{B.s, B.q}, nf, B.dot_tmp, EPI_CURV, sc, st, launches);
                (*launches)++;
            }
            static const int upd_minb = getenv("FLIPB200_UPDATE_MINB") ? atoi(getenv("FLIPB200_UPDATE_MINB")) : 1;
            auto kupd = upd_minb == 6 ? k_pcg_update<6> : upd_minb == 8 ? k_pcg_update<8> : k_pcg_update<1>;
            launch_pdl(kupd, wave_blocks(kupd, n), kThreads, 0, st, n,
                       B.r + o, (const double *)(B.q + o), sc,
                       (lane && !sl) ? LV.lane->rL : nullptr,
                       (lane && !sl) ? (const int *)LV.lane->posL : nullptr,
                       (int64_t)cfg.max_iters, cfg.history, sl ? 0 : 1,
                       lane ? LV.lane->hr : HaloReset{});
            if (sl) {
                slab_max(cfg, &sc->res_bits);
                k_iter_check<<<1, 1, 0, st>>>(sc, cfg.max_iters, cfg.history);
                (*launches)++;
            }
            apply_pc(S, cfg, B, LV, B.r, B.z, sc, st, launches, lane);
            if (lane && st_zr) {
                const RowLaneDot f{LV.lane->zL, LV.lane->posL, B.z, B.r,
                                   lane_entries(LV.lane->args.geom)};
                // 5 CTAs/SM (48 registers): PROJECT 37.86 -> 37.47 ms vs 66
                // registers at 4; 6 (40, spills) 37.8
                launch_dot_staged<RowLaneDot, 4, 5>(f, n, B.dot_tmp, EPI_SIGMA_NEW, sc, st, launches);
            }
            else if (lane)
                solver_dot(cfg, LdLaneDot{LV.lane->zL, LV.lane->posL, B.z, B.r, lane_entries(LV.lane->args.geom)}, nf, B.dot_tmp,
                           EPI_SIGMA_NEW, sc, st, launches);
            else
                solver_dot(cfg, LdProd{B.z, B.r}, nf, B.dot_tmp, EPI_SIGMA_NEW, sc, st,
                           launches);
            launch_pdl(k_pcg_dir, wave_blocks(k_pcg_dir, n), kThreads, 0, st, n, B.s + o,
                       (const double *)(B.z + o), B.x + o, sc);
            if (sl) slab_halo(cfg, B.s);
            *launches += 2;  // update (with the convergence test) + dir
        } else {  // pressure.py:209-213
            if (cfg.solver == FLIP_SOLVER_JACOBI && jfast) {
                // ping-pong iterates (the reference's x = sweep(x) makes a new
                // array): iteration k reads buf[(k-1)%2], writes buf[k%2]
                double *xin = (jit & 1) ? B.xtmp : B.x, *xout = (jit & 1) ? B.x : B.xtmp;
                jit++;
                launch_pdl(k_jacobi_c, wave_blocks(k_jacobi_c, n), kThreads, 0, st, S,
                           (const double *)xin, xout, (const DevScalars *)sc);
                launch_pdl(k_resid_c, wave_blocks(k_resid_c, n), kThreads, 0, st, S,
                           (const double *)xout, sc, (int64_t)cfg.max_iters, cfg.history);
                *launches += 2;
                return;  // the convergence test ran in k_resid_c
            }
            if (cfg.solver == FLIP_SOLVER_JACOBI) {
                k_jacobi<<<nblocks(n), kThreads, 0, st>>>(S, B.x, B.xtmp, sc, 1);
                if (sl) slab_halo(cfg, B.xtmp);
                k_matvec<<<nblocks(n), kThreads, 0, st>>>(S, B.xtmp, nullptr, S.rhs, &sc->res_bits,
                                                          B.x, sc, 1);
                if (sl) {  // the halo rows of x follow xtmp's
                    cudaMemcpyAsync(B.x + SL->Rlo, B.xtmp + SL->Rlo,
                                    sizeof(double) * (SL->R0 - SL->Rlo), cudaMemcpyDeviceToDevice, st);
                    cudaMemcpyAsync(B.x + SL->R1, B.xtmp + SL->R1,
                                    sizeof(double) * (SL->Rhi - SL->R1), cudaMemcpyDeviceToDevice, st);
                }
                *launches += 2;
            } else {
                bool gs_oop = cfg.solver == FLIP_SOLVER_GS && LV.wave;
                if (cfg.solver == FLIP_SOLVER_GS) {
                    const SysView &F = sl ? *cfg.full : S;
                    if (LV.wave) {  // out of place: old x in, new x out, copied back below
                        do_sweep<SW_GS>(F, LV, B.x, B.xtmp, nullptr, sc, st, launches);
                    } else {
                        do_sweep<SW_GS>(F, LV, nullptr, B.x, nullptr, sc, st, launches);
                    }
                } else {
                    k_gs_rows<<<nblocks(cfg.red ? cfg.nred : n), kThreads, 0, st>>>(
                        S, cfg.red, cfg.nred, 0, cfg.d, B.x, sc, 1);
                    if (sl) slab_halo(cfg, B.x);
                    k_gs_rows<<<nblocks(cfg.black ? cfg.nblack : n), kThreads, 0, st>>>(
                        S, cfg.black, cfg.nblack, 1, cfg.d, B.x, sc, 1);
                    if (sl) slab_halo(cfg, B.x);
                    *launches += 2;
                }
                k_matvec<<<nblocks(n), kThreads, 0, st>>>(S, gs_oop ? B.xtmp : B.x, nullptr,
                                                          S.rhs, &sc->res_bits,
                                                          (gs_oop && !sl) ? B.x : nullptr, sc, 1);
                if (gs_oop && sl)  // the replicated iterate, every row
                    cudaMemcpyAsync(B.x, B.xtmp, sizeof(double) * nf, cudaMemcpyDeviceToDevice, st);
                (*launches)++;
            }
            if (sl) slab_max(cfg, &sc->res_bits);
            k_iter_check<<<1, 1, 0, st>>>(sc, cfg.max_iters, cfg.history);
            (*launches)++;
        }
    };
    int64_t it = 0, nbatch = 0, seen = 0;
    // FLIPB200_GRAPH=1 (one GPU): the whole loop is one CUDA graph -- a WHILE
    // conditional node whose body is `unroll` iterations and whose condition
    // (!done) is set on the device by the body's last kernel, so the host is
    // not involved until the solve ends.  Measured 0.6 ms/step slower than
    // the stream loop below at 256^3 (62.3 vs 61.7 ms; the per-solve capture
    // and instantiation, and the WHILE round trips), so it is opt-in; the
    // stream loop never drains the stream either (its done-flag reads are
    // asynchronous).  The event probe needs the stream loop; the quad
    // sweeps' device-stamp probe works in both.
    static const bool graph_env = [] {
        const char *e = getenv("FLIPB200_GRAPH");
        return e ? atoi(e) != 0 : false;
    }();
    int64_t graph_per_iter = 0, graph_l0 = 0, graph_unroll = 1;  // launch accounting (graph mode)
    const bool stamps = LV.probe && LV.probe->kind == 1 && LV.lane && LV.lane->hr.on && LV.probe->ts &&
                        cfg.precond == FLIP_PRECOND_MIC0;
    if (nf > 0 && !sl && graph_env && !(LV.probe && LV.probe->kind == 1 && !stamps)) {
        // a body of `unroll` iterations: fewer WHILE round trips per solve
        static const int unroll = [] {
            const char *e = getenv("FLIPB200_GRAPH_UNROLL");
            const int v = e ? atoi(e) : 4;
            return v < 1 ? 1 : v > 64 ? 64 : v;
        }();
        graph_l0 = *launches;
        graph_unroll = unroll;
        cudaError_t ge = loop_graph(st, sc, unroll, one_iter);
        graph_per_iter = (*launches - graph_l0) / unroll;
        if (ge != cudaSuccess) {
            set_error(std::string("solver graph: ") + cudaGetErrorString(ge));
            return FLIP_E_CUDA;
        }
        it = cfg.max_iters;  // the device ran the loop to its end
    }
    while (nf > 0 && it < cfg.max_iters) {
        int64_t batch = std::min<int64_t>(every, cfg.max_iters - it);
        for (int64_t b = 0; b < batch; b++) one_iter();
        it += batch;
        if (sl) {  // every rank polls after the same batch (the batches hold collectives)
            cudaMemcpyAsync(sch, sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st);
            FLIP_CUDA_OK(cudaStreamSynchronize(st));
            if (g_slab_err) return g_slab_err;
            if (sch->done) break;
            continue;
        }
        // one GPU: the done flag is read back asynchronously (pinned slot +
        // event per batch), so the stream never drains at a poll; at most
        // kPollDepth batches are in flight past the newest flag seen (after
        // convergence their kernels exit at once on the device flag)
        PollRing &pr = poll_ring();
        const int slot = (int)(nbatch % kPollDepth);
        cudaMemcpyAsync(&pr.h[slot], sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st);
        cudaEventRecord(pr.ev[slot], st);
        nbatch++;
        bool stop = false;
        while (seen < nbatch) {
            const int q = (int)(seen % kPollDepth);
            if (nbatch - seen < kPollDepth && cudaEventQuery(pr.ev[q]) == cudaErrorNotReady) break;
            FLIP_CUDA_OK(cudaEventSynchronize(pr.ev[q]));
            seen++;
            if (pr.h[q].done) {
                stop = true;
                break;
            }
        }
        if (stop) break;
    }
    if (sl && nf > 0 && !relax) slab_halo(cfg, B.x);  // pressure_field reads planes k0-1, k1
    if (g_slab_err) return g_slab_err;
    cudaMemcpyAsync(sch, sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st);
    FLIP_CUDA_OK(cudaStreamSynchronize(st));
    FLIP_CUDA_OK(cudaGetLastError());
    if (jfast && (sch->iter & 1)) {  // iteration K wrote buf[K % 2]: xtmp for odd K
        FLIP_CUDA_OK(cudaMemcpyAsync(B.x, B.xtmp, sizeof(double) * nf, cudaMemcpyDeviceToDevice, st));
    }
    if (graph_per_iter) {  // body executions x (its iterations' kernels + the loop test)
        const int64_t bodies = std::max<int64_t>(1, (sch->iter + graph_unroll - 1) / graph_unroll);
        *launches = graph_l0 + bodies * (graph_unroll * graph_per_iter + 1);
    }
    if (stamps && !relax) {  // this solve's sweep durations, then re-arm the slots
        Probe &pb = *LV.probe;
        const int used = (int)std::min<int64_t>(2 * (sch->iter + 1), kProbeSlots);
        FLIP_CUDA_OK(cudaMemcpyAsync(pb.ts_host, pb.ts, sizeof(unsigned long long) * used,
                                     cudaMemcpyDeviceToHost, st));
        FLIP_CUDA_OK(cudaMemcpyAsync(pb.ts_host + kProbeSlots, pb.ts + kProbeSlots,
                                     sizeof(unsigned long long) * used, cudaMemcpyDeviceToHost, st));
        FLIP_CUDA_OK(cudaStreamSynchronize(st));
        for (int k = 0; k < used; k++) {
            const unsigned long long a = pb.ts_host[k], b = pb.ts_host[kProbeSlots + k];
            if (a == ~0ull || b == 0ull || b < a) continue;
            pb.stamp_ms += (double)(b - a) * 1e-6;
            pb.stamp_launches++;
            pb.stamp_bytes += 24.0 * (double)nf;  // src + precon read, dst written per row
        }
        cudaMemsetAsync(pb.ts, 0xff, sizeof(unsigned long long) * kProbeSlots, st);
        cudaMemsetAsync(pb.ts + kProbeSlots, 0, sizeof(unsigned long long) * kProbeSlots, st);
    }
    out->iterations = sch->iter;
    out->residual = sch->res;
    out->converged = sch->converged;
    out->status = sch->status;
    out->err_cell = sch->err_cell;
    out->err_it = sch->err_it;
    out->err_value = sch->err_value;
    return 0;
}


// ============================================================ step: project
// assemble (pressure.py:76-166) + SOLVERS[cfg.solver] (sim.py:266-270) +
// grid.p = pressure_field(x) (sim.py:274).  Syncs to learn the row count.
// Sealed-region pinning (union-find over the labels), row numbering and
// compaction, reset of the row box (pressure.py:76-166 before the rhs).
static void project_rows(Ctx &c, cudaStream_t st) {
    int64_t nc = c.ncells;
    cudaMemsetAsync(&c.sc->npinned, 0, sizeof(int), st);
    static const bool uf_plain = getenv("FLIPB200_UF_PLAIN") != nullptr;
    if (uf_plain) {
        k_uf_init<<<nblocks(nc), kThreads, 0, st>>>(c.label, nc, c.parent, c.has_air);
        k_uf_link<<<nblocks(nc), kThreads, 0, st>>>(c.label, c.d, c.parent);
    } else {
        const int64_t rows = (int64_t)c.d.ny * c.d.nz;
        k_uf_runs<<<nblocks(rows * 32), kThreads, 0, st>>>(c.label, c.d, c.parent, c.has_air);
        k_uf_link_runs<<<nblocks(nc), kThreads, 0, st>>>(c.label, c.d, c.parent);
    }
    k_uf_finish<<<nblocks(nc), kThreads, 0, st>>>(c.label, c.d, c.parent, c.has_air);
    IsRowIn in{c.label, c.parent, c.has_air};
    exclusive_scan(in, nc, c.rowscan, &c.sc->nrows, c.scan_tmp, st);
    k_rows_compact<<<nblocks(nc), kThreads, 0, st>>>(in, nc, c.rowscan, c.isrow, c.cell_of_row, c.sc);
    k_bbox_reset<<<1, 1, 0, st>>>(c.sc);
    c.launches += 6;
}

// The rows, their neighbours and diagonal depend on the labels only, so
// they are built on the side stream while P2G runs on the main stream (one
// GPU; FLIPB200_PROJECT_OVERLAP=0 keeps them inside stage_project).  The
// rhs needs the P2G velocities and is assembled by stage_project.
void project_prefetch(Ctx &c) {
    static const bool env = !getenv("FLIPB200_PROJECT_OVERLAP") ||
                            atoi(getenv("FLIPB200_PROJECT_OVERLAP"));
    if (c.slab.on || !env) return;
    cudaEventRecord(c.ev_fork, c.st);  // labels final (classify)
    cudaStreamWaitEvent(c.st2, c.ev_fork, 0);
    project_rows(c, c.st2);
    k_assemble_rows<true, false><<<nblocks(c.ncells), kThreads, 0, c.st2>>>(
        c.d, c.label, c.isrow, c.rowscan, c.cell_of_row, c.sc, c.u, c.v, c.w, c.nbr, c.ncells,
        c.diagd, c.rhs, &c.sc->rhsmax_bits, c.sc, (int64_t)0, (int64_t)-1, (int64_t)0, (int64_t)-1);
    c.launches++;
    cudaMemcpyAsync(c.sch, c.sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, c.st2);
    cudaEventRecord(c.ev_side, c.st2);
    c.proj_pre = 1;
}

int stage_project(Ctx &c, const flip_step_params &prm, flip_step_report *rep) {
    cudaStream_t st = c.st;
    int64_t nc = c.ncells;
    cudaMemsetAsync(&c.sc->rhsmax_bits, 0, sizeof(unsigned long long), st);
    const bool pre = c.proj_pre != 0;
    c.proj_pre = 0;
    if (!pre) project_rows(c, st);
    bool need_sweeps = prm.solver == FLIP_SOLVER_GS ||
                       (prm.solver == FLIP_SOLVER_PCG && prm.precond == FLIP_PRECOND_MIC0);
    Slab &SL = c.slab;
    SlabDot SD{&c};
    if (pre) {
        // structure from project_prefetch; the rhs from the P2G velocities
        FLIP_CUDA_OK(cudaEventSynchronize(c.ev_side));
        cudaStreamWaitEvent(st, c.ev_side, 0);
        k_assemble_rows<false, true><<<nblocks(nc), kThreads, 0, st>>>(
            c.d, c.label, c.isrow, c.rowscan, c.cell_of_row, c.sc, c.u, c.v, c.w, c.nbr, nc, c.diagd,
            c.rhs, &c.sc->rhsmax_bits, c.sc, (int64_t)0, (int64_t)-1, (int64_t)0, (int64_t)-1);
        c.launches++;
    } else if (!SL.on) {
        k_assemble_rows<true, true><<<nblocks(nc), kThreads, 0, st>>>(c.d, c.label, c.isrow, c.rowscan,
                                                          c.cell_of_row, c.sc, c.u, c.v, c.w, c.nbr,
                                                          nc, c.diagd, c.rhs, &c.sc->rhsmax_bits,
                                                          c.sc, (int64_t)0, (int64_t)-1,
                                                          (int64_t)0, (int64_t)-1);
        c.launches += 2;
    } else {
        // the rows are numbered globally (every rank labelled every plane):
        // own rows [R0, R1) and the halo rows of planes k0-1 / k1
        if (int rc = slab_rows(c)) return rc;
        const bool full = need_sweeps || (prm.solver == FLIP_SOLVER_PCG &&
                                          prm.precond == FLIP_PRECOND_MG);
        // structure (diag, neighbours, bounding box) of every row when a
        // replicated sweep needs it, else of the window; rhs of the own rows
        const int64_t a_lo = full ? 0 : SL.Rlo, a_hi = full ? SL.rstart[SL.world] : SL.Rhi;
        k_assemble_rows<true, true><<<nblocks(std::max<int64_t>(a_hi - a_lo, 1)), kThreads, 0, st>>>(
            c.d, c.label, c.isrow, c.rowscan, c.cell_of_row, c.sc, c.u, c.v, c.w, c.nbr, nc,
            c.diagd, c.rhs, &c.sc->rhsmax_bits, c.sc, a_lo, a_hi, SL.R0, SL.R1);
        c.launches++;
        if (int rc = slab_allreduce(c, (int64_t *)&c.sc->rhsmax_bits, 1, FLIP_OP_MAX)) return rc;
    }
    if (!pre) {
        cudaMemcpyAsync(c.sch, c.sc, sizeof(DevScalars), cudaMemcpyDeviceToHost, st);
        FLIP_CUDA_OK(cudaStreamSynchronize(st));
    }
    int64_t n = c.sch->nrows;
    double dt = c.sch->dt;
    rep->nrows = n;
    rep->npinned = c.sch->npinned;
    // scale = dt / (rho * dtau**2) (pressure.py:164), same IEEE division as the reference
    double scale = dt / prm.rho_dtau2_h;
    SysView S{n, c.cell_of_row, c.nbr, nc, c.diagd, c.rhs, scale};
    SysView Sfull = S;
    if (SL.on) {  // this rank computes its own rows
        S.r0 = SL.R0;
        S.n = SL.R1 - SL.R0;
    }
    static const bool plain_mv = getenv("FLIPB200_PLAIN_MATVEC") != nullptr;
    if ((prm.solver == FLIP_SOLVER_PCG || prm.solver == FLIP_SOLVER_JACOBI) && n > 0 &&
        c.d.nx < 32768 && !plain_mv) {
        k_compact_nbr<<<nblocks(S.n), kThreads, 0, st>>>(S, c.nb_meta, c.nb_dy, c.nb_dz);
        c.launches++;
        S.meta = c.nb_meta;
        S.dy = c.nb_dy;
        S.dz = c.nb_dz;
    }
    // sequential sweeps (GS, MIC(0)) run as the pipelined wavefront over the
    // rows' bounding box; FLIPB200_LEVEL_SWEEPS=1 selects the level-scheduled
    // cooperative fallback (same results, used to cross-check)
    static const bool level_sweeps = getenv("FLIPB200_LEVEL_SWEEPS") != nullptr && !SL.on;
    Levels L{c.lvl, c.lvl_cnt, c.lvl_off, c.lvl_rows, &c.sc->nlevels, 0};
    WaveArgs W{};
    bool use_wave = need_sweeps && n > 0 && !level_sweeps;
    if (use_wave) {
        W.d = c.d;
        W.geom = wave_geom(c.sch->row_lo, c.sch->row_hi);
        W.rowscan = c.rowscan;
        W.cflags = c.cflags;
        W.n = n;
        W.diag = c.diagd;
        W.rhs = c.rhs;
        W.scale = scale;
        W.tau = 0.97;   // pressure.py:288
        W.sigma = 0.25;
        W.halo_y = c.wave_halo;
        W.halo_z = c.wave_halo + (int64_t)W.geom.TB * W.geom.TC * W.geom.tz * W.geom.ispan_pad;
        W.ticket = c.wave_prog;
        W.trace = getenv("FLIPB200_WAVE_TRACE") ? c.wave_trace : nullptr;
        launch_cell_flags(c.d, c.isrow, c.cflags, st);
        c.launches++;
    } else if (need_sweeps && n > 0) {
        int maxl = c.d.nx + c.d.ny + c.d.nz - 2;
        cudaMemsetAsync(c.lvl_cnt, 0, sizeof(int) * (maxl + 1), st);
        k_lvl_geom<<<nblocks(n), kThreads, 0, st>>>(c.cell_of_row, n, c.d, c.lvl, c.lvl_cnt);
        bucket_levels(L, n, maxl, c.scan_tmp, st, &c.launches);
        k_set_nlevels<<<1, 1, 0, st>>>(c.sc, maxl);
        c.launches += 2;
    }
    LaneBufs LB{};
    static const bool no_lane = getenv("FLIPB200_NO_LANE") != nullptr;
    bool use_lane = use_wave && prm.solver == FLIP_SOLVER_PCG && prm.precond == FLIP_PRECOND_MIC0 &&
                    !no_lane && lane_entries(W.geom) <= c.lane_cap;
    // the substitutions run 2 x 2 pencils per thread (k_mic_quad) when their
    // lane layout and halos fit the buffers sized for the 16 x 16 geometry
    WaveGeom LG = W.geom;
    if (use_lane && mic_quad_enabled()) {
        WaveGeom qg = quad_geom(c.sch->row_lo, c.sch->row_hi);
        const int64_t halo_need = (int64_t)qg.TB * qg.TC * qg.nsteps * 2 * qg.ty;
        if (lane_entries(qg) <= c.lane_cap &&
            halo_need <= wave_halo_doubles(c.d.nx, c.d.ny, c.d.nz) - 64 &&
            mic_quad_supported(qg.nsteps))
            LG = qg;
    }
    if (use_lane) {
        LB.args.geom = LG;
        LB.args.halo_y = W.halo_y;
        LB.args.halo_z = W.halo_z;
        LB.args.scale = scale;
        LB.args.ticket = W.ticket;
        LB.args.trace = getenv("FLIPB200_WAVE_TRACE") ? c.wave_trace : nullptr;
        if (LB.args.trace) cudaMemsetAsync(c.wave_trace, 0, 8 * 32768, st);  // (trace buffer: 32768 u64)
        LB.args.dbg = getenv("FLIPB200_LANE_DBG") ? atoi(getenv("FLIPB200_LANE_DBG")) : 0;
        if (LG.quad) {
            int cy = 0, cz = 0;
            quad_cluster_shape(&cy, &cz);
            const int64_t per = (int64_t)LG.TB * LG.TC * LG.nsteps * 2 * LG.ty;
            if (2 * per + 64 <= wave_halo_doubles(c.d.nx, c.d.ny, c.d.nz)) {
                LB.hr = HaloReset{{c.wave_halo, c.wave_halo + per}, {c.wave_prog, c.wave_prog + 1},
                                  LG.TB, LG.TC, LG.nsteps, LG.ty, cy, cz, 1};
            }
        }
        LB.posL = c.posL;
        LB.rL = c.laneA;
        LB.tqL = c.laneB;
        LB.zL = c.laneC;
        LB.preL = c.laneD;
        launch_lane_map(LG, c.d, c.isrow, c.rowscan, c.lrow, c.posL, c.laneA, c.laneB, st);
        c.launches++;
    }
    SweepLevels LV{&L, &L, &L, 1, use_wave ? &W : nullptr, &c.probe, use_lane ? &LB : nullptr, &c};
    if (prm.solver == FLIP_SOLVER_PCG && prm.precond == FLIP_PRECOND_MG && n > 0)
        if (int rc = mg_setup(c, scale, c.sch->row_lo, c.sch->row_hi, st)) return rc;
    SolveCfg cfg{prm.solver, prm.precond, prm.max_iters, prm.tol, prm.solver_check_every, nullptr,
                 nullptr, nullptr, 0, 0, c.d};
    if (SL.on) {
        cfg.slab = &SD;
        cfg.full = &Sfull;
    }
    SolveBufs B{c.x, c.r, c.z, c.s, c.q, c.tq, c.precon, c.xtmp, c.dot_part, c.scan_tmp,
                c.u64_scratch};
    SolveOut o{};
    g_sweep_launch_err = cudaSuccess;
    int rc = run_solve(S, cfg, B, LV, c.sc, c.sch, st, &c.launches, &o);
    if (rc) return rc;
    if (g_sweep_launch_err != cudaSuccess) {
        set_error(std::string("MIC(0) sweep launch failed: ") + cudaGetErrorString(g_sweep_launch_err));
        return FLIP_E_CUDA;
    }
    rep->solver_iterations = o.iterations;
    rep->solver_residual = o.residual;
    rep->solver_converged = o.converged;
    rep->status = o.status;
    rep->err_cell = o.err_cell;
    rep->err_iteration = o.err_it;
    rep->err_value = o.err_value;
    if (o.status) return 0;
    if (SL.on) {  // own planes and the two next to them (the gradient reads them)
        const int64_t pc = (int64_t)c.d.nx * c.d.ny;
        const int64_t c0 = std::max<int64_t>(SL.k0 - 1, 0) * pc;
        const int64_t c1 = std::min<int64_t>(SL.k1 + 1, c.d.nz) * pc;
        k_pressure_field<<<nblocks(c1 - c0), kThreads, 0, st>>>(c.p + c0, c1 - c0, c.isrow + c0,
                                                               c.rowscan + c0, c.x);
        c.launches++;
        return 0;
    }
    k_pressure_field<<<nblocks(nc), kThreads, 0, st>>>(c.p, nc, c.isrow, c.rowscan, c.x);
    c.launches++;
    return 0;
}

// ======================================================= plugin API solves
__global__ void k_i64_to_i32(const long long *__restrict__ a, int *__restrict__ b, int64_t n) {
    for (int64_t i = gtid(); i < n; i += gstride()) b[i] = (int)a[i];
}

// (n,6) row-major int64 -> [6][n] int32
__global__ void k_nbr_transpose(const long long *__restrict__ a, int *__restrict__ b, int64_t n) {
    for (int64_t i = gtid(); i < n * 6; i += gstride()) {
        int64_t r = i / 6, q = i % 6;
        b[q * n + r] = (int)a[i];
    }
}

__global__ void k_absmax(const double *__restrict__ a, int64_t n, unsigned long long *out) {
    double m = 0.0;
    for (int64_t i = gtid(); i < n; i += gstride()) m = fmax(m, fabs(a[i]));
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomic_max_nonneg(out, m);
}

// Device scratch for one plugin-API call, freed on scope exit.
struct DevArena {
    cudaStream_t st;  // the call's stream: the zero-fill is ordered before its kernels
    std::vector<void *> ptrs;
    explicit DevArena(cudaStream_t s) : st(s) {}
    ~DevArena() {
        for (void *p : ptrs) cudaFree(p);
    }
    template <class T>
    T *get(int64_t n) {
        void *p = nullptr;
        if (cudaMalloc(&p, sizeof(T) * (size_t)(n > 0 ? n : 1)) != cudaSuccess) return nullptr;
        // zeroed on the call's stream: dot scratch carries the fused dot's ticket word
        cudaMemsetAsync(p, 0, sizeof(T) * (size_t)(n > 0 ? n : 1), st);
        ptrs.push_back(p);
        return (T *)p;
    }
};

// Generic levels by relaxation; returns 0 or a CUDA error code.
static int generic_levels(DevArena &ar, const SysView &S, int mode, Levels &L, cudaStream_t st,
                          int *scan_tmp) {
    int64_t n = S.n;
    L.lvl = ar.get<int>(n);
    L.rows = ar.get<int>(n);
    L.cnt = ar.get<int>(n + 1);
    L.off = ar.get<int>(n + 2);
    L.nlev = ar.get<int>(2);
    L.reverse = 0;
    int *changed = ar.get<int>(1);
    if (!L.lvl || !L.rows || !L.cnt || !L.off || !L.nlev || !changed) {
        set_error("cudaMalloc failed (levels)");
        return FLIP_E_CUDA;
    }
    cudaMemsetAsync(L.lvl, 0, sizeof(int) * n, st);
    int h = 1;
    int64_t guard = 0;
    while (h) {
        cudaMemsetAsync(changed, 0, sizeof(int), st);
        k_lvl_relax<<<nblocks(n), kThreads, 0, st>>>(S, mode, L.lvl, changed);
        FLIP_CUDA_OK(cudaMemcpyAsync(&h, changed, sizeof(int), cudaMemcpyDeviceToHost, st));
        FLIP_CUDA_OK(cudaStreamSynchronize(st));
        if (++guard > 4 * n + 8) {
            set_error("level schedule did not converge");
            return FLIP_E_ARG;
        }
    }
    cudaMemsetAsync(L.cnt, 0, sizeof(int) * (n + 1), st);
    cudaMemsetAsync(L.nlev + 1, 0xff, sizeof(int), st);
    k_lvl_count<<<nblocks(n), kThreads, 0, st>>>(L.lvl, n, L.cnt, L.nlev + 1);
    int64_t dummy = 0;
    bucket_levels(L, n, (int)n, scan_tmp, st, &dummy);
    k_nlev_from_max<<<1, 1, 0, st>>>(L.nlev);
    return 0;
}


}  // namespace flip

using namespace flip;

// ---------------------------------------------------- extern "C" plugin API
namespace {

struct ApiStream {
    cudaStream_t st = nullptr;
    ApiStream() { cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking); }
    ~ApiStream() {
        if (st) cudaStreamDestroy(st);
    }
};

#define API_CHECK(expr) FLIP_CUDA_OK(expr)

// Uploads an (n,6) int64 neighbour table as [6][n] int32.
int upload_nbr(DevArena &ar, const int64_t *nbr_rows, int64_t n, int **out, cudaStream_t st) {
    long long *tmp = ar.get<long long>(n * 6);
    int *d = ar.get<int>(n * 6);
    if (!tmp || !d) {
        set_error("cudaMalloc failed");
        return FLIP_E_CUDA;
    }
    API_CHECK(cudaMemcpyAsync(tmp, nbr_rows, sizeof(int64_t) * n * 6, cudaMemcpyHostToDevice, st));
    if (n > 0) k_nbr_transpose<<<nblocks(n * 6), kThreads, 0, st>>>(tmp, d, n);
    *out = d;
    return 0;
}

double *upload_d(DevArena &ar, const double *h, int64_t n, cudaStream_t st) {
    double *d = ar.get<double>(n);
    if (d && n > 0) cudaMemcpyAsync(d, h, sizeof(double) * n, cudaMemcpyHostToDevice, st);
    return d;
}

}  // namespace

extern "C" int flip_k_laplacian_matvec(int64_t n, const double *diag, const int64_t *nbr_rows,
                                       const double *x, double scale, double *y) {
    ApiStream S;
    DevArena ar(S.st);
    int *nb = nullptr;
    if (int rc = upload_nbr(ar, nbr_rows, n, &nb, S.st)) return rc;
    double *dd = upload_d(ar, diag, n, S.st), *dx = upload_d(ar, x, n, S.st), *dy = ar.get<double>(n);
    SysView V{n, nullptr, nb, n, dd, nullptr, scale};
    if (n > 0) k_matvec<<<nblocks(n), kThreads, 0, S.st>>>(V, dx, dy, nullptr, nullptr, nullptr, nullptr, 0);
    API_CHECK(cudaMemcpyAsync(y, dy, sizeof(double) * n, cudaMemcpyDeviceToHost, S.st));
    API_CHECK(cudaStreamSynchronize(S.st));
    API_CHECK(cudaGetLastError());
    return 0;
}

extern "C" int flip_k_jacobi_iter(int64_t n, const double *diag, const int64_t *nbr_rows,
                                  const double *rhs, const double *x, double scale, double *out) {
    ApiStream S;
    DevArena ar(S.st);
    int *nb = nullptr;
    if (int rc = upload_nbr(ar, nbr_rows, n, &nb, S.st)) return rc;
    double *dd = upload_d(ar, diag, n, S.st), *dr = upload_d(ar, rhs, n, S.st),
           *dx = upload_d(ar, x, n, S.st), *dout = ar.get<double>(n);
    SysView V{n, nullptr, nb, n, dd, dr, scale};
    if (n > 0) k_jacobi<<<nblocks(n), kThreads, 0, S.st>>>(V, dx, dout, nullptr, 0);
    API_CHECK(cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, S.st));
    API_CHECK(cudaStreamSynchronize(S.st));
    API_CHECK(cudaGetLastError());
    return 0;
}

extern "C" int flip_k_gs_sweep_rows(int64_t m, const int64_t *rows, int64_t n, const double *diag,
                                    const int64_t *nbr_rows, const double *rhs, double *x,
                                    double scale) {
    ApiStream S;
    DevArena ar(S.st);
    int *nb = nullptr;
    if (int rc = upload_nbr(ar, nbr_rows, n, &nb, S.st)) return rc;
    double *dd = upload_d(ar, diag, n, S.st), *dr = upload_d(ar, rhs, n, S.st),
           *dx = upload_d(ar, x, n, S.st);
    long long *r64 = ar.get<long long>(m);
    int *r32 = ar.get<int>(m);
    API_CHECK(cudaMemcpyAsync(r64, rows, sizeof(int64_t) * m, cudaMemcpyHostToDevice, S.st));
    if (m > 0) {
        k_i64_to_i32<<<nblocks(m), kThreads, 0, S.st>>>(r64, r32, m);
        SysView V{n, nullptr, nb, n, dd, dr, scale};
        k_gs_rows<<<nblocks(m), kThreads, 0, S.st>>>(V, r32, m, 0, Dims{}, dx, nullptr, 0);
    }
    API_CHECK(cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, S.st));
    API_CHECK(cudaStreamSynchronize(S.st));
    API_CHECK(cudaGetLastError());
    return 0;
}

// Wavefront kernels of the plugin API use generic (relaxed) level schedules.
static int api_sweep(int mode, int64_t n, const double *diag, const int64_t *nbr_rows,
                     const double *rhs, const double *src_h, const double *precon_h, double scale,
                     double *out_h, const double *xin_h) {
    ApiStream S;
    DevArena ar(S.st);
    int *nb = nullptr;
    if (int rc = upload_nbr(ar, nbr_rows, n, &nb, S.st)) return rc;
    double *dd = diag ? upload_d(ar, diag, n, S.st) : nullptr;
    double *dr = rhs ? upload_d(ar, rhs, n, S.st) : nullptr;
    double *dsrc = src_h ? upload_d(ar, src_h, n, S.st) : nullptr;
    double *dpc = precon_h ? upload_d(ar, precon_h, n, S.st) : nullptr;
    double *tq = ar.get<double>(n), *dout = xin_h ? upload_d(ar, xin_h, n, S.st) : ar.get<double>(n);
    int *scan_tmp = ar.get<int>(scan_tmp_ints(n + 2) + 8);
    if (n == 0) return 0;
    SysView V{n, nullptr, nb, n, dd, dr, scale};
    if (mode == SW_MIC_FWD) {  // full apply: forward into tq, backward into out
        Levels Lf{}, Lb{};
        if (int rc = generic_levels(ar, V, 0, Lf, S.st, scan_tmp)) return rc;
        if (int rc = generic_levels(ar, V, 1, Lb, S.st, scan_tmp)) return rc;
        SweepArgs A{V, Lf.rows, Lf.off, Lf.nlev, 0, 0.97, 0.25, dsrc, tq, dpc, nullptr, 0};
        API_CHECK(launch_sweep<SW_MIC_FWD>(A, S.st));
        SweepArgs B{V, Lb.rows, Lb.off, Lb.nlev, 0, 0.97, 0.25, tq, dout, dpc, nullptr, 0};
        API_CHECK(launch_sweep<SW_MIC_BWD>(B, S.st));
    } else {
        Levels L{};  // SW_GS
        if (int rc = generic_levels(ar, V, 2, L, S.st, scan_tmp)) return rc;
        SweepArgs A{V, L.rows, L.off, L.nlev, 0, 0.97, 0.25, dsrc, dout, dpc, nullptr, 0};
        API_CHECK(launch_sweep<SW_GS>(A, S.st));
    }
    API_CHECK(cudaMemcpyAsync(out_h, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, S.st));
    API_CHECK(cudaStreamSynchronize(S.st));
    API_CHECK(cudaGetLastError());
    return 0;
}

extern "C" int flip_k_gs_sweep(int64_t n, const double *diag, const int64_t *nbr_rows,
                               const double *rhs, double *x, double scale) {
    return api_sweep(SW_GS, n, diag, nbr_rows, rhs, nullptr, nullptr, scale, x, x);
}

extern "C" int flip_k_mic0_apply(int64_t n, const double *precon, const int64_t *nbr_rows,
                                 const double *r, double scale, double *z) {
    return api_sweep(SW_MIC_FWD, n, nullptr, nbr_rows, nullptr, r, precon, scale, z, nullptr);
}

extern "C" int flip_k_mic0_build(int64_t n, const double *diag, const int64_t *nbr_rows,
                                 double scale, double tau, double sigma, double *precon) {
    ApiStream S;
    DevArena ar(S.st);
    int *nb = nullptr;
    if (int rc = upload_nbr(ar, nbr_rows, n, &nb, S.st)) return rc;
    double *dd = upload_d(ar, diag, n, S.st), *dout = ar.get<double>(n);
    int *scan_tmp = ar.get<int>(scan_tmp_ints(n + 2) + 8);
    if (n == 0) return 0;
    SysView V{n, nullptr, nb, n, dd, nullptr, scale};
    Levels L{};
    if (int rc = generic_levels(ar, V, 0, L, S.st, scan_tmp)) return rc;
    SweepArgs A{V, L.rows, L.off, L.nlev, 0, tau, sigma, nullptr, dout, nullptr, nullptr, 0};
    API_CHECK(launch_sweep<SW_MIC_BUILD>(A, S.st));
    API_CHECK(cudaMemcpyAsync(precon, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, S.st));
    API_CHECK(cudaStreamSynchronize(S.st));
    API_CHECK(cudaGetLastError());
    return 0;
}

extern "C" int flip_k_pairwise_dot(int64_t n, const double *a, const double *b, double *out) {
    ApiStream S;
    DevArena ar(S.st);
    double *da = upload_d(ar, a, n, S.st), *db = b ? upload_d(ar, b, n, S.st) : nullptr;
    double *tmp = ar.get<double>(dot_tmp_doubles(n)), *res = ar.get<double>(1);
    int64_t l = 0;
    if (n == 0) {
        *out = 0.0;
        return 0;
    }
    launch_pairwise_dot(da, db, n, tmp, res, S.st, &l);
    API_CHECK(cudaMemcpyAsync(out, res, sizeof(double), cudaMemcpyDeviceToHost, S.st));
    API_CHECK(cudaStreamSynchronize(S.st));
    API_CHECK(cudaGetLastError());
    return 0;
}

extern "C" int flip_solve_system(int32_t solver, int32_t precond, int64_t n, const int64_t *cells,
                                 const double *diag, const int64_t *nbr_rows, const double *rhs,
                                 double scale, int64_t max_iters, double tol,
                                 const int64_t *red_rows, int64_t nred, const int64_t *black_rows,
                                 int64_t nblack, double *x, int64_t *iterations, double *residual,
                                 int32_t *converged, int64_t *err_cell, int64_t *err_iteration,
                                 double *err_value) {
    if (solver < 0 || solver > 3 || precond < 0 || precond > FLIP_PRECOND_MG) {
        set_error("unknown solver or preconditioner");
        return FLIP_E_CONFIG;
    }
    ApiStream S;
    DevArena ar(S.st);
    int *nb = nullptr;
    if (int rc = upload_nbr(ar, nbr_rows, n, &nb, S.st)) return rc;
    double *dd = upload_d(ar, diag, n, S.st), *dr = upload_d(ar, rhs, n, S.st);
    long long *c64 = ar.get<long long>(n);
    int *c32 = ar.get<int>(n);
    API_CHECK(cudaMemcpyAsync(c64, cells, sizeof(int64_t) * n, cudaMemcpyHostToDevice, S.st));
    if (n > 0) k_i64_to_i32<<<nblocks(n), kThreads, 0, S.st>>>(c64, c32, n);
    int *red = nullptr, *black = nullptr;
    if (solver == FLIP_SOLVER_RBGS) {
        long long *t = ar.get<long long>(nred + nblack);
        red = ar.get<int>(nred);
        black = ar.get<int>(nblack);
        API_CHECK(cudaMemcpyAsync(t, red_rows, sizeof(int64_t) * nred, cudaMemcpyHostToDevice, S.st));
        API_CHECK(cudaMemcpyAsync(t + nred, black_rows, sizeof(int64_t) * nblack,
                                  cudaMemcpyHostToDevice, S.st));
        if (nred) k_i64_to_i32<<<nblocks(nred), kThreads, 0, S.st>>>(t, red, nred);
        if (nblack) k_i64_to_i32<<<nblocks(nblack), kThreads, 0, S.st>>>(t + nred, black, nblack);
    }
    DevScalars *sc = ar.get<DevScalars>(1);
    DevScalars *sch = nullptr;
    API_CHECK(cudaMallocHost(&sch, sizeof(DevScalars)));
    struct HostFree {
        void *p;
        ~HostFree() { cudaFreeHost(p); }
    } hf{sch};
    API_CHECK(cudaMemsetAsync(sc, 0, sizeof(DevScalars), S.st));
    if (n > 0) k_absmax<<<nblocks(n), kThreads, 0, S.st>>>(dr, n, &sc->rhsmax_bits);
    SysView V{n, c32, nb, n, dd, dr, scale};
    int *scan_tmp = ar.get<int>(scan_tmp_ints(n + 2) + 8);
    Levels Lf{}, Lb{}, Lg{};
    if (precond == FLIP_PRECOND_MG) {
        set_error("the multigrid preconditioner needs the grid (use it through flip_step)");
        return FLIP_E_ARG;
    }
    bool mic = solver == FLIP_SOLVER_PCG && precond == FLIP_PRECOND_MIC0;
    if (n > 0 && mic) {
        if (int rc = generic_levels(ar, V, 0, Lf, S.st, scan_tmp)) return rc;
        if (int rc = generic_levels(ar, V, 1, Lb, S.st, scan_tmp)) return rc;
    }
    if (n > 0 && solver == FLIP_SOLVER_GS)
        if (int rc = generic_levels(ar, V, 2, Lg, S.st, scan_tmp)) return rc;
    SweepLevels LV{&Lf, &Lb, &Lg, 0, nullptr, nullptr, nullptr};
    SolveCfg cfg{solver, precond, max_iters, tol, 0, nullptr, red, black, nred, nblack, Dims{}};
    SolveBufs B{ar.get<double>(n), ar.get<double>(n), ar.get<double>(n), ar.get<double>(n),
                ar.get<double>(n), ar.get<double>(n), ar.get<double>(n), ar.get<double>(n),
                ar.get<double>(dot_tmp_doubles(n)), scan_tmp, ar.get<unsigned long long>(1)};
    SolveOut o{};
    int64_t api_launches = 0;
    if (int rc = run_solve(V, cfg, B, LV, sc, sch, S.st, &api_launches, &o)) return rc;
    if (n > 0) API_CHECK(cudaMemcpyAsync(x, B.x, sizeof(double) * n, cudaMemcpyDeviceToHost, S.st));
    API_CHECK(cudaStreamSynchronize(S.st));
    API_CHECK(cudaGetLastError());
    *iterations = o.iterations;
    *residual = o.residual;
    *converged = o.converged;
    *err_cell = o.err_cell;
    *err_iteration = o.err_it;
    *err_value = o.err_value;
    if (o.status == FLIP_E_SINGULAR) {
        set_error("singular pressure system");
        set_error_cell(o.err_cell);
    } else if (o.status == FLIP_E_BREAKDOWN) {
        set_error("conjugate-gradient breakdown");
    }
    return o.status;
}
