"""Slab decomposition of the FLIP step over ranks (one process per GPU).

SURVEY §8(e); north star: "the domain is slab-decomposed ... particle
migration ... ghost layers ... reductions allreduced".

Decomposition
-------------
Rank r owns the cell z-planes ``[k0, k1)`` of :class:`SlabPlan`.  Every grid
array is x-fastest with z slowest (``flipsim/grid.py:47-72``), so a slab is a
contiguous range of each cell and face array, and the particles of a slab are
a contiguous range of the cell-sorted particle set.  Each rank holds the
particles of its own slab, in global order, and the whole grid.

Per step (``flipsim/sim.py:226-300``), with the exchange that makes each
stage exact:

1. dt (``particles.py:214-224``): local, then allreduce MIN.  dt is a
   monotone function of max|v|^2, so the MIN of the local values is the
   global value bit for bit.
2. advect: local.
3. migration: particles whose cell left the slab go to the owning rank
   (``all_to_all``).  The receive buffer is ordered by source rank, and the
   global order is rank order, so the stable sort of step 4 reproduces the
   1-GPU order.
4. bin: local.
5. classify: local (FLUID needs count > 0), then allreduce MIN of the labels
   (SOLID 0 < FLUID 1 < AIR 2).
6. ghost planes: each rank sends its first/last particle plane to its
   neighbours.  P2G (``transfer.py:35-57``) of a face in the slab reads cells
   one plane beyond it.
7. P2G + force on [ghost_lo, own, ghost_hi], then the ghosts are dropped and
   the slab re-binned.
8. owned faces of grid, grid_old and the known masks are all-gathered.
   Every rank then holds the 1-GPU grid.
9. assemble / solve / gradient / extrapolation: replicated (see below).
10. G2P: local.
11. reseed: local, restricted to the slab's cells (``flip_set_slab``).

The result on every rank is the 1-GPU grid, and the concatenation of the
ranks' particles in rank order is the 1-GPU particle set, bit for bit
(``tests/test_dist_*``).

Why the solve is replicated.  Every PCG iteration applies MIC(0), a
sequential recurrence across the whole grid (``_core.pyx:311-347``).  Its
critical path (≈ nx + ny + nz dependent hyperplanes) does not shorten when
split over GPUs.  The pipelined wavefront could cross slab boundaries over
peer memory, but each such boundary adds NVLink latency to that path.
Splitting only the vector kernels (≈ 20% of the solve) would need a
distributed pairwise-dot tree and per-iteration halo exchanges for a
fraction of the step.  The replicated solve keeps the reference's
arithmetic and costs no communication.  The particle-side stages are the
part that scales.

Transport
---------
Exchanges run on torch tensors that alias the ctx's device buffers:
``backend="nccl"`` uses them directly, ``"gloo"`` stages through host memory
(CPU tests, or two ranks sharing one GPU with no cross-process waits in any
kernel).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import LIB, check
from . import rng
from . import sim as _sim

__all__ = ["SlabPlan", "Transport", "make_scene", "step", "gather_particles",
           "migrate_rows", "ghost_rows", "face_ranges"]


# ----------------------------------------------------------------- plan ----
@dataclass(frozen=True)
class SlabPlan:
    """Contiguous z-plane ranges: rank r owns planes [k0(r), k1(r))."""
    nx: int
    ny: int
    nz: int
    world: int

    def __post_init__(self):
        if self.world < 1 or self.world > self.nz:
            raise ValueError(f"cannot split {self.nz} planes over {self.world} ranks")

    def planes(self, rank: int) -> tuple:
        return (rank * self.nz) // self.world, ((rank + 1) * self.nz) // self.world

    def owner_of_plane(self, k: int) -> int:
        for r in range(self.world):
            k0, k1 = self.planes(r)
            if k0 <= k < k1:
                return r
        raise ValueError(f"plane {k} outside the grid")

    def plane_owners(self) -> np.ndarray:
        """owner rank of every cell z-plane (int64[nz])."""
        out = np.empty(self.nz, dtype=np.int64)
        for r in range(self.world):
            k0, k1 = self.planes(r)
            out[k0:k1] = r
        return out

    @property
    def plane_cells(self) -> int:
        return self.nx * self.ny


def face_ranges(plan: SlabPlan, comp: int, rank: int) -> tuple:
    """[lo, hi) flat indices of the faces of component ``comp`` that rank
    owns: the faces of its cell planes, plus the top w plane (k = nz) on the
    last rank (``grid.py:65-72`` layouts)."""
    k0, k1 = plan.planes(rank)
    nx, ny = plan.nx, plan.ny
    if comp == 0:
        per = (nx + 1) * ny
    elif comp == 1:
        per = nx * (ny + 1)
    else:
        per = nx * ny
        if rank == plan.world - 1:
            k1 += 1
    return k0 * per, k1 * per


# ------------------------------------------------------------ transport ----
class Transport:
    """torch.distributed collectives on device tensors (NCCL) or staged
    through host memory (gloo)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.staged = dist.get_backend(group) != "nccl"

    def _out(self, t):
        return t.cpu() if self.staged else t

    def _back(self, t, like):
        return t.to(like.device) if self.staged else t

    def allreduce_min_(self, t):
        x = self._out(t)
        self.dist.all_reduce(x, op=self.dist.ReduceOp.MIN, group=self.group)
        if self.staged:
            t.copy_(x)
        return t

    def allreduce_sum_int(self, v: int) -> int:
        t = self.torch.tensor([int(v)], dtype=self.torch.int64)
        if not self.staged:
            t = t.cuda()
        self.dist.all_reduce(t, group=self.group)
        return int(t.item())

    def all_to_all_rows(self, rows, send_counts):
        """rows: (n, k) grouped by destination rank in rank order; returns the
        received rows grouped by source rank in rank order, and the counts."""
        torch = self.torch
        sc = torch.tensor([int(c) for c in send_counts], dtype=torch.int64)
        rc = torch.empty(self.world, dtype=torch.int64)
        if not self.staged:
            sc, rc = sc.cuda(), rc.cuda()
        self.dist.all_to_all_single(rc, sc, group=self.group)
        recv_counts = [int(c) for c in rc.tolist()]
        k = rows.shape[1]
        src = self._out(rows.contiguous())
        dst = torch.empty((sum(recv_counts), k), dtype=rows.dtype, device=src.device)
        self.dist.all_to_all_single(dst.view(-1), src.view(-1),
                                    [c * k for c in recv_counts],
                                    [int(c) * k for c in send_counts], group=self.group)
        return self._back(dst, rows), recv_counts

    def allgather_var(self, local, sizes):
        """all-gather of 1-D tensors of per-rank lengths ``sizes``."""
        torch = self.torch
        m = max(max(sizes), 1)
        x = self._out(local)
        pad = torch.zeros(m, dtype=x.dtype, device=x.device)
        pad[:x.numel()] = x
        parts = [torch.empty(m, dtype=x.dtype, device=x.device) for _ in range(self.world)]
        self.dist.all_gather(parts, pad, group=self.group)
        return [self._back(p[:s], local) for p, s in zip(parts, sizes)]


# ------------------------------------------------- host-logic pieces ----
def migrate_rows(rows, plane_of_row, owners, tr: Transport):
    """Send each row to the rank owning its z-plane.  ``rows`` (n, k) in the
    rank's current order; returns the rows this rank now owns, in global
    order (source ranks ascending, each source's order kept)."""
    torch = tr.torch
    dest = owners[plane_of_row.long()]
    order = torch.argsort(dest, stable=True)
    counts = torch.bincount(dest, minlength=tr.world).tolist()
    return tr.all_to_all_rows(rows[order], counts)[0]


def ghost_rows(rows, first_plane, last_plane, tr: Transport):
    """Exchange boundary planes with the neighbours.  ``first_plane`` /
    ``last_plane`` are (start, end) row ranges of the rank's first and last
    cell plane in ``rows``.  Returns (ghost_lo, ghost_hi): the previous
    rank's last plane and the next rank's first plane."""
    torch = tr.torch
    r, w = tr.rank, tr.world
    parts, counts = [], [0] * w
    if r > 0:
        parts.append(rows[first_plane[0]:first_plane[1]])
        counts[r - 1] = first_plane[1] - first_plane[0]
    if r + 1 < w:
        parts.append(rows[last_plane[0]:last_plane[1]])
        counts[r + 1] = last_plane[1] - last_plane[0]
    send = torch.cat(parts) if parts else rows[:0]
    recv, rc = tr.all_to_all_rows(send, counts)
    nlo = rc[r - 1] if r > 0 else 0
    return recv[:nlo], recv[nlo:]


# ------------------------------------------------------- device views ----
class _CAI:
    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def _view(ptr, n: int, dtype):
    import torch
    typestr = {torch.float64: "<f8", torch.int32: "<i4", torch.uint8: "|u1"}[dtype]
    if n == 0:
        return torch.empty(0, dtype=dtype, device="cuda")
    return torch.as_tensor(_CAI(ptr, n, typestr), device="cuda")


def _ptrs(dev):
    p = _lib.DevPtrs()
    check(LIB.flip_get_dev_ptrs(dev.ctx, C.byref(p)), "flip_get_dev_ptrs")
    return p


def _particle_rows(dev):
    import torch
    p = _ptrs(dev)
    n = int(p.n)
    cols = [_view(p.pos[a], n, torch.float64) for a in range(3)]
    cols += [_view(p.vel[a], n, torch.float64) for a in range(3)]
    return torch.stack(cols, dim=1) if n else torch.empty((0, 6), dtype=torch.float64, device="cuda")


def _write_particles(dev, rows) -> None:
    import torch
    p = _ptrs(dev)
    m = int(rows.shape[0])
    torch.cuda.synchronize()
    if m > p.capacity:  # grow first (keeps nothing we need: rows is a copy)
        check(LIB.flip_reserve_particles(dev.ctx, m), "flip_reserve_particles")
        p = _ptrs(dev)
    for a in range(6):
        ptr = p.pos[a] if a < 3 else p.vel[a - 3]
        if m:
            _view(ptr, m, torch.float64).copy_(rows[:, a])
    torch.cuda.synchronize()
    check(LIB.flip_set_particle_count(dev.ctx, m), "flip_set_particle_count")
    dev.bump()


def _particle_planes(dev, plan: SlabPlan):
    import torch
    n = dev.count()
    cells = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    check(LIB.flip_particle_cells(dev.ctx, C.c_void_p(cells.data_ptr())), "flip_particle_cells")
    check(LIB.flip_synchronize(dev.ctx))
    return (cells[:n].long() // plan.plane_cells)


# ---------------------------------------------------------- the step ----
class SlabContext:
    def __init__(self, plan: SlabPlan, tr: Transport):
        import torch
        self.plan = plan
        self.tr = tr
        self.owners = torch.as_tensor(plan.plane_owners(), device="cuda")


def make_scene(spec, rng_seed: int = 0, group=None, device: int = 0, capacity: int = 0):
    """make_scene on every rank (the scene builder is deterministic), then
    each rank keeps the particles of its own slab."""
    tr = Transport(group)
    state = _sim.make_scene(spec, rng_seed, device=device, capacity=capacity)
    dev = state.device
    plan = SlabPlan(dev.dims.nx, dev.dims.ny, dev.dims.nz, tr.world)
    ctx = SlabContext(plan, tr)
    k0, k1 = plan.planes(tr.rank)
    check(LIB.flip_set_slab(dev.ctx, k0, k1), "flip_set_slab")
    planes = _particle_planes(dev, plan)
    rows = _particle_rows(dev)
    keep = (planes >= k0) & (planes < k1)
    _write_particles(dev, rows[keep])
    rc, _ = dev.run_stages(_sim._params(spec, dev.dims.dtau), _lib.STAGE["bin"], _lib.STAGE["bin"])
    check(rc, "slab bin")
    state.slab = ctx
    return state


def _stages(state, params, first: str, last: str, acc: dict):
    dev = state.device
    rc, rep = dev.run_stages(params, _lib.STAGE[first], _lib.STAGE[last])
    if rc in (_lib.FLIP_E_SINGULAR, _lib.FLIP_E_BREAKDOWN):
        _sim._raise_solver(state, rep)
    check(rc, f"flip_run_stages {first}..{last}")
    for i in range(_lib.STAGE[first], _lib.STAGE[last] + 1):
        name = _lib.STAGE_NAMES[i]
        acc[name] = acc.get(name, 0.0) + float(rep.stage_ms[i])
    acc["_launches"] = acc.get("_launches", 0) + int(rep.gpu_launches)
    return rep


def step(state, cfg):
    """One slab-decomposed timestep; same StepReport as ``sim.step``."""
    import torch
    ctx: SlabContext = state.slab
    plan, tr = ctx.plan, ctx.tr
    dev = state.device
    seed = rng.derive_seed(state.rng_seed, state.step_count + 1)
    params = _sim._params(cfg, dev.dims.dtau, seed)
    acc: dict = {}
    k0, k1 = plan.planes(tr.rank)
    pc = plan.plane_cells

    # 1. dt: local, allreduce MIN
    _stages(state, params, "dt_compute", "dt_compute", acc)
    dt = torch.tensor([dev.dt()], dtype=torch.float64, device="cuda")
    tr.allreduce_min_(dt)
    dev.set_dt(float(dt.item()))
    # 2-3. advect, migration
    _stages(state, params, "advect", "advect", acc)
    rows = migrate_rows(_particle_rows(dev), _particle_planes(dev, plan), ctx.owners, tr)
    _write_particles(dev, rows)
    # 4-5. bin, classify + label MIN
    _stages(state, params, "bin", "classify", acc)
    p = _ptrs(dev)
    label = _view(p.label, dev.dims.ncells, torch.uint8)
    tr.allreduce_min_(label)
    torch.cuda.synchronize()
    # 6. ghost planes
    offset = _view(p.offset, dev.dims.ncells + 1, torch.int32)
    bounds = offset[torch.tensor([k0 * pc, (k0 + 1) * pc, (k1 - 1) * pc, k1 * pc],
                                 device="cuda")].tolist()
    own = _particle_rows(dev)
    n_own = int(own.shape[0])
    glo, ghi = ghost_rows(own, (bounds[0], bounds[1]), (bounds[2], bounds[3]), tr)
    _write_particles(dev, torch.cat([glo, own, ghi]))
    # 7. bin the extended set, P2G + force, drop the ghosts, re-bin
    _stages(state, params, "bin", "bin", acc)
    _stages(state, params, "p2g", "force", acc)
    _write_particles(dev, own)
    _stages(state, params, "bin", "bin", acc)
    # 8. owned faces of grid, grid_old, known masks
    p = _ptrs(dev)
    nfaces = dev.nfaces
    arrays = [(p.u, 0, torch.float64), (p.v, 1, torch.float64), (p.w, 2, torch.float64),
              (p.uo, 0, torch.float64), (p.vo, 1, torch.float64), (p.wo, 2, torch.float64),
              (p.ku, 0, torch.uint8), (p.kv, 1, torch.uint8), (p.kw, 2, torch.uint8)]
    for ptr, comp, dtype in arrays:
        full = _view(ptr, nfaces[comp], dtype)
        rngs = [face_ranges(plan, comp, r) for r in range(tr.world)]
        lo, hi = rngs[tr.rank]
        parts = tr.allgather_var(full[lo:hi], [b - a for a, b in rngs])
        for r, (a, b) in enumerate(rngs):
            if r != tr.rank and b > a:
                full[a:b].copy_(parts[r])
    torch.cuda.synchronize()
    dev.bump()
    # 9-11. replicated grid stages, then G2P + reseed on the slab
    rep = _stages(state, params, "project", "apply_gradient", acc)
    solver = (int(rep.solver_iterations), float(rep.solver_residual), bool(rep.solver_converged),
              int(rep.nrows), int(rep.npinned))
    rep2 = _stages(state, params, "g2p", "reseed", acc)
    total = tr.allreduce_sum_int(int(rep2.particle_count))
    timings = _sim.StageTimings(**{n: acc.get(n, 0.0) for n in _lib.STAGE_NAMES})
    state.time += float(dt.item())
    state.step_count += 1
    return _sim.StepReport(timings=timings, dt=float(dt.item()), particle_count=total,
                           solver_iterations=solver[0], solver_residual=solver[1],
                           solver_converged=solver[2], nrows=solver[3], npinned=solver[4],
                           gpu_launches=int(acc["_launches"]))


def gather_particles(state):
    """The global particle set (host arrays, every rank), concatenated in
    rank order = the 1-GPU order."""
    import torch
    tr: Transport = state.slab.tr
    rows = _particle_rows(state.device)
    sizes = [0] * tr.world
    n = torch.tensor([rows.shape[0]], dtype=torch.int64)
    if not tr.staged:
        n = n.cuda()
    lst = [torch.zeros_like(n) for _ in range(tr.world)]
    tr.dist.all_gather(lst, n, group=tr.group)
    sizes = [int(x.item()) for x in lst]
    cols = []
    for a in range(6):
        parts = tr.allgather_var(rows[:, a].contiguous(), sizes)
        cols.append(torch.cat(parts).cpu().numpy())
    return tuple(cols)
