"""Slab decomposition of the FLIP step over ranks (one process per GPU).

SURVEY §8(e); north star: "the domain is slab-decomposed across the 8 GPUs
of one box, with ghost-layer pressure/velocity halo exchange and particle
migration over NVLink (NCCL or P2P), and the CG dot products are
allreduced".

Decomposition
-------------
Rank r owns the cell z-planes ``[k0, k1)`` of :class:`SlabPlan`.  The flat
index is x-fastest with z slowest (``flipsim/grid.py:47-72``), so the rank's
cells, the faces of its planes, the pressure rows of its cells (rows ascend
with the cell index, ``pressure.py:76-166``) and its cell-sorted particles
are each one contiguous range of the global arrays.  Every device array
keeps its full-grid size and global indexing; the library computes only the
rank's range and calls back into :class:`Transport` for each exchange
(``flip_comm`` in ``include/flipb200.h``, driven from inside
``flip_step``).  Per step, all on the device and stream-ordered:

==================  ======================================================
stage               sharding / exchange (``csrc/slab.cu``, ``pressure.cu``)
==================  ======================================================
dt                  own particles; MAX-allreduce of max|v|^2 (8 B)
advect + migrate    own particles; particles whose cell left the slab go
                    to its owner (all-to-all, order kept)
bin, classify       own particles / own cells; the label planes are
                    all-gathered (1 B/cell: sealed-region pinning is global)
P2G + force         own face planes; the neighbours' boundary particle
                    planes are the ghosts; then 1-plane face halos
assemble            own rows' rhs (global row numbering); MAX of max|rhs|
solve               own rows; 1-plane row halo before every stencil pass,
                    MAX-allreduced residuals, distributed bit-exact
                    pairwise dots; MIC(0) / GS / multigrid sweeps are
                    global recurrences: replicated on the all-gathered r
gradient, extrap.   own face planes; 1-plane face halos between passes
G2P, reseed         own particles / own cells
==================  ======================================================

The concatenation of the ranks' particles (rank order) is the 1-GPU particle
array and every rank's own planes hold the 1-GPU grid, bit for bit
(``tests/test_dist_gpu.py``).

Transport
---------
``backend="nccl"``: collectives on the ctx stream (``torch.cuda.ExternalStream``)
over device tensors aliasing the ctx's buffers, no host sync.  ``"gloo"``:
staged through host memory (CPU tests; ranks sharing the one GPU of this
pool, where no kernel waits on another process).
"""

from __future__ import annotations

import ctypes as C
import traceback
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import LIB, check
from . import rng
from . import sim as _sim

__all__ = ["SlabPlan", "Transport", "make_scene", "step", "gather_particles", "gather_grid",
           "face_ranges", "pairwise_tree_plan", "distributed_pairwise_sum", "exchange_stats"]

FLIP_OP_MAX, FLIP_OP_MIN, FLIP_OP_SUM = 0, 1, 2


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

    def starts(self) -> list:
        return [self.planes(r)[0] for r in range(self.world)] + [self.nz]

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
    last rank (``grid.py:65-72`` layouts; ``slab_face_range`` in slab.cu)."""
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


# ------------------------------------- distributed pairwise tree (mirror) ---
def _split(n: int) -> int:
    n2 = n // 2
    return n2 - n2 % 8


def _pairwise(a) -> float:
    """numpy DOUBLE_pairwise_sum (np.add.reduce, pressure.py:269-271)."""
    n = len(a)
    if n < 8:
        s = 0.0
        for v in a:
            s += float(v)
        return s
    if n <= 128:
        r = [float(a[i]) for i in range(8)]
        for i in range(8, n - n % 8, 8):
            for k in range(8):
                r[k] += float(a[i + k])
        s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for i in range(n - n % 8, n):
            s += float(a[i])
        return s
    n2 = _split(n)
    return _pairwise(a[:n2]) + _pairwise(a[n2:])


def pairwise_tree_plan(n: int):
    """(cut, node spans) of the deepest tree level at which every node
    exists (pw_cut in pressure.cu)."""
    spans = [(0, n)]
    cut = 0
    while spans and all(l > 128 for _, l in spans):
        nxt = []
        for s, l in spans:
            n2 = _split(l)
            nxt += [(s, n2), (s + n2, l - n2)]
        spans = nxt
        cut += 1
    return cut, spans


def distributed_pairwise_sum(parts) -> float:
    """Host restatement of the slab dot (launch_dot_slab, pressure.cu):
    ``parts`` are the ranks' contiguous pieces of one vector.  Each rank sums
    the cut-level nodes that start in its rows (reading the next ranks'
    leading elements), reduces them to maximal aligned blocks, and the
    blocks are merged in index order -- bit-identical to np.add.reduce of the
    concatenation (tests/test_dist_host.py)."""
    full = np.concatenate(parts) if parts else np.zeros(0)
    n = len(full)
    cut, spans = pairwise_tree_plan(max(n, 1))
    starts = np.cumsum([0] + [len(p) for p in parts])
    blocks = []
    for q in range(len(parts)):
        r0, r1 = int(starts[q]), int(starts[q + 1])
        mine = [k for k, (s, _) in enumerate(spans) if r0 <= s < r1 or (q == len(parts) - 1 and s >= r1)]
        if n == 0 or not mine:
            continue
        na, nb = mine[0], mine[-1] + 1
        v = {k: _pairwise(full[spans[k][0]:spans[k][0] + spans[k][1]]) for k in range(na, nb)}
        st = 1
        while st < nb - na:
            for g in range(na, nb):
                if g % (2 * st) == 0 and g + 2 * st <= nb:
                    v[g] = v[g] + v[g + st]
            st *= 2
        g = na
        while g < nb:
            lvl = 0
            while (g >> lvl) & 1 == 0 and g + (2 << lvl) <= nb:
                lvl += 1
            blocks.append((lvl, g >> lvl, v[g]))
            g += 1 << lvl
    stack = []
    for b in blocks:
        stack.append(list(b))
        while (len(stack) >= 2 and stack[-1][0] == stack[-2][0] and stack[-2][1] % 2 == 0
               and stack[-1][1] == stack[-2][1] + 1):
            top = stack.pop()
            stack[-1] = [top[0] + 1, stack[-1][1] >> 1, stack[-1][2] + top[2]]
    return stack[0][2] if stack else 0.0


# ------------------------------------------------------------ transport ----
_NEIGH = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                     C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64)
_ALLRED = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32)
_ALLGV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64))
_A2AV = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64),
                    C.c_void_p, C.POINTER(C.c_int64))


class FlipComm(C.Structure):
    _fields_ = [("user", C.c_void_p), ("neighbors", _NEIGH), ("allreduce", _ALLRED),
                ("allgatherv", _ALLGV), ("alltoallv", _A2AV)]


class _CAI:
    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def _dview(ptr, nbytes: int, typestr: str = "|u1", itemsize: int = 1):
    """A torch tensor aliasing device memory (no copy)."""
    import torch
    n = int(nbytes) // itemsize
    if n == 0 or not ptr:
        return torch.empty(0, dtype={"|u1": torch.uint8, "<i8": torch.int64}[typestr],
                           device="cuda")
    return torch.as_tensor(_CAI(ptr, n, typestr), device="cuda")


class Transport:
    """The flip_comm callbacks over torch.distributed.

    Each collective also has a tensor-level form (``*_t``) used directly by
    the CPU tests.  With NCCL the tensors are device views and the ops run
    on the library's stream; with gloo they are staged through host memory
    (the stream is synchronised first and the results copied back before
    the callback returns)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch = torch
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.staged = dist.get_backend(group) != "nccl"
        self._cbs = None

    # ---- tensor level -------------------------------------------------
    def neighbors_t(self, send_lo, send_hi, recv_lo, recv_hi):
        """send_lo -> rank-1, send_hi -> rank+1; recv_lo <- rank-1,
        recv_hi <- rank+1 (empty tensors skip)."""
        d, ops = self.dist, []
        r, w = self.rank, self.world
        if r > 0 and send_lo.numel():
            ops.append(d.P2POp(d.isend, send_lo, r - 1, self.group))
        if r > 0 and recv_lo.numel():
            ops.append(d.P2POp(d.irecv, recv_lo, r - 1, self.group))
        if r + 1 < w and send_hi.numel():
            ops.append(d.P2POp(d.isend, send_hi, r + 1, self.group))
        if r + 1 < w and recv_hi.numel():
            ops.append(d.P2POp(d.irecv, recv_hi, r + 1, self.group))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()

    def allreduce_t(self, t, op: int):
        d = self.dist
        red = {FLIP_OP_MAX: d.ReduceOp.MAX, FLIP_OP_MIN: d.ReduceOp.MIN,
               FLIP_OP_SUM: d.ReduceOp.SUM}[int(op)]
        d.all_reduce(t, op=red, group=self.group)

    def allgatherv_t(self, buf, offsets):
        """In place: bytes [offsets[q], offsets[q+1]) of rank q everywhere."""
        torch = self.torch
        sizes = [int(offsets[q + 1] - offsets[q]) for q in range(self.world)]
        m = max(max(sizes), 1)
        mine = torch.zeros(m, dtype=buf.dtype, device=buf.device)
        a, b = int(offsets[self.rank]), int(offsets[self.rank + 1])
        mine[:b - a] = buf[a:b]
        out = torch.empty(m * self.world, dtype=buf.dtype, device=buf.device)
        self.dist.all_gather_into_tensor(out, mine, group=self.group)
        for q in range(self.world):
            if q != self.rank and sizes[q]:
                buf[int(offsets[q]):int(offsets[q + 1])] = out[q * m:q * m + sizes[q]]

    def alltoallv_t(self, send, sbytes, recv, rbytes):
        self.dist.all_to_all_single(recv, send, [int(x) for x in rbytes],
                                    [int(x) for x in sbytes], group=self.group)

    # ---- flip_comm callbacks (device pointers) -------------------------
    def _stage(self, views):
        """gloo: host copies of device views (after the ctx stream drained)."""
        return [v.cpu() for v in views]

    def _run(self, stream, fn):
        torch = self.torch
        try:
            if self.staged:
                torch.cuda.synchronize()
                fn()
                torch.cuda.synchronize()
            else:
                with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0))):
                    fn()
            return 0
        except Exception:  # reported through the C status
            traceback.print_exc()
            return 1

    def comm(self) -> FlipComm:
        """The callback table for flip_set_slab_comm (kept alive here)."""
        if self._cbs is not None:
            return self._cbs[0]

        def neighbors(user, stream, slo, nslo, shi, nshi, rlo, nrlo, rhi, nrhi):
            def go():
                views = [_dview(slo, nslo), _dview(shi, nshi), _dview(rlo, nrlo), _dview(rhi, nrhi)]
                if self.staged:
                    h = self._stage(views)
                    self.neighbors_t(*h)
                    views[2].copy_(h[2])
                    views[3].copy_(h[3])
                else:
                    self.neighbors_t(*views)
            return self._run(stream, go)

        def allreduce(user, stream, buf, n, op):
            def go():
                v = _dview(buf, 8 * n, "<i8", 8)
                t = v.cpu() if self.staged else v
                self.allreduce_t(t, op)
                if self.staged:
                    v.copy_(t)
            return self._run(stream, go)

        def allgatherv(user, stream, buf, offsets):
            def go():
                off = [int(offsets[q]) for q in range(self.world + 1)]
                v = _dview(buf, off[-1])
                t = v.cpu() if self.staged else v
                self.allgatherv_t(t, off)
                if self.staged:
                    v.copy_(t)
            return self._run(stream, go)

        def alltoallv(user, stream, send, sbytes, recv, rbytes):
            def go():
                sb = [int(sbytes[q]) for q in range(self.world)]
                rb = [int(rbytes[q]) for q in range(self.world)]
                s, r = _dview(send, sum(sb)), _dview(recv, sum(rb))
                if self.staged:
                    hs = s.cpu()
                    hr = self.torch.empty(sum(rb), dtype=self.torch.uint8)
                    self.alltoallv_t(hs, sb, hr, rb)
                    if sum(rb):
                        r.copy_(hr)
                else:
                    self.alltoallv_t(s, sb, r, rb)
            return self._run(stream, go)

        fns = (_NEIGH(neighbors), _ALLRED(allreduce), _ALLGV(allgatherv), _A2AV(alltoallv))
        cs = FlipComm(None, *fns)
        self._cbs = (cs, fns)
        return cs

    def allreduce_sum_int(self, v: int) -> int:
        t = self.torch.tensor([int(v)], dtype=self.torch.int64)
        if not self.staged:
            t = t.cuda()
        self.dist.all_reduce(t, group=self.group)
        return int(t.item())

    def allgather_obj(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


# ---------------------------------------------------------- the step ----
class SlabContext:
    def __init__(self, plan: SlabPlan, tr: Transport):
        self.plan = plan
        self.tr = tr


def make_scene(spec, rng_seed: int = 0, group=None, device: int = 0, capacity: int = 0):
    """make_scene on every rank (the scene builder is deterministic), then
    each rank keeps the particles of its own planes (a contiguous range of
    the binned set) and enters slab mode."""
    import torch
    if getattr(spec, "advection", "euler") != "euler":
        raise _sim.ConfigError("RK2 advection is not supported with a slab decomposition")
    tr = Transport(group)
    state = _sim.make_scene(spec, rng_seed, device=device, capacity=capacity)
    dev = state.device
    plan = SlabPlan(dev.dims.nx, dev.dims.ny, dev.dims.nz, tr.world)
    k0, k1 = plan.planes(tr.rank)
    pc = plan.plane_cells
    p = _lib.DevPtrs()
    check(LIB.flip_get_dev_ptrs(dev.ctx, C.byref(p)), "flip_get_dev_ptrs")
    off, _cnt = dev.hash_arrays()
    a = int(off[k0 * pc])
    b = int(off[k1 * pc]) if k1 * pc < len(off) else int(p.n)
    torch.cuda.synchronize()
    for ptr in list(p.pos) + list(p.vel):
        v = _dview(ptr, 8 * int(p.n), "<i8", 8)
        keep = v[a:b].clone()
        v[:b - a].copy_(keep)
    torch.cuda.synchronize()
    check(LIB.flip_set_particle_count(dev.ctx, b - a), "flip_set_particle_count")
    dev.bump()
    rc, _ = dev.run_stages(_sim._params(spec, dev.dims.dtau), _lib.STAGE["bin"], _lib.STAGE["bin"])
    check(rc, "slab bin")
    starts = (C.c_int64 * (tr.world + 1))(*plan.starts())
    comm = tr.comm()
    check(LIB.flip_set_slab_comm(dev.ctx, tr.rank, tr.world, C.addressof(starts),
                                 C.addressof(comm)), "flip_set_slab_comm")
    state.slab = SlabContext(plan, tr)
    return state


def step(state, cfg):
    """One slab-decomposed timestep (the whole step runs inside
    flip_step); same StepReport as ``sim.step`` with the global particle
    count."""
    dev = state.device
    tr = state.slab.tr
    seed = rng.derive_seed(state.rng_seed, state.step_count + 1)
    params = _sim._params(cfg, dev.dims.dtau, seed)
    rc, rep = dev.run_stages(params, 0, _lib.NSTAGES - 1)
    if rc in (_lib.FLIP_E_SINGULAR, _lib.FLIP_E_BREAKDOWN):
        _sim._raise_solver(state, rep)
    check(rc, "flip_step (slab)")
    total = tr.allreduce_sum_int(int(rep.particle_count))
    timings = _sim.StageTimings(**{n: float(rep.stage_ms[i])
                                   for i, n in enumerate(_lib.STAGE_NAMES)})
    state.time += float(rep.dt)
    state.step_count += 1
    return _sim.StepReport(timings=timings, dt=float(rep.dt), particle_count=total,
                           solver_iterations=int(rep.solver_iterations),
                           solver_residual=float(rep.solver_residual),
                           solver_converged=bool(rep.solver_converged), nrows=int(rep.nrows),
                           npinned=int(rep.npinned), gpu_launches=int(rep.gpu_launches))


def exchange_stats(state) -> dict:
    """Bytes this rank sent and collective calls since the last query."""
    sent, calls = C.c_int64(0), C.c_int64(0)
    check(LIB.flip_slab_bytes(state.device.ctx, C.byref(sent), C.byref(calls)))
    return {"bytes_sent": int(sent.value), "calls": int(calls.value)}


def gather_particles(state):
    """The global particle set (host arrays, every rank), concatenated in
    rank order = the 1-GPU order."""
    tr: Transport = state.slab.tr
    parts = state.particles.arrays()
    allp = tr.allgather_obj([np.asarray(a) for a in parts])
    return tuple(np.concatenate([allp[q][a] for q in range(tr.world)]) for a in range(6))


def gather_grid(state):
    """The global grid / grid_old / hash as one GPU holds them: every array
    assembled from its owners' planes (host arrays, every rank)."""
    tr: Transport = state.slab.tr
    plan = state.slab.plan
    g, go = state.grid, state.grid_old
    pc = plan.plane_cells
    k0, k1 = plan.planes(tr.rank)
    mine = {}
    for name, arr in (("u", g.u), ("v", g.v), ("w", g.w), ("uo", go.u), ("vo", go.v),
                      ("wo", go.w)):
        comp = "uvw".index(name[0])
        a, b = face_ranges(plan, comp, tr.rank)
        mine[name] = np.asarray(arr)[a:b]
    for name, arr in (("p", g.p), ("label", g.label), ("count", state.hash.count)):
        mine[name] = np.asarray(arr)[k0 * pc:k1 * pc]
    every = tr.allgather_obj(mine)
    return {k: np.concatenate([every[q][k] for q in range(tr.world)]) for k in mine}
