"""CPU oracle for the FLIP timestep: ctypes glue over ``oracle/flip_oracle.c``.

TEST INFRASTRUCTURE ONLY.  Imported by ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` leg, and nowhere else.
The product package never imports this module.

It restates the reference step (``flipsim.sim.step``,
/root/reference/pkg/src/flipsim/sim.py:226-300) stage by stage, calling the C
restatement of each reference function.  Scene construction restates
``sim.py:96-223`` (scene_regions, _fit_box, make_scene).  Parity of this
oracle with the real reference is pinned by ``tests/golden/`` fixtures
(generated from the reference by ``tests/golden/make_golden.py``) and, in the
build container, by ``tests/test_oracle_pins.py::test_oracle_equals_live_reference_40cubed``
(the live reference, skipped where /root/reference is absent).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
import time
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(HERE, "liboracle.so")

SOLID, FLUID, AIR = 0, 1, 2
SCENE_NAMES = ("dam-break", "double-dam-break", "water-drop", "double-dam-break-obstacle")
SOLVER_KIND = {"jacobi": 0, "gs": 1, "rbgs": 2, "pcg": 3}
PRECOND = {"mic0": 0, "jacobi": 1, "none": 2}
STAGES = ("dt_compute", "advect", "bin", "classify", "p2g", "force", "project",
          "apply_gradient", "g2p", "reseed")

_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)
_u8 = C.POINTER(C.c_uint8)


class Dims(C.Structure):
    _fields_ = [("nx", C.c_int64), ("ny", C.c_int64), ("nz", C.c_int64),
                ("dtau", C.c_double), ("ox", C.c_double), ("oy", C.c_double),
                ("oz", C.c_double)]


class SolveRes(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("residual", C.c_double),
                ("converged", C.c_int), ("err_cell", C.c_int64),
                ("err_it", C.c_int64), ("err_value", C.c_double)]


def build() -> None:
    src = os.path.join(HERE, "flip_oracle.c")
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src)):
        cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
        subprocess.run(["make", "-s", "-C", HERE, f"CC={cc}", "liboracle.so"], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        P = C.POINTER
        sig = {
            "orc_uniform01": (C.c_double, [C.c_uint64, C.c_uint64, C.c_uint64]),
            "orc_derive_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "orc_covered_cells_box": (C.c_int64, [P(Dims), _d, _d, _i64]),
            "orc_covered_cells_sphere": (C.c_int64, [P(Dims), _d, C.c_double, _i64]),
            "orc_jittered_positions": (None, [P(Dims), C.c_int64, _i64, _i64, C.c_int64,
                                              C.c_uint64, _d, _d, _d]),
            "orc_compute_dt": (C.c_double, [C.c_int64, _d, _d, _d, C.c_double, C.c_double,
                                            C.c_double]),
            "orc_interior_box": (C.c_int, [P(Dims), _u8, _d, _d]),
            "orc_advect_rk2": (None, [P(Dims), _d, _d, _d, C.c_int64, _d, _d, _d, C.c_double,
                                      _d, _d, C.c_double]),
            "orc_advect": (None, [C.c_int64, _d, _d, _d, _d, _d, _d, C.c_double, _d, _d,
                                  C.c_double]),
            "orc_cell_index_many": (None, [P(Dims), C.c_int64, _d, _d, _d, _i64]),
            "orc_exclusive_scan": (None, [C.c_int64, _i64, _i64]),
            "orc_counting_sort_perm": (None, [C.c_int64, _i64, _i64, C.c_int64, _i64]),
            "orc_bin_particles": (None, [P(Dims), C.c_int64, P(_d), _d, _i64, _i64, _i64,
                                         _i64]),
            "orc_classify_cells": (None, [C.c_int64, _i64, _u8]),
            "orc_sample_velocity_many": (None, [P(Dims), _d, _d, _d, C.c_int64, _d, _d, _d,
                                                _d, _d, _d]),
            "orc_p2g_component": (None, [P(Dims), C.c_int, _d, _d, _d, _d, _i64, _i64, _d,
                                         _d]),
            "orc_add_body_force": (None, [P(Dims), _d, _d, _d, _d, C.c_double]),
            "orc_enforce_solid_boundaries": (None, [P(Dims), _u8, _d, _d, _d]),
            "orc_extrapolate_component": (None, [C.c_int64, C.c_int64, C.c_int64, _d, _u8,
                                                 C.c_int, _d, _i64, _u8]),
            "orc_assemble": (C.c_int64, [P(Dims), _u8, _d, _d, _d, _i64, _i64, _d, _i64, _d,
                                         _i64, _i64]),
            "orc_laplacian_matvec": (None, [C.c_int64, _d, _i64, _d, C.c_double, _d]),
            "orc_jacobi_iter": (None, [C.c_int64, _d, _i64, _d, _d, C.c_double, _d]),
            "orc_gs_sweep": (None, [C.c_int64, _d, _i64, _d, _d, C.c_double]),
            "orc_gs_sweep_rows": (None, [C.c_int64, _i64, _d, _i64, _d, _d, C.c_double]),
            "orc_mic0_build": (None, [C.c_int64, _d, _i64, C.c_double, C.c_double,
                                      C.c_double, _d]),
            "orc_mic0_apply": (None, [C.c_int64, _d, _i64, _d, C.c_double, _d, _d]),
            "orc_pairwise_dot": (C.c_double, [C.c_int64, _d, _d]),
            "orc_pairwise_sum": (C.c_double, [C.c_int64, _d]),
            "orc_solve": (C.c_int, [C.c_int, C.c_int, C.c_int64, _i64, _d, _i64, _d,
                                    C.c_double, C.c_int64, C.c_double, _i64, C.c_int64, _i64,
                                    C.c_int64, _d, _d, P(SolveRes)]),
            "orc_apply_pressure_gradient": (None, [P(Dims), _u8, _d, C.c_double, C.c_double,
                                                   _d, _d, _d]),
            "orc_g2p": (None, [P(Dims), _d, _d, _d, _d, _d, _d, C.c_int64, _d, _d, _d, _d,
                               _d, _d, C.c_double]),
            "orc_reseed_counts": (C.c_int64, [C.c_int64, _i64, _u8, C.c_int64, _i64, _i64,
                                              _i64]),
            "orc_reseed_fill": (None, [P(Dims), C.c_int64, _i64, _i64, _i64, _i64, C.c_int64,
                                       C.c_uint64, P(_d), P(_d), _d, _d, _d]),
            "orc_divergence_field": (None, [P(Dims), _d, _d, _d, _d]),
            "orc_num_threads": (C.c_int, []),
            "orc_set_num_threads": (None, [C.c_int]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _p(a, kind=_d):
    return a.ctypes.data_as(kind)


def set_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().orc_num_threads())


# --------------------------------------------------------------- config ---
@dataclass
class Spec:
    """Restates SceneSpec (sim.py:50-72)."""
    name: str = "dam-break"
    res: int = 32
    density: int = 2
    particle_target: int | None = None
    gravity: tuple = (0.0, -9.81, 0.0)
    solver: str = "pcg"
    tol: float = 1e-6
    max_iters: int | None = None
    flip_fraction: float = 0.95
    alpha: float = 3.0
    dt_max: float = 1.0 / 30.0
    rho_fluid: float = 1000.0
    skin_fraction: float = 1e-3
    extrapolation_layers: int = 2
    steps: int = 50
    precond: str = "mic0"   # not in SceneSpec; the reference hard-wires mic0 (pressure.py:274)
    obstacles: tuple = ()   # extension: SOLID cell boxes after the shell
    advection: str = "euler"  # extension: "rk2" = orc_advect_rk2 (the reference is Euler only)

    def resolved_max_iters(self) -> int:
        if self.max_iters is not None:
            return self.max_iters
        return 100 if self.solver == "pcg" else 2000


@dataclass
class Dimz:
    nx: int
    ny: int
    nz: int
    dtau: float
    origin: tuple = (0.0, 0.0, 0.0)

    @property
    def ncells(self):
        return self.nx * self.ny * self.nz

    def c(self) -> Dims:
        return Dims(self.nx, self.ny, self.nz, self.dtau, *[float(x) for x in self.origin])


@dataclass
class Region:
    kind: str
    a: tuple
    b: object
    density: int


def _box_region(dims, i0, i1, j0, j1, k0, k1, density):     # sim.py:105-109
    o = np.asarray(dims.origin, dtype=np.float64)
    lo = o + np.array([i0, j0, k0]) * dims.dtau
    hi = o + np.array([i1 + 1, j1 + 1, k1 + 1]) * dims.dtau
    return Region("box", tuple(float(x) for x in lo), tuple(float(x) for x in hi), density)


def _fit_box(target, ni, nj, nk, frac_x, frac_y):             # sim.py:112-132
    best = None
    for rho in range(1, 11):
        per_cell = rho ** 3
        need = target / per_cell / nk
        ratio = (frac_x * ni) / (frac_y * nj)
        cx0 = np.sqrt(need * ratio)
        for cx in range(max(1, int(cx0) - 2), min(ni, int(cx0) + 3)):
            cy_mid = need / cx
            for cy in range(max(1, int(cy_mid) - 1), min(nj, int(cy_mid) + 3)):
                count = cx * cy * nk * per_cell
                err = abs(count - target) / target
                distort = abs(cx / (frac_x * ni) - 1.0) + abs(cy / (frac_y * nj) - 1.0)
                key = (err > 0.05, round(err, 6), round(distort, 6), rho)
                if best is None or key < best[0]:
                    best = (key, rho, cx, cy)
    return best[1], best[2], best[3]


def covered_cells(region: Region, dims: Dimz) -> np.ndarray:  # particles.py:103-110
    out = np.empty(dims.ncells, dtype=np.int64)
    if region.kind == "box":
        lo = np.asarray(region.a, dtype=np.float64)
        hi = np.asarray(region.b, dtype=np.float64)
        m = lib().orc_covered_cells_box(C.byref(dims.c()), _p(lo), _p(hi), _p(out, _i64))
    else:
        c = np.asarray(region.a, dtype=np.float64)
        m = lib().orc_covered_cells_sphere(C.byref(dims.c()), _p(c), float(region.b),
                                           _p(out, _i64))
    return out[:m].copy()


def scene_regions(spec: Spec, dims: Dimz):                    # sim.py:140-201
    lo_c, hi_c = 1, spec.res - 2
    ni = nj = nk = hi_c - lo_c + 1
    if ni < 1:
        raise ValueError(f"resolution {spec.res} leaves no interior cells")
    edge = dims.nx * dims.dtau
    o = np.asarray(dims.origin, dtype=np.float64)
    if spec.name == "dam-break":
        if spec.particle_target:
            rho, cx, cy = _fit_box(spec.particle_target, ni, nj, nk, 0.25, 0.75)
        else:
            rho, cx, cy = spec.density, max(1, round(0.25 * ni)), max(1, round(0.75 * nj))
        return [_box_region(dims, lo_c, lo_c + cx - 1, lo_c, lo_c + cy - 1, lo_c, hi_c, rho)]
    if spec.name in ("double-dam-break", "double-dam-break-obstacle"):
        if spec.particle_target:
            rho, cx, cy = _fit_box(spec.particle_target // 2, ni, nj, nk, 0.25, 0.75)
        else:
            rho, cx, cy = spec.density, max(1, round(0.25 * ni)), max(1, round(0.75 * nj))
        cx = min(cx, ni // 2)
        return [_box_region(dims, lo_c, lo_c + cx - 1, lo_c, lo_c + cy - 1, lo_c, hi_c, rho),
                _box_region(dims, hi_c - cx + 1, hi_c, lo_c, lo_c + cy - 1, lo_c, hi_c, rho)]
    if spec.name == "water-drop":
        center = tuple(o + (0.5 * edge, 0.6 * edge, 0.5 * edge))
        radius = 0.125 * edge
        pool_cap = max(1, int(0.40 * nj))
        if spec.particle_target:
            sphere_n = len(covered_cells(Region("sphere", center, radius, 1), dims))
            best = None
            for rho in range(1, 11):
                need = spec.particle_target / rho ** 3 - sphere_n
                py = min(pool_cap, max(1, round(need / (ni * nk))))
                count = (py * ni * nk + sphere_n) * rho ** 3
                err = abs(count - spec.particle_target) / spec.particle_target
                key = (err > 0.05, round(err, 6), rho)
                if best is None or key < best[0]:
                    best = (key, rho, py)
            rho, py = best[1], best[2]
        else:
            rho, py = spec.density, max(1, round(0.25 * nj))
        return [_box_region(dims, lo_c, hi_c, lo_c, lo_c + py - 1, lo_c, hi_c, rho),
                Region("sphere", tuple(float(x) for x in center), float(radius), rho)]
    raise ValueError(f"unknown scene {spec.name!r}")


# ---------------------------------------------------------------- state ---
@dataclass
class OState:
    dims: Dimz
    u: np.ndarray
    v: np.ndarray
    w: np.ndarray
    p: np.ndarray
    label: np.ndarray
    uo: np.ndarray
    vo: np.ndarray
    wo: np.ndarray
    parts: list            # six float64 arrays pos_x..vel_z
    count: np.ndarray
    offset: np.ndarray
    time: float = 0.0
    step_count: int = 0
    rng_seed: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return len(self.parts[0])

    def copy(self) -> "OState":
        return OState(self.dims, self.u.copy(), self.v.copy(), self.w.copy(), self.p.copy(),
                      self.label.copy(), self.uo.copy(), self.vo.copy(), self.wo.copy(),
                      [a.copy() for a in self.parts], self.count.copy(), self.offset.copy(),
                      self.time, self.step_count, self.rng_seed)

    def fluid_cells(self) -> np.ndarray:
        return np.flatnonzero(self.count > 0).astype(np.int64)


def empty_grid(dims: Dimz):
    nx, ny, nz = dims.nx, dims.ny, dims.nz
    return (np.zeros((nx + 1) * ny * nz), np.zeros(nx * (ny + 1) * nz),
            np.zeros(nx * ny * (nz + 1)), np.zeros(nx * ny * nz),
            np.full(nx * ny * nz, AIR, dtype=np.uint8))


def scene_obstacles(spec: Spec, dims: Dimz):
    """Extension (no reference counterpart): SOLID boxes of the scene, same
    rule as paper_2404_01931_b200.sim.scene_obstacles."""
    boxes = [tuple(int(x) for x in b) for b in spec.obstacles]
    if spec.name == "double-dam-break-obstacle":
        lo_c, hi_c = 1, spec.res - 2
        n = hi_c - lo_c + 1
        i0 = lo_c + round(0.45 * n)
        i1 = max(i0, lo_c + round(0.55 * n) - 1)
        j1 = lo_c + max(1, round(0.35 * n)) - 1
        k0 = lo_c + round(0.25 * n)
        k1 = max(k0, lo_c + round(0.75 * n) - 1)
        boxes.append((i0, i1, lo_c, j1, k0, k1))
    return boxes


def solid_boxes(dims: Dimz, label: np.ndarray, boxes) -> None:
    lab = label.reshape(dims.nz, dims.ny, dims.nx)
    for i0, i1, j0, j1, k0, k1 in boxes:
        lab[max(k0, 0):k1 + 1, max(j0, 0):j1 + 1, max(i0, 0):i1 + 1] = SOLID


def solid_shell(dims: Dimz, label: np.ndarray) -> None:       # grid.py:110-118
    lab = label.reshape(dims.nz, dims.ny, dims.nx)
    lab[0] = SOLID
    lab[-1] = SOLID
    lab[:, 0] = SOLID
    lab[:, -1] = SOLID
    lab[:, :, 0] = SOLID
    lab[:, :, -1] = SOLID


def seed_region(region: Region, dims: Dimz, rng_seed: int):   # particles.py:133-149
    rho = region.density
    cells = covered_cells(region, dims)
    nsub = rho ** 3
    if len(cells) == 0:
        return [np.zeros(0) for _ in range(6)]
    cells_rep = np.repeat(cells, nsub)
    subs = np.tile(np.arange(nsub, dtype=np.int64), len(cells))
    px, py, pz = jittered_positions(cells_rep, subs, rho, dims, rng_seed)
    z = np.zeros(len(px))
    return [px, py, pz, z, z.copy(), z.copy()]


def jittered_positions(cells, subs, density, dims, rng_seed):
    m = len(cells)
    px, py, pz = np.empty(m), np.empty(m), np.empty(m)
    cells = np.ascontiguousarray(cells, dtype=np.int64)
    subs = np.ascontiguousarray(subs, dtype=np.int64)
    lib().orc_jittered_positions(C.byref(dims.c()), m, _p(cells, _i64), _p(subs, _i64),
                                 int(density), C.c_uint64(int(rng_seed) & (2**64 - 1)),
                                 _p(px), _p(py), _p(pz))
    return px, py, pz


def bin_particles(dims: Dimz, parts):
    n = len(parts[0])
    nc = dims.ncells
    count = np.zeros(nc, dtype=np.int64)
    offset = np.zeros(nc, dtype=np.int64)
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in parts]
    ptrs = (_d * 6)(*[_p(a) for a in arrs])
    scratch = np.empty(max(n, 1))
    cells = np.empty(max(n, 1), dtype=np.int64)
    perm = np.empty(max(n, 1), dtype=np.int64)
    lib().orc_bin_particles(C.byref(dims.c()), n, ptrs, _p(scratch), _p(count, _i64),
                            _p(offset, _i64), _p(cells, _i64), _p(perm, _i64))
    return arrs, count, offset


def classify(state: OState) -> None:
    lib().orc_classify_cells(state.dims.ncells, _p(state.count, _i64), _p(state.label, _u8))


def make_scene(spec: Spec, rng_seed: int = 0) -> OState:      # sim.py:204-223
    if spec.name not in SCENE_NAMES:
        raise ValueError(f"unknown scene {spec.name!r}")
    if spec.solver not in SOLVER_KIND:
        raise ValueError(f"unknown solver {spec.solver!r}")
    dims = Dimz(spec.res, spec.res, spec.res, 1.0 / spec.res)
    u, v, w, p, label = empty_grid(dims)
    solid_shell(dims, label)
    solid_boxes(dims, label, scene_obstacles(spec, dims))
    regions = scene_regions(spec, dims)
    parts = [np.zeros(0) for _ in range(6)]
    for region in regions:
        add = seed_region(region, dims, rng_seed)
        parts = [np.concatenate([a, b]) for a, b in zip(parts, add)]
    spec.density = regions[0].density
    parts, count, offset = bin_particles(dims, parts)
    st = OState(dims, u, v, w, p, label, u.copy(), v.copy(), w.copy(), parts, count, offset,
                rng_seed=rng_seed)
    classify(st)
    return st


# -------------------------------------------------------------- stages ----
def compute_dt(st: OState, spec: Spec) -> float:
    vx, vy, vz = st.parts[3], st.parts[4], st.parts[5]
    return float(lib().orc_compute_dt(st.n, _p(vx), _p(vy), _p(vz), st.dims.dtau,
                                      spec.alpha, spec.dt_max))


def interior_box(st: OState):
    lo, hi = np.empty(3), np.empty(3)
    if lib().orc_interior_box(C.byref(st.dims.c()), _p(st.label, _u8), _p(lo), _p(hi)):
        raise ValueError("grid has no non-solid cells")
    return lo, hi


def advect(st: OState, dt: float, skin: float, scheme: str = "euler") -> None:
    lo, hi = interior_box(st)
    P = st.parts
    if scheme == "rk2":
        lib().orc_advect_rk2(C.byref(st.dims.c()), _p(st.u), _p(st.v), _p(st.w), st.n,
                             _p(P[0]), _p(P[1]), _p(P[2]), dt, _p(lo), _p(hi), skin)
        return
    lib().orc_advect(st.n, _p(P[0]), _p(P[1]), _p(P[2]), _p(P[3]), _p(P[4]), _p(P[5]),
                     dt, _p(lo), _p(hi), skin)


def sample_velocity_many(dims, u, v, w, px, py, pz):
    n = len(px)
    vx, vy, vz = np.empty(n), np.empty(n), np.empty(n)
    px, py, pz = (np.ascontiguousarray(a, dtype=np.float64) for a in (px, py, pz))
    lib().orc_sample_velocity_many(C.byref(dims.c()), _p(u), _p(v), _p(w), n, _p(px), _p(py),
                                   _p(pz), _p(vx), _p(vy), _p(vz))
    return vx, vy, vz


def p2g_component(dims, comp, vel, px, py, pz, offset, count):
    nx, ny, nz = dims.nx, dims.ny, dims.nz
    nf = [(nx + 1) * ny * nz, nx * (ny + 1) * nz, nx * ny * (nz + 1)][comp]
    out, den = np.empty(nf), np.empty(nf)
    lib().orc_p2g_component(C.byref(dims.c()), comp, _p(vel), _p(px), _p(py), _p(pz),
                            _p(offset, _i64), _p(count, _i64), _p(out), _p(den))
    return out, den


def p2g(st: OState):
    P = st.parts
    known = []
    for comp, dst in ((0, st.u), (1, st.v), (2, st.w)):
        vals, den = p2g_component(st.dims, comp, P[3 + comp], P[0], P[1], P[2], st.offset,
                                  st.count)
        dst[:] = vals
        known.append((den > 0.0).astype(np.uint8))
    return known


def body_force(st: OState, g, dt: float) -> None:
    gg = np.asarray(g, dtype=np.float64)
    lib().orc_add_body_force(C.byref(st.dims.c()), _p(st.u), _p(st.v), _p(st.w), _p(gg), dt)


def enforce(dims, label, u, v, w) -> None:
    lib().orc_enforce_solid_boundaries(C.byref(dims.c()), _p(label, _u8), _p(u), _p(v), _p(w))


@dataclass
class System:
    cells: np.ndarray
    row_of: np.ndarray
    diag: np.ndarray
    nbr_rows: np.ndarray
    rhs: np.ndarray
    scale: float
    pinned: np.ndarray
    red_rows: np.ndarray
    black_rows: np.ndarray

    @property
    def nrows(self):
        return len(self.cells)


def assemble(dims: Dimz, label, u, v, w, dt: float, rho: float) -> System:
    nc = dims.ncells
    row_of = np.empty(nc, dtype=np.int64)
    cells = np.empty(nc, dtype=np.int64)
    diag = np.empty(nc)
    nbr = np.empty(nc * 6, dtype=np.int64)
    rhs = np.empty(nc)
    pinned = np.empty(nc, dtype=np.int64)
    npin = C.c_int64(0)
    n = lib().orc_assemble(C.byref(dims.c()), _p(label, _u8), _p(u), _p(v), _p(w),
                           _p(row_of, _i64), _p(cells, _i64), _p(diag), _p(nbr, _i64), _p(rhs),
                           _p(pinned, _i64), C.byref(npin))
    cells = cells[:n].copy()
    i = cells % dims.nx
    j = (cells // dims.nx) % dims.ny
    k = cells // (dims.nx * dims.ny)
    parity = (i + j + k) & 1
    return System(cells, row_of, diag[:n].copy(), nbr[:n * 6].reshape(n, 6).copy(),
                  rhs[:n].copy(), dt / (rho * dims.dtau ** 2), pinned[:npin.value].copy(),
                  np.flatnonzero(parity == 0).astype(np.int64),
                  np.flatnonzero(parity == 1).astype(np.int64))


class OracleSolverError(Exception):
    def __init__(self, kind, msg, cell=None):
        super().__init__(msg)
        self.kind = kind
        self.cell = cell


def solve(sys: System, solver: str, max_iters: int, tol: float, precond: str = "mic0"):
    n = sys.nrows
    x = np.zeros(max(n, 1))
    hist = np.zeros(max(max_iters, 1))
    res = SolveRes()
    nbr = np.ascontiguousarray(sys.nbr_rows.reshape(-1), dtype=np.int64)
    if nbr.size == 0:
        nbr = np.zeros(6, dtype=np.int64)
    red = sys.red_rows if len(sys.red_rows) else np.zeros(1, dtype=np.int64)
    black = sys.black_rows if len(sys.black_rows) else np.zeros(1, dtype=np.int64)
    cells = sys.cells if n else np.zeros(1, dtype=np.int64)
    diag = sys.diag if n else np.zeros(1)
    rhs = sys.rhs if n else np.zeros(1)
    rc = lib().orc_solve(SOLVER_KIND[solver], PRECOND[precond], n, _p(cells, _i64), _p(diag),
                         _p(nbr, _i64), _p(rhs), sys.scale, max_iters, tol, _p(red, _i64),
                         len(sys.red_rows), _p(black, _i64), len(sys.black_rows), _p(x),
                         _p(hist), C.byref(res))
    if rc == 1:
        raise OracleSolverError("singular", f"zero diagonal at cell {res.err_cell}",
                                res.err_cell)
    if rc == 2:
        raise OracleSolverError("breakdown", f"curvature {res.err_value:.3e} at iteration "
                                f"{res.err_it}")
    it = res.iterations
    return dict(p=x[:n].copy(), iterations=int(it), residual=float(res.residual),
                converged=bool(res.converged), history=hist[:min(it, max_iters)].copy())


def pressure_field(sys: System, x, ncells):
    p = np.zeros(ncells)
    p[sys.cells] = x
    return p


def apply_gradient(st: OState, p, dt, rho) -> None:
    lib().orc_apply_pressure_gradient(C.byref(st.dims.c()), _p(st.label, _u8), _p(p), dt, rho,
                                      _p(st.u), _p(st.v), _p(st.w))


def extrapolate(dims, u, v, w, known, layers):
    nx, ny, nz = dims.nx, dims.ny, dims.nz
    shapes = [(nx + 1, ny, nz), (nx, ny + 1, nz), (nx, ny, nz + 1)]
    for arr, kn, (mx, my, mz) in zip((u, v, w), known, shapes):
        k = kn.astype(np.uint8).copy()
        n = mx * my * mz
        lib().orc_extrapolate_component(mx, my, mz, _p(arr), _p(k, _u8), int(layers),
                                        _p(np.empty(n)), _p(np.zeros(n, dtype=np.int64), _i64),
                                        _p(np.empty(n, dtype=np.uint8), _u8))


def g2p(st: OState, flip: float) -> None:
    P = st.parts
    lib().orc_g2p(C.byref(st.dims.c()), _p(st.u), _p(st.v), _p(st.w), _p(st.uo), _p(st.vo),
                  _p(st.wo), st.n, _p(P[0]), _p(P[1]), _p(P[2]), _p(P[3]), _p(P[4]), _p(P[5]),
                  float(flip))


def derive_seed(base: int, stream: int) -> int:
    return int(lib().orc_derive_seed(C.c_uint64(base & (2**64 - 1)),
                                     C.c_uint64(stream & (2**64 - 1))))


def reseed(st: OState, density: int, seed: int) -> None:
    nc = st.dims.ncells
    n_add = np.empty(nc, dtype=np.int64)
    new_count = np.empty(nc, dtype=np.int64)
    new_offset = np.empty(nc, dtype=np.int64)
    total = lib().orc_reseed_counts(nc, _p(st.count, _i64), _p(st.label, _u8), int(density),
                                    _p(n_add, _i64), _p(new_count, _i64), _p(new_offset, _i64))
    out = [np.zeros(total) for _ in range(6)]
    src = [np.ascontiguousarray(a) for a in st.parts]
    pin = (_d * 6)(*[_p(a) for a in src])
    pout = (_d * 6)(*[_p(a) if total else _p(np.zeros(1)) for a in out])
    lib().orc_reseed_fill(C.byref(st.dims.c()), nc, _p(st.count, _i64), _p(st.offset, _i64),
                          _p(n_add, _i64), _p(new_offset, _i64), int(density),
                          C.c_uint64(seed & (2**64 - 1)), pin, pout, _p(st.u), _p(st.v),
                          _p(st.w))
    st.parts = out
    st.count = new_count
    st.offset = new_offset


def divergence_field(dims, u, v, w):
    out = np.empty(dims.ncells)
    lib().orc_divergence_field(C.byref(dims.c()), _p(u), _p(v), _p(w), _p(out))
    return out


# ----------------------------------------------------------------- step ---
def step(st: OState, spec: Spec, hook=None) -> dict:
    """Restates sim.py:226-300.  `hook(stage_name, state, extras)` is called
    after each stage (for per-stage parity checks)."""
    t = {}
    clock = time.perf_counter

    def mark(name, t0, **extra):
        t[name] = (clock() - t0) * 1e3
        if hook is not None:
            hook(name, st, extra)

    t0 = clock()
    dt = compute_dt(st, spec)
    mark("dt_compute", t0, dt=dt)

    t0 = clock()
    advect(st, dt, spec.skin_fraction * st.dims.dtau, spec.advection)
    mark("advect", t0)

    t0 = clock()
    st.parts, st.count, st.offset = bin_particles(st.dims, st.parts)
    mark("bin", t0)

    t0 = clock()
    classify(st)
    mark("classify", t0)

    t0 = clock()
    known = p2g(st)
    st.uo[:] = st.u
    st.vo[:] = st.v
    st.wo[:] = st.w
    mark("p2g", t0, known=known)

    t0 = clock()
    body_force(st, spec.gravity, dt)
    enforce(st.dims, st.label, st.u, st.v, st.w)
    mark("force", t0)

    t0 = clock()
    sys = assemble(st.dims, st.label, st.u, st.v, st.w, dt, spec.rho_fluid)
    try:
        result = solve(sys, spec.solver, spec.resolved_max_iters(), spec.tol, spec.precond)
    except OracleSolverError as exc:
        raise OracleSolverError(exc.kind, f"step {st.step_count}: {exc}", exc.cell) from exc
    mark("project", t0, system=sys, result=result)

    t0 = clock()
    st.p[:] = pressure_field(sys, result["p"], st.dims.ncells)
    apply_gradient(st, st.p, dt, spec.rho_fluid)
    extrapolate(st.dims, st.u, st.v, st.w, known, spec.extrapolation_layers)
    extrapolate(st.dims, st.uo, st.vo, st.wo, known, spec.extrapolation_layers)
    enforce(st.dims, st.label, st.u, st.v, st.w)
    mark("apply_gradient", t0)

    t0 = clock()
    g2p(st, spec.flip_fraction)
    mark("g2p", t0)

    t0 = clock()
    reseed(st, spec.density, derive_seed(st.rng_seed, st.step_count + 1))
    mark("reseed", t0)

    st.time += dt
    st.step_count += 1
    return dict(timings=t, dt=dt, particle_count=st.n, solver_iterations=result["iterations"],
                solver_residual=result["residual"], solver_converged=result["converged"])
