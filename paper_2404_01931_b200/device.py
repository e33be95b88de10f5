"""Owner of one device context (``flip_ctx``) plus lazily downloaded views.

All simulation state lives in HBM inside the C library's context; the views
handed out by ``MacGrid`` / ``ParticleSet`` / ``SpaceHash`` are read-only
NumPy copies fetched on first access after each mutation (``version``
bump).  Writing goes through explicit setters that upload, so host copies can
never silently diverge from the device state.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import LIB, check, ptr


def _ro(a: np.ndarray) -> np.ndarray:
    a.flags.writeable = False
    return a


class Device:
    """One ``flip_ctx``: grid + grid_old velocities, particles, hash, solver."""

    def __init__(self, dims, capacity: int = 0, device: int = 0):
        self.dims = dims
        ctx = C.c_void_p()
        origin = (C.c_double * 3)(*[float(x) for x in dims.origin])
        check(LIB.flip_create(int(device), dims.nx, dims.ny, dims.nz, float(dims.dtau), origin,
                              int(capacity), C.byref(ctx)), "flip_create")
        self.ctx = ctx
        self.device = device
        self.version = 0
        self._cache: dict = {}
        nx, ny, nz = dims.nx, dims.ny, dims.nz
        self.nfaces = ((nx + 1) * ny * nz, nx * (ny + 1) * nz, nx * ny * (nz + 1))

    # -- lifecycle ---------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "ctx", None):
            LIB.flip_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bump(self) -> None:
        self.version += 1
        self._cache.clear()

    def stream_ptr(self) -> int:
        sp = C.c_void_p()
        check(LIB.flip_get_stream(self.ctx, C.byref(sp)))
        return int(sp.value or 0)

    # -- grid --------------------------------------------------------------
    def grid_array(self, name: str) -> np.ndarray:
        key = ("grid", name)
        if key not in self._cache:
            nc = self.dims.ncells
            size = {"u": self.nfaces[0], "v": self.nfaces[1], "w": self.nfaces[2], "p": nc,
                    "label": nc}[name]
            out = np.empty(size, dtype=np.uint8 if name == "label" else np.float64)
            args = [None] * 5
            args[("u", "v", "w", "p", "label").index(name)] = ptr(
                out, _lib._u8 if name == "label" else _lib._d)
            check(LIB.flip_get_grid(self.ctx, *args), "flip_get_grid")
            self._cache[key] = _ro(out)
        return self._cache[key]

    def set_grid(self, **arrays) -> None:
        args = []
        for name in ("u", "v", "w", "p", "label"):
            a = arrays.get(name)
            if a is None:
                args.append(None)
                continue
            dt = np.uint8 if name == "label" else np.float64
            a = np.ascontiguousarray(a, dtype=dt)
            exp = {"u": self.nfaces[0], "v": self.nfaces[1], "w": self.nfaces[2],
                   "p": self.dims.ncells, "label": self.dims.ncells}[name]
            if a.size != exp:
                raise ValueError(f"{name} needs {exp} values, got {a.size}")
            arrays[name] = a
            args.append(ptr(a, _lib._u8 if name == "label" else _lib._d))
        check(LIB.flip_set_grid(self.ctx, *args), "flip_set_grid")
        self.bump()

    def old_array(self, name: str) -> np.ndarray:
        key = ("old", name)
        if key not in self._cache:
            out = np.empty(self.nfaces["uvw".index(name)])
            args = [None] * 3
            args["uvw".index(name)] = ptr(out)
            check(LIB.flip_get_grid_old(self.ctx, *args), "flip_get_grid_old")
            self._cache[key] = _ro(out)
        return self._cache[key]

    def set_grid_old(self, u=None, v=None, w=None) -> None:
        arrs = [None if a is None else np.ascontiguousarray(a, dtype=np.float64) for a in (u, v, w)]
        for a, n in zip(arrs, self.nfaces):
            if a is not None and a.size != n:
                raise ValueError("grid_old array has the wrong length")
        check(LIB.flip_set_grid_old(self.ctx, *[ptr(a) for a in arrs]), "flip_set_grid_old")
        self.bump()

    # -- particles ---------------------------------------------------------
    def count(self) -> int:
        n = C.c_int64(0)
        check(LIB.flip_particle_count(self.ctx, C.byref(n)))
        return int(n.value)

    def particles(self):
        if "parts" not in self._cache:
            n = self.count()
            arrs = [np.empty(n) for _ in range(6)]
            check(LIB.flip_get_particles(self.ctx, *[ptr(a) for a in arrs]), "flip_get_particles")
            self._cache["parts"] = tuple(_ro(a) for a in arrs)
        return self._cache["parts"]

    def set_particles(self, arrays) -> None:
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in arrays]
        n = len(arrs[0])
        if any(len(a) != n for a in arrs):
            raise ValueError("particle arrays must share one length")
        check(LIB.flip_set_particles(self.ctx, n, *[ptr(a) for a in arrs]), "flip_set_particles")
        self.bump()

    # -- hash --------------------------------------------------------------
    def hash_arrays(self):
        if "hash" not in self._cache:
            nc = self.dims.ncells
            off = np.empty(nc, dtype=np.int64)
            cnt = np.empty(nc, dtype=np.int64)
            check(LIB.flip_get_hash(self.ctx, ptr(off, _lib._i64), ptr(cnt, _lib._i64)))
            self._cache["hash"] = (_ro(off), _ro(cnt))
        return self._cache["hash"]

    def set_hash(self, offset, count) -> None:
        off = np.ascontiguousarray(offset, dtype=np.int64)
        cnt = np.ascontiguousarray(count, dtype=np.int64)
        if off.size != self.dims.ncells or cnt.size != self.dims.ncells:
            raise ValueError("hash arrays need one entry per cell")
        check(LIB.flip_set_hash(self.ctx, ptr(off, _lib._i64), ptr(cnt, _lib._i64)))
        self.bump()

    def fluid_cells(self) -> np.ndarray:
        if "fluid" not in self._cache:
            out = np.empty(self.dims.ncells, dtype=np.int64)
            m = C.c_int64(0)
            check(LIB.flip_get_fluid_cells(self.ctx, ptr(out, _lib._i64), C.byref(m)))
            self._cache["fluid"] = _ro(out[:m.value].copy())
        return self._cache["fluid"]

    # -- inter-stage data --------------------------------------------------
    def dt(self) -> float:
        v = C.c_double(0.0)
        check(LIB.flip_get_dt(self.ctx, C.byref(v)))
        return float(v.value)

    def set_dt(self, dt: float) -> None:
        check(LIB.flip_set_dt(self.ctx, float(dt)))
        self.bump()

    def known(self):
        out = [np.empty(n, dtype=np.uint8) for n in self.nfaces]
        check(LIB.flip_get_known(self.ctx, *[ptr(a, _lib._u8) for a in out]))
        return tuple(a.astype(bool) for a in out)

    def set_known(self, ku, kv, kw) -> None:
        arrs = [np.ascontiguousarray(a, dtype=np.uint8) for a in (ku, kv, kw)]
        check(LIB.flip_set_known(self.ctx, *[ptr(a, _lib._u8) for a in arrs]))
        self.bump()

    # -- stages ------------------------------------------------------------
    def run_stages(self, params, first: int, last: int):
        rep = _lib.StepReportC()
        rc = LIB.flip_run_stages(self.ctx, C.byref(params), int(first), int(last), C.byref(rep))
        self.bump()
        return rc, rep

    def debug_buffer(self, name: str, count: int, dtype=np.float64) -> np.ndarray:
        out = np.empty(count, dtype=dtype)
        check(LIB.flip_debug_copy(self.ctx, name.encode(), out.ctypes.data_as(C.c_void_p),
                                  out.nbytes))
        return out

    def divergence_field(self) -> np.ndarray:
        out = np.empty(self.dims.ncells)
        check(LIB.flip_divergence_field(self.ctx, ptr(out)))
        return out

    def energy_sums(self, floor_y: float):
        ke, pe = C.c_double(0.0), C.c_double(0.0)
        check(LIB.flip_energy_sums(self.ctx, float(floor_y), C.byref(ke), C.byref(pe)))
        return float(ke.value), float(pe.value)
