"""MAC grid dimensions, labels and the device-backed grid view.

Layout matches the reference exactly (flipsim/grid.py:62-93): flat x-fastest
arrays, u (nx+1)*ny*nz, v nx*(ny+1)*nz, w nx*ny*(nz+1), p and label nx*ny*nz,
3-D views indexed [k, j, i].  The arrays themselves live in HBM; attribute
reads return read-only host copies, assignments upload.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SOLID = 0
FLUID = 1
AIR = 2


@dataclass(frozen=True)
class GridDims:
    """Cells per axis, cell edge length and world position of the min corner."""

    nx: int
    ny: int
    nz: int
    dtau: float
    origin: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise ValueError("grid needs at least one cell per axis")
        if not self.dtau > 0:
            raise ValueError("cell size must be positive")

    @property
    def ncells(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def shape(self) -> tuple:
        return (self.nx, self.ny, self.nz)


def flat_index(i: int, j: int, k: int, dims: GridDims) -> int:
    """x-fastest flat cell index (flipsim/grid.py:47-50)."""
    assert 0 <= i < dims.nx and 0 <= j < dims.ny and 0 <= k < dims.nz, (i, j, k)
    return i + dims.nx * (j + dims.ny * k)


def cell_coords(index: int, dims: GridDims) -> tuple:
    """Inverse of flat_index (flipsim/grid.py:53-59)."""
    assert 0 <= index < dims.ncells, index
    k, rem = divmod(index, dims.nx * dims.ny)
    j, i = divmod(rem, dims.nx)
    return i, j, k


class MacGrid:
    """Device-resident MAC grid (``which`` = "grid" or "old").

    grid_old only ever receives velocities from the step
    (copy_velocities_from, flipsim/grid.py:104-107); its p and label are the
    snapshot taken when it was cloned in make_scene, kept on the host.
    """

    def __init__(self, device, which: str = "grid", old_p=None, old_label=None):
        self._dev = device
        self._which = which
        self.dims = device.dims
        self._old_p = old_p
        self._old_label = old_label

    def _get(self, name):
        if self._which == "grid":
            return self._dev.grid_array(name)
        if name in ("u", "v", "w"):
            return self._dev.old_array(name)
        return self._old_p if name == "p" else self._old_label

    def _set(self, name, value):
        if self._which == "grid":
            self._dev.set_grid(**{name: value})
        elif name in ("u", "v", "w"):
            self._dev.set_grid_old(**{name: value})
        else:
            arr = np.array(value, dtype=np.uint8 if name == "label" else np.float64)
            arr.flags.writeable = False
            if name == "p":
                self._old_p = arr
            else:
                self._old_label = arr

    u = property(lambda s: s._get("u"), lambda s, a: s._set("u", a))
    v = property(lambda s: s._get("v"), lambda s, a: s._set("v", a))
    w = property(lambda s: s._get("w"), lambda s, a: s._set("w", a))
    p = property(lambda s: s._get("p"), lambda s, a: s._set("p", a))
    label = property(lambda s: s._get("label"), lambda s, a: s._set("label", a))

    def u3(self):
        d = self.dims
        return self.u.reshape(d.nz, d.ny, d.nx + 1)

    def v3(self):
        d = self.dims
        return self.v.reshape(d.nz, d.ny + 1, d.nx)

    def w3(self):
        d = self.dims
        return self.w.reshape(d.nz + 1, d.ny, d.nx)

    def p3(self):
        d = self.dims
        return self.p.reshape(d.nz, d.ny, d.nx)

    def label3(self):
        d = self.dims
        return self.label.reshape(d.nz, d.ny, d.nx)

    def to_host(self) -> dict:
        """Writable host copies of every field."""
        return {k: np.array(getattr(self, k)) for k in ("u", "v", "w", "p", "label")}


def interior_box_from_labels(label: np.ndarray, dims: GridDims):
    """Bounding box of non-SOLID cells in world units (flipsim/grid.py:121-132).

    Host helper for callers holding labels; the step computes it on device.
    """
    lab = np.asarray(label).reshape(dims.nz, dims.ny, dims.nx)
    ks, js, is_ = np.nonzero(lab != SOLID)
    if len(is_) == 0:
        raise ValueError("grid has no non-solid cells")
    o = np.asarray(dims.origin, dtype=np.float64)
    lo = o + np.array([is_.min(), js.min(), ks.min()]) * dims.dtau
    hi = o + (np.array([is_.max(), js.max(), ks.max()]) + 1) * dims.dtau
    return lo, hi
