"""Particle set view, seed regions and the reseeding constants.

The particle state is structure-of-arrays float64 in HBM (double-buffered
by the C library, like ParticleSet.reorder's spare buffer,
flipsim/particles.py:13-64).  ``ParticleSet`` is either a read-only view of
a device context or a plain host container (for callers that build sets by
hand, e.g. total_energy on host data).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

# Bridson's bounds on particles per FLUID cell (flipsim/particles.py:151-152)
MIN_PER_CELL = 3
MAX_PER_CELL = 12

_NAMES = ("pos_x", "pos_y", "pos_z", "vel_x", "vel_y", "vel_z")


class ParticleSet:
    """pos_x..vel_z float64 arrays of one length."""

    def __init__(self, *arrays, device=None):
        self._dev = device
        if device is None:
            if len(arrays) != 6:
                raise TypeError("ParticleSet needs six arrays")
            self._host = tuple(np.asarray(a, dtype=np.float64) for a in arrays)
            if len({len(a) for a in self._host}) != 1:
                raise ValueError("particle arrays must share one length")
        else:
            self._host = None

    @classmethod
    def empty(cls) -> "ParticleSet":
        return cls(*(np.zeros(0) for _ in range(6)))

    def arrays(self):
        return self._dev.particles() if self._dev is not None else self._host

    @property
    def count(self) -> int:
        return self._dev.count() if self._dev is not None else len(self._host[0])

    def copy(self) -> "ParticleSet":
        return ParticleSet(*(np.array(a) for a in self.arrays()))

    def extend(self, other: "ParticleSet") -> "ParticleSet":
        return ParticleSet(*(np.concatenate([a, b]) for a, b in zip(self.arrays(), other.arrays())))


for _i, _n in enumerate(_NAMES):
    setattr(ParticleSet, _n, property(lambda self, i=_i: self.arrays()[i]))


@dataclass(frozen=True)
class SeedRegion:
    """Box [a, b] or sphere (center a, radius b) with `density` subcells per
    axis per covered cell (flipsim/particles.py:67-100)."""

    kind: str
    a: tuple
    b: object
    density: int = 2

    def __post_init__(self):
        if self.kind not in ("box", "sphere"):
            raise ValueError(f"unknown region kind {self.kind!r}")
        if self.density < 1:
            raise ValueError("seed density must be >= 1")

    @classmethod
    def box(cls, lo, hi, density: int = 2) -> "SeedRegion":
        return cls("box", tuple(map(float, lo)), tuple(map(float, hi)), density)

    @classmethod
    def sphere(cls, center, radius: float, density: int = 2) -> "SeedRegion":
        return cls("sphere", tuple(map(float, center)), float(radius), density)

    def contains(self, px, py, pz) -> np.ndarray:
        if self.kind == "box":
            lo, hi = self.a, self.b
            return ((px >= lo[0]) & (px <= hi[0]) & (py >= lo[1]) & (py <= hi[1])
                    & (pz >= lo[2]) & (pz <= hi[2]))
        cx, cy, cz = self.a
        return ((px - cx) ** 2 + (py - cy) ** 2 + (pz - cz) ** 2) <= self.b * self.b

    def to_c(self):
        from ._lib import Region
        r = Region()
        r.kind = 0 if self.kind == "box" else 1
        r.density = int(self.density)
        r.a[:] = [float(x) for x in self.a]
        if self.kind == "box":
            r.b[:] = [float(x) for x in self.b]
            r.radius = 0.0
        else:
            r.b[:] = [0.0, 0.0, 0.0]
            r.radius = float(self.b)
        return r


def covered_cells(region: SeedRegion, dims) -> np.ndarray:
    """Cells whose center lies in the region (flipsim/particles.py:103-110).

    Host helper used only by scene sizing (particle_target); seeding itself
    evaluates the same predicate on the device.
    """
    idx = np.arange(dims.ncells, dtype=np.int64)
    ox, oy, oz = dims.origin
    cx = ox + (idx % dims.nx + 0.5) * dims.dtau
    cy = oy + ((idx // dims.nx) % dims.ny + 0.5) * dims.dtau
    cz = oz + (idx // (dims.nx * dims.ny) + 0.5) * dims.dtau
    return idx[region.contains(cx, cy, cz)]
