"""Counter-based RNG (flipsim/rng.py:19-41).

Particle jitter is drawn on the device (common.cuh ``uniform01``); the host
only forks per-step seeds with ``derive_seed`` (sim.py:291).  ``uniform01``
is provided for host-side checks and is bit-identical to the device draw.
"""

from __future__ import annotations

import numpy as np

GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1


def _finalize(z: int) -> int:
    z = ((z ^ (z >> 30)) * MIX1) & MASK64
    z = ((z ^ (z >> 27)) * MIX2) & MASK64
    return z ^ (z >> 31)


def derive_seed(base: int, stream: int) -> int:
    """Fork a 64-bit seed from (base, stream)."""
    return _finalize((base + (stream + 1) * GOLDEN) & MASK64)


def uniform01(seed: int, stream, lane) -> np.ndarray:
    """U[0,1) draw per (stream, lane); lane < 2**20."""
    s = np.asarray(stream, dtype=np.uint64)
    ln = np.asarray(lane, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & MASK64) + ((s << np.uint64(20)) + ln + np.uint64(1)) * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
