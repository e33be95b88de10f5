"""Data formats on either side of the step: FLIP v1 particle
snapshots (flipsim/io.py:1-75), flat key = value configs, and the CSV
column contracts of the reference CLI's timing and bench outputs
(flipsim/cli.py:31-35, 253-292).

Snapshots of device-resident state are converted on the GPU: the float64
particle arrays narrow to float32 with round-to-nearest-even (numpy's
``astype('<f4')``) in one kernel, so the host copy is 24 instead of 48 bytes
per particle.  Reading widens exactly.  Files are byte-identical to the
reference's ``write_snapshot`` (tests/test_formats.py).
"""

from __future__ import annotations

import csv
import ctypes as C
import struct

import numpy as np

from ._lib import LIB, check
from .errors import SnapshotFormatError
from .particles import ParticleSet
from .sim import StageTimings

MAGIC = b"FLIP"
VERSION = 1

TIMINGS_COLUMNS = ("step", "dt", "particles", "solver_iters", "solver_residual") + tuple(
    f"{name}_ms" for name in StageTimings.stage_names()) + ("total_ms",)      # cli.py:31-33
ENERGY_COLUMNS = ("step", "sim_time", "kinetic_and_potential")              # cli.py:34
BENCH_COLUMNS = ("scene", "res", "particles", "stage", "ms")                # cli.py:35


def _header(n: int) -> bytes:
    return MAGIC + struct.pack("<I", VERSION) + struct.pack("<Q", int(n))


def write_snapshot(path, particles) -> None:
    """io.py:23-30.  ``particles``: a device-backed ParticleSet (state.particles:
    converted on the GPU) or anything with ``arrays()``/``count`` on the host."""
    dev = getattr(particles, "_dev", None)
    n = int(particles.count)
    if dev is not None:
        buf = np.empty(6 * max(n, 1), dtype="<f4")
        check(LIB.flip_get_particles_f32(dev.ctx, buf.ctypes.data_as(C.POINTER(C.c_float))),
              "flip_get_particles_f32")
        payload = buf[:6 * n].tobytes()
    else:
        payload = b"".join(np.asarray(a).astype("<f4").tobytes() for a in particles.arrays())
    with open(path, "wb") as fh:
        fh.write(_header(n))
        fh.write(payload)


def _parse(path, data: bytes) -> tuple:
    if data[:4] != MAGIC:
        raise SnapshotFormatError(path, 0, "bad magic")
    if len(data) < 16:
        raise SnapshotFormatError(path, len(data), "truncated header")
    (version,) = struct.unpack_from("<I", data, 4)
    if version != VERSION:
        raise SnapshotFormatError(path, 4, f"unsupported version {version}")
    (count,) = struct.unpack_from("<Q", data, 8)
    need = 16 + 6 * 4 * count
    if len(data) != need:
        raise SnapshotFormatError(path, min(len(data), need),
                                  f"expected {need} bytes for {count} particles, got {len(data)}")
    return count, np.frombuffer(data, dtype="<f4", count=6 * count, offset=16)


def read_snapshot(path) -> ParticleSet:
    """io.py:33-55: a host ParticleSet (float64), same errors as the reference."""
    with open(path, "rb") as fh:
        data = fh.read()
    count, f32 = _parse(path, data)
    arrays = [f32[a * count:(a + 1) * count].astype(np.float64) for a in range(6)]
    return ParticleSet(*arrays)


def load_snapshot_to_device(path, state) -> int:
    """Replace ``state``'s particles with a snapshot, widened on the GPU.
    The set is unbinned afterwards (run the bin stage, as after
    flip_set_particles)."""
    with open(path, "rb") as fh:
        data = fh.read()
    count, f32 = _parse(path, data)
    buf = np.ascontiguousarray(f32)
    dev = state.device
    check(LIB.flip_set_particles_f32(dev.ctx, int(count),
                                     buf.ctypes.data_as(C.POINTER(C.c_float))),
          "flip_set_particles_f32")
    dev.bump()
    return int(count)


def parse_config(text: str) -> dict:
    """io.py:58-69: flat ``key = value`` lines, '#' comments, blanks ignored."""
    out: dict = {}
    for lineno, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ValueError(f"line {lineno}: expected 'key = value', got {raw!r}")
        key, value = line.split("=", 1)
        out[key.strip()] = value.strip()
    return out


def format_config(values: dict) -> str:
    """io.py:72-73."""
    return "".join(f"{k} = {v}\n" for k, v in values.items())


def timings_row(step: int, report) -> tuple:
    """One TIMINGS_COLUMNS row for a StepReport (cli.py's per-step CSV)."""
    t = report.timings
    return ((step, report.dt, report.particle_count, report.solver_iterations,
             report.solver_residual)
            + tuple(getattr(t, n) for n in StageTimings.stage_names()) + (t.total(),))


def write_csv(path, columns, rows) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(columns)
        w.writerows(rows)


def bench_rows(name: str, res: int, target, stage_ms: dict) -> list:
    """cli.py:262-281: one (scene, res, particles, stage, ms) row per stage
    with the mean over the run's steps, formatted as the reference does."""
    return [(name, res, target, n, f"{np.mean(stage_ms[n]):.3f}")
            for n in StageTimings.stage_names()]
