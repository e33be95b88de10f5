"""Pressure solves on an assembled system (flipsim/pressure.py:200-340).

Inside ``step`` assembly and the solve run fused on the device (stage
PROJECT).  ``solve`` exposes the same solvers for a system assembled
elsewhere (any object with the LaplacianSystem fields cells, diag, nbr_rows,
rhs, scale, red_rows, black_rows), e.g. for the pressure-only benchmark.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import LIB, ptr
from .errors import SingularSystemError, SolverBreakdownError

SOLVERS = ("jacobi", "gs", "rbgs", "pcg")


@dataclass
class SolveResult:
    p: np.ndarray
    iterations: int
    residual: float
    converged: bool


def solve(system, solver: str = "pcg", max_iters: int | None = None, tol: float = 1e-6,
          precond: str = "mic0") -> SolveResult:
    """SOLVERS[solver](system, max_iters, tol) on the device."""
    if solver not in SOLVERS:
        raise KeyError(solver)
    if precond not in _lib.PRECOND_ID:
        raise ValueError(f"unknown preconditioner {precond!r}")
    if max_iters is None:
        max_iters = 100 if solver == "pcg" else 2000
    cells = np.ascontiguousarray(system.cells, dtype=np.int64)
    n = len(cells)
    diag = np.ascontiguousarray(system.diag, dtype=np.float64)
    nbr = np.ascontiguousarray(system.nbr_rows, dtype=np.int64).reshape(-1)
    rhs = np.ascontiguousarray(system.rhs, dtype=np.float64)
    red = np.ascontiguousarray(getattr(system, "red_rows", np.zeros(0)), dtype=np.int64)
    black = np.ascontiguousarray(getattr(system, "black_rows", np.zeros(0)), dtype=np.int64)
    x = np.zeros(max(n, 1))
    it, cv = C.c_int64(0), C.c_int32(0)
    res, ev = C.c_double(0.0), C.c_double(0.0)
    ec, ei = C.c_int64(-1), C.c_int64(0)
    one = np.zeros(1, dtype=np.int64)
    rc = LIB.flip_solve_system(
        _lib.SOLVER_ID[solver], _lib.PRECOND_ID[precond], n, ptr(cells if n else one, _lib._i64),
        ptr(diag if n else np.zeros(1)), ptr(nbr if n else np.zeros(6, dtype=np.int64), _lib._i64),
        ptr(rhs if n else np.zeros(1)), float(system.scale), int(max_iters), float(tol),
        ptr(red if len(red) else one, _lib._i64), len(red),
        ptr(black if len(black) else one, _lib._i64), len(black), ptr(x), C.byref(it),
        C.byref(res), C.byref(cv), C.byref(ec), C.byref(ei), C.byref(ev))
    if rc == _lib.FLIP_E_SINGULAR:
        raise SingularSystemError(int(ec.value))
    if rc == _lib.FLIP_E_BREAKDOWN:
        raise SolverBreakdownError(f"conjugate-gradient breakdown: curvature {ev.value:.3e} "
                                   f"at iteration {int(ei.value)}")
    _lib.check(rc, "flip_solve_system")
    return SolveResult(x[:n].copy(), int(it.value), float(res.value), bool(cv.value))
