"""``cuda`` backend: the reference kernel signatures on sm_100a.

Signatures, argument meaning, return conventions and in-place semantics
follow flipsim/_kernels/_core.pyx (cited per function).  ``workers`` is
accepted and ignored.  Arrays are coerced to C-contiguous float64 / int64
like the Cython memoryviews require.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from .. import _lib
from .._lib import LIB, check, ptr

_d, _i64 = _lib._d, _lib._i64


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _nbr(nbr_rows, n):
    nb = _i(nbr_rows).reshape(-1)
    if nb.size != 6 * n:
        raise ValueError("nbr_rows must have shape (n, 6)")
    return nb


def sample_velocity_many(u, v, w, nx, ny, nz, dtau, ox, oy, oz, px, py, pz, workers=1):
    """_core.pyx:68-90 — trilinear staggered samples at each position."""
    px, py, pz = _f64(px), _f64(py), _f64(pz)
    n = len(px)
    out = [np.empty(n) for _ in range(3)]
    check(LIB.flip_k_sample_velocity_many(ptr(_f64(u)), ptr(_f64(v)), ptr(_f64(w)), nx, ny, nz,
                                          dtau, ox, oy, oz, n, ptr(px), ptr(py), ptr(pz),
                                          *[ptr(a) for a in out]))
    return tuple(out)


def p2g_component(comp, vel_p, px, py, pz, offset, count, nx, ny, nz, dtau, ox, oy, oz,
                  workers=1):
    """_core.pyx:93-176 — per-face Kahan gather; returns (values, weights)."""
    vel_p, px, py, pz = _f64(vel_p), _f64(px), _f64(py), _f64(pz)
    off, cnt = _i(offset), _i(count)
    nf = [(nx + 1) * ny * nz, nx * (ny + 1) * nz, nx * ny * (nz + 1)][comp]
    vals, wts = np.empty(nf), np.empty(nf)
    check(LIB.flip_k_p2g_component(int(comp), len(px), ptr(vel_p), ptr(px), ptr(py), ptr(pz),
                                   ptr(off, _i64), ptr(cnt, _i64), nx, ny, nz, dtau, ox, oy, oz,
                                   ptr(vals), ptr(wts)))
    return vals, wts


def counting_sort_perm(cells, offset, workers=1):
    """_core.pyx:179-193 — stable permutation ordering particles by cell."""
    cells, off = _i(cells), _i(offset)
    perm = np.empty(len(cells), dtype=np.int64)
    check(LIB.flip_k_counting_sort_perm(len(cells), ptr(cells, _i64), len(off), ptr(off, _i64),
                                        ptr(perm, _i64)))
    return perm


def laplacian_matvec(diag, nbr_rows, x, scale, workers=1):
    """_core.pyx:196-213 — y = scale * (diag*x - sum of neighbour x)."""
    diag, x = _f64(diag), _f64(x)
    n = len(diag)
    y = np.empty(n)
    check(LIB.flip_k_laplacian_matvec(n, ptr(diag), ptr(_nbr(nbr_rows, n), _i64), ptr(x),
                                      float(scale), ptr(y)))
    return y


def jacobi_iter(diag, nbr_rows, rhs, x, scale, workers=1):
    """_core.pyx:216-234 — one Jacobi sweep (out of place)."""
    diag, rhs, x = _f64(diag), _f64(rhs), _f64(x)
    n = len(diag)
    out = np.empty(n)
    check(LIB.flip_k_jacobi_iter(n, ptr(diag), ptr(_nbr(nbr_rows, n), _i64), ptr(rhs), ptr(x),
                                 float(scale), ptr(out)))
    return out


def _inplace(x):
    if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous):
        raise TypeError("x must be a C-contiguous float64 array (updated in place)")
    return x


def gs_sweep(diag, nbr_rows, rhs, x, scale):
    """_core.pyx:237-252 — lexicographic Gauss-Seidel, x updated in place
    (a hyperplane wavefront on the device, same per-row arithmetic)."""
    x = _inplace(x)
    diag, rhs = _f64(diag), _f64(rhs)
    n = len(diag)
    check(LIB.flip_k_gs_sweep(n, ptr(diag), ptr(_nbr(nbr_rows, n), _i64), ptr(rhs), ptr(x),
                              float(scale)))


def gs_sweep_rows(rows, diag, nbr_rows, rhs, x, scale, workers=1):
    """_core.pyx:255-272 — update of a mutually uncoupled row subset, in place."""
    x = _inplace(x)
    rows, diag, rhs = _i(rows), _f64(diag), _f64(rhs)
    n = len(diag)
    check(LIB.flip_k_gs_sweep_rows(len(rows), ptr(rows, _i64), n, ptr(diag),
                                   ptr(_nbr(nbr_rows, n), _i64), ptr(rhs), ptr(x), float(scale)))


def mic0_build(diag, nbr_rows, scale, tau=0.97, sigma=0.25, workers=1):
    """_core.pyx:275-308 — MIC(0) scaling vector."""
    diag = _f64(diag)
    n = len(diag)
    out = np.empty(n)
    check(LIB.flip_k_mic0_build(n, ptr(diag), ptr(_nbr(nbr_rows, n), _i64), float(scale),
                                float(tau), float(sigma), ptr(out)))
    return out


def mic0_apply(precon, nbr_rows, r_vec, scale, workers=1):
    """_core.pyx:311-347 — forward then backward substitution."""
    precon, r_vec = _f64(precon), _f64(r_vec)
    n = len(precon)
    z = np.empty(n)
    check(LIB.flip_k_mic0_apply(n, ptr(precon), ptr(_nbr(nbr_rows, n), _i64), ptr(r_vec),
                                float(scale), ptr(z)))
    return z


def pairwise_dot(a, b=None) -> float:
    """np.add.reduce(a * b) with numpy's pairwise order (pressure.py:269-271)."""
    a = _f64(a)
    out = C.c_double(0.0)
    check(LIB.flip_k_pairwise_dot(len(a), ptr(a), ptr(_f64(b)) if b is not None else None,
                                  C.byref(out)))
    return float(out.value)
