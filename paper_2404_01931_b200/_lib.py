"""ctypes binding of libflipb200.so (the C ABI declared in include/flipb200.h).

The library is built in-tree (``paper_2404_01931_b200/libflipb200.so``) by
``paper_2404_01931_b200.build.build()``.  There is no fallback: if the shared
object is missing or fails to load, importing the package raises.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# FLIPB200_CHECKED=1: the bounds-checked build (FLIP_CHECK sites trap on an
# out-of-range index; `make -C paper_2404_01931_b200/csrc checked`)
LIB_PATH = os.path.join(HERE, "libflipb200_checked.so" if os.environ.get("FLIPB200_CHECKED") == "1"
                        else "libflipb200.so")

FLIP_OK = 0
FLIP_E_CONFIG = 1
FLIP_E_SINGULAR = 2
FLIP_E_BREAKDOWN = 3
FLIP_E_CUDA = 4
FLIP_E_ARG = 5
FLIP_E_CAPACITY = 6

STAGE_NAMES = ("dt_compute", "advect", "bin", "classify", "p2g", "force", "project",
               "apply_gradient", "g2p", "reseed")
NSTAGES = len(STAGE_NAMES)
STAGE = {name: i for i, name in enumerate(STAGE_NAMES)}

SOLVER_ID = {"jacobi": 0, "gs": 1, "rbgs": 2, "pcg": 3}
PRECOND_ID = {"mic0": 0, "jacobi": 1, "none": 2, "mg": 3}


class StepParams(C.Structure):
    _fields_ = [
        ("gravity", C.c_double * 3),
        ("dt_max", C.c_double),
        ("flip_fraction", C.c_double),
        ("tol", C.c_double),
        ("alpha_dtau_h", C.c_double),
        ("rho_dtau2_h", C.c_double),
        ("rho_dtau_h", C.c_double),
        ("skin_h", C.c_double),
        ("max_iters", C.c_int64),
        ("solver", C.c_int32),
        ("precond", C.c_int32),
        ("extrapolation_layers", C.c_int32),
        ("density", C.c_int32),
        ("reseed_seed", C.c_uint64),
        ("solver_check_every", C.c_int32),
        ("advection", C.c_int32),
    ]


class StepReportC(C.Structure):
    _fields_ = [
        ("dt", C.c_double),
        ("particle_count", C.c_int64),
        ("solver_iterations", C.c_int64),
        ("solver_residual", C.c_double),
        ("solver_converged", C.c_int32),
        ("status", C.c_int32),
        ("err_cell", C.c_int64),
        ("err_iteration", C.c_int64),
        ("err_value", C.c_double),
        ("nrows", C.c_int64),
        ("npinned", C.c_int64),
        ("stage_ms", C.c_double * NSTAGES),
        ("gpu_launches", C.c_int64),
    ]


class Region(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("density", C.c_int32),
        ("a", C.c_double * 3),
        ("b", C.c_double * 3),
        ("radius", C.c_double),
    ]


class DevPtrs(C.Structure):
    """flip_dev_ptrs: device pointers of a ctx's state (slab decomposition)."""
    _fields_ = [
        ("pos", C.c_void_p * 3),
        ("vel", C.c_void_p * 3),
        ("count", C.c_void_p),
        ("offset", C.c_void_p),
        ("label", C.c_void_p),
        ("u", C.c_void_p), ("v", C.c_void_p), ("w", C.c_void_p), ("p", C.c_void_p),
        ("uo", C.c_void_p), ("vo", C.c_void_p), ("wo", C.c_void_p),
        ("ku", C.c_void_p), ("kv", C.c_void_p), ("kw", C.c_void_p),
        ("capacity", C.c_int64),
        ("n", C.c_int64),
    ]


_d = C.POINTER(C.c_double)
_i64 = C.POINTER(C.c_int64)
_u8 = C.POINTER(C.c_uint8)
_i32 = C.POINTER(C.c_int32)
_vp = C.c_void_p

# name -> (restype, argtypes)
_SIGNATURES = {
    "flip_last_error": (C.c_char_p, []),
    "flip_device_count": (C.c_int, [_i32]),
    "flip_create": (C.c_int, [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_double, _d,
                              C.c_int64, C.POINTER(_vp)]),
    "flip_destroy": (None, [_vp]),
    "flip_synchronize": (C.c_int, [_vp]),
    "flip_get_stream": (C.c_int, [_vp, C.POINTER(_vp)]),
    "flip_set_grid": (C.c_int, [_vp, _d, _d, _d, _d, _u8]),
    "flip_get_grid": (C.c_int, [_vp, _d, _d, _d, _d, _u8]),
    "flip_set_grid_old": (C.c_int, [_vp, _d, _d, _d]),
    "flip_get_grid_old": (C.c_int, [_vp, _d, _d, _d]),
    "flip_set_particles": (C.c_int, [_vp, C.c_int64, _d, _d, _d, _d, _d, _d]),
    "flip_get_particles": (C.c_int, [_vp, _d, _d, _d, _d, _d, _d]),
    "flip_particle_count": (C.c_int, [_vp, _i64]),
    "flip_get_particles_f32": (C.c_int, [_vp, C.POINTER(C.c_float)]),
    "flip_set_particles_f32": (C.c_int, [_vp, C.c_int64, C.POINTER(C.c_float)]),
    "flip_set_hash": (C.c_int, [_vp, _i64, _i64]),
    "flip_get_hash": (C.c_int, [_vp, _i64, _i64]),
    "flip_get_fluid_cells": (C.c_int, [_vp, _i64, _i64]),
    "flip_set_dt": (C.c_int, [_vp, C.c_double]),
    "flip_get_dt": (C.c_int, [_vp, _d]),
    "flip_set_known": (C.c_int, [_vp, _u8, _u8, _u8]),
    "flip_get_known": (C.c_int, [_vp, _u8, _u8, _u8]),
    "flip_set_solid_shell": (C.c_int, [_vp]),
    "flip_set_solid_box": (C.c_int, [_vp, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                     C.c_int64, C.c_int64]),
    "flip_seed_regions": (C.c_int, [_vp, C.c_int32, C.POINTER(Region), C.c_uint64]),
    "flip_step": (C.c_int, [_vp, C.POINTER(StepParams), C.POINTER(StepReportC)]),
    "flip_run_stages": (C.c_int, [_vp, C.POINTER(StepParams), C.c_int32, C.c_int32,
                                  C.POINTER(StepReportC)]),
    "flip_divergence_field": (C.c_int, [_vp, _d]),
    "flip_debug_copy": (C.c_int, [_vp, C.c_char_p, _vp, C.c_int64]),
    "flip_set_probe": (C.c_int, [_vp, C.c_int32]),
    "flip_get_probe": (C.c_int, [_vp, _d, _i64, _d]),
    "flip_energy_sums": (C.c_int, [_vp, C.c_double, _d, _d]),
    "flip_get_dev_ptrs": (C.c_int, [_vp, C.POINTER(DevPtrs)]),
    "flip_set_particle_count": (C.c_int, [_vp, C.c_int64]),
    "flip_reserve_particles": (C.c_int, [_vp, C.c_int64]),
    "flip_set_slab_comm": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "flip_slab_bytes": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "flip_last_error_cell": (C.c_int64, []),
    "flip_set_slab": (C.c_int, [_vp, C.c_int64, C.c_int64]),
    "flip_particle_cells": (C.c_int, [_vp, _vp]),
    "flip_k_sample_velocity_many": (C.c_int, [_d, _d, _d, C.c_int64, C.c_int64, C.c_int64,
                                              C.c_double, C.c_double, C.c_double, C.c_double,
                                              C.c_int64, _d, _d, _d, _d, _d, _d]),
    "flip_k_p2g_component": (C.c_int, [C.c_int32, C.c_int64, _d, _d, _d, _d, _i64, _i64,
                                       C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_double,
                                       C.c_double, C.c_double, _d, _d]),
    "flip_k_counting_sort_perm": (C.c_int, [C.c_int64, _i64, C.c_int64, _i64, _i64]),
    "flip_k_laplacian_matvec": (C.c_int, [C.c_int64, _d, _i64, _d, C.c_double, _d]),
    "flip_k_jacobi_iter": (C.c_int, [C.c_int64, _d, _i64, _d, _d, C.c_double, _d]),
    "flip_k_gs_sweep": (C.c_int, [C.c_int64, _d, _i64, _d, _d, C.c_double]),
    "flip_k_gs_sweep_rows": (C.c_int, [C.c_int64, _i64, C.c_int64, _d, _i64, _d, _d,
                                       C.c_double]),
    "flip_k_mic0_build": (C.c_int, [C.c_int64, _d, _i64, C.c_double, C.c_double, C.c_double,
                                    _d]),
    "flip_k_mic0_apply": (C.c_int, [C.c_int64, _d, _i64, _d, C.c_double, _d]),
    "flip_k_pairwise_dot": (C.c_int, [C.c_int64, _d, _d, _d]),
    "flip_solve_system": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, _i64, _d, _i64, _d,
                                    C.c_double, C.c_int64, C.c_double, _i64, C.c_int64, _i64,
                                    C.c_int64, _d, _i64, _d, _i32, _i64, _i64, _d]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: the CUDA library is the only implementation "
            "(no CPU fallback). Build it with `python -c \"import __graft_entry__ as g; "
            "g.build()\"` or `make -C paper_2404_01931_b200/csrc`.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()


def last_error() -> str:
    msg = LIB.flip_last_error()
    return msg.decode() if msg else ""


def ptr(a, kind=_d):
    return a.ctypes.data_as(kind) if a is not None else None


def check(rc: int, what: str = "") -> None:
    """Map a status code to the exception hierarchy (errors.py)."""
    if rc == FLIP_OK:
        return
    from . import errors
    msg = last_error() or what
    if rc == FLIP_E_CONFIG:
        raise errors.ConfigError(msg)
    if rc == FLIP_E_ARG:
        raise ValueError(msg)
    if rc == FLIP_E_CAPACITY:
        raise MemoryError(msg)
    if rc == FLIP_E_SINGULAR:
        cell = int(LIB.flip_last_error_cell())
        if cell >= 0:
            raise errors.SingularSystemError(cell)
        raise errors.SolverError(msg)
    if rc == FLIP_E_BREAKDOWN:
        raise errors.SolverBreakdownError(msg)
    raise RuntimeError(f"libflipb200: {msg} (code {rc})")


def device_count() -> int:
    n = C.c_int32(0)
    rc = LIB.flip_device_count(C.byref(n))
    return int(n.value) if rc == 0 else 0
