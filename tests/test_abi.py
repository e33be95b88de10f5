"""CPU checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/flipb200.h declares; host-side API mirrors the reference."""

import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "flipb200.h")).read()
    return sorted(set(re.findall(r"\b(flip_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol(pkg):
    out = subprocess.run(["nm", "-D", "--defined-only", pkg.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (flip_[a-z0-9_]+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    assert len(header_symbols()) >= 30


def test_checked_library_exports_the_same_symbols(pkg):
    """The bounds-checked variant (FLIPB200_CHECKED=1) is a drop-in copy of the ABI."""
    path = os.path.join(ROOT, "paper_2404_01931_b200", "libflipb200_checked.so")
    if not os.path.exists(path):
        pytest.skip("checked library not built (make -C paper_2404_01931_b200/csrc checked)")
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (flip_[a-z0-9_]+)", out))
    assert not [s for s in header_symbols() if s not in exported]


def test_ctypes_binds_every_header_symbol(pkg):
    from paper_2404_01931_b200 import _lib
    for s in header_symbols():
        assert hasattr(_lib.LIB, s), s


def test_library_is_sm100a_only(pkg):
    out = subprocess.run(["cuobjdump", "--list-elf", pkg.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_kernel_registry_mirrors_reference(pkg):
    from paper_2404_01931_b200 import _kernels
    assert _kernels.available_backends() == ("cuda",)
    assert _kernels.backend_name() == "cuda"
    mod = _kernels.active()
    for name in ("sample_velocity_many", "p2g_component", "counting_sort_perm",
                 "laplacian_matvec", "jacobi_iter", "gs_sweep", "gs_sweep_rows", "mic0_build",
                 "mic0_apply"):
        assert callable(getattr(mod, name)), name
    with pytest.raises(ValueError):
        _kernels.set_backend("python")
    with pytest.raises(ValueError):
        _kernels.set_workers(-1)
    _kernels.set_workers(0)
    assert _kernels.workers() >= 1


def test_scene_spec_defaults_and_config_errors(pkg):
    spec = pkg.SceneSpec()
    assert (spec.res, spec.density, spec.solver, spec.tol) == (32, 2, "pcg", 1e-6)
    assert spec.resolved_max_iters() == 100
    assert pkg.SceneSpec(solver="jacobi").resolved_max_iters() == 2000
    with pytest.raises(pkg.ConfigError):
        pkg.make_scene(pkg.SceneSpec(name="tsunami"))
    with pytest.raises(pkg.ConfigError):
        pkg.make_scene(pkg.SceneSpec(solver="multigrid"))


def test_stage_timings_keys_match_reference(pkg):
    assert pkg.StageTimings.stage_names() == (
        "dt_compute", "advect", "bin", "classify", "p2g", "force", "project",
        "apply_gradient", "g2p", "reseed")


def test_errors_hierarchy(pkg):
    e = pkg.SingularSystemError(17)
    assert isinstance(e, pkg.SolverError) and e.cell == 17
    assert issubclass(pkg.SolverBreakdownError, pkg.SolverError)
    assert issubclass(pkg.ConfigError, pkg.FlipsimError)
