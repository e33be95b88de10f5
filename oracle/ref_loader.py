"""Import the REAL reference package (`flipsim`) for parity checking.

Test infrastructure only (never imported by the product package). The
reference's pure-Python modules are imported in place from
``/root/reference/pkg/src``; its compiled core ``_core.pyx`` is built by
``oracle/build_ref.sh`` into ``oracle/_ref/`` and injected into
``sys.modules`` as ``flipsim._kernels._core`` before ``flipsim._kernels``
imports it (``flipsim/_kernels/__init__.py:17-20``), so the Cython backend
(the bit-deterministic oracle) is active.

Only available where ``/root/reference`` exists (the build container). On the
GPU box `available()` is False and callers fall back to the committed golden
fixtures plus the C restatement in ``oracle/flip_oracle.c``.
"""

from __future__ import annotations

import importlib.util
import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = os.path.join(os.environ.get("FLIPSIM_REF_ROOT", "/root/reference"),
                       "pkg", "src")
_SO = os.path.join(HERE, "_ref", "_core" + sysconfig.get_config_var("EXT_SUFFIX"))


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "flipsim"))


def build() -> None:
    if available():
        subprocess.run(["bash", os.path.join(HERE, "build_ref.sh")], check=True)


def load():
    """Return the reference `flipsim` package with the Cython backend active."""
    if "flipsim" in sys.modules:
        return sys.modules["flipsim"]
    if not available():
        raise RuntimeError("reference sources not present (only in the build container)")
    build()
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    spec = importlib.util.spec_from_file_location("flipsim._kernels._core", _SO)
    core = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(core)
    sys.modules["flipsim._kernels._core"] = core
    import flipsim  # noqa: E402
    from flipsim import _kernels
    assert "cython" in _kernels.available_backends(), "reference Cython core not loaded"
    _kernels.set_backend("cython")
    return flipsim
