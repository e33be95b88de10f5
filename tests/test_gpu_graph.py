"""The device-driven solver loop (FLIPB200_GRAPH=1: one CUDA graph per solve,
a WHILE conditional node over the iteration body) against the oracle, in a
subprocess because the mode is read once per process.  Same checks as
test_gpu_parity: every array bit-identical after every step, iterations equal
(reference loop: /root/reference/pkg/src/flipsim/pressure.py:200-213, 314-331)."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {oracle!r})
import numpy as np
import oracle as O
import paper_2404_01931_b200 as P
from paper_2404_01931_b200 import _lib
for name, res, solver, precond in [("dam-break", 24, "pcg", "mic0"), ("water-drop", 20, "pcg", "jacobi"),
                                   ("dam-break", 20, "jacobi", "mic0"), ("double-dam-break", 16, "rbgs", "mic0"),
                                   ("dam-break", 16, "gs", "mic0"), ("dam-break", 20, "pcg", "none")]:
    spec = P.SceneSpec(name=name, res=res, solver=solver, precond=precond)
    ospec = O.Spec(name=name, res=res, solver=solver, precond=precond)
    st = P.make_scene(spec, rng_seed=0, device=0)
    os_ = O.make_scene(ospec, rng_seed=0)
    if {probe}:
        _lib.check(_lib.LIB.flip_set_probe(st.device.ctx, 1))
    for k in range(3):
        rep = P.step(st, spec)
        ref = O.step(os_, ospec)
        assert rep.solver_iterations == ref["solver_iterations"], (name, k, rep.solver_iterations)
        assert rep.solver_residual == ref["solver_residual"], (name, k)
        for got, want in zip(st.particles.arrays(), os_.parts):
            assert np.array_equal(got, want), (name, k)
        for a in ("u", "v", "w", "p"):
            assert np.array_equal(getattr(st.grid, a), getattr(os_, a)), (name, k, a)
    print("ok", name, solver, precond, rep.solver_iterations, rep.gpu_launches)
print("graph ok")
"""


@pytest.mark.gpu
@pytest.mark.parametrize("probe", [0, 1])
def test_graph_loop_bit_exact(probe):
    env = dict(os.environ, FLIPB200_GRAPH="1")
    code = SCRIPT.format(root=HERE, oracle=os.path.join(HERE, "oracle"), probe=probe)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "graph ok" in r.stdout
