"""Small cases for compute-sanitizer (one tool per run): the MIC(0) wavefront
sweeps (k_mic_quad, k_wave BUILD), the pairwise dots, Jacobi / RBGS / GS and
the particle stages at 20^3-24^3, each step checked against the oracle.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py
"""
import os
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(HERE, "oracle"))
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
import paper_2404_01931_b200 as P  # noqa: E402

cases = [("dam-break", 24, "pcg", "mic0"), ("double-dam-break", 20, "gs", "mic0"),
         ("water-drop", 20, "rbgs", "mic0"), ("dam-break", 20, "jacobi", "mic0"),
         ("dam-break", 20, "pcg", "jacobi")]
if len(sys.argv) > 1:
    cases = cases[: int(sys.argv[1])]
for name, res, solver, precond in cases:
    spec = P.SceneSpec(name=name, res=res, solver=solver, precond=precond)
    ospec = O.Spec(name=name, res=res, solver=solver, precond=precond)
    st = P.make_scene(spec, rng_seed=0, device=0)
    os_ = O.make_scene(ospec, rng_seed=0)
    for k in range(2):
        rep = P.step(st, spec)
        ref = O.step(os_, ospec)
        assert rep.solver_iterations == ref["solver_iterations"], (name, k)
    for got, want in zip(st.particles.arrays(), os_.parts):
        assert np.array_equal(got, want), name
    assert np.array_equal(st.grid.p, os_.p), name
    print(f"{name} {res}^3 {solver}/{precond}: 2 steps bit-exact, "
          f"{rep.solver_iterations} iterations", flush=True)
print("sanitize cases ok")
