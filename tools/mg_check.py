"""Multigrid-preconditioned PCG (precond="mg", extension) against MIC(0)-PCG,
both run to convergence: iterations, residual, relative pressure difference,
post-step max |div| over FLUID, project time."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import sys
import numpy as np
import paper_2404_01931_b200 as P

res = int(sys.argv[1]) if len(sys.argv) > 1 else 64
scene = sys.argv[2] if len(sys.argv) > 2 else "dam-break"
out = {}
for pc in ("mic0", "mg"):
    spec = P.SceneSpec(name=scene, res=res, precond=pc, max_iters=1000)
    st = P.make_scene(spec, 0)
    P.step(st, spec)
    r = P.step(st, spec)
    div = P.divergence_field(st)
    fl = np.asarray(st.grid.label) == P.FLUID
    out[pc] = (np.array(st.grid.p), r)
    print(f"{scene} {res}^3 {pc:5s}: its {r.solver_iterations:4d} res {r.solver_residual:.2e} "
          f"conv {r.solver_converged} project {r.timings.project:8.2f} ms  max|div| {np.abs(div[fl]).max():.2e}")
pm, pg = out["mic0"][0], out["mg"][0]
print("relative pressure difference (inf norm):", float(np.abs(pm - pg).max() / max(np.abs(pm).max(), 1e-300)))
