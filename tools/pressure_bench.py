"""Pressure-only benchmark (BASELINE config 5): the dam-break
system at step 2 for R in {64, 128, 256, 512}, solved by Jacobi, MIC(0)-PCG
(the reference's) and multigrid-PCG (extension) to tol 1e-6.  Reports
iterations, residual, converged, PROJECT time (assembly + solve, CUDA
events) and ms per iteration.  The system is rebuilt from the same grid
state for every solve (run_stages("project") only writes p)."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import argparse
import json

import paper_2404_01931_b200 as P

try:
    PEAK = json.load(open(_os.path.join(_os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    PEAK = 6552.6
# SURVEY 8(d) algorithmic bytes per iteration (per row): Jacobi 25, MIC(0)-PCG 147
# (+17 once for the build); the multigrid V-cycle has no such formula here
BYTES_PER_ROW_IT = {("jacobi", None): 25.0, ("pcg", "mic0"): 147.0}

ap = argparse.ArgumentParser()
ap.add_argument("--res", default="64,128,256,512")
ap.add_argument("--jacobi-cap", type=int, default=20000)
ap.add_argument("--pcg-cap", type=int, default=2000)
a = ap.parse_args()

for res in [int(r) for r in a.res.split(",")]:
    spec = P.SceneSpec(name="dam-break", res=res)
    cap = int(1.5 * 24_709_120 * (res / 256) ** 3) + 4096   # grows on demand if exceeded
    st = P.make_scene(spec, 0, capacity=cap)
    for _ in range(2):
        P.step(st, spec)
    for solver, precond, mi in (("jacobi", "mic0", a.jacobi_cap), ("pcg", "mic0", a.pcg_cap),
                                ("pcg", "mg", a.pcg_cap)):
        s2 = P.SceneSpec(name="dam-break", res=res, solver=solver, precond=precond,
                         max_iters=mi, tol=1e-6)
        P.run_stages(st, s2, "project", "project")          # warm-up (allocations, MG setup)
        rep = P.run_stages(st, s2, "project", "project")
        ms = float(rep.stage_ms[P._lib.STAGE["project"]])
        it = int(rep.solver_iterations)
        pc = precond if solver == "pcg" else None
        roof = None
        if (solver, pc) in BYTES_PER_ROW_IT:
            b = BYTES_PER_ROW_IT[(solver, pc)] * int(rep.nrows) * it
            if pc == "mic0":
                b += 17.0 * int(rep.nrows)
            gbs = b / (ms * 1e-3) / 1e9
            roof = {"alg_bytes": b, "achieved_gbs": round(gbs, 1), "peak_gbs": PEAK,
                    "frac": round(gbs / PEAK, 4), "note": "PROJECT stage incl. assembly"}
        print(json.dumps({"res": res, "rows": int(rep.nrows), "solver": solver,
                          "precond": pc, "iterations": it,
                          "residual": float(rep.solver_residual),
                          "converged": bool(rep.solver_converged), "project_ms": round(ms, 2),
                          "ms_per_iteration": round(ms / max(it, 1), 4), "roofline": roof}),
              flush=True)
    del st
