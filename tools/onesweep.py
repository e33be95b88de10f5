"""Two 256^3 dam-break steps (for profiling the pressure sweeps)."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os
import paper_2404_01931_b200 as P
spec = P.SceneSpec(name="dam-break", res=int(os.environ.get("RES", "256")),
                   max_iters=int(os.environ.get("ITERS", "100")))
st = P.make_scene(spec, 0)
for _ in range(2):
    r = P.step(st, spec)
print("project ms", r.timings.project, r.solver_iterations)
