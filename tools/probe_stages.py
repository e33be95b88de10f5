import sys, time
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import paper_2404_01931_b200 as P
res = int(sys.argv[1]) if len(sys.argv) > 1 else 256
solver = sys.argv[2] if len(sys.argv) > 2 else "pcg"
spec = P.SceneSpec(name="dam-break", res=res, solver=solver)
t0 = time.time(); st = P.make_scene(spec, 0); t1 = time.time()
print("make_scene", round(t1 - t0, 3), "N", st.particles.count, flush=True)
for k in range(6):
    t0 = time.time(); r = P.step(st, spec); t1 = time.time()
    print(k, "wall", round((t1 - t0) * 1e3, 1), "ms N", r.particle_count, "it", r.solver_iterations,
          "res", r.solver_residual, "rows", r.nrows, "launches", r.gpu_launches,
          {a: round(b, 2) for a, b in r.timings.as_dict().items()}, flush=True)
