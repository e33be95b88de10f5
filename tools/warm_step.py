"""One 256^3 step inside a cudaProfilerStart/Stop range after warm-up steps,
for `ncu --profile-from-start off --cache-control none` (warm-cache
per-kernel durations; their sum against the step's event time gives the
launch-gap overhead)."""
import sys
import time

import torch

import os as _o, sys as _s
_s.path.insert(0, _o.path.dirname(_o.path.dirname(_o.path.abspath(__file__))))
import paper_2404_01931_b200 as P

res = int(sys.argv[1]) if len(sys.argv) > 1 else 256
precond = sys.argv[2] if len(sys.argv) > 2 else "mic0"
spec = P.SceneSpec(res=res, precond=precond)
st = P.make_scene(spec)
for _ in range(3):
    P.step(st, spec)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
t0 = time.perf_counter()
rep = P.step(st, spec)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(f"step wall {1e3 * (time.perf_counter() - t0):.2f} ms project {rep.timings.project:.2f} ms "
      f"iters {rep.solver_iterations} rows {rep.nrows} launches {rep.gpu_launches}")
