"""A/B timing of the 256^3 step under the current FLIPB200_* environment:
mean device ms/step and PROJECT ms over K steps after W warm-up steps, the
MIC(0) sweep's mean launch time (flip_set_probe), bit-exactness digest of
the final state (so variants can be compared for identical results).

    FLIPB200_QUAD=0 python tools/ab_step.py [res] [K] [W]

AB_CAP=n sets the particle capacity (default: the 12-per-cell bound); AB_PAD_GB=g holds g GB
of extra device memory (footprint / placement experiments: the MIC(0) sweep time moves by
~1.5 % with the allocation layout).
"""
import ctypes as C
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_2404_01931_b200 as P
from paper_2404_01931_b200._lib import LIB, check

res = int(sys.argv[1]) if len(sys.argv) > 1 else 256
K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
W = int(sys.argv[3]) if len(sys.argv) > 3 else 3
spec = P.SceneSpec(name="dam-break", res=res, precond=os.environ.get("AB_PRECOND", "mic0"))
st = P.make_scene(spec, capacity=int(os.environ.get("AB_CAP", "0")))
_pad_gb = float(os.environ.get("AB_PAD_GB", "0"))  # footprint experiment: extra device memory held
_pad = torch.empty(int(_pad_gb * 2**30), dtype=torch.uint8, device="cuda") if _pad_gb > 0 else None
for _ in range(W):
    P.step(st, spec)
check(LIB.flip_set_probe(st.device.ctx, 1))
stream = torch.cuda.ExternalStream(st.device.stream_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(stream)
proj = 0.0
stages = {}
for _ in range(K):
    rep = P.step(st, spec)
    proj += rep.timings.project
    for k, v in vars(rep.timings).items():
        stages[k] = stages.get(k, 0.0) + v
e1.record(stream)
e1.synchronize()
ms = e0.elapsed_time(e1) / K
pms, pl, pb = C.c_double(0), C.c_int64(0), C.c_double(0)
check(LIB.flip_get_probe(st.device.ctx, C.byref(pms), C.byref(pl), C.byref(pb)))
h = hashlib.sha256()
for a in st.particles.arrays():
    h.update(np.ascontiguousarray(a).tobytes())
h.update(np.ascontiguousarray(st.grid.p).tobytes())
env = {k: v for k, v in os.environ.items() if k.startswith("FLIPB200_")}
print(f"{env} res {res}: {ms:.2f} ms/step, project {proj / K:.2f} ms, "
      f"mic sweep {pms.value / max(pl.value, 1) * 1e3:.1f} us x {pl.value // K}/step, "
      f"its {rep.solver_iterations}, digest {h.hexdigest()[:16]}", flush=True)
print("  stages (ms): " + ", ".join(f"{k} {v / K:.3f}" for k, v in stages.items() if k != "project"),
      flush=True)
