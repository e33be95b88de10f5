"""k_mic_cl forward sweep, tile FLIPB200_LANE_DBG, thread 0 (a y- and z-face
consumer): clock64 before/after the DSMEM face polls per step."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os
import numpy as np
import paper_2404_01931_b200 as P
spec = P.SceneSpec(name="dam-break", res=int(os.environ.get("RES", "256")), max_iters=1)
st = P.make_scene(spec, 0)
for _ in range(2):
    P.step(st, spec)
tr = st.device.debug_buffer("wave_trace", 32768, dtype=np.uint64).astype(np.int64)
c0 = tr[16384:17384]; c1 = tr[17408:18408]
n = int((c0 > 0).sum())
step = np.diff(c0[:n]); wait = (c1 - c0)[:n - 1]
print("steps", n, "median step cycles", np.median(step), "median poll wait", np.median(wait),
      "mean step", step.mean(), "mean wait", wait.mean())
print("step:", step[:40].tolist())
print("wait:", wait[:40].tolist())
