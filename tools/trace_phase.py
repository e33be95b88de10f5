"""k_mic_lane2 forward sweep, tile FLIPB200_LANE_DBG: compute-thread phases per step
(barrier exit -> body done -> next barrier exit) next to the helper's halo timeline."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os
import numpy as np
import paper_2404_01931_b200 as P
spec = P.SceneSpec(name="dam-break", res=int(os.environ.get("RES", "256")), max_iters=1)
st = P.make_scene(spec, 0)
for _ in range(2):
    try:
        P.step(st, spec)
    except Exception as e:  # ablation runs break the solve
        print('step error', type(e).__name__)
tr = st.device.debug_buffer("wave_trace", 24576, dtype=np.uint64).astype(np.int64)
a = tr[16384:17384]; bdone = tr[17500:18500]
n = int((a > 0).sum())
t0 = a[0]
print("step  (clock64 cycles) body wait")
for s in range(min(n - 1, 60)):
    print(f"{s:3d} {(a[s]-t0)/1e3:7.2f} {(bdone[s]-t0)/1e3:7.2f} {bdone[s]-a[s]:6d} {a[s+1]-bdone[s]:6d}")
body = bdone[:n-1] - a[:n-1]; wait = a[1:n] - bdone[:n-1]
polls = tr[16384 + 1024:16384 + 2024]
print("median body", np.median(body), "median wait", np.median(wait), "sync polls", int(polls.sum()), "first steps", polls[:24].tolist())
