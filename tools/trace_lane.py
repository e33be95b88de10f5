"""Per-step clock of k_mic_lane tile 0 / lane 0 (FLIPB200_WAVE_TRACE=1)."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os
import numpy as np
import paper_2404_01931_b200 as P
RES = int(os.environ.get("RES", "20"))
spec = P.SceneSpec(name="dam-break", res=RES, max_iters=1)
st = P.make_scene(spec, 0)
P.step(st, spec)
P.step(st, spec)   # last lane sweep launched: backward substitution
ck = st.device.debug_buffer("wave_trace", 256, dtype=np.uint64).astype(np.int64)
ck = ck[ck > 0]
d = np.diff(ck)
print(os.environ.get("FLIPB200_LANE_DBG", "0"), RES, "steps", len(ck), "median cycles/step", np.median(d))
