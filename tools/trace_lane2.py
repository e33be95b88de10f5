"""Per-step globaltimer of one k_mic_lane2 tile + count of synchronous halo polls."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os
import numpy as np
import paper_2404_01931_b200 as P
from paper_2404_01931_b200 import _lib
RES = int(os.environ.get("RES", "256"))
spec = P.SceneSpec(name="dam-break", res=RES, max_iters=1)
st = P.make_scene(spec, 0)
P.step(st, spec)
P.step(st, spec)
tr = st.device.debug_buffer("wave_trace", 16384 + 2048, dtype=np.uint64).astype(np.int64)[16384:]
ts = tr[:1000]; ts = ts[ts > 0]
polls = tr[1024:2024]
d = np.diff(ts)
print("tile", os.environ.get("FLIPB200_LANE_DBG"), "steps", len(ts), "span us", (ts[-1] - ts[0]) / 1e3,
      "median ns/step", np.median(d), "sync polls", int(polls.sum()))
print("ns per step (first 60):", d[:60].tolist())
print("polls per step (first 60):", polls[:60].tolist())
