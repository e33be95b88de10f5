import os, sys
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import numpy as np
import paper_2404_01931_b200 as P
RES = int(os.environ.get("RES", "12"))
spec = P.SceneSpec(name="dam-break", res=RES, max_iters=1)
st = P.make_scene(spec, 0)
P.step(st, spec)
r = P.step(st, spec)  # last sweep launched: MIC backward (k_mic_sweep)
full = st.device.debug_buffer("wave_trace", 4 * 4096 + 1024, dtype=np.uint64)
ck = full[4 * 4096: 4 * 4096 + 200].astype(np.int64)
ck = ck[ck > 0]
d = np.diff(ck)
print(RES, "steps", len(ck), "cycles/step median", np.median(d), "list", d[:40].tolist())
