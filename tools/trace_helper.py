"""k_mic_lane2 helper-warp phases (first z-face lane) per step, clock64 cycles:
barrier exit -> publish done -> ring value in hand -> staged + next fetch issued -> next exit."""
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
    except Exception as e:
        print("step error", type(e).__name__)
tr = st.device.debug_buffer("wave_trace", 32768, dtype=np.uint64).astype(np.int64)
h = tr[28000:28512].reshape(4, 128)
print("step  publish  ringwait  stage+fetch  to-next-exit")
rows = []
for s in range(1, 100):
    if h[0, s] == 0 or h[0, s + 1] == 0:
        continue
    r = (h[1, s] - h[0, s], (h[2, s] - h[1, s]) if h[2, s] else -1, h[3, s] - max(h[2, s], h[1, s]), h[0, s + 1] - h[3, s])
    rows.append(r)
    if s < 40:
        print(f"{s:3d}", " ".join(f"{v:8d}" for v in r))
rows = np.array(rows)
print("median", np.median(rows, axis=0))
