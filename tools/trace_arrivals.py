"""Which warp reaches each step barrier last in k_mic_lane2 (tile FLIPB200_LANE_DBG)?
Compute warps stamp after their step body, the helper after its staging."""
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
nw = int(os.environ.get("NW", "9"))
A = tr[25600:25600 + nw * 128].reshape(nw, 128)
ok = (A > 0).all(axis=0)
steps = np.nonzero(ok)[0]
t0 = A[:, steps[0]].min()
print("step  arrival cycles rel. to earliest warp (warps 0..%d, last = helper)" % (nw - 1))
for s in steps[:40]:
    col = A[:, s]
    print(f"{s:3d}", " ".join(f"{v - col.min():5d}" for v in col), "  last:", int(np.argmax(col)),
          " step len", int(col.max() - A[:, s - 1].max()) if s - 1 in steps else "")
