"""Per-tile start/end/sync-poll trace of the forward k_mic_lane2 sweep (last launch)."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os
import numpy as np
import paper_2404_01931_b200 as P
RES = int(os.environ.get("RES", "256"))
spec = P.SceneSpec(name="dam-break", res=RES, max_iters=int(os.environ.get("ITERS", "1")))
st = P.make_scene(spec, 0)
P.step(st, spec)
P.step(st, spec)
tr = st.device.debug_buffer("wave_trace", 4 * 4096, dtype=np.uint64).astype(np.int64).reshape(-1, 4)
m = tr[:, 1] > 0
tr = tr[m]
t0 = tr[:, 0].min()
b = tr[:, 3] // 65536; c = tr[:, 3] % 65536
start = (tr[:, 0] - t0) / 1e3; end = (tr[:, 1] - t0) / 1e3; dur = end - start
print("tiles", len(tr), "sweep span us", end.max())
TB, TC = b.max() + 1, c.max() + 1
S = np.full((TB, TC), np.nan); D = np.full((TB, TC), np.nan); Q = np.zeros((TB, TC))
S[b, c] = start; D[b, c] = dur; Q[b, c] = (tr[:, 2] - t0) / 1e3
np.set_printoptions(linewidth=250, precision=0, suppress=True)
print("start us (rows b, cols c):"); print(S)
print("end us:"); print(D)
print("real start (step 0) us:"); print(Q)
R = (end - (tr[:, 2] - t0) / 1e3)
print("run time us (end - real start):"); RR = np.full((TB, TC), np.nan); RR[b, c] = R; print(RR)
