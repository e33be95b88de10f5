"""k_mic_cl forward sweep: per-step globaltimer (after the face polls) of
tiles 0..7 in one launch -> per-tile step rate and lag to the previous tile."""
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
        print("step error", type(e).__name__)
tr = st.device.debug_buffer("wave_trace", 32768, dtype=np.uint64).astype(np.int64)
T = tr[20000:20000 + 8 * 300].reshape(8, 300)
nzr = np.nonzero(tr[18500:])[0]
print("nz beyond 18500:", len(nzr), (nzr[:5] + 18500).tolist(), (nzr[-5:] + 18500).tolist() if len(nzr) else [])
print("nonzero per tile", (T > 0).sum(axis=1).tolist(), "nonzero 16384..", int((tr[16384:17384] > 0).sum()), "nz 0..1024", int((tr[:1024] > 0).sum()))
n = int((T[0] > 0).sum())
t0 = T[0, 0]
for k in range(8):
    row = T[k, :n]
    d = np.diff(row)
    lag = (row - T[k - 1, :n]) / 1e3 if k else np.zeros(n)
    print(f"tile {k}: start {(row[0]-t0)/1e3:7.2f} us  median ns/step {np.median(d):6.0f}  "
          f"last-first {(row[-1]-row[0])/1e3:7.2f} us  lag to prev tile (us) at s=0,20,50,90: "
          f"{[round(float(lag[i]),2) for i in (0, 20, 50, min(90, n - 1))]}")
