"""Per-x timeline of one z-face hop in k_mic_lane2 (tile dbg-1 -> tile dbg, lane jj=0):
producer publish, consumer fetch issue, consumer use begin, value in hand."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os
import numpy as np
import paper_2404_01931_b200 as P
spec = P.SceneSpec(name="dam-break", res=int(os.environ.get("RES", "256")), max_iters=1)
st = P.make_scene(spec, 0)
P.step(st, spec)
P.step(st, spec)
tr = st.device.debug_buffer("wave_trace", 24576, dtype=np.uint64).astype(np.int64)
pub, use, got, iss = tr[20000:21000], tr[21000:22000], tr[22000:23000], tr[23000:24000]
m = (pub > 0) & (use > 0) & (got > 0) & (iss > 0)
x = np.nonzero(m)[0]
t0 = min(pub[m].min(), iss[m].min())
print(" x   issue  publish   use    got   (us, rel)   got-pub  issue-pub")
for i in x[:80]:
    print(f"{i:3d} {(iss[i]-t0)/1e3:7.2f} {(pub[i]-t0)/1e3:7.2f} {(use[i]-t0)/1e3:7.2f} {(got[i]-t0)/1e3:7.2f}  {(got[i]-pub[i]):6d} {(iss[i]-pub[i]):6d}")
tr2 = st.device.debug_buffer("wave_trace", 24576 + 1024, dtype=np.uint64).astype(np.int64)
lat = tr2[24000:24256]
lat = lat[lat > 0]
print("in-situ synchronous halo reload latency (cycles): median", np.median(lat), "p10", np.percentile(lat, 10), "p90", np.percentile(lat, 90))
