import os, sys
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import numpy as np
import paper_2404_01931_b200 as P
RES = int(os.environ.get("RES", "256"))
spec = P.SceneSpec(name="dam-break", res=RES, max_iters=2)
st = P.make_scene(spec, 0)
P.step(st, spec)
r = P.step(st, spec)   # the last wave launched is the backward sweep of the first PCG iteration
tr = st.device.debug_buffer("wave_trace", 4 * 4000, dtype=np.uint64).reshape(-1, 4)
tr = tr[tr[:, 1] > 0]
t0 = tr[:, 0].min()
b = (tr[:, 3] >> 32).astype(int); c = (tr[:, 3] & 0xffffffff).astype(int)
start = (tr[:, 0] - t0) / 1e3; end = (tr[:, 1] - t0) / 1e3; spin = tr[:, 2] / 1.9e3
print("tiles", len(tr), "span us", end.max(), "TB", b.max() + 1, "TC", c.max() + 1)
o = np.argsort(start)
for x in list(o[:5]) + list(o[-5:]):
    print(f"tile b={b[x]:3d} c={c[x]:3d} start {start[x]:8.1f} end {end[x]:8.1f} dur {end[x]-start[x]:8.1f} spin {spin[x]:8.1f} us")
dur = end - start
print("mean dur", dur.mean(), "mean spin", spin.mean())
# along the diagonal path
for bb, cc in [(0, 0), (0, 10), (0, 30), (5, 0), (5, 30)]:
    m = (b == bb) & (c == cc)
    if m.any():
        x = np.flatnonzero(m)[0]; print("tile", bb, cc, "start", start[x], "end", end[x], "spin", spin[x])
full = st.device.debug_buffer("wave_trace", 4 * 4096 + 1024, dtype=np.uint64)
ck = full[4 * 4096: 4 * 4096 + 200].astype(np.int64)
ck = ck[ck > 0]
d = np.diff(ck)
print("tile0 steps", len(ck), "cycles/step median", np.median(d), "mean", d.mean(), "first", d[:12].tolist(), "last", d[-12:].tolist())
bw = full[4 * 4096 + 200: 4 * 4096 + 400].astype(np.int64)[:len(ck)]
print("barrier wait cycles median", np.median(bw), "body+wait", np.median(d))
T = full[4 * 4096 + 400: 4 * 4096 + 600].astype(np.int64).reshape(50, 4)
st_ = full[4 * 4096: 4 * 4096 + 50].astype(np.int64)
for s in range(min(8, len(ck) - 10), min(18, len(ck) - 2)):
    print("step", s, "bar->compute_done", T[s,0]-st_[s], "halo", T[s,1]-T[s,0], "load2", T[s,2]-T[s,1], "e_load", T[s,3]-T[s,2], "->next bar", st_[s+1]-T[s,3])
AB = full[4 * 4096 + 700: 4 * 4096 + 800].astype(np.int64).reshape(50, 2)
for s in range(8, 18):
    print("step", s, "bar->tcA", AB[s,0]-st_[s], "tcA->operand_ready", AB[s,1]-AB[s,0], "->compute_done", T[s,0]-AB[s,1])
