"""Per-tile timeline of the forward k_mic_cl sweep (last launch; 256^3 dam-break
after STEPS steps, PCG capped at one iteration so the traced launch is the
last forward sweep): kernel entry, first step, end of the compute loop."""
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import os
import numpy as np
import paper_2404_01931_b200 as P
os.environ.setdefault("FLIPB200_WAVE_TRACE", "1")
RES = int(os.environ.get("RES", "256"))
spec = P.SceneSpec(name="dam-break", res=RES, max_iters=1)
st = P.make_scene(spec, 0)
for _ in range(int(os.environ.get("STEPS", "8"))):
    try:
        P.step(st, spec)
    except P.SolverError:  # timing experiments (FLIPB200_QUAD_EXP) break the numerics
        pass
tr = st.device.debug_buffer("wave_trace", 32768, dtype=np.uint64).astype(np.int64)
t4 = tr[:4 * 4096].reshape(-1, 4)
m = t4[:, 1] > 0
t4 = t4[m]
t0 = t4[:, 0].min()
b, c = t4[:, 3] >> 16, t4[:, 3] & 0xffff
TB, TC = b.max() + 1, c.max() + 1
ent, first, end = [(t4[:, k] - t0) / 1e3 for k in (0, 2, 1)]
print(f"tiles {len(t4)} grid {TB}x{TC}; entry spread {ent.max():.1f} us; "
      f"sweep span {end.max():.1f} us; first step of tile (0,0) at {first[(b == 0) & (c == 0)][0]:.1f} us")
np.set_printoptions(linewidth=250, precision=1, suppress=True)
F = np.full((TB, TC), np.nan); E = np.full((TB, TC), np.nan)
F[b, c] = first; E[b, c] = end
print("first step (us), rows b, cols c:"); print(F)
print("end (us):"); print(E)
print("end - first (us):"); print(E - F)
steps = tr[20000:20300]
n = int((steps > 0).sum())
if n > 1:
    d = np.diff(steps[:n]) / 1e3
    print(f"tile 0: {n} steps, median step {np.median(d) * 1e3:.0f} ns, mean {d.mean() * 1e3:.0f} ns")
# per-step stamps of tiles 0..7 (row b = 0 when TC >= 8): each consumes
# tile c-1's z face at the producer's step s + 15
S = tr[20000:20000 + 8 * 300].reshape(8, 300).astype(np.float64)
for c in range(8):
    n = int((S[c] > 0).sum())
    if n < 20:
        continue
    d = np.diff(S[c, :n])
    msg = f"tile {c}: steps {n}, step ns median {np.median(d):.0f} p90 {np.percentile(d, 90):.0f}"
    if c > 0:
        m = min(n, int((S[c - 1] > 0).sum()) - 15)
        slack = S[c, :m] - S[c - 1, 15:15 + m]   # consumer step s minus producer step s+15
        msg += f"; slack vs producer step s+15: median {np.median(slack):.0f} ns, min {slack.min():.0f}"
    print(msg)
