"""Per-tile timeline of the forward k_mic_quad sweep (256^3 dam-break after
STEPS steps, PCG capped at one iteration so the traced launch is the last
forward sweep): first-step and end stamps per tile (%globaltimer), the
per-tile step period, and each tile's start lag behind its producers."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("FLIPB200_WAVE_TRACE", "1")
import numpy as np  # noqa: E402

import paper_2404_01931_b200 as P  # noqa: E402

RES = int(os.environ.get("RES", "256"))
spec = P.SceneSpec(name="dam-break", res=RES, max_iters=1)
st = P.make_scene(spec, 0)
for _ in range(int(os.environ.get("STEPS", "6"))):
    try:
        P.step(st, spec)
    except P.SolverError:
        pass
tr = st.device.debug_buffer("wave_trace", 32768, dtype=np.uint64).astype(np.int64)
t4 = tr[:4 * 4096].reshape(-1, 4)
t4 = t4[t4[:, 1] > 0]
t0 = t4[:, 0].min()
b, c = (t4[:, 3] >> 16) & 0xffff, t4[:, 3] & 0xffff
smid = t4[:, 3] >> 32
TB, TC = b.max() + 1, c.max() + 1
ent, first, end = [(t4[:, k] - t0) / 1e3 for k in (0, 2, 1)]
F = np.full((TB, TC), np.nan)
E = np.full((TB, TC), np.nan)
N = np.full((TB, TC), np.nan)
F[b, c] = first
E[b, c] = end
nsteps = int(os.environ.get("NSTEPS", "0"))
print(f"tiles {len(t4)} grid {TB}x{TC}; sweep span {end.max():.1f} us (entry spread {ent.max():.1f})")
np.set_printoptions(linewidth=250, precision=2, suppress=True)
print("first step (us):")
print(F)
print("end - first (us) = nsteps x period:")
print(E - F)
# start lag of each tile behind the later of its producers' first steps
lag = np.full((TB, TC), np.nan)
for i in range(TB):
    for j in range(TC):
        p = []
        if i > 0:
            p.append(F[i - 1, j])
        if j > 0:
            p.append(F[i, j - 1])
        if p:
            lag[i, j] = F[i, j] - max(p)
print("start lag behind the later producer (us):")
print(lag)
# SM of each tile (%smid) and the lag split by whether a tile's later producer sits on the
# same half of the SM ids (a proxy for the same die) or the other half
SM = np.full((TB, TC), -1)
SM[b, c] = smid
half = int(os.environ.get("SM_HALF", "74"))
print("SM id per tile:")
print(SM)
same, cross = [], []
for i in range(TB):
    for j in range(TC):
        cand = []
        if i > 0:
            cand.append((F[i - 1, j], (i - 1, j)))
        if j > 0:
            cand.append((F[i, j - 1], (i, j - 1)))
        if cand and not np.isnan(lag[i, j]):
            pi, pj = max(cand)[1]
            (same if (SM[i, j] < half) == (SM[pi, pj] < half) else cross).append(lag[i, j])
if same and cross:
    print(f"lag behind the later producer: same SM half {np.median(same):.2f} us (n={len(same)}), "
          f"other half {np.median(cross):.2f} us (n={len(cross)})")
print(f"median lag {np.nanmedian(lag):.2f} us; median busy span {np.nanmedian(E - F):.1f} us; "
      f"last tile first step {F[-1, -1]:.1f} us, end {E[-1, -1]:.1f} us")
T0 = int(os.environ.get("FLIPB200_TRACE_TILE0", "0"))
S = tr[20000:20000 + 8 * 300].reshape(8, 300).astype(np.float64)
SP = tr[24000:24000 + 8 * 300].reshape(8, 300)
for k in range(8):
    n = int((S[k] > 0).sum())
    if n > 20:
        d = np.diff(S[k, :n])
        sp = SP[k, :n]
        print(f"tile {T0 + k} (b={(T0 + k) // TC}, c={(T0 + k) % TC}): {n} steps, step ns median "
              f"{np.median(d):.0f} mean {d.mean():.0f} p90 {np.percentile(d, 90):.0f} max {d.max():.0f}; "
              f"spins: global y {int((sp & 1 > 0).sum())} z {int((sp & 2 > 0).sum())}, "
              f"dsmem y {int((sp & 4 > 0).sum())} z {int((sp & 8 > 0).sum())}")
        if os.environ.get("VERBOSE"):
            print("  dt ns:", " ".join(f"{x:.0f}{'*' if sp[i + 1] else ''}" for i, x in enumerate(d)))
