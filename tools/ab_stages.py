"""Per-stage device ms at 256^3 (mean over K steps after W warm-ups) under
the current FLIPB200_* environment, plus a state digest."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2404_01931_b200 as P

res = int(sys.argv[1]) if len(sys.argv) > 1 else 256
K = int(sys.argv[2]) if len(sys.argv) > 2 else 5
W = int(sys.argv[3]) if len(sys.argv) > 3 else 3
spec = P.SceneSpec(name="dam-break", res=res)
st = P.make_scene(spec)
for _ in range(W):
    P.step(st, spec)
acc = {}
for _ in range(K):
    rep = P.step(st, spec)
    for k, v in rep.timings.as_dict().items():
        acc[k] = acc.get(k, 0.0) + v / K
h = hashlib.sha256()
for a in st.particles.arrays():
    h.update(np.ascontiguousarray(a).tobytes())
env = {k: v for k, v in os.environ.items() if k.startswith("FLIPB200_")}
print(env, " ".join(f"{k} {v:.2f}" for k, v in acc.items()), f"total {sum(acc.values()):.2f}",
      h.hexdigest()[:16], flush=True)
