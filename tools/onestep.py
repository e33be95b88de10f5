import sys
import os as _os, sys as _sys
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
import paper_2404_01931_b200 as P
res = int(sys.argv[1]) if len(sys.argv) > 1 else 256
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = P.SceneSpec(name="dam-break", res=res)
st = P.make_scene(spec, 0)
for _ in range(steps):
    r = P.step(st, spec)
print({k: round(v, 2) for k, v in r.timings.as_dict().items()}, r.gpu_launches, flush=True)
