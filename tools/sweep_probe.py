import os, sys, time
sys.path.insert(0, '/root/repo')
import paper_2404_01931_b200 as P
from paper_2404_01931_b200 import _lib
import ctypes as C
spec = P.SceneSpec(res=256)
st = P.make_scene(spec)
for _ in range(3):
    try: P.step(st, spec)
    except P.SolverError: pass
_lib.check(_lib.LIB.flip_set_probe(st.device.ctx, 1))
for _ in range(3):
    try: P.step(st, spec)
    except P.SolverError: pass
ms, n, b = C.c_double(), C.c_int64(), C.c_double()
_lib.check(_lib.LIB.flip_get_probe(st.device.ctx, C.byref(ms), C.byref(n), C.byref(b)))
print(os.environ.get("FLIPB200_QUAD_EXP", "0"), "sweep avg ms", ms.value / max(n.value, 1), n.value)
