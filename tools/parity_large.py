"""One-off bit-exact check at a large configuration (default: BASELINE
config 4's scene, double-dam-break + obstacle at 512^3, ~200M particles):
make_scene and STEPS steps on the device and in the oracle (all host
threads), every array compared.  Too slow for the default test suite."""
import os as _os, sys as _sys
ROOT = _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))
_sys.path.insert(0, ROOT)
_sys.path.insert(0, _os.path.join(ROOT, "oracle"))
_sys.path.insert(0, _os.path.join(ROOT, "tests"))
import argparse
import time

import oracle as O
import paper_2404_01931_b200 as P
from helpers import device_arrays, diff_report, oracle_arrays

ap = argparse.ArgumentParser()
ap.add_argument("--res", type=int, default=512)
ap.add_argument("--scene", default="double-dam-break-obstacle")
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
O.set_threads(_os.cpu_count() or 1)
spec, ospec = P.SceneSpec(name=a.scene, res=a.res), O.Spec(name=a.scene, res=a.res)
t0 = time.perf_counter()
st = P.make_scene(spec, 0, capacity=int(1.5 * 8 * 0.21 * a.res ** 3) + 4096)
os_ = O.make_scene(ospec, 0)
print(f"make_scene {a.scene} {a.res}^3: N0 = {st.particles.count} (oracle {os_.n}), "
      f"{time.perf_counter() - t0:.1f} s", flush=True)
bad = diff_report(device_arrays(st), oracle_arrays(os_))
print("make_scene:", "bit-exact" if not bad else bad, flush=True)
for k in range(a.steps):
    t0 = time.perf_counter()
    rep = P.step(st, spec)
    t1 = time.perf_counter()
    ref = O.step(os_, ospec)
    t2 = time.perf_counter()
    bad = diff_report(device_arrays(st), oracle_arrays(os_))
    same = (rep.solver_iterations == ref["solver_iterations"] and
            rep.solver_residual == ref["solver_residual"])
    print(f"step {k + 1}: device {1e3 * (t1 - t0):.0f} ms, oracle {t2 - t1:.1f} s, "
          f"N={rep.particle_count}, its={rep.solver_iterations}: "
          f"{'bit-exact' if not bad and same else bad}", flush=True)
