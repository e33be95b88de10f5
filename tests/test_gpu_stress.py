"""Timing-perturbation stress of the MIC(0) wavefront protocol (stands in for
compute-sanitizer racecheck, which this pool does not allow): with
FLIPB200_QUAD_EXP=16 every compute thread and helper lane of k_mic_quad
sleeps pseudo-randomly (up to ~2 us at ~1 in 8 steps), which reorders every
producer/consumer pair of the face rings (DSMEM inside clusters, the global
step-major halo across them).  The step must stay bit-identical to the
CPU oracle.  Runs in a subprocess (the flag is read once per process)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
sys.path[:0] = [ROOT, ROOT + "/oracle", ROOT + "/tests"]
import oracle as O
import paper_2404_01931_b200 as P
from helpers import device_arrays, diff_report, oracle_arrays
case = json.loads(sys.argv[1])
d, o = P.SceneSpec(**case), O.Spec(**case)
st, os_ = P.make_scene(d, 1), O.make_scene(o, 1)
for k in range(2):
    rep = P.step(st, d)
    ref = O.step(os_, o)
    bad = diff_report(device_arrays(st), oracle_arrays(os_))
    assert not bad, (k, bad)
    assert rep.solver_residual == ref["solver_residual"], k
print("stress ok", rep.solver_iterations)
""".replace("ROOT", repr(ROOT))


@pytest.mark.parametrize("case", [dict(name="dam-break", res=128, solver="pcg"),
                                  dict(name="double-dam-break-obstacle", res=96, solver="pcg")],
                         ids=["dam-break-128", "obstacle-96"])
def test_mic_wavefront_under_random_delays(case):
    env = dict(os.environ, FLIPB200_QUAD_EXP="16")
    r = subprocess.run([sys.executable, "-c", SCRIPT, json.dumps(case)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]
    assert "stress ok" in r.stdout
