"""The bounds-checked build (libflipb200_checked.so, FLIP_CHECK sites in the
quad wavefront's chunk copies / halo publishes and reads / DSMEM ring slots /
group stores / cluster tickets, the update's lane scatter, the z.r dot's lane
gather, the lane map) on the sanitizer cases of tools/sanitize_case.py, in a
subprocess (the library is chosen at import).  compute-sanitizer is closed on
the GPU pool (profiles/r02_compute_sanitizer_refused.log); a failed check
traps, which fails the launch and this test."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_checked_build_sanitizer_cases():
    lib = os.path.join(HERE, "paper_2404_01931_b200", "libflipb200_checked.so")
    assert os.path.exists(lib), "build the checked library: make -C paper_2404_01931_b200/csrc checked"
    env = dict(os.environ, FLIPB200_CHECKED="1")
    r = subprocess.run([sys.executable, os.path.join(HERE, "tools", "sanitize_case.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "sanitize cases ok" in r.stdout
    assert "FLIP_CHECK failed" not in r.stdout + r.stderr
