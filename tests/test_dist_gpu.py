"""Slab-decomposed step (paper_2404_01931_b200/dist.py) vs the 1-GPU step:
2 and 3 ranks sharing the one GPU, gloo transport.  Particles gathered in
rank order, grid, grid_old and the StepReport must be bit-identical."""
import hashlib
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [
    dict(spec=dict(name="dam-break", res=16, solver="pcg"), seed=3, steps=3),
    dict(spec=dict(name="double-dam-break", res=20, solver="jacobi"), seed=1, steps=2),
    dict(spec=dict(name="water-drop", res=16, solver="pcg"), seed=2, steps=3),
    # larger: several clusters in the sweep, heavy slab-crossing migration
    dict(spec=dict(name="dam-break", res=64, solver="pcg"), seed=0, steps=4),
]


def digest(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + a.tobytes()).hexdigest()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _single(case):
    import paper_2404_01931_b200 as P
    spec = P.SceneSpec(**case["spec"])
    st = P.make_scene(spec, case["seed"])
    recs = []
    for _ in range(case["steps"]):
        rep = P.step(st, spec)
        g, go = st.grid, st.grid_old
        rec = {f"part{i}": digest(a) for i, a in enumerate(st.particles.arrays())}
        rec.update({k: digest(getattr(g, k)) for k in ("u", "v", "w", "p", "label")})
        rec.update({"uo": digest(go.u), "vo": digest(go.v), "wo": digest(go.w)})
        rec.update({"n": int(rep.particle_count), "dt": float(rep.dt).hex(),
                    "its": int(rep.solver_iterations), "res": float(rep.solver_residual).hex()})
        recs.append(rec)
    st.device.close()
    return recs


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("ci", range(len(CASES)))
def test_slab_step_matches_single_gpu(tmp_path, world, ci):
    case = CASES[ci]
    out = tmp_path / "digests.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.join(HERE, "_dist_gpu_worker.py"),
           str(out), json.dumps(case)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, MASTER_ADDR="127.0.0.1"))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    got = json.load(open(out))
    exp = _single(case)
    assert len(got) == len(exp)
    for s, (g, e) in enumerate(zip(got, exp)):
        bad = [k for k in e if g[k] != e[k]]
        assert not bad, f"step {s + 1}: {bad}"
