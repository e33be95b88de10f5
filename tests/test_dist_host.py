"""Slab-decomposition host logic (paper_2404_01931_b200/dist.py) on CPU:
plane plan and face ownership in-process, and the exchanges (migration
order, ghost planes, owned-face all-gather, label/dt reductions) with two
gloo ranks (tests/_dist_host_worker.py)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_slab_plan_partitions_planes(pkg):
    from paper_2404_01931_b200.dist import SlabPlan, face_ranges
    for nz, world in ((16, 2), (17, 3), (256, 8), (5, 5)):
        plan = SlabPlan(4, 3, nz, world)
        owners = plan.plane_owners()
        ranges = [plan.planes(r) for r in range(world)]
        assert ranges[0][0] == 0 and ranges[-1][1] == nz
        assert all(ranges[r][1] == ranges[r + 1][0] for r in range(world - 1))
        assert all(b - a >= 1 for a, b in ranges)
        assert all(owners[k] == plan.owner_of_plane(k) for k in range(nz))
        for comp, nf in enumerate(((4 + 1) * 3 * nz, 4 * (3 + 1) * nz, 4 * 3 * (nz + 1))):
            rr = [face_ranges(plan, comp, r) for r in range(world)]
            assert rr[0][0] == 0 and rr[-1][1] == nf
            assert all(rr[r][1] == rr[r + 1][0] for r in range(world - 1))
    with pytest.raises(ValueError):
        SlabPlan(4, 4, 3, 4)


@pytest.mark.parametrize("world", [2, 3])
def test_slab_exchanges_gloo(world):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.join(HERE, "_dist_host_worker.py")]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-4000:]
    for r in range(world):
        assert f"rank {r} ok" in out.stdout
