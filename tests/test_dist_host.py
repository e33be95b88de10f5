"""Slab-decomposition host logic (paper_2404_01931_b200/dist.py) on CPU:
plane plan and face ownership in-process, the distributed pairwise-dot
algorithm against numpy on ragged partitions, the C-ABI entry points, and
the transport's collectives with 2 and 3 gloo ranks
(tests/_dist_host_worker.py)."""
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


@pytest.mark.parametrize("n", [0, 1, 7, 8, 127, 128, 129, 1000, 4097, 65536, 300001])
def test_distributed_pairwise_sum_is_numpy(pkg, n):
    """The slab dot's algorithm (csrc/pressure.cu launch_dot_slab, mirrored in
    dist.distributed_pairwise_sum): any contiguous partition, including empty
    and single-row pieces, gives np.add.reduce bit for bit."""
    from paper_2404_01931_b200.dist import distributed_pairwise_sum
    rng = np.random.default_rng(n)
    v = rng.normal(size=n) * rng.choice([1e-8, 1.0, 1e8], size=n)
    want = float(np.add.reduce(v))
    for world in (1, 2, 3, 8):
        for trial in range(3):
            cuts = sorted(rng.integers(0, n + 1, size=world - 1)) if n else [0] * (world - 1)
            if trial == 0:
                cuts = np.linspace(0, n, world + 1).astype(int)[1:-1]
            assert distributed_pairwise_sum(np.split(v, cuts)) == want, (world, cuts)


def test_slab_abi_exports(pkg):
    from paper_2404_01931_b200._lib import LIB
    for name in ("flip_set_slab_comm", "flip_slab_bytes", "flip_reserve_particles"):
        assert hasattr(LIB, name)


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
