"""Worker for tests/test_dist_host.py (launched with torch.distributed.run,
gloo, CPU tensors): checks the slab-exchange host logic of
paper_2404_01931_b200.dist against a single-process restatement."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
import torch.distributed as dist


def main():
    dist.init_process_group("gloo")
    # import the host-logic pieces without loading the CUDA library
    from paper_2404_01931_b200 import dist as D
    rank, world = dist.get_rank(), dist.get_world_size()
    tr = D.Transport()
    plan = D.SlabPlan(6, 5, 11, world)
    owners = torch.as_tensor(plan.plane_owners())
    rng = np.random.default_rng(7)
    # global particle sequence: each rank starts with a contiguous chunk
    n = 400
    G = rng.normal(size=(n, 6))
    planes = rng.integers(0, plan.nz, size=n)
    cuts = np.linspace(0, n, world + 1).astype(int)
    mine = slice(cuts[rank], cuts[rank + 1])
    got = D.migrate_rows(torch.as_tensor(G[mine]), torch.as_tensor(planes[mine]), owners, tr)
    own = plan.plane_owners()[planes] == rank
    assert np.array_equal(got.numpy(), G[own]), "migration order"
    # ghost planes: rows of the slab sorted by plane
    order = np.argsort(planes, kind="stable")
    Gs, Ps = G[order], planes[order]
    k0, k1 = plan.planes(rank)
    sel = (Ps >= k0) & (Ps < k1)
    rows, pl = Gs[sel], Ps[sel]
    first = (int(np.searchsorted(pl, k0)), int(np.searchsorted(pl, k0 + 1)))
    last = (int(np.searchsorted(pl, k1 - 1)), int(np.searchsorted(pl, k1)))
    lo, hi = D.ghost_rows(torch.as_tensor(rows), first, last, tr)
    exp_lo = Gs[Ps == k0 - 1] if rank > 0 else Gs[:0]
    exp_hi = Gs[Ps == k1] if rank + 1 < world else Gs[:0]
    assert np.array_equal(lo.numpy(), exp_lo), "ghost_lo"
    assert np.array_equal(hi.numpy(), exp_hi), "ghost_hi"
    # owned faces cover every face exactly once
    for comp in range(3):
        nf = [(plan.nx + 1) * plan.ny * plan.nz, plan.nx * (plan.ny + 1) * plan.nz,
              plan.nx * plan.ny * (plan.nz + 1)][comp]
        full = np.arange(nf, dtype=np.float64) * (rank + 1)
        rngs = [D.face_ranges(plan, comp, r) for r in range(world)]
        a, b = rngs[rank]
        parts = tr.allgather_var(torch.as_tensor(full[a:b]), [y - x for x, y in rngs])
        out = np.concatenate([p.numpy() for p in parts])
        exp = np.concatenate([np.arange(x, y) * (r + 1.0) for r, (x, y) in enumerate(rngs)])
        assert out.shape[0] == nf and np.array_equal(out, exp), f"faces comp {comp}"
    # reductions
    t = torch.tensor([3.0 + rank, 1.0 - rank], dtype=torch.float64)
    tr.allreduce_min_(t)
    assert t.tolist() == [3.0, 1.0 - (world - 1)]
    lab = torch.tensor([0, 2, 2, 1], dtype=torch.uint8) if rank == 0 else torch.tensor([0, 1, 2, 2], dtype=torch.uint8)
    tr.allreduce_min_(lab)
    assert lab.tolist() == ([0, 1, 2, 1] if world > 1 else [0, 2, 2, 1])
    assert tr.allreduce_sum_int(rank + 1) == world * (world + 1) // 2
    print(f"rank {rank} ok", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
