"""Worker for tests/test_dist_host.py (launched with torch.distributed.run,
gloo, CPU tensors): the slab transport's collectives (the flip_comm
callbacks' tensor-level forms in paper_2404_01931_b200.dist.Transport)
against their specification, and the distributed pairwise dot across real
ranks."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
import torch.distributed as dist


def main():
    dist.init_process_group("gloo")
    from paper_2404_01931_b200 import dist as D
    rank, world = dist.get_rank(), dist.get_world_size()
    tr = D.Transport()
    # neighbours: rank r sends (r, lo) down and (r, hi) up, sizes agree pairwise
    sz = lambda a, b: 3 + a + 2 * b          # bytes from rank a to rank b
    send_lo = torch.full((sz(rank, rank - 1) if rank > 0 else 0,), 10 * rank + 1, dtype=torch.uint8)
    send_hi = torch.full((sz(rank, rank + 1) if rank + 1 < world else 0,), 10 * rank + 2,
                         dtype=torch.uint8)
    recv_lo = torch.zeros(sz(rank - 1, rank) if rank > 0 else 0, dtype=torch.uint8)
    recv_hi = torch.zeros(sz(rank + 1, rank) if rank + 1 < world else 0, dtype=torch.uint8)
    tr.neighbors_t(send_lo, send_hi, recv_lo, recv_hi)
    if rank > 0:
        assert (recv_lo == 10 * (rank - 1) + 2).all(), "neighbors lo"
    if rank + 1 < world:
        assert (recv_hi == 10 * (rank + 1) + 1).all(), "neighbors hi"
    # allreduce MAX / MIN / SUM on int64 (max of non-negative double bits)
    bits = torch.tensor([np.float64(0.5 + rank).view(np.int64)], dtype=torch.int64)
    tr.allreduce_t(bits, D.FLIP_OP_MAX)
    assert bits.numpy().view(np.float64)[0] == 0.5 + world - 1
    t = torch.tensor([7 - rank, rank], dtype=torch.int64)
    tr.allreduce_t(t, D.FLIP_OP_MIN)
    assert t.tolist() == [7 - (world - 1), 0]
    t = torch.tensor([rank + 1], dtype=torch.int64)
    tr.allreduce_t(t, D.FLIP_OP_SUM)
    assert t.item() == world * (world + 1) // 2
    # allgatherv in place, uneven and empty contributions
    sizes = [(5 * q + 3) % 7 for q in range(world)]
    off = np.concatenate([[0], np.cumsum(sizes)]).tolist()
    buf = torch.zeros(off[-1], dtype=torch.uint8)
    buf[off[rank]:off[rank + 1]] = rank + 1
    tr.allgatherv_t(buf, off)
    exp = np.concatenate([np.full(sizes[q], q + 1, dtype=np.uint8) for q in range(world)])
    assert np.array_equal(buf.numpy(), exp), "allgatherv"
    # all-to-all with uneven splits, received in source-rank order
    sb = [(rank + 2 * q) % 4 for q in range(world)]
    send = torch.cat([torch.full((sb[q],), 16 * rank + q, dtype=torch.uint8) for q in range(world)])
    rb = [(q + 2 * rank) % 4 for q in range(world)]
    recv = torch.zeros(sum(rb), dtype=torch.uint8)
    tr.alltoallv_t(send, sb, recv, rb)
    exp = np.concatenate([np.full(rb[q], 16 * q + rank, dtype=np.uint8) for q in range(world)])
    assert np.array_equal(recv.numpy(), exp), "alltoallv"
    # the distributed pairwise dot with real ranks: each rank contributes its
    # piece, the pieces travel with the transport, every rank gets numpy's sum
    rng = np.random.default_rng(11)
    for n in (0, 5, 129, 4099, 100003):
        v = rng.normal(size=n)
        cuts = np.linspace(0, n, world + 1).astype(int)
        pieces = tr.allgather_obj(v[cuts[rank]:cuts[rank + 1]])
        assert D.distributed_pairwise_sum(pieces) == float(np.add.reduce(v)), n
    print(f"rank {rank} ok", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
