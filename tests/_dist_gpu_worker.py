"""Worker for tests/test_dist_gpu.py: the slab-decomposed step on ranks that
share one GPU, exchanging through gloo (host-staged; no kernel waits on
another process).  Rank 0 writes digests of the gathered state after every
step, and every rank's exchange volume, to argv[1]."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
import torch.distributed as dist


def digest(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + a.tobytes()).hexdigest()


def main():
    out_path, case = sys.argv[1], json.loads(sys.argv[2])
    dist.init_process_group("gloo")
    import paper_2404_01931_b200 as P
    from paper_2404_01931_b200 import dist as D
    torch.cuda.set_device(0)
    spec = P.SceneSpec(**case["spec"])
    st = D.make_scene(spec, rng_seed=case["seed"])
    recs, xfer = [], []
    for _ in range(case["steps"]):
        rep = D.step(st, spec)
        xfer.append(D.exchange_stats(st))
        parts = D.gather_particles(st)
        g = D.gather_grid(st)
        rec = {f"part{i}": digest(a) for i, a in enumerate(parts)}
        rec.update({k: digest(g[k]) for k in ("u", "v", "w", "p", "label", "uo", "vo", "wo")})
        rec["count"] = digest(g["count"].astype(np.int64))
        rec.update({"n": int(rep.particle_count), "dt": float(rep.dt).hex(),
                    "its": int(rep.solver_iterations), "res": float(rep.solver_residual).hex(),
                    "conv": bool(rep.solver_converged), "nrows": int(rep.nrows)})
        recs.append(rec)
    every = st.slab.tr.allgather_obj(xfer)
    if dist.get_rank() == 0:
        json.dump({"steps": recs, "exchange": every}, open(out_path, "w"))
    print(f"rank {dist.get_rank()} ok", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
