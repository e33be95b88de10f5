"""Worker for tests/test_dist_gpu.py: the slab-decomposed step on ranks that
share one GPU, exchanging through gloo (host-staged; no kernel waits on
another process).  Rank 0 writes digests of the gathered state after every
step to argv[1]."""
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
    recs = []
    for _ in range(case["steps"]):
        rep = D.step(st, spec)
        parts = D.gather_particles(st)
        g, go = st.grid, st.grid_old
        rec = {f"part{i}": digest(a) for i, a in enumerate(parts)}
        rec.update({k: digest(getattr(g, k)) for k in ("u", "v", "w", "p", "label")})
        rec.update({"uo": digest(go.u), "vo": digest(go.v), "wo": digest(go.w)})
        rec.update({"n": int(rep.particle_count), "dt": float(rep.dt).hex(),
                    "its": int(rep.solver_iterations), "res": float(rep.solver_residual).hex()})
        recs.append(rec)
    if dist.get_rank() == 0:
        json.dump(recs, open(out_path, "w"))
    print(f"rank {dist.get_rank()} ok", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
