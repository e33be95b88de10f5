"""Stage-by-stage comparison of the slab step with the 1-GPU step (debug).
    python -m torch.distributed.run --nproc-per-node 3 --master-addr 127.0.0.1 \
        tools/dist_stage_debug.py '{"name": "dam-break", "res": 64, "solver": "pcg"}' 0 2
runs STEPS full steps, then the next step stage by stage; rank 0 reports
the first stage whose gathered state differs from the 1-GPU state."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch
import torch.distributed as dist


def main():
    spec_kw, seed, steps = json.loads(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    dist.init_process_group("gloo")
    import paper_2404_01931_b200 as P
    from paper_2404_01931_b200 import dist as D, _lib, rng
    from paper_2404_01931_b200 import sim as S
    torch.cuda.set_device(0)
    rank = dist.get_rank()
    spec = P.SceneSpec(**spec_kw)
    st = D.make_scene(spec, rng_seed=seed)
    ref = P.make_scene(spec, seed) if rank == 0 else None
    for _ in range(steps):
        D.step(st, spec)
        if ref is not None:
            P.step(ref, spec)
    seed3 = rng.derive_seed(st.rng_seed, st.step_count + 1)
    params = S._params(spec, st.device.dims.dtau, seed3)
    for s in range(_lib.NSTAGES):
        rc, rep = st.device.run_stages(params, s, s)
        assert rc == 0, (s, rc)
        g = D.gather_grid(st)
        parts = D.gather_particles(st)
        if ref is not None:
            rc2, rep2 = ref.device.run_stages(params, s, s)
            e = {"u": ref.grid.u, "v": ref.grid.v, "w": ref.grid.w, "p": ref.grid.p,
                 "label": ref.grid.label, "uo": ref.grid_old.u, "vo": ref.grid_old.v,
                 "wo": ref.grid_old.w, "count": np.asarray(ref.hash.count)}
            bad = [k for k in e if np.asarray(e[k]).tobytes() != np.asarray(g[k]).astype(np.asarray(e[k]).dtype).tobytes()]
            pb = [i for i, (a, b) in enumerate(zip(parts, ref.particles.arrays())) if a.tobytes() != b.tobytes()]
            extra = ""
            if s == 6:
                extra = f" its {rep.solver_iterations}/{rep2.solver_iterations} res {rep.solver_residual.hex()}/{rep2.solver_residual.hex()} rows {rep.nrows}/{rep2.nrows}"
                for k in ("p",):
                    a, b = np.asarray(g[k]), np.asarray(e[k])
                    d = np.flatnonzero(a != b)
                    if len(d):
                        nxy = spec.res * spec.res
                        extra += f" {k}: {len(d)} differ, planes {sorted(set((d // nxy).tolist()))[:20]}"
            print(f"stage {_lib.STAGE_NAMES[s]}: grid {bad or 'OK'} particles {pb or 'OK'}{extra}", flush=True)
            ref.device.bump()
        st.device.bump()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
