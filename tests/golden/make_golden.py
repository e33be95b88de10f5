"""Generate golden fixtures from the REAL reference (flipsim, Cython backend).

Run in the build container (needs /root/reference):
    python tests/golden/make_golden.py

Writes tests/golden/reference_steps.json: for each case, SHA-256 digests of
every state array (grid u/v/w/p/label, grid_old u/v/w, hash count/offset,
six particle arrays) after make_scene and after each of the first steps,
plus the StepReport scalars; and tests/golden/reference_kernels.json with
digests of the kernel-level API outputs on the seeded inputs of the
reference's own tests (test_binning.py, test_transfer.py, test_pressure.py).
The oracle (oracle/flip_oracle.c) must reproduce every digest bit for bit
(tests/test_oracle_pins.py), and the GPU must reproduce the oracle
(tests/test_gpu_*.py).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

CASES = [
    dict(name="dam-break", res=12, solver="pcg", seed=3, steps=4),
    dict(name="dam-break", res=16, solver="jacobi", seed=3, steps=3),
    dict(name="double-dam-break", res=16, solver="rbgs", seed=3, steps=3),
    dict(name="water-drop", res=16, solver="gs", seed=3, steps=3),
    dict(name="water-drop", res=20, solver="pcg", seed=1, steps=3, particle_target=20000),
    dict(name="dam-break", res=32, solver="pcg", seed=0, steps=3),
    dict(name="dam-break", res=12, solver="pcg", seed=2, steps=2, gravity=(0.0, 0.0, 0.0)),
    dict(name="double-dam-break", res=20, solver="pcg", seed=7, steps=3, flip_fraction=0.0),
    # scene extension: the reference scene with SOLID boxes
    # injected into its labels after make_scene (the seeding never touches them)
    dict(name="double-dam-break-obstacle", res=20, solver="pcg", seed=2, steps=3),
    dict(name="dam-break", res=16, solver="jacobi", seed=4, steps=2,
         obstacles=((8, 10, 1, 5, 4, 11),)),
]


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + a.tobytes()).hexdigest()


def ref_state_digests(st) -> dict:
    g, go = st.grid, st.grid_old
    out = {k: digest(getattr(g, k)) for k in ("u", "v", "w", "p", "label")}
    out.update({"uo": digest(go.u), "vo": digest(go.v), "wo": digest(go.w),
                "count": digest(st.hash.count.astype(np.int64)),
                "offset": digest(st.hash.offset.astype(np.int64))})
    for i, a in enumerate(st.particles.arrays()):
        out[f"part{i}"] = digest(a)
    out["n"] = int(st.particles.count)
    return out


def case_key(c) -> str:
    return ",".join(f"{k}={v}" for k, v in sorted(c.items()))


def main():
    import ref_loader
    ref_loader.load()
    from flipsim import _kernels
    from flipsim import sim as RS
    _kernels.set_workers(os.cpu_count() or 1)

    steps_out = {}
    for c in CASES:
        kw = {k: v for k, v in c.items() if k not in ("seed", "steps", "obstacles")}
        boxes = []
        if kw["name"] == "double-dam-break-obstacle" or c.get("obstacles"):
            import oracle as O
            boxes = O.scene_obstacles(O.Spec(**{k: v for k, v in c.items()
                                                if k not in ("seed", "steps")}), None)
            if kw["name"] == "double-dam-break-obstacle":
                kw["name"] = "double-dam-break"
        spec = RS.SceneSpec(**kw)
        st = RS.make_scene(spec, rng_seed=c["seed"])
        if boxes:
            lab = st.grid.label3()
            for i0, i1, j0, j1, k0, k1 in boxes:
                lab[k0:k1 + 1, j0:j1 + 1, i0:i1 + 1] = 0      # SOLID (grid.py:17)
        rec = {"density": spec.density, "states": [ref_state_digests(st)], "reports": []}
        for _ in range(c["steps"]):
            r = RS.step(st, spec)
            rec["states"].append(ref_state_digests(st))
            rec["reports"].append({"dt": r.dt.hex() if isinstance(r.dt, float) else float(r.dt).hex(),
                                   "particle_count": r.particle_count,
                                   "solver_iterations": r.solver_iterations,
                                   "solver_residual": float(r.solver_residual).hex(),
                                   "solver_converged": bool(r.solver_converged)})
        steps_out[case_key(c)] = rec
        print("case", case_key(c), "ok")
    json.dump({"generator": "tests/golden/make_golden.py", "reference": "flipsim 0.1.0 cython",
               "cases": steps_out}, open(os.path.join(HERE, "reference_steps.json"), "w"),
              indent=1)

    # ---- kernel-level goldens (inputs = the reference tests' seeded inputs)
    from flipsim._kernels import _core as K
    from flipsim.binning import bin_particles, cell_index_many
    from flipsim.grid import (GridDims, MacGrid, divergence_field, enforce_solid_boundaries,
                              set_solid_shell, FLUID)
    from flipsim.particles import ParticleSet
    from flipsim.pressure import assemble, SOLVERS, solve_pcg
    import functools

    kout = {}
    dims = GridDims(6, 6, 6, 1.0 / 6.0)

    def random_set(n, seed):
        rng = np.random.default_rng(seed)
        pos = rng.random((n, 3))
        vel = rng.normal(size=(n, 3))
        return ParticleSet(pos[:, 0].copy(), pos[:, 1].copy(), pos[:, 2].copy(),
                           vel[:, 0].copy(), vel[:, 1].copy(), vel[:, 2].copy())

    # test_binning.py:114-121 input (10^5 particles, seed 5)
    ps = random_set(10 ** 5, 5)
    ps, h = bin_particles(ps, dims)
    kout["bin_1e5_seed5"] = {f"part{i}": digest(a) for i, a in enumerate(ps.arrays())}
    kout["bin_1e5_seed5"]["count"] = digest(h.count.astype(np.int64))
    # test_transfer.py:106-116 input (1000 particles, seed 3)
    ps = random_set(1000, 3)
    ps, h = bin_particles(ps, dims)
    for comp in range(3):
        vel = ps.arrays()[3 + comp]
        vals, w = K.p2g_component(comp, vel, ps.pos_x, ps.pos_y, ps.pos_z, h.offset, h.count,
                                  6, 6, 6, 1.0 / 6.0, 0.0, 0.0, 0.0, 1)
        kout[f"p2g_1000_seed3_comp{comp}"] = {"values": digest(vals), "weights": digest(w)}
    # sample_velocity_many on random fields (seed 23, test_grid.py:145-151 style)
    rng = np.random.default_rng(23)
    u = rng.normal(size=7 * 6 * 6)
    v = rng.normal(size=6 * 7 * 6)
    w = rng.normal(size=6 * 6 * 7)
    pos = rng.random((500, 3)) * 1.4 - 0.2
    sv = K.sample_velocity_many(u, v, w, 6, 6, 6, 1.0 / 6.0, 0.0, 0.0, 0.0,
                                pos[:, 0].copy(), pos[:, 1].copy(), pos[:, 2].copy(), 1)
    kout["sample_500_seed23"] = {f"v{i}": digest(a) for i, a in enumerate(sv)}

    # pressure systems: random masks (test_pressure.py:98-109, seeds 7 and 14)
    def random_mask_grid(n, seed):
        r = np.random.default_rng(seed)
        g = MacGrid(GridDims(n, n, n, 1.0 / n))
        set_solid_shell(g)
        lab = g.label3()
        mask = r.random(lab[1:-1, 1:-1, 1:-1].shape) < 0.4
        lab[1:-1, 1:-1, 1:-1][mask] = FLUID
        r2 = np.random.default_rng(seed + 1)
        g.u[:] = r2.normal(size=g.u.shape)
        g.v[:] = r2.normal(size=g.v.shape)
        g.w[:] = r2.normal(size=g.w.shape)
        enforce_solid_boundaries(g)
        return g

    for n, seed in ((8, 7), (8, 14), (12, 300)):
        g = random_mask_grid(n, seed)
        sys_ = assemble(g, 0.01, 1000.0)
        key = f"system_{n}_seed{seed}"
        rec = {"nrows": sys_.nrows, "cells": digest(sys_.cells.astype(np.int64)),
               "nbr_rows": digest(sys_.nbr_rows.astype(np.int64)), "diag": digest(sys_.diag),
               "rhs": digest(sys_.rhs), "scale": float(sys_.scale).hex(),
               "pinned": digest(sys_.pinned.astype(np.int64))}
        pc = K.mic0_build(sys_.diag, sys_.nbr_rows, sys_.scale, 0.97, 0.25, 1)
        rec["mic0_build"] = digest(pc)
        rec["mic0_apply_rhs"] = digest(K.mic0_apply(pc, sys_.nbr_rows, sys_.rhs, sys_.scale, 1))
        for solver in ("jacobi", "gs", "rbgs", "pcg"):
            res = SOLVERS[solver](sys_, 400, 1e-9)
            rec[f"solve_{solver}"] = {"p": digest(res.p), "iterations": res.iterations,
                                      "residual": float(res.residual).hex(),
                                      "converged": bool(res.converged)}
        for pre in ("jacobi", "none"):
            res = solve_pcg(sys_, 400, 1e-9, precond=pre)
            rec[f"solve_pcg_{pre}"] = {"p": digest(res.p), "iterations": res.iterations,
                                       "residual": float(res.residual).hex(),
                                       "converged": bool(res.converged)}
        kout[key] = rec
        # divergence_field (grid.py:147-156) of the same random velocity field
        kout[f"divergence_{n}_seed{seed}"] = digest(divergence_field(g))
    # divergence_field of a scene state after two steps (non-trivial u/v/w)
    spec = RS.SceneSpec(name="dam-break", res=20, solver="pcg")
    st = RS.make_scene(spec, rng_seed=6)
    for _ in range(2):
        RS.step(st, spec)
    kout["divergence_dam_break_20_seed6_step2"] = {"grid": digest(divergence_field(st.grid)),
                                                   "u": digest(st.grid.u)}
    json.dump({"generator": "tests/golden/make_golden.py", "kernels": kout},
              open(os.path.join(HERE, "reference_kernels.json"), "w"), indent=1)
    print("wrote goldens")


if __name__ == "__main__":
    main()
