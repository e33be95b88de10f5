"""The CPU oracle against golden fixtures produced by the REAL reference
(tests/golden/make_golden.py), bit for bit, plus direct checks against the
reference when its sources are present (build container only)."""

import os

import numpy as np
import pytest

import oracle as O
from golden_util import load, oracle_digests, parse_case, report_tuple

STEPS = load("reference_steps.json")["cases"]
KERN = load("reference_kernels.json")["kernels"]


@pytest.mark.parametrize("key", sorted(STEPS))
def test_oracle_steps_match_reference_digests(key):
    c = parse_case(key)
    seed, steps = c.pop("seed"), c.pop("steps")
    spec = O.Spec(**c)
    st = O.make_scene(spec, rng_seed=seed)
    want = STEPS[key]
    assert spec.density == want["density"]
    assert oracle_digests(st) == want["states"][0], "make_scene"
    for k in range(steps):
        r = O.step(st, spec)
        assert oracle_digests(st) == want["states"][k + 1], f"step {k}"
        rep = want["reports"][k]
        got = report_tuple(r["dt"], r["particle_count"], r["solver_iterations"],
                           r["solver_residual"], r["solver_converged"])
        assert got == (rep["dt"], rep["particle_count"], rep["solver_iterations"],
                       rep["solver_residual"], rep["solver_converged"])


def _random_set(n, seed):
    rng = np.random.default_rng(seed)
    pos = rng.random((n, 3))
    vel = rng.normal(size=(n, 3))
    return [pos[:, 0].copy(), pos[:, 1].copy(), pos[:, 2].copy(),
            vel[:, 0].copy(), vel[:, 1].copy(), vel[:, 2].copy()]


def test_oracle_binning_and_p2g_match_reference():
    from golden_util import digest
    dims = O.Dimz(6, 6, 6, 1.0 / 6.0)
    parts, count, offset = O.bin_particles(dims, _random_set(10 ** 5, 5))
    g = KERN["bin_1e5_seed5"]
    assert {f"part{i}": digest(a) for i, a in enumerate(parts)} == \
        {k: v for k, v in g.items() if k != "count"}
    assert digest(count) == g["count"]
    parts, count, offset = O.bin_particles(dims, _random_set(1000, 3))
    for comp in range(3):
        vals, w = O.p2g_component(dims, comp, parts[3 + comp], parts[0], parts[1], parts[2],
                                  offset, count)
        assert digest(vals) == KERN[f"p2g_1000_seed3_comp{comp}"]["values"]
        assert digest(w) == KERN[f"p2g_1000_seed3_comp{comp}"]["weights"]


def test_oracle_sampling_matches_reference():
    from golden_util import digest
    rng = np.random.default_rng(23)
    u = rng.normal(size=7 * 6 * 6)
    v = rng.normal(size=6 * 7 * 6)
    w = rng.normal(size=6 * 6 * 7)
    pos = rng.random((500, 3)) * 1.4 - 0.2
    out = O.sample_velocity_many(O.Dimz(6, 6, 6, 1.0 / 6.0), u, v, w, pos[:, 0], pos[:, 1],
                                 pos[:, 2])
    assert {f"v{i}": digest(a) for i, a in enumerate(out)} == KERN["sample_500_seed23"]


def random_mask_system(n, seed):
    dims = O.Dimz(n, n, n, 1.0 / n)
    u, v, w, p, label = O.empty_grid(dims)
    O.solid_shell(dims, label)
    r = np.random.default_rng(seed)
    lab = label.reshape(n, n, n)
    mask = r.random(lab[1:-1, 1:-1, 1:-1].shape) < 0.4
    inner = lab[1:-1, 1:-1, 1:-1]
    inner[mask] = O.FLUID
    r2 = np.random.default_rng(seed + 1)
    u[:], v[:], w[:] = r2.normal(size=u.size), r2.normal(size=v.size), r2.normal(size=w.size)
    O.enforce(dims, label, u, v, w)
    return O.assemble(dims, label, u, v, w, 0.01, 1000.0)


@pytest.mark.parametrize("n,seed", [(8, 7), (8, 14), (12, 300)])
def test_oracle_assembly_and_solvers_match_reference(n, seed):
    from golden_util import digest
    sys_ = random_mask_system(n, seed)
    g = KERN[f"system_{n}_seed{seed}"]
    assert sys_.nrows == g["nrows"]
    assert digest(sys_.cells) == g["cells"]
    assert digest(sys_.nbr_rows) == g["nbr_rows"]
    assert digest(sys_.diag) == g["diag"] and digest(sys_.rhs) == g["rhs"]
    assert float(sys_.scale).hex() == g["scale"]
    assert digest(sys_.pinned) == g["pinned"]
    nb = sys_.nbr_rows.reshape(-1)
    pc = np.empty(sys_.nrows)
    O.lib().orc_mic0_build(sys_.nrows, O._p(sys_.diag), O._p(nb, O._i64), sys_.scale, 0.97, 0.25,
                           O._p(pc))
    assert digest(pc) == g["mic0_build"]
    z = np.empty(sys_.nrows)
    O.lib().orc_mic0_apply(sys_.nrows, O._p(pc), O._p(nb, O._i64), O._p(sys_.rhs), sys_.scale,
                           O._p(np.empty(sys_.nrows)), O._p(z))
    assert digest(z) == g["mic0_apply_rhs"]
    for solver in ("jacobi", "gs", "rbgs", "pcg"):
        r = O.solve(sys_, solver, 400, 1e-9)
        want = g[f"solve_{solver}"]
        assert (digest(r["p"]), r["iterations"], float(r["residual"]).hex(), r["converged"]) == \
            (want["p"], want["iterations"], want["residual"], want["converged"]), solver
    for pre in ("jacobi", "none"):
        r = O.solve(sys_, "pcg", 400, 1e-9, pre)
        want = g[f"solve_pcg_{pre}"]
        assert (digest(r["p"]), r["iterations"], float(r["residual"]).hex(), r["converged"]) == \
            (want["p"], want["iterations"], want["residual"], want["converged"]), pre


def random_mask_velocities(n, seed):
    """The random velocity field of random_mask_system (before assembly)."""
    dims = O.Dimz(n, n, n, 1.0 / n)
    u, v, w, p, label = O.empty_grid(dims)
    O.solid_shell(dims, label)
    r = np.random.default_rng(seed)
    lab = label.reshape(n, n, n)
    mask = r.random(lab[1:-1, 1:-1, 1:-1].shape) < 0.4
    lab[1:-1, 1:-1, 1:-1][mask] = O.FLUID
    r2 = np.random.default_rng(seed + 1)
    u[:], v[:], w[:] = r2.normal(size=u.size), r2.normal(size=v.size), r2.normal(size=w.size)
    O.enforce(dims, label, u, v, w)
    return dims, u, v, w, label


@pytest.mark.parametrize("n,seed", [(8, 7), (8, 14), (12, 300)])
def test_oracle_divergence_matches_reference(n, seed):
    """orc_divergence_field == flipsim.grid.divergence_field (grid.py:147-156)."""
    from golden_util import digest
    dims, u, v, w, _ = random_mask_velocities(n, seed)
    assert digest(O.divergence_field(dims, u, v, w)) == KERN[f"divergence_{n}_seed{seed}"]


def test_oracle_divergence_after_steps_matches_reference():
    from golden_util import digest
    spec = O.Spec(name="dam-break", res=20, solver="pcg")
    st = O.make_scene(spec, rng_seed=6)
    for _ in range(2):
        O.step(st, spec)
    g = KERN["divergence_dam_break_20_seed6_step2"]
    assert digest(st.u) == g["u"]
    assert digest(O.divergence_field(st.dims, st.u, st.v, st.w)) == g["grid"]


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 127, 128, 129, 1000, 8193, 100003, 1_000_001])
def test_pairwise_sum_is_numpy_add_reduce(n):
    rng = np.random.default_rng(n)
    a = rng.normal(size=n) * np.exp(rng.normal(size=n) * 5)
    b = rng.normal(size=n)
    assert O.lib().orc_pairwise_dot(n, O._p(a), O._p(b)) == float(np.add.reduce(a * b))


def test_rng_known_values():
    # splitmix64-finalised Weyl counter (flipsim/rng.py:19-41)
    from paper_2404_01931_b200 import rng
    assert rng.derive_seed(123, 0) == O.derive_seed(123, 0)
    d = [O.derive_seed(123, s) for s in range(100)]
    assert len(set(d)) == 100
    full = rng.uniform01(7, np.arange(100), 3)
    assert full[57] == rng.uniform01(7, 57, 3)
    assert all(O.lib().orc_uniform01(7, s, 3) == full[s] for s in range(100))


def test_threads_do_not_change_oracle_results():
    spec = O.Spec(name="dam-break", res=16)
    outs = []
    for t in (1, max(2, os.cpu_count() or 2)):
        O.set_threads(t)
        st = O.make_scene(spec, 4)
        for _ in range(2):
            O.step(st, spec)
        outs.append(oracle_digests(st))
    O.set_threads(os.cpu_count() or 1)
    assert outs[0] == outs[1]


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src/flipsim"),
                    reason="reference sources only exist in the build container")
def test_oracle_equals_live_reference_40cubed():
    import ref_loader
    ref_loader.load()
    from flipsim import sim as RS
    rspec = RS.SceneSpec(name="dam-break", res=40)
    ospec = O.Spec(name="dam-break", res=40)
    rs = RS.make_scene(rspec, 0)
    os_ = O.make_scene(ospec, 0)
    from golden_util import digest
    for _ in range(3):
        RS.step(rs, rspec)
        O.step(os_, ospec)
    for a, b in zip(rs.particles.arrays(), os_.parts):
        assert a.tobytes() == b.tobytes()
    assert rs.grid.p.tobytes() == os_.p.tobytes()


def test_oracle_rk2_is_midpoint_through_the_grid():
    """orc_advect_rk2 (extension) against a numpy restatement on a random
    grid: k1 = sample(p), m = p + k1*(dt/2), k2 = sample(m), p' = clamp(p + k2*dt)."""
    dims = O.Dimz(6, 5, 7, 1.0 / 8.0)
    rng = np.random.default_rng(4)
    u = rng.normal(size=7 * 5 * 7)
    v = rng.normal(size=6 * 6 * 7)
    w = rng.normal(size=6 * 5 * 8)
    n = 300
    P = [rng.random(n) * (m / 8.0) for m in (6, 5, 7)] + [np.zeros(n)] * 3
    lo, hi, dt, skin = np.array([0.125] * 3), np.array([0.625, 0.5, 0.75]), 0.05, 1e-4
    k1 = O.sample_velocity_many(dims, u, v, w, *P[:3])
    m = [P[a] + k1[a] * (0.5 * dt) for a in range(3)]
    k2 = O.sample_velocity_many(dims, u, v, w, *m)
    want = []
    for a in range(3):
        q = P[a] + k2[a] * dt
        q = np.where(q <= lo[a], lo[a] + skin, np.where(q >= hi[a], hi[a] - skin, q))
        want.append(q)
    got = [a.copy() for a in P[:3]]
    O.lib().orc_advect_rk2(O.C.byref(dims.c()), O._p(u), O._p(v), O._p(w), n, O._p(got[0]),
                           O._p(got[1]), O._p(got[2]), dt, O._p(lo), O._p(hi), skin)
    for a in range(3):
        assert got[a].tobytes() == want[a].tobytes()
