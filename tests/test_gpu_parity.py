"""GPU parity: the CUDA step against the CPU oracle, bit for bit.

The oracle (oracle/flip_oracle.c) is itself pinned to the reference
(tests/test_oracle_pins.py).  Everything here compares raw bytes: labels,
hash counts/offsets, particle order and every float64 field.
"""

import numpy as np
import pytest

import oracle as O
from helpers import device_arrays, diff_report, oracle_arrays, spec_pair, upload

pytestmark = pytest.mark.gpu

STEP_CASES = [
    dict(name="dam-break", res=12, solver="pcg"),
    dict(name="dam-break", res=16, solver="jacobi"),
    dict(name="double-dam-break", res=16, solver="rbgs"),
    dict(name="water-drop", res=16, solver="gs"),
    dict(name="dam-break", res=24, solver="pcg"),
    dict(name="water-drop", res=20, solver="pcg", particle_target=20000),
    dict(name="dam-break", res=20, solver="pcg", precond="jacobi"),
    dict(name="double-dam-break", res=18, solver="pcg", precond="none", flip_fraction=0.0),
    dict(name="double-dam-break-obstacle", res=24, solver="pcg"),
    dict(name="water-drop", res=20, solver="rbgs", obstacles=((3, 6, 1, 3, 3, 16), (12, 14, 2, 8, 5, 9))),
    # extension: RK2 (explicit midpoint through the grid) vs orc_advect_rk2
    dict(name="dam-break", res=16, solver="pcg", advection="rk2"),
    dict(name="double-dam-break-obstacle", res=20, solver="jacobi", advection="rk2"),
]


def _ids(c):
    return "-".join(f"{v}" for v in c.values())


@pytest.mark.parametrize("case", STEP_CASES, ids=[_ids(c) for c in STEP_CASES])
def test_make_scene_and_steps_bit_exact(pkg, case):
    dspec, ospec = spec_pair(**case)
    st = pkg.make_scene(dspec, rng_seed=3)
    os_ = O.make_scene(ospec, rng_seed=3)
    assert dspec.density == ospec.density
    bad = diff_report(device_arrays(st), oracle_arrays(os_))
    assert not bad, f"make_scene: {bad}"
    for k in range(5):
        rep = pkg.step(st, dspec)
        ref = O.step(os_, ospec)
        bad = diff_report(device_arrays(st), oracle_arrays(os_))
        assert not bad, f"step {k}: {bad}"
        assert rep.dt == ref["dt"]
        assert rep.particle_count == ref["particle_count"]
        assert rep.solver_iterations == ref["solver_iterations"]
        assert rep.solver_residual == ref["solver_residual"]
        assert rep.solver_converged == ref["solver_converged"]
        assert st.time == os_.time and st.step_count == os_.step_count


def _stage_snapshots(os_, ospec):
    snaps = {"start": os_.copy()}
    extras = {}

    def hook(name, st, extra):
        snaps[name] = st.copy()
        extras[name] = extra

    O.step(os_, ospec, hook=hook)
    return snaps, extras


@pytest.mark.parametrize("case", STEP_CASES[:5], ids=[_ids(c) for c in STEP_CASES[:5]])
def test_each_stage_bit_exact(pkg, case):
    """Upload the oracle's state before each stage, run that stage alone on
    the device, compare with the oracle's state after it."""
    dspec, ospec = spec_pair(**case)
    st = pkg.make_scene(dspec, rng_seed=5)
    os_ = O.make_scene(ospec, rng_seed=5)
    for _ in range(2):  # get off the degenerate all-zero first step
        O.step(os_, ospec)
    snaps, extras = _stage_snapshots(os_, ospec)
    dt = extras["dt_compute"]["dt"]
    known = extras["p2g"]["known"]
    order = ["start"] + list(O.STAGES)
    for prev, name in zip(order[:-1], order[1:]):
        before = snaps[prev].copy()
        after = snaps[name]
        if name == "apply_gradient":
            sys_, res = extras["project"]["system"], extras["project"]["result"]
            before.p = O.pressure_field(sys_, res["p"], before.dims.ncells)
        st.step_count = before.step_count
        upload(st, before, dt=None if name == "dt_compute" else dt,
               known=known if name == "apply_gradient" else None)
        rep = pkg.run_stages(st, dspec, name, name)
        ref = oracle_arrays(after)
        if name == "project":  # the device writes p = pressure_field(x) here
            sys_, res = extras["project"]["system"], extras["project"]["result"]
            ref["p"] = O.pressure_field(sys_, res["p"], after.dims.ncells)
            assert rep.solver_iterations == res["iterations"]
            assert rep.solver_residual == res["residual"]
            assert rep.nrows == sys_.nrows
        if name == "advect":
            # the device fuses cell_index + bincount into advect, so count
            # already holds the BIN stage's histogram of the moved particles
            cells = np.empty(after.n, dtype=np.int64)
            O.lib().orc_cell_index_many(after.dims.c(), after.n, O._p(after.parts[0]),
                                        O._p(after.parts[1]), O._p(after.parts[2]),
                                        O._p(cells, O._i64))
            ref["count"] = np.bincount(cells, minlength=after.dims.ncells)
        bad = diff_report(device_arrays(st), ref)
        assert not bad, f"stage {name}: {bad}"
        if name == "dt_compute":
            assert st.device.dt() == dt
        if name == "p2g":
            got = st.device.known()
            for g, k in zip(got, known):
                assert np.array_equal(g, k.astype(bool))


def test_gpu_reseed_fast_path_keeps_state(pkg):
    """A rest state with zero gravity is a bit-exact fixed point (test_sim.py:69-77)."""
    dspec, _ = spec_pair(name="dam-break", res=12, gravity=(0.0, 0.0, 0.0))
    st = pkg.make_scene(dspec, rng_seed=2)
    before = [a.tobytes() for a in st.particles.arrays()]
    rep = pkg.step(st, dspec)
    assert [a.tobytes() for a in st.particles.arrays()] == before
    assert rep.dt == dspec.dt_max
    assert not st.particles.vel_x.any() and not st.particles.vel_y.any()


def test_post_step_divergence_small(pkg):
    """Projection leaves max|div| <= 1e-4 over FLUID cells (test_sim.py:79-86)."""
    dspec, _ = spec_pair(name="dam-break", res=16)
    st = pkg.make_scene(dspec, rng_seed=3)
    for _ in range(3):
        pkg.step(st, dspec)
        div = pkg.divergence_field(st)
        fluid = st.grid.label == pkg.FLUID
        assert np.abs(div[fluid]).max() <= 1e-4


def test_hash_accounts_for_every_particle(pkg):
    dspec, _ = spec_pair(name="dam-break", res=12)
    st = pkg.make_scene(dspec, rng_seed=6)
    pkg.step(st, dspec)
    assert st.hash.count.sum() == st.particles.count
    assert np.array_equal(st.hash.fluid_cells, np.flatnonzero(st.hash.count > 0))


def test_energy_matches_oracle_pairwise(pkg):
    dspec, ospec = spec_pair(name="dam-break", res=16)
    st = pkg.make_scene(dspec, rng_seed=1)
    os_ = O.make_scene(ospec, rng_seed=1)
    for _ in range(3):
        pkg.step(st, dspec)
        O.step(os_, ospec)
    e_dev = pkg.total_energy(st.particles, dspec.gravity, pkg.energy_floor(st))
    P = os_.parts
    g = float(np.linalg.norm(np.asarray(dspec.gravity)))
    floor = 1.0 / 16
    e_ref = (0.5 * float(np.add.reduce(P[3] ** 2 + P[4] ** 2 + P[5] ** 2))
             + g * float(np.add.reduce(P[1] - floor)))
    assert e_dev == e_ref


@pytest.mark.parametrize("case", [dict(name="dam-break", res=128, solver="pcg"),
                                  dict(name="double-dam-break-obstacle", res=96, solver="pcg")],
                         ids=["dam-break-128", "double-dam-break-obstacle-96"])
def test_multicluster_sweep_bit_exact(pkg, case):
    """The MIC(0) sweep with more than one 4x4 cluster of 16x16 tiles (rows
    spanning > 64 cells in y or z): tile faces then also cross clusters
    through the global halo (helper polls, selective halo prep), a path the
    small cases above never reach."""
    dspec, ospec = spec_pair(**case)
    st = pkg.make_scene(dspec, rng_seed=1)
    os_ = O.make_scene(ospec, rng_seed=1)
    lab = np.asarray(st.grid.label).reshape(case["res"], case["res"], case["res"])
    k, j, _ = np.nonzero(lab == pkg.FLUID)
    assert max(np.ptp(j), np.ptp(k)) + 1 > 64
    for step in range(2):
        rep = pkg.step(st, dspec)
        ref = O.step(os_, ospec)
        bad = diff_report(device_arrays(st), oracle_arrays(os_))
        assert not bad, f"step {step}: {bad}"
        assert rep.solver_iterations == ref["solver_iterations"]
        assert rep.solver_residual == ref["solver_residual"]


def test_full_size_steps_bit_exact(pkg):
    """BASELINE's full size: the 256^3 dam-break (24.7M particles) make_scene
    and three steps, every byte equal to the oracle's after each step.  Step 1
    starts from zero velocities (advect and the P2G values are trivial);
    steps 2 and 3 exercise advect, binning of moved particles, P2G, the FLIP
    blend and reseed on non-degenerate data at the BASELINE size."""
    dspec, ospec = spec_pair(name="dam-break", res=256, solver="pcg")
    st = pkg.make_scene(dspec, rng_seed=0)
    os_ = O.make_scene(ospec, rng_seed=0)
    assert st.particles.count == os_.parts[0].size > 24_000_000
    for k in range(3):
        rep = pkg.step(st, dspec)
        ref = O.step(os_, ospec)
        bad = diff_report(device_arrays(st), oracle_arrays(os_))
        assert not bad, f"256^3 step {k + 1}: {bad}"
        assert rep.dt == ref["dt"]
        assert rep.particle_count == ref["particle_count"]
        assert rep.solver_iterations == ref["solver_iterations"]
        assert rep.solver_residual == ref["solver_residual"]
        if k:
            assert np.abs(st.particles.vel_y).max() > 0      # non-degenerate


def test_full_size_step_from_oracle_state(pkg):
    """One device step from the ORACLE's 256^3 state after step 2 (uploaded),
    compared with the oracle's step 3: the device step is checked on the
    reference's own non-degenerate input, independently of its own history."""
    dspec, ospec = spec_pair(name="dam-break", res=256, solver="pcg")
    os_ = O.make_scene(ospec, rng_seed=0)
    for _ in range(2):
        O.step(os_, ospec)
    st = pkg.make_scene(dspec, rng_seed=0)
    for _ in range(2):                       # step_count / time / reseed stream
        st.step_count += 1
    st.time = os_.time
    upload(st, os_)
    rep = pkg.step(st, dspec)
    ref = O.step(os_, ospec)
    bad = diff_report(device_arrays(st), oracle_arrays(os_))
    assert not bad, f"256^3 step 3 from the oracle state: {bad}"
    assert rep.solver_iterations == ref["solver_iterations"]
    assert rep.solver_residual == ref["solver_residual"]


def test_divergence_field_bit_exact(pkg):
    """divergence_field (grid.py:147-156) on the device == the oracle's
    orc_divergence_field, byte for byte, on scene states after each step."""
    dspec, ospec = spec_pair(name="double-dam-break-obstacle", res=24, solver="pcg")
    st = pkg.make_scene(dspec, rng_seed=2)
    os_ = O.make_scene(ospec, rng_seed=2)
    for k in range(3):
        pkg.step(st, dspec)
        O.step(os_, ospec)
        want = O.divergence_field(os_.dims, os_.u, os_.v, os_.w)
        got = pkg.divergence_field(st)
        assert got.tobytes() == want.tobytes(), f"step {k}"


@pytest.mark.parametrize("n,seed", [(8, 7), (8, 14), (12, 300)])
def test_divergence_field_reference_golden(pkg, n, seed):
    """The device divergence of the reference tests' random velocity fields
    against the digests produced by the real reference (make_golden.py)."""
    from golden_util import digest, load
    from test_oracle_pins import random_mask_velocities
    dims, u, v, w, label = random_mask_velocities(n, seed)
    dspec, _ = spec_pair(name="dam-break", res=n)
    st = pkg.make_scene(dspec, rng_seed=0)
    st.device.set_grid(u=u, v=v, w=w, label=label)
    want = load("reference_kernels.json")["kernels"][f"divergence_{n}_seed{seed}"]
    assert digest(pkg.divergence_field(st)) == want


@pytest.mark.slow
def test_config4_512_obstacle_bit_exact(pkg):
    """BASELINE config 4's scene at full size: double-dam-break + obstacle at
    512^3 (399M particles), make_scene and one step, every byte equal to the
    oracle's (all host threads; several minutes).  Selected with -m slow."""
    import os
    O.set_threads(os.cpu_count() or 1)
    dspec, ospec = spec_pair(name="double-dam-break-obstacle", res=512, solver="pcg")
    st = pkg.make_scene(dspec, rng_seed=0, capacity=int(1.5 * 8 * 0.21 * 512 ** 3) + 4096)
    os_ = O.make_scene(ospec, rng_seed=0)
    assert st.particles.count == os_.n == 398_991_360
    bad = diff_report(device_arrays(st), oracle_arrays(os_))
    assert not bad, f"make_scene: {bad}"
    rep = pkg.step(st, dspec)
    ref = O.step(os_, ospec)
    bad = diff_report(device_arrays(st), oracle_arrays(os_))
    assert not bad, f"512^3 step: {bad}"
    assert rep.solver_iterations == ref["solver_iterations"]
    assert rep.solver_residual == ref["solver_residual"]


def test_config2_jacobi_128_bit_exact(pkg):
    """BASELINE config 2: dam-break 128^3 with solver="jacobi" (cap 2000),
    make_scene and one step, every byte equal to the oracle's."""
    dspec, ospec = spec_pair(name="dam-break", res=128, solver="jacobi")
    st = pkg.make_scene(dspec, rng_seed=0)
    os_ = O.make_scene(ospec, rng_seed=0)
    assert st.particles.count == 3_032_064
    rep = pkg.step(st, dspec)
    ref = O.step(os_, ospec)
    bad = diff_report(device_arrays(st), oracle_arrays(os_))
    assert not bad, f"128^3 jacobi step: {bad}"
    assert rep.solver_iterations == ref["solver_iterations"]
    assert rep.solver_residual == ref["solver_residual"]
    assert rep.solver_converged == ref["solver_converged"]


def test_config1_64_hundred_steps_bit_exact(pkg):
    """BASELINE config 1 (`flipsim run --res 64 --steps 100`): 100 steps of
    the 64^3 dam-break, state compared every 10 steps -- no drift."""
    dspec, ospec = spec_pair(name="dam-break", res=64, solver="pcg")
    st = pkg.make_scene(dspec, rng_seed=0)
    os_ = O.make_scene(ospec, rng_seed=0)
    assert st.particles.count == 365_056
    for k in range(100):
        rep = pkg.step(st, dspec)
        ref = O.step(os_, ospec)
        assert rep.solver_iterations == ref["solver_iterations"], k
        if k % 10 == 9:
            bad = diff_report(device_arrays(st), oracle_arrays(os_))
            assert not bad, f"step {k}: {bad}"
