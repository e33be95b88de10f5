"""The reference's own behavioural tests (flipsim tests/test_sim.py,
test_particles.py, test_grid.py), restated against the device
implementation: scene setup, stepping invariants, advect, reseed thresholds,
classification, body force, solid boundaries and extrapolation.  Each test
names the reference test it mirrors.  The stages run on the GPU through
``run_stages``; states are set through the Device setters, so these exercise
the same kernels as a full step."""
import numpy as np
import pytest

import paper_2404_01931_b200 as P
from paper_2404_01931_b200 import _lib, sim
from paper_2404_01931_b200.binning import SpaceHash
from paper_2404_01931_b200.device import Device
from paper_2404_01931_b200.grid import GridDims, MacGrid
from paper_2404_01931_b200.particles import ParticleSet

pytestmark = pytest.mark.gpu


def small_spec(**kw):
    base = dict(name="dam-break", res=12, steps=1)
    base.update(kw)
    return P.SceneSpec(**base)


def shell_state(res=8, shell=True):
    """A bare device state like the reference's shell_grid fixture (8^3,
    dtau 1/8, one-cell SOLID shell, every other cell AIR, no particles)."""
    dims = GridDims(res, res, res, 1.0 / res)
    dev = Device(dims)
    if shell:
        _lib.check(_lib.LIB.flip_set_solid_shell(dev.ctx))
    dev.bump()
    old_p = np.zeros(dims.ncells)
    old_label = np.array(dev.grid_array("label"))
    return sim.SimState(grid=MacGrid(dev, "grid"), grid_old=MacGrid(dev, "old", old_p, old_label),
                        particles=ParticleSet(device=dev), hash=SpaceHash(device=dev), device=dev)


def set_parts(st, pos, vel=None):
    pos = np.asarray(pos, dtype=np.float64).reshape(-1, 3)
    vel = np.zeros_like(pos) if vel is None else np.asarray(vel, dtype=np.float64).reshape(-1, 3)
    st.device.set_particles([pos[:, 0], pos[:, 1], pos[:, 2], vel[:, 0], vel[:, 1], vel[:, 2]])


def stages(st, first, last, **kw):
    return sim.run_stages(st, small_spec(**kw), first, last)


def snapshot(st):
    return [np.array(a) for a in st.particles.arrays()]


# ------------------------------------------------------------- test_sim ----
class TestScene:
    def test_same_spec_identical_states(self):              # test_sim.py:61-65
        a = P.make_scene(small_spec(), rng_seed=9)
        b = P.make_scene(small_spec(), rng_seed=9)
        for x, y in zip(snapshot(a), snapshot(b)):
            assert np.array_equal(x, y)
        assert np.array_equal(a.grid.label, b.grid.label)

    def test_dam_break_against_wall(self):                  # test_sim.py:30-38
        spec = small_spec()
        st = P.make_scene(spec, rng_seed=1)
        assert st.particles.count > 0
        i = st.hash.fluid_cells % spec.res
        assert i.min() == 1 and i.max() < spec.res // 2

    def test_double_dam_break_two_mirrored_boxes(self):     # test_sim.py:56-60
        spec = small_spec(name="double-dam-break")
        i = P.make_scene(spec).hash.fluid_cells % spec.res
        assert i.min() == 1 and i.max() == spec.res - 2

    def test_water_drop_pool_and_sphere(self):              # test_sim.py:45-54
        spec = small_spec(name="water-drop", res=16)
        st = P.make_scene(spec)
        pool, sphere = P.scene_regions(spec, st.device.dims)
        from paper_2404_01931_b200.particles import covered_cells
        pc = set(covered_cells(pool, st.device.dims).tolist())
        sc = set(covered_cells(sphere, st.device.dims).tolist())
        assert pc and sc and not pc & sc

    def test_particle_target_within_5_percent(self):        # test_sim.py:40-43
        st = P.make_scene(P.SceneSpec(name="dam-break", res=32, particle_target=100_000))
        assert abs(st.particles.count - 100_000) <= 5_000


class TestStep:
    def test_rest_state_zero_gravity_fixed_point(self):     # test_sim.py:69-77
        spec = small_spec(gravity=(0.0, 0.0, 0.0))
        st = P.make_scene(spec, rng_seed=2)
        before = snapshot(st)
        rep = P.step(st, spec)
        for x, y in zip(before, snapshot(st)):
            assert np.array_equal(x, y)
        assert not np.any(st.particles.vel_x) and not np.any(st.particles.vel_y)
        assert rep.dt == spec.dt_max

    def test_post_step_divergence_small(self):              # test_sim.py:79-86
        spec = small_spec(res=16, steps=3)
        st = P.make_scene(spec, rng_seed=3)
        for _ in range(3):
            P.step(st, spec)
            fluid = np.asarray(st.grid.label) == P.FLUID
            assert np.abs(P.divergence_field(st)[fluid]).max() <= 1e-4

    def test_determinism_across_runs(self):                 # test_sim.py:88-96
        snaps = []
        for _ in range(2):
            spec = small_spec(steps=10)
            st = P.make_scene(spec, rng_seed=5)
            for _ in range(10):
                P.step(st, spec)
            snaps.append(snapshot(st))
        for x, y in zip(*snaps):
            assert np.array_equal(x, y)

    def test_hash_accounts_for_every_particle(self):        # test_sim.py:98-105
        spec = small_spec()
        st = P.make_scene(spec, rng_seed=6)
        P.step(st, spec)
        assert int(np.asarray(st.hash.count).sum()) == st.particles.count

    def test_stage_timings_nonnegative_and_complete(self):  # test_sim.py:107-114
        spec = small_spec()
        st = P.make_scene(spec, rng_seed=7)
        rep = P.step(st, spec)
        d = rep.timings.as_dict()
        assert set(d) == set(P.StageTimings.stage_names())
        assert all(v >= 0 for v in d.values())
        assert rep.timings.total() == pytest.approx(sum(d.values()))

    def test_time_advances_by_dt(self):                     # test_sim.py:116-121
        spec = small_spec()
        st = P.make_scene(spec, rng_seed=8)
        rep = P.step(st, spec)
        assert st.time == rep.dt and st.step_count == 1


# -------------------------------------------------------- test_particles ----
class TestAdvect:
    def _advect(self, st, dt, skin_fraction):
        st.device.set_dt(dt)
        stages(st, "advect", "advect", skin_fraction=skin_fraction)

    def test_zero_velocity_fixed(self):                     # test_particles.py:196-201
        st = shell_state()
        pos = np.array([[0.5, 0.5, 0.5], [0.3, 0.6, 0.2]])
        set_parts(st, pos)
        self._advect(st, 0.5, 1e-4 * 8)
        assert np.array_equal(st.particles.pos_x, pos[:, 0])
        assert np.array_equal(st.particles.pos_y, pos[:, 1])

    def test_forward_euler_arithmetic(self):                # test_particles.py:203-208
        dims = GridDims(8, 8, 8, 1.0)
        dev = Device(dims)          # open grid: every cell AIR
        st = sim.SimState(grid=MacGrid(dev, "grid"),
                          grid_old=MacGrid(dev, "old", np.zeros(dims.ncells),
                                           np.array(dev.grid_array("label"))),
                          particles=ParticleSet(device=dev), hash=SpaceHash(device=dev),
                          device=dev)
        set_parts(st, [[1.0, 1.0, 1.0]], [[2.0, 0.0, 0.0]])
        dev.set_dt(0.5)
        sim.run_stages(st, P.SceneSpec(res=8, skin_fraction=1e-3), "advect", "advect")
        p = st.particles
        assert (p.pos_x[0], p.pos_y[0], p.pos_z[0]) == (2.0, 1.0, 1.0)

    def test_wall_clamp_exact_skin(self):                   # test_particles.py:210-215
        st = shell_state()
        skin = 1e-3 * (1.0 / 8)
        set_parts(st, [[0.5, 0.5, 0.5]], [[10.0, 0.0, 0.0]])
        self._advect(st, 1.0, 1e-3)
        assert st.particles.pos_x[0] == 0.875 - skin
        assert st.particles.pos_y[0] == 0.5

    def test_no_particle_in_solid_after_advect(self):       # test_particles.py:217-225
        st = shell_state()
        rng = np.random.default_rng(8)
        set_parts(st, 0.125 + rng.random((200, 3)) * 0.75, rng.normal(size=(200, 3)) * 5.0)
        self._advect(st, 0.1, 1e-4 * 8)
        p = st.particles
        i, j, k = (np.floor(np.asarray(a) * 8).astype(np.int64) for a in (p.pos_x, p.pos_y, p.pos_z))
        cells = i + 8 * (j + 8 * k)
        assert (np.asarray(st.grid.label)[cells] != P.SOLID).all()


class TestReseed:
    def _seeded(self, density=2):
        st = shell_state()
        spec = small_spec(res=8, density=density)
        regions = [P.SeedRegion.box((0.125, 0.125, 0.125), (0.5, 0.5, 0.5), density)]
        arr = (_lib.Region * 1)(*[r.to_c() for r in regions])
        _lib.check(_lib.LIB.flip_seed_regions(st.device.ctx, 1, arr, 5))
        st.device.bump()
        sim.run_stages(st, spec, "bin", "classify")
        return st, spec

    def _reseed(self, st, spec, seed):
        p = sim._params(spec, st.device.dims.dtau, seed)
        rc, rep = st.device.run_stages(p, _lib.STAGE["reseed"], _lib.STAGE["reseed"])
        _lib.check(rc)
        return rep

    def _rebin(self, st, spec, keep):
        arrs = [np.asarray(a)[keep] for a in st.particles.arrays()]
        st.device.set_particles(arrs)
        sim.run_stages(st, spec, "bin", "classify")

    def test_cell_within_thresholds_unchanged(self):        # test_particles.py:80-87
        st, spec = self._seeded()
        before = snapshot(st)
        cnt0 = np.array(st.hash.count)
        self._reseed(st, spec, 10)
        for x, y in zip(before, snapshot(st)):
            assert np.array_equal(x, y)
        assert np.array_equal(np.array(st.hash.count), cnt0)

    def test_underfull_fluid_cell_refilled_to_density_cubed(self):  # :89-102
        st, spec = self._seeded()
        cell = int(st.hash.fluid_cells[0])
        off, cnt = int(st.hash.offset[cell]), int(st.hash.count[cell])
        keep = np.ones(st.particles.count, dtype=bool)
        keep[off + 1:off + cnt] = False
        self._rebin(st, spec, keep)
        assert int(st.hash.count[cell]) == 1
        self._reseed(st, spec, 11)
        assert int(st.hash.count[cell]) == 8

    def test_overfull_cell_culled_to_max_keeping_lowest_indices(self):  # :104-118
        st = shell_state()
        spec = small_spec(res=8)
        pos = np.tile([0.4, 0.4, 0.4], (20, 1))
        pos[:, 1] += np.linspace(0.001, 0.02, 20)
        set_parts(st, pos)
        sim.run_stages(st, spec, "bin", "classify")
        cell = int(st.hash.fluid_cells[0])
        assert int(st.hash.count[cell]) == 20
        marker = np.array(st.particles.pos_y[:P.MAX_PER_CELL])
        self._reseed(st, spec, 12)
        assert int(st.hash.count[cell]) == P.MAX_PER_CELL
        assert np.array_equal(np.array(st.particles.pos_y), marker)

    def test_new_particles_sample_grid_velocity(self):      # :120-137
        st, spec = self._seeded()
        d = st.device.dims
        st.device.set_grid(u=np.full(st.device.nfaces[0], 1.5), v=np.full(st.device.nfaces[1], -0.5),
                           w=np.full(st.device.nfaces[2], 0.25))
        cell = int(st.hash.fluid_cells[3])
        off, cnt = int(st.hash.offset[cell]), int(st.hash.count[cell])
        keep = np.ones(st.particles.count, dtype=bool)
        keep[off + 2:off + cnt] = False
        self._rebin(st, spec, keep)
        self._reseed(st, spec, 13)
        vx = np.array(st.particles.vel_x)
        new = vx != 0
        assert new.sum() == 6
        assert np.allclose(vx[new], 1.5, atol=1e-12)
        assert np.allclose(np.array(st.particles.vel_y)[new], -0.5, atol=1e-12)

    def test_counts_land_in_thresholds_when_target_inside(self):  # :147-159
        st, spec = self._seeded()
        keep = np.random.default_rng(0).random(st.particles.count) > 0.8
        self._rebin(st, spec, keep)
        self._reseed(st, spec, 15)
        cnt = np.array(st.hash.count)
        occ = cnt[cnt > 0]
        assert (occ >= P.MIN_PER_CELL).all() and (occ <= P.MAX_PER_CELL).all()
        assert int(cnt.sum()) == st.particles.count


# ------------------------------------------------------------- test_grid ----
class TestClassify:
    def test_all_zero_counts_no_fluid(self):                # test_grid.py:123-125
        st = shell_state()
        set_parts(st, np.zeros((0, 3)))
        stages(st, "bin", "classify", res=8)
        assert not (np.asarray(st.grid.label) == P.FLUID).any()

    def test_single_occupied_cell(self):                    # test_grid.py:127-131
        st = shell_state()
        set_parts(st, np.tile([3.5 / 8, 3.5 / 8, 3.5 / 8], (5, 1)))
        stages(st, "bin", "classify", res=8)
        lab = np.asarray(st.grid.label)
        cell = P.flat_index(3, 3, 3, st.device.dims)
        assert lab[cell] == P.FLUID and (lab == P.FLUID).sum() == 1

    def test_solid_cells_never_change(self):                # test_grid.py:133-137
        st = shell_state()
        set_parts(st, np.tile([0.5 / 8, 3.5 / 8, 3.5 / 8], (9, 1)))
        stages(st, "bin", "classify", res=8)
        assert np.asarray(st.grid.label)[P.flat_index(0, 3, 3, st.device.dims)] == P.SOLID


class TestBodyForceAndWalls:
    def _random(self, st, seed):
        r = np.random.default_rng(seed)
        st.device.set_grid(**{c: r.normal(size=n) for c, n in zip("uvw", st.device.nfaces)})

    def test_zero_gravity_no_change_on_interior(self):      # test_grid.py:140-145
        st = shell_state()
        self._random(st, 1)
        st.device.set_dt(0.1)
        before = [np.array(st.grid.u), np.array(st.grid.v)]
        stages(st, "force", "force", res=8, gravity=(0.0, 0.0, 0.0))
        u3 = np.array(st.grid.u).reshape(8, 8, 9)
        assert np.array_equal(u3[3:5, 3:5, 3:5], before[0].reshape(8, 8, 9)[3:5, 3:5, 3:5])

    def test_gravity_applied_to_v_only(self):               # test_grid.py:147-155
        st = shell_state()
        self._random(st, 2)
        st.device.set_dt(0.1)
        u0, v0 = np.array(st.grid.u).reshape(8, 8, 9), np.array(st.grid.v).reshape(8, 9, 8)
        w0 = np.array(st.grid.w).reshape(9, 8, 8)
        stages(st, "force", "force", res=8, gravity=(0.0, -9.81, 0.0))
        u3, v3 = np.array(st.grid.u).reshape(8, 8, 9), np.array(st.grid.v).reshape(8, 9, 8)
        assert np.array_equal(u3[3:5, 3:5, 3:5], u0[3:5, 3:5, 3:5])
        assert np.allclose(v3[3:5, 3:5, 3:5], v0[3:5, 3:5, 3:5] - 0.981, atol=1e-12)
        w3 = np.array(st.grid.w).reshape(9, 8, 8)
        assert np.array_equal(w3[3:5, 3:5, 3:5], w0[3:5, 3:5, 3:5])

    def test_domain_wall_faces_zeroed_and_idempotent(self):  # test_grid.py:158-179
        st = shell_state()
        self._random(st, 3)
        st.device.set_dt(0.1)
        stages(st, "force", "force", res=8, gravity=(0.0, 0.0, 0.0))
        u3 = np.array(st.grid.u).reshape(8, 8, 9)
        v3 = np.array(st.grid.v).reshape(8, 9, 8)
        w3 = np.array(st.grid.w).reshape(9, 8, 8)
        assert np.all(u3[:, :, :2] == 0) and np.all(u3[:, :, -2:] == 0)
        assert np.all(v3[:, :2, :] == 0) and np.all(v3[:, -2:, :] == 0)
        assert np.all(w3[:2, :, :] == 0) and np.all(w3[-2:, :, :] == 0)
        once = [np.array(getattr(st.grid, c)) for c in "uvw"]
        stages(st, "force", "force", res=8, gravity=(0.0, 0.0, 0.0))
        for a, c in zip(once, "uvw"):
            assert np.array_equal(a, np.array(getattr(st.grid, c)))


class TestExtrapolation:
    def test_fills_two_layers_from_known(self):             # test_grid.py:182-197
        st = shell_state()
        dev = st.device
        u = np.zeros(dev.nfaces[0])
        u.reshape(8, 8, 9)[4, 4, 4] = 7.0
        dev.set_grid(u=u, v=np.zeros(dev.nfaces[1]), w=np.zeros(dev.nfaces[2]),
                     p=np.zeros(dev.dims.ncells))
        dev.set_grid_old(np.zeros(dev.nfaces[0]), np.zeros(dev.nfaces[1]), np.zeros(dev.nfaces[2]))
        ku = np.zeros(dev.nfaces[0], dtype=np.uint8)
        ku.reshape(8, 8, 9)[4, 4, 4] = 1
        dev.set_known(ku, np.ones(dev.nfaces[1], np.uint8), np.ones(dev.nfaces[2], np.uint8))
        dev.set_dt(0.01)
        stages(st, "apply_gradient", "apply_gradient", res=8, extrapolation_layers=2)
        u3 = np.array(st.grid.u).reshape(8, 8, 9)
        assert u3[4, 4, 5] == 7.0 and u3[4, 4, 3] == 7.0      # layer 1
        assert u3[4, 4, 6] == 7.0 and u3[4, 5, 5] == 7.0      # layer 2
        assert u3[4, 4, 7] == 0.0                              # beyond fill depth
        assert u3[4, 6, 4] == 7.0 and u3[4, 7, 4] == 0.0       # wall row stays zero
