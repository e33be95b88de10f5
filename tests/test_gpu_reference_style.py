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


def shell_state(res=8, shell=True, dtau=None):
    """A bare device state like the reference's shell_grid fixture (8^3,
    dtau 1/8, one-cell SOLID shell, every other cell AIR, no particles)."""
    dims = GridDims(res, res, res, 1.0 / res if dtau is None else dtau)
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


# --------------------------------------------------------- test_transfer ----
def _random_parts(n, seed):
    rng = np.random.default_rng(seed)
    pos, vel = rng.random((n, 3)), rng.normal(size=(n, 3))
    return pos, vel


class TestP2G:
    def _p2g(self, pos, vel):
        st = shell_state(6, shell=False)
        set_parts(st, pos, vel)
        stages(st, "bin", "p2g", res=6)
        return st, st.device.known()

    def test_constant_velocity_everywhere(self):            # test_transfer.py:82-93
        pos, vel = _random_parts(500, 1)
        vel[:] = (2.5, -1.0, 0.75)
        st, (ku, kv, kw) = self._p2g(pos, vel)
        u, v, w = (np.array(getattr(st.grid, c)) for c in "uvw")
        assert np.allclose(u[ku], 2.5, atol=1e-12)
        assert np.allclose(v[kv], -1.0, atol=1e-12)
        assert np.allclose(w[kw], 0.75, atol=1e-12)
        assert (u[~ku] == 0).all()

    def test_single_particle_at_face_sample(self):          # test_transfer.py:95-105
        h = 1.0 / 6.0
        st, _ = self._p2g([[2 * h, 2.5 * h, 2.5 * h]], [[3.3, 0.0, 0.0]])
        assert st.grid.u3()[2, 2, 2] == pytest.approx(3.3, rel=1e-15)

    def test_max_principle_per_component(self):             # test_transfer.py:118-124
        pos, vel = _random_parts(2000, 4)
        st, (ku, _, _) = self._p2g(pos, vel)
        u = np.array(st.grid.u)
        assert u[ku].min() >= vel[:, 0].min() - 1e-12
        assert u[ku].max() <= vel[:, 0].max() + 1e-12

    def test_far_particle_contributes_zero(self):           # test_transfer.py:126-136
        st, (ku, _, _) = self._p2g([[0.9, 0.9, 0.9]], [[100.0, 0.0, 0.0]])
        assert not ku.reshape(6, 6, 7)[0, 0, 0]
        assert st.grid.u3()[0, 0, 0] == 0.0


class TestG2P:
    def _state(self, seed_new=5):
        st = shell_state(6, shell=False)
        dev = st.device
        rng = np.random.default_rng(seed_new)
        z = [np.zeros(n) for n in dev.nfaces]
        dev.set_grid(u=rng.normal(size=dev.nfaces[0]), v=z[1], w=z[2])
        dev.set_grid_old(rng.normal(size=dev.nfaces[0]), z[1], z[2])
        return st

    def _g2p(self, st, flip):
        stages(st, "g2p", "g2p", res=6, flip_fraction=flip)

    def test_pure_pic_equals_new_field_sample(self):        # test_transfer.py:147-153
        import oracle as O
        st = self._state()
        pos, vel = _random_parts(100, 6)
        set_parts(st, pos, vel)
        g = st.grid
        expect = O.sample_velocity_many(O.Dimz(6, 6, 6, 1.0 / 6.0), np.array(g.u), np.array(g.v),
                                        np.array(g.w), pos[:, 0], pos[:, 1], pos[:, 2])[0]
        self._g2p(st, 0.0)
        assert np.allclose(st.particles.vel_x, expect, atol=1e-14)

    def test_pure_flip_with_equal_grids_is_identity(self):  # test_transfer.py:155-161
        st = self._state()
        st.device.set_grid_old(np.array(st.grid.u), np.array(st.grid.v), np.array(st.grid.w))
        pos, vel = _random_parts(100, 7)
        set_parts(st, pos, vel)
        self._g2p(st, 1.0)
        assert np.allclose(st.particles.vel_x, vel[:, 0], atol=1e-12)

    def test_blend_arithmetic(self):                        # test_transfer.py:163-172
        st = shell_state(6, shell=False)
        dev = st.device
        z = [np.zeros(n) for n in dev.nfaces]
        dev.set_grid(u=np.full(dev.nfaces[0], 2.0), v=z[1], w=z[2])
        dev.set_grid_old(*z)
        set_parts(st, [[0.5, 0.5, 0.5]], [[4.0, 0.0, 0.0]])
        self._g2p(st, 0.5)
        assert st.particles.vel_x[0] == pytest.approx(4.0, abs=1e-14)

    def test_blend_params_validation(self):                 # test_transfer.py:199-203
        st = self._state()
        for bad in (1.5, -0.1):
            with pytest.raises(ValueError):
                self._g2p(st, bad)


class TestRoundTrip:
    def test_constant_field_recovered_pure_pic(self):       # test_transfer.py:182-196
        st = shell_state(6)
        region = P.SeedRegion.box((1 / 6, 1 / 6, 1 / 6), (5 / 6, 5 / 6, 5 / 6), 2)
        arr = (_lib.Region * 1)(region.to_c())
        _lib.check(_lib.LIB.flip_seed_regions(st.device.ctx, 1, arr, 1))
        st.device.bump()
        c = (1.25, -0.5, 2.0)
        pos = np.stack([np.array(a) for a in st.particles.arrays()[:3]], axis=1)
        set_parts(st, pos, np.tile(c, (len(pos), 1)))
        stages(st, "bin", "p2g", res=6)
        g = st.grid
        st.device.set_grid_old(np.array(g.u), np.array(g.v), np.array(g.w))
        stages(st, "g2p", "g2p", res=6, flip_fraction=0.0)
        p = st.particles
        for comp, arr_ in zip(c, (p.vel_x, p.vel_y, p.vel_z)):
            assert (np.abs(np.asarray(arr_) - comp) / abs(comp)).max() < 1e-6


# --------------------------------------------------------- test_pressure ----
DT, RHO = 0.01, 1000.0
_NB6 = ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1))


def dense_pressure(label3, u3, v3, w3, dtau, dt=DT, rho=RHO):
    """Independent dense restatement of assemble + solve (pressure.py:147-199):
    rows are FLUID cells in flat order; a component that touches no AIR
    loses its lowest-index cell (pinned to zero); out-of-domain is SOLID."""
    from scipy import ndimage
    nz, ny, nx = label3.shape
    fl = label3 == P.FLUID
    comp, ncomp = ndimage.label(fl)
    air = np.pad(label3 == P.AIR, 1)
    near_air = np.zeros_like(fl)
    for di, dj, dk in _NB6:
        near_air |= air[1 + dk:1 + dk + nz, 1 + dj:1 + dj + ny, 1 + di:1 + di + nx]
    flat = np.arange(label3.size).reshape(label3.shape)
    pinned = set()
    for c in range(1, ncomp + 1):
        m = comp == c
        if not (near_air & m).any():
            pinned.add(int(flat[m].min()))
    rows = [int(f) for f in flat[fl] if int(f) not in pinned]
    index = {f: r for r, f in enumerate(rows)}
    scale = dt / (rho * dtau * dtau)
    A = np.zeros((len(rows), len(rows)))
    b = np.zeros(len(rows))
    for r, f in enumerate(rows):
        k, j, i = np.unravel_index(f, label3.shape)
        for di, dj, dk in _NB6:
            a, bb, cc = i + di, j + dj, k + dk
            inside = 0 <= a < nx and 0 <= bb < ny and 0 <= cc < nz
            lab = label3[cc, bb, a] if inside else P.SOLID
            if lab != P.SOLID:
                A[r, r] += scale
            nf = int(flat[cc, bb, a]) if inside else -1
            if lab == P.FLUID and nf in index:
                A[r, index[nf]] -= scale
        b[r] = -(u3[k, j, i + 1] - u3[k, j, i] + v3[k, j + 1, i] - v3[k, j, i]
                 + w3[k + 1, j, i] - w3[k, j, i]) / dtau
    p = np.zeros(label3.size)
    if rows:
        p[rows] = np.linalg.solve(A, b)
    return p, rows, len(pinned)


def grid_state(label3, seed, dtau):
    """Device state with the given labels and random velocities, walls
    enforced (random_mask_grid / single_cell_grid, test_pressure.py:100-120)."""
    n = label3.shape[0]
    st = shell_state(n, shell=False, dtau=dtau)
    dev = st.device
    rng = np.random.default_rng(seed)
    dev.set_grid(label=label3.reshape(-1), u=rng.normal(size=dev.nfaces[0]),
                 v=rng.normal(size=dev.nfaces[1]), w=rng.normal(size=dev.nfaces[2]),
                 p=np.zeros(dev.dims.ncells))
    dev.set_dt(DT)
    if (label3 == P.SOLID).any():
        dev.set_known(*[np.ones(nf, np.uint8) for nf in dev.nfaces])
        stages(st, "apply_gradient", "apply_gradient", res=n, extrapolation_layers=0)
    return st


def random_mask(n, seed, fraction=0.4):
    lab = np.full((n, n, n), P.SOLID, dtype=np.uint8)
    interior = np.full((n - 2,) * 3, P.AIR, dtype=np.uint8)
    interior[np.random.default_rng(seed).random(interior.shape) < fraction] = P.FLUID
    lab[1:-1, 1:-1, 1:-1] = interior
    return lab


def single_cell(neighbors):
    lab = np.full((5, 5, 5), neighbors, dtype=np.uint8)
    lab[2, 2, 2] = P.FLUID
    return lab


def project(st, solver, tol, max_iters, **kw):
    n = st.device.dims.nx
    rep = stages(st, "project", "project", res=n, solver=solver, tol=tol, max_iters=max_iters,
                 **kw)
    return rep, np.array(st.grid.p)


SOLVER_NAMES = ("jacobi", "gs", "rbgs", "pcg")


class TestSolvers:
    @pytest.mark.parametrize("solver", SOLVER_NAMES)
    def test_zero_rhs_zero_solution(self, solver):          # test_pressure.py:187-199
        st = grid_state(single_cell(P.AIR), 0, 0.2)
        z = [np.zeros(n) for n in st.device.nfaces]
        st.device.set_grid(u=z[0], v=z[1], w=z[2])
        rep, p = project(st, solver, 1e-6, 2000)
        assert rep.solver_converged and (p == 0).all()
        assert rep.solver_iterations == (0 if solver == "pcg" else 1)

    @pytest.mark.parametrize("solver", SOLVER_NAMES)
    def test_two_cell_system_matches_dense(self, solver):   # test_pressure.py:201-209
        lab = single_cell(P.AIR)
        lab[2, 2, 3] = P.FLUID
        st = grid_state(lab, 0, 0.2)
        g = st.grid
        x, rows, _ = dense_pressure(lab, g.u3(), g.v3(), g.w3(), 0.2)
        rep, p = project(st, solver, 1e-10, 2000)
        assert rep.solver_converged
        assert np.allclose(p[rows], x[rows], atol=1e-8 * max(1, np.abs(x).max()))

    @pytest.mark.parametrize("solver", SOLVER_NAMES)
    def test_8cubed_random_mask_matches_dense(self, solver):  # test_pressure.py:211-218
        lab = random_mask(8, 7)
        st = grid_state(lab, 8, 1 / 8)
        g = st.grid
        x, rows, _ = dense_pressure(lab, g.u3(), g.v3(), g.w3(), 1 / 8)
        rep, p = project(st, solver, 1e-9, 5000)
        assert rep.solver_converged
        assert (np.abs(p - x) / max(1.0, np.abs(x).max())).max() < 1e-6

    def test_mg_preconditioner_matches_dense(self):         # extension, same bar
        lab = random_mask(16, 21, 0.6)
        st = grid_state(lab, 22, 1 / 16)
        g = st.grid
        x, rows, _ = dense_pressure(lab, g.u3(), g.v3(), g.w3(), 1 / 16)
        rep, p = project(st, "pcg", 1e-9, 500, precond="mg")
        assert rep.solver_converged
        assert (np.abs(p - x) / max(1.0, np.abs(x).max())).max() < 1e-6

    def test_iteration_ordering(self):                      # test_pressure.py:220-236
        its = {}
        for solver in SOLVER_NAMES:
            lab = random_mask(8, 9)
            rep, _ = project(grid_state(lab, 10, 1 / 8), solver, 1e-8,
                             200 if solver == "pcg" else 5000)
            assert rep.solver_converged
            its[solver] = rep.solver_iterations
        assert its["gs"] < its["jacobi"]
        assert its["pcg"] <= its["gs"] and its["pcg"] <= its["rbgs"]

    def test_pcg_single_cell_one_iteration(self):          # test_pressure.py:238-243
        lab = single_cell(P.AIR)
        st = grid_state(lab, 0, 0.2)
        g = st.grid
        x, _, _ = dense_pressure(lab, g.u3(), g.v3(), g.w3(), 0.2)
        rep, p = project(st, "pcg", 1e-6, 100)
        assert rep.solver_converged and rep.solver_iterations == 1
        assert p[P.flat_index(2, 2, 2, st.device.dims)] == pytest.approx(x[62], rel=1e-12)

    def test_convergence_across_random_masks(self):         # test_pressure.py:245-253
        for s in range(20):
            lab = random_mask(6, 100 + s)
            if not (lab == P.FLUID).any():
                continue
            for solver in ("jacobi", "gs"):
                rep, _ = project(grid_state(lab, 101 + s, 1 / 6), solver, 1e-7, 5000)
                assert rep.solver_converged

    def test_sealed_two_cell_component_solvable_after_pinning(self):  # :285-292
        lab = single_cell(P.SOLID)
        lab[2, 2, 3] = P.FLUID
        st = grid_state(lab, 0, 0.2)
        rep, p = project(st, "pcg", 1e-6, 100)
        assert rep.nrows == 1 and rep.npinned == 1 and rep.solver_converged
        assert p[P.flat_index(2, 2, 2, st.device.dims)] == 0.0

    def test_all_four_agree_on_random_masks(self):          # test_pressure.py:341-352
        for s in range(3):
            lab = random_mask(6, 300 + s)
            if not (lab == P.FLUID).any():
                continue
            sols = [project(grid_state(lab, 301 + s, 1 / 6), sv, 1e-8, 8000)[1]
                    for sv in SOLVER_NAMES]
            scale = max(1.0, max(np.abs(q).max() for q in sols))
            for a in sols:
                for b in sols:
                    assert (np.abs(a - b) / scale).max() < 1e-5


class TestApplyGradient:
    def _apply(self, st, p):
        dev = st.device
        dev.set_grid(p=p)
        dev.set_known(*[np.ones(nf, np.uint8) for nf in dev.nfaces])
        stages(st, "apply_gradient", "apply_gradient", res=dev.dims.nx, extrapolation_layers=0)

    def test_uniform_pressure_all_fluid_no_change(self):    # test_pressure.py:296-306
        lab = np.full((5, 5, 5), P.SOLID, dtype=np.uint8)
        lab[1:-1, 1:-1, 1:-1] = P.FLUID
        st = grid_state(lab, 12, 0.2)
        before = np.array(st.grid.u)
        self._apply(st, np.where(lab.reshape(-1) == P.FLUID, 3.7, 0.0))
        assert np.allclose(st.grid.u, before, atol=1e-12)

    def test_two_cell_column_face_update(self):             # test_pressure.py:308-319
        lab = np.full((5, 5, 5), P.AIR, dtype=np.uint8)
        lab[2, 2, 2] = lab[2, 2, 3] = P.FLUID
        st = grid_state(lab, 0, 0.2)
        z = [np.zeros(n) for n in st.device.nfaces]
        st.device.set_grid(u=z[0], v=z[1], w=z[2])
        p = np.zeros(125)
        p.reshape(5, 5, 5)[2, 2, 3] = 50.0
        self._apply(st, p)
        assert st.grid.u3()[2, 2, 3] == pytest.approx(-DT / RHO * 50.0 / 0.2)

    def test_solid_adjacent_faces_zeroed(self):             # test_pressure.py:321-326
        st = grid_state(random_mask(6, 13), 14, 1 / 6)
        self._apply(st, np.zeros(216))
        u3 = st.grid.u3()
        assert np.all(u3[:, :, :2] == 0) and np.all(u3[:, :, -2:] == 0)

    def test_projection_kills_divergence(self):             # test_pressure.py:328-338
        lab = random_mask(8, 14)
        st = grid_state(lab, 15, 1 / 8)
        fl = (lab.reshape(-1) == P.FLUID)
        rhs_max = max(1.0, np.abs(P.divergence_field(st)[fl]).max())
        tol = 1e-8
        rep = stages(st, "project", "project", res=8, tol=tol, max_iters=500)
        assert rep.solver_converged
        self._apply(st, np.array(st.grid.p))
        div = P.divergence_field(st)
        assert np.abs(div[fl]).max() <= 100 * tol * rhs_max


# ---------------------------------------------------------- test_binning ----
class TestBinParticles:
    def _bin(self, pos):
        st = shell_state(6, shell=False)
        set_parts(st, pos)
        stages(st, "bin", "classify", res=6)
        return st

    def test_single_cell_keeps_order(self):                 # test_binning.py:98-107
        pos = 0.05 + np.random.default_rng(3).random((20, 3)) * 0.05
        st = self._bin(pos)
        assert np.array_equal(st.particles.pos_x, pos[:, 0])
        assert st.hash.offset[0] == 0 and st.hash.count[0] == 20
        assert np.asarray(st.hash.fluid_cells).tolist() == [0]

    def test_empty_set(self):                               # test_binning.py:109-112
        st = self._bin(np.zeros((0, 3)))
        assert st.particles.count == 0
        assert int(np.asarray(st.hash.count).sum()) == 0 and len(st.hash.fluid_cells) == 0

    def test_matches_stable_sort_byte_identical(self):      # test_binning.py:114-121
        pos, vel = _random_parts(10**5, 5)
        st = shell_state(6, shell=False)
        set_parts(st, pos, vel)
        stages(st, "bin", "classify", res=6)
        i, j, k = (np.minimum(np.floor(pos[:, a] * 6).astype(np.int64), 5) for a in range(3))
        perm = np.argsort(i + 6 * (j + 6 * k), kind="stable")
        want = np.concatenate([pos, vel], axis=1)[perm]
        for a, got in enumerate(st.particles.arrays()):
            assert np.asarray(got).tobytes() == np.ascontiguousarray(want[:, a]).tobytes()

    def test_hash_invariants(self):                         # test_binning.py:123-139
        pos, _ = _random_parts(5000, 6)
        st = self._bin(pos)
        h = st.hash
        cnt, off = np.asarray(h.count), np.asarray(h.offset)
        assert np.array_equal(off[1:], np.cumsum(cnt)[:-1]) and off[0] == 0
        assert off[-1] + cnt[-1] == st.particles.count
        assert np.array_equal(h.fluid_cells, np.flatnonzero(cnt > 0))
        assert np.array_equal(np.sort(st.particles.pos_x), np.sort(pos[:, 0]))
        p = st.particles
        i, j, k = (np.minimum(np.floor(np.asarray(a) * 6).astype(np.int64), 5)
                   for a in (p.pos_x, p.pos_y, p.pos_z))
        cells = i + 6 * (j + 6 * k)
        for c in np.asarray(h.fluid_cells)[:50]:
            assert (cells[h.segment(int(c))] == c).all()


def test_particle_buffers_grow_past_initial_capacity():
    """The reference's ParticleSet has no capacity; the device context grows
    its particle buffers on set/seed, keeping live particles."""
    dims = GridDims(8, 8, 8, 1.0 / 8)
    dev = Device(dims, capacity=16)
    _lib.check(_lib.LIB.flip_set_solid_shell(dev.ctx))
    pos, vel = _random_parts(40, 11)
    pos = 0.125 + pos * 0.75
    dev.set_particles([*pos.T, *vel.T])
    region = P.SeedRegion.box((0.125, 0.125, 0.125), (0.5, 0.5, 0.5), 2)
    _lib.check(_lib.LIB.flip_seed_regions(dev.ctx, 1, (_lib.Region * 1)(region.to_c()), 3))
    dev.bump()
    parts = dev.particles()
    assert len(parts[0]) == 40 + 27 * 8
    assert np.array_equal(parts[0][:40], pos[:, 0]) and np.array_equal(parts[3][:40], vel[:, 0])
    st = sim.SimState(grid=MacGrid(dev, "grid"),
                      grid_old=MacGrid(dev, "old", np.zeros(dims.ncells),
                                       np.array(dev.grid_array("label"))),
                      particles=ParticleSet(device=dev), hash=SpaceHash(device=dev), device=dev)
    P.step(st, small_spec(res=8))
    assert int(np.asarray(st.hash.count).sum()) == st.particles.count


def test_solver_api_independent_of_call_order():
    """Standalone solves with different n back to back (the fused dot's
    scratch must not carry state from an earlier call)."""
    for n, seed in ((8, 1), (6, 2), (8, 3), (5, 4), (8, 5)):
        lab = random_mask(n, seed)
        if not (lab == P.FLUID).any():
            continue
        st = grid_state(lab, seed + 50, 1.0 / n)
        g = st.grid
        x, _, _ = dense_pressure(lab, g.u3(), g.v3(), g.w3(), 1.0 / n)
        for pre in ("jacobi", "mic0", "none"):
            rep, p = project(st, "pcg", 1e-10, 500, precond=pre)
            assert rep.solver_converged
            assert (np.abs(p - x) / max(1.0, np.abs(x).max())).max() < 1e-6


def test_reseed_grows_past_user_capacity():
    """A capacity below the 12-per-cell bound: reseed grows the buffers
    instead of writing past them, and matches the default-capacity run."""
    dims = GridDims(8, 8, 8, 1.0 / 8)
    region = P.SeedRegion.box((0.125, 0.125, 0.125), (0.625, 0.625, 0.625), 1)
    outs = []
    for cap in (64, 0):
        dev = Device(dims, capacity=cap)
        _lib.check(_lib.LIB.flip_set_solid_shell(dev.ctx))
        _lib.check(_lib.LIB.flip_seed_regions(dev.ctx, 1, (_lib.Region * 1)(region.to_c()), 4))
        dev.bump()
        st = sim.SimState(grid=MacGrid(dev, "grid"),
                          grid_old=MacGrid(dev, "old", np.zeros(dims.ncells),
                                           np.array(dev.grid_array("label"))),
                          particles=ParticleSet(device=dev), hash=SpaceHash(device=dev),
                          device=dev)
        spec = small_spec(res=8, density=2)
        sim.run_stages(st, spec, "bin", "classify")
        assert st.particles.count == 64
        sim.run_stages(st, spec, "reseed", "reseed")
        assert st.particles.count == 64 * 8 > 64
        assert int(np.asarray(st.hash.count).sum()) == st.particles.count
        outs.append([np.array(a) for a in st.particles.arrays()])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
