"""Host-side logic of the drop-in API (runs on CPU): scene construction
mirrors flipsim.sim.scene_regions / _fit_box exactly (checked against the
oracle's restatement, which the golden fixtures pin to the reference)."""

import numpy as np
import pytest

import oracle as O


CASES = [dict(name="dam-break", res=12), dict(name="dam-break", res=256),
         dict(name="double-dam-break", res=16), dict(name="double-dam-break", res=511),
         dict(name="water-drop", res=16), dict(name="water-drop", res=64),
         dict(name="dam-break", res=32, particle_target=100_000),
         dict(name="double-dam-break", res=64, particle_target=500_000),
         dict(name="water-drop", res=32, particle_target=60_000)]


@pytest.mark.parametrize("c", CASES, ids=[str(c) for c in CASES])
def test_scene_regions_match_oracle(pkg, c):
    spec = pkg.SceneSpec(**c)
    ospec = O.Spec(**c)
    dims = pkg.GridDims(spec.res, spec.res, spec.res, 1.0 / spec.res)
    odims = O.Dimz(spec.res, spec.res, spec.res, 1.0 / spec.res)
    mine = pkg.scene_regions(spec, dims)
    ref = O.scene_regions(ospec, odims)
    assert len(mine) == len(ref)
    for a, b in zip(mine, ref):
        assert a.kind == b.kind and a.density == b.density
        assert tuple(a.a) == tuple(b.a)
        assert (tuple(a.b) if a.kind == "box" else a.b) == (tuple(b.b) if b.kind == "box" else b.b)


def test_particle_target_within_5_percent(pkg):
    # test_sim.py:70-73: the fitted box lands within 5% of the target
    spec = pkg.SceneSpec(name="dam-break", res=32, particle_target=100_000)
    dims = pkg.GridDims(32, 32, 32, 1 / 32)
    (r,) = pkg.scene_regions(spec, dims)
    cells = pkg.particles.covered_cells(r, dims)
    assert abs(len(cells) * r.density ** 3 - 100_000) <= 5_000


def test_flat_index_and_coords(pkg):
    d = pkg.GridDims(4, 4, 4, 1.0)
    assert pkg.flat_index(0, 0, 0, d) == 0 and pkg.flat_index(1, 0, 0, d) == 1
    assert pkg.flat_index(3, 3, 3, d) == 63
    d8 = pkg.GridDims(8, 8, 8, 1.0)
    seen = {pkg.flat_index(i, j, k, d8) for k in range(8) for j in range(8) for i in range(8)}
    assert seen == set(range(512))
    assert all(pkg.cell_coords(pkg.flat_index(i, j, k, d8), d8) == (i, j, k)
               for (i, j, k) in [(0, 0, 0), (3, 2, 1), (7, 7, 7)])


def test_grid_dims_validation(pkg):
    with pytest.raises(ValueError):
        pkg.GridDims(0, 4, 4, 1.0)
    with pytest.raises(ValueError):
        pkg.GridDims(4, 4, 4, 0.0)


def test_seed_region_validation(pkg):
    with pytest.raises(ValueError):
        pkg.SeedRegion("cone", (0, 0, 0), 1.0)
    with pytest.raises(ValueError):
        pkg.SeedRegion.box((0, 0, 0), (1, 1, 1), 0)


def test_host_particle_set_energy(pkg):
    # test_sim.py:154-172 on a host-side ParticleSet
    ps = pkg.ParticleSet(np.array([0.3]), np.array([0.125]), np.array([0.3]),
                         np.zeros(1), np.zeros(1), np.zeros(1))
    assert pkg.total_energy(ps, (0, -9.81, 0), floor_y=0.125) == 0.0
    ps = pkg.ParticleSet(np.array([0.0]), np.array([1.0]), np.array([0.0]),
                         np.zeros(1), np.zeros(1), np.zeros(1))
    assert pkg.total_energy(ps, (0, -9.81, 0), floor_y=0.25) == pytest.approx(9.81 * 0.75)
    assert pkg.total_energy(pkg.ParticleSet.empty(), (0, -9.81, 0)) == 0.0


def test_params_match_reference_host_arithmetic(pkg):
    from paper_2404_01931_b200 import sim
    spec = pkg.SceneSpec(res=48)
    dtau = 1.0 / 48
    p = sim._params(spec, dtau, 5)
    assert p.alpha_dtau_h == spec.alpha * dtau
    assert p.rho_dtau2_h == spec.rho_fluid * dtau ** 2
    assert p.rho_dtau_h == spec.rho_fluid * dtau
    assert p.skin_h == spec.skin_fraction * dtau
    assert p.max_iters == 100
    with pytest.raises(ValueError):
        sim._params(pkg.SceneSpec(flip_fraction=1.5), dtau)
    with pytest.raises(pkg.ConfigError):
        sim._params(pkg.SceneSpec(solver="multigrid"), dtau)
    assert sim._params(spec, dtau).advection == 0                    # forward Euler default
    assert sim._params(pkg.SceneSpec(advection="rk2"), dtau).advection == 1
    with pytest.raises(pkg.ConfigError):
        sim._params(pkg.SceneSpec(advection="rk4"), dtau)
