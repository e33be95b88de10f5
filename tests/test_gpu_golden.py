"""The CUDA step against the REAL reference's digests (tests/golden/), bit
for bit: labels, hash, particle order, every float64 field, StepReport."""

import pytest

from golden_util import device_digests, load, parse_case, report_tuple

pytestmark = pytest.mark.gpu
STEPS = load("reference_steps.json")["cases"]


@pytest.mark.parametrize("key", sorted(STEPS))
def test_device_steps_match_reference_digests(pkg, key):
    c = parse_case(key)
    seed, steps = c.pop("seed"), c.pop("steps")
    spec = pkg.SceneSpec(**c)
    st = pkg.make_scene(spec, rng_seed=seed)
    want = STEPS[key]
    assert spec.density == want["density"]
    assert device_digests(st) == want["states"][0], "make_scene"
    for k in range(steps):
        r = pkg.step(st, spec)
        assert device_digests(st) == want["states"][k + 1], f"step {k}"
        rep = want["reports"][k]
        assert report_tuple(r.dt, r.particle_count, r.solver_iterations, r.solver_residual,
                            r.solver_converged) == (rep["dt"], rep["particle_count"],
                                                    rep["solver_iterations"],
                                                    rep["solver_residual"],
                                                    rep["solver_converged"])
