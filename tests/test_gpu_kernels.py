"""GPU parity of the kernel-backend plugin API (flipsim._kernels signatures)
against the oracle's restatement of _kernels/_core.pyx, on seeded inputs —
the same inputs the reference's own tests use (test_binning.py,
test_transfer.py, test_pressure.py)."""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2404_01931_b200 import _kernels
    return _kernels.active()


def random_set(n, dims, seed):
    rng = np.random.default_rng(seed)
    o = np.asarray(dims.origin)
    ext = np.array([dims.nx, dims.ny, dims.nz]) * dims.dtau
    pos = o + rng.random((n, 3)) * ext
    vel = rng.normal(size=(n, 3))
    return [pos[:, 0].copy(), pos[:, 1].copy(), pos[:, 2].copy(),
            vel[:, 0].copy(), vel[:, 1].copy(), vel[:, 2].copy()]


@pytest.mark.parametrize("n,res,seed", [(10**5, 6, 5), (3000, 6, 9), (0, 6, 1), (20, 6, 3),
                                        (200000, 32, 11)])
def test_counting_sort_perm_matches(K, n, res, seed):
    dims = O.Dimz(res, res, res, 1.0 / res)
    parts = random_set(n, dims, seed)
    cells = np.empty(n, dtype=np.int64)
    O.lib().orc_cell_index_many(dims.c(), n, O._p(parts[0]), O._p(parts[1]), O._p(parts[2]),
                                O._p(cells, O._i64))
    count = np.bincount(cells, minlength=dims.ncells).astype(np.int64)
    offset = np.zeros_like(count)
    np.cumsum(count[:-1], out=offset[1:])
    expect = np.argsort(cells, kind="stable")
    got = K.counting_sort_perm(cells, offset)
    assert np.array_equal(got, expect)


@pytest.mark.parametrize("comp", [0, 1, 2])
@pytest.mark.parametrize("res,n,seed", [(6, 1000, 3), (6, 2000, 4), (12, 30000, 7), (16, 500, 8)])
def test_p2g_component_bit_exact(K, comp, res, n, seed):
    dims = O.Dimz(res, res, res, 1.0 / res)
    parts, count, offset = O.bin_particles(dims, random_set(n, dims, seed))
    v_ref, w_ref = O.p2g_component(dims, comp, parts[3 + comp], parts[0], parts[1], parts[2],
                                   offset, count)
    v, w = K.p2g_component(comp, parts[3 + comp], parts[0], parts[1], parts[2], offset, count,
                           res, res, res, 1.0 / res, 0.0, 0.0, 0.0)
    assert v.tobytes() == v_ref.tobytes()
    assert w.tobytes() == w_ref.tobytes()


def test_p2g_non_power_of_two_cell(K):
    dims = O.Dimz(12, 9, 7, 0.1)
    parts, count, offset = O.bin_particles(dims, random_set(5000, dims, 2))
    for comp in range(3):
        v_ref, w_ref = O.p2g_component(dims, comp, parts[3 + comp], parts[0], parts[1],
                                       parts[2], offset, count)
        v, w = K.p2g_component(comp, parts[3 + comp], parts[0], parts[1], parts[2], offset,
                               count, 12, 9, 7, 0.1, 0.0, 0.0, 0.0)
        assert v.tobytes() == v_ref.tobytes() and w.tobytes() == w_ref.tobytes()


@pytest.mark.parametrize("res,n", [(6, 100), (8, 5000), (13, 7000)])
def test_sample_velocity_many_bit_exact(K, res, n):
    dims = O.Dimz(res, res, res, 1.0 / res)
    rng = np.random.default_rng(res)
    u = rng.normal(size=(res + 1) * res * res)
    v = rng.normal(size=res * (res + 1) * res)
    w = rng.normal(size=res * res * (res + 1))
    pos = rng.random((n, 3)) * 1.4 - 0.2  # includes clamped queries outside
    ref = O.sample_velocity_many(dims, u, v, w, pos[:, 0], pos[:, 1], pos[:, 2])
    got = K.sample_velocity_many(u, v, w, res, res, res, 1.0 / res, 0.0, 0.0, 0.0,
                                 pos[:, 0], pos[:, 1], pos[:, 2])
    for a, b in zip(got, ref):
        assert a.tobytes() == b.tobytes()


def _system(res, seed, frac=0.4):
    """Random FLUID/AIR interior in a solid shell (test_pressure.py:98-109)."""
    dims = O.Dimz(res, res, res, 1.0 / res)
    u, v, w, p, label = O.empty_grid(dims)
    O.solid_shell(dims, label)
    rng = np.random.default_rng(seed)
    lab = label.reshape(res, res, res)
    mask = rng.random((res - 2,) * 3) < frac
    inner = lab[1:-1, 1:-1, 1:-1]
    inner[mask] = O.FLUID
    r2 = np.random.default_rng(seed + 1)
    u[:], v[:], w[:] = r2.normal(size=u.size), r2.normal(size=v.size), r2.normal(size=w.size)
    O.enforce(dims, label, u, v, w)
    return O.assemble(dims, label, u, v, w, 0.01, 1000.0)


@pytest.mark.parametrize("res,seed", [(8, 7), (12, 3), (16, 9)])
def test_solver_kernels_bit_exact(K, res, seed):
    sys_ = _system(res, seed)
    n = sys_.nrows
    nbr = sys_.nbr_rows.reshape(-1)
    rng = np.random.default_rng(seed)
    x = rng.normal(size=n)
    L = O.lib()
    y_ref = np.empty(n)
    L.orc_laplacian_matvec(n, O._p(sys_.diag), O._p(nbr, O._i64), O._p(x), sys_.scale, O._p(y_ref))
    assert K.laplacian_matvec(sys_.diag, sys_.nbr_rows, x, sys_.scale).tobytes() == y_ref.tobytes()
    j_ref = np.empty(n)
    L.orc_jacobi_iter(n, O._p(sys_.diag), O._p(nbr, O._i64), O._p(sys_.rhs), O._p(x), sys_.scale,
                      O._p(j_ref))
    assert K.jacobi_iter(sys_.diag, sys_.nbr_rows, sys_.rhs, x, sys_.scale).tobytes() == j_ref.tobytes()
    g_ref = x.copy()
    L.orc_gs_sweep(n, O._p(sys_.diag), O._p(nbr, O._i64), O._p(sys_.rhs), O._p(g_ref), sys_.scale)
    g = x.copy()
    K.gs_sweep(sys_.diag, sys_.nbr_rows, sys_.rhs, g, sys_.scale)
    assert g.tobytes() == g_ref.tobytes()
    r_ref = x.copy()
    L.orc_gs_sweep_rows(len(sys_.red_rows), O._p(sys_.red_rows, O._i64), O._p(sys_.diag),
                        O._p(nbr, O._i64), O._p(sys_.rhs), O._p(r_ref), sys_.scale)
    r = x.copy()
    K.gs_sweep_rows(sys_.red_rows, sys_.diag, sys_.nbr_rows, sys_.rhs, r, sys_.scale)
    assert r.tobytes() == r_ref.tobytes()
    pc_ref = np.empty(n)
    L.orc_mic0_build(n, O._p(sys_.diag), O._p(nbr, O._i64), sys_.scale, 0.97, 0.25, O._p(pc_ref))
    pc = K.mic0_build(sys_.diag, sys_.nbr_rows, sys_.scale, 0.97, 0.25)
    assert pc.tobytes() == pc_ref.tobytes()
    z_ref = np.empty(n)
    L.orc_mic0_apply(n, O._p(pc_ref), O._p(nbr, O._i64), O._p(x), sys_.scale, O._p(np.empty(n)),
                     O._p(z_ref))
    assert K.mic0_apply(pc_ref, sys_.nbr_rows, x, sys_.scale).tobytes() == z_ref.tobytes()


@pytest.mark.parametrize("n", [0, 1, 5, 7, 8, 9, 100, 127, 128, 129, 1000, 8193, 100003, 3_000_001])
def test_pairwise_dot_matches_numpy(K, n):
    rng = np.random.default_rng(n)
    a = rng.normal(size=n) * np.exp(rng.normal(size=n) * 4)
    b = rng.normal(size=n)
    assert K.pairwise_dot(a, b) == float(np.add.reduce(a * b))
    assert K.pairwise_dot(a) == float(np.add.reduce(a))


@pytest.mark.parametrize("solver,precond", [("jacobi", "mic0"), ("gs", "mic0"), ("rbgs", "mic0"),
                                            ("pcg", "mic0"), ("pcg", "jacobi"), ("pcg", "none")])
@pytest.mark.parametrize("res,seed", [(8, 7), (12, 300)])
def test_whole_solvers_bit_exact(pkg, solver, precond, res, seed):
    sys_ = _system(res, seed)
    max_iters, tol = 400, 1e-9
    ref = O.solve(sys_, solver, max_iters, tol, precond)
    got = pkg.solve(sys_, solver, max_iters, tol, precond)
    assert got.iterations == ref["iterations"]
    assert got.residual == ref["residual"]
    assert got.converged == ref["converged"]
    assert got.p.tobytes() == ref["p"].tobytes()


def test_zero_diagonal_raises_naming_cell(pkg):
    sys_ = _system(8, 7)
    sys_.diag[3] = 0.0
    for solver in ("jacobi", "gs", "rbgs", "pcg"):
        with pytest.raises(pkg.SingularSystemError) as exc:
            pkg.solve(sys_, solver)
        assert exc.value.cell == int(sys_.cells[3])


def test_zero_rhs_iterations(pkg):
    sys_ = _system(8, 7)
    sys_.rhs[:] = 0.0
    assert pkg.solve(sys_, "pcg").iterations == 0
    for s in ("jacobi", "gs", "rbgs"):
        r = pkg.solve(sys_, s)
        assert r.iterations == 1 and r.converged and not r.p.any()
