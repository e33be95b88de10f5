"""FLIP v1 snapshots, configs and CSV columns (paper_2404_01931_b200/formats.py)
against the reference's io.py / cli.py (live when its sources are present)."""
import os

import numpy as np
import pytest

HAVE_REF = os.path.isdir("/root/reference/pkg/src/flipsim")


def _parts(n, seed):
    from paper_2404_01931_b200.particles import ParticleSet
    r = np.random.default_rng(seed)
    return ParticleSet(*(r.normal(size=n) * s for s in (1.0, 1e-3, 1e5, 3.0, 1e-30, 7.0)))


def test_snapshot_host_roundtrip_and_layout(pkg, tmp_path):
    from paper_2404_01931_b200 import formats as F
    ps = _parts(1001, 3)
    path = tmp_path / "a.flip"
    F.write_snapshot(path, ps)
    data = path.read_bytes()
    assert data[:4] == b"FLIP" and len(data) == 16 + 24 * 1001
    back = F.read_snapshot(path)
    for a, b in zip(ps.arrays(), back.arrays()):
        assert np.array_equal(a.astype(np.float32).astype(np.float64), b)


@pytest.mark.parametrize("mutate,offset", [
    (lambda d: b"FLOP" + d[4:], 0),
    (lambda d: d[:12], 12),
    (lambda d: d[:4] + (2).to_bytes(4, "little") + d[8:], 4),
    (lambda d: d[:-4], None),
])
def test_snapshot_errors(pkg, tmp_path, mutate, offset):
    from paper_2404_01931_b200 import formats as F
    from paper_2404_01931_b200.errors import SnapshotFormatError
    path = tmp_path / "b.flip"
    F.write_snapshot(path, _parts(10, 1))
    path.write_bytes(mutate(path.read_bytes()))
    with pytest.raises(SnapshotFormatError) as ei:
        F.read_snapshot(path)
    if offset is not None:
        assert ei.value.offset == offset
    if HAVE_REF:
        import ref_loader
        ref_loader.load()
        from flipsim import io as RIO
        from flipsim.errors import SnapshotFormatError as RefErr
        with pytest.raises(RefErr) as ej:
            RIO.read_snapshot(path)
        assert ej.value.offset == ei.value.offset
        assert str(ej.value) == str(ei.value)


@pytest.mark.skipif(not HAVE_REF, reason="reference sources absent")
def test_snapshot_bytes_equal_reference(pkg, tmp_path):
    import ref_loader
    ref_loader.load()
    from flipsim import io as RIO
    from flipsim.particles import ParticleSet as RPS
    from paper_2404_01931_b200 import formats as F
    ps = _parts(777, 9)
    F.write_snapshot(tmp_path / "ours.flip", ps)
    RIO.write_snapshot(tmp_path / "ref.flip", RPS(*ps.arrays()))
    assert (tmp_path / "ours.flip").read_bytes() == (tmp_path / "ref.flip").read_bytes()


def test_config_roundtrip(pkg):
    from paper_2404_01931_b200 import formats as F
    text = "# c\nres = 64\n  solver=pcg  # trailing\n\nsteps = 10\n"
    d = F.parse_config(text)
    assert d == {"res": "64", "solver": "pcg", "steps": "10"}
    assert F.parse_config(F.format_config(d)) == d
    with pytest.raises(ValueError):
        F.parse_config("res 64")
    if HAVE_REF:
        import ref_loader
        ref_loader.load()
        from flipsim import io as RIO
        assert RIO.parse_config(text) == d and RIO.format_config(d) == F.format_config(d)


def test_csv_columns_match_reference_cli(pkg, tmp_path):
    from paper_2404_01931_b200 import formats as F
    assert F.TIMINGS_COLUMNS[:5] == ("step", "dt", "particles", "solver_iters", "solver_residual")
    assert F.TIMINGS_COLUMNS[-1] == "total_ms" and len(F.TIMINGS_COLUMNS) == 16
    rows = F.bench_rows("dam-break", 64, None, {n: [1.0, 2.0] for n in
                                                 pkg.StageTimings.stage_names()})
    F.write_csv(tmp_path / "b.csv", F.BENCH_COLUMNS, rows)
    assert (tmp_path / "b.csv").read_text().splitlines()[1] == "dam-break,64,,dt_compute,1.500"
    if HAVE_REF:
        import ref_loader
        ref_loader.load()
        from flipsim import cli as RCLI
        assert F.TIMINGS_COLUMNS == RCLI.TIMINGS_COLUMNS
        assert F.ENERGY_COLUMNS == RCLI.ENERGY_COLUMNS
        assert F.BENCH_COLUMNS == RCLI.BENCH_COLUMNS


@pytest.mark.gpu
def test_device_snapshot_matches_host_conversion(pkg, tmp_path):
    from paper_2404_01931_b200 import formats as F
    spec = pkg.SceneSpec(name="water-drop", res=16)
    st = pkg.make_scene(spec, 1)
    pkg.step(st, spec)
    pkg.step(st, spec)
    F.write_snapshot(tmp_path / "dev.flip", st.particles)            # converted on the GPU
    host = pkg.particles.ParticleSet(*st.particles.arrays())
    F.write_snapshot(tmp_path / "host.flip", host)                     # numpy astype
    assert (tmp_path / "dev.flip").read_bytes() == (tmp_path / "host.flip").read_bytes()
    n = F.load_snapshot_to_device(tmp_path / "dev.flip", st)
    assert n == host.count
    for a, b in zip(host.arrays(), st.particles.arrays()):
        assert np.array_equal(a.astype(np.float32).astype(np.float64), b)
