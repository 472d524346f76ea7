"""The rest of the reference's public API (growsurf/__init__.py:50-87).

CPU: OFF / XYZ readers and writers (byte-identical to the reference's own
writers, same parse errors), ExecConfig validation.  GPU: the single-signal
engine ``run`` against the reference's own run (tests/golden/run_single.npz,
made by tests/golden/make_single_golden.py), quantization_error and the
parallel find entry points.
"""

import os
import sys

import numpy as np
import pytest

from cases import GOLDEN, load_golden, same_numpy

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


def _reference():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        import growsurf.sampling as rs

        return rs
    except ImportError:
        pytest.skip("reference package not built (oracle/build_ref.sh)")


def test_off_xyz_writers_match_reference(tmp_path):
    from paper_1503_08294_b200 import TriMesh, load_off, load_xyz, save_off, save_xyz

    rs = _reference()
    rng = np.random.default_rng(5)
    verts = rng.random((40, 3)) * 3 - 1.5
    verts[0] = [1e-300, -0.0, 123456789.123456789]
    faces = rng.integers(0, 40, (30, 3))
    mesh = TriMesh(verts, faces)
    save_off(tmp_path / "a.off", mesh)
    rs.save_off(tmp_path / "b.off", mesh)
    assert (tmp_path / "a.off").read_bytes() == (tmp_path / "b.off").read_bytes()
    save_xyz(tmp_path / "a.xyz", verts)
    rs.save_xyz(tmp_path / "b.xyz", verts)
    assert (tmp_path / "a.xyz").read_bytes() == (tmp_path / "b.xyz").read_bytes()
    assert np.array_equal(load_xyz(tmp_path / "a.xyz"), verts)
    got, want = load_off(tmp_path / "a.off"), rs.load_off(tmp_path / "a.off")
    assert np.array_equal(got.vertices, want.vertices) and np.array_equal(got.faces, want.faces)


@pytest.mark.parametrize("text", [
    "", "OFX\n1 0 0\n", "OFF\n", "OFF\n2\n", "OFF\n1 x 0\n", "OFF\n-1 0 0\n",
    "OFF\n2 0 0\n0 0 0\n", "OFF\n1 0 0\n0 0\n", "OFF\n1 0 0\n0 0 nan\n",
    "OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n4 0 1 2\n", "OFF\n3 1 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 3\n",
    "# c\nOFF # header\n3 2 0\n0 0 0\n1 0 0\n0 1 0\n3 0 1 2\n3 0 0 1\n",
])
def test_off_parse_errors_match_reference(tmp_path, text):
    from paper_1503_08294_b200 import ParseError, load_off

    rs = _reference()
    p = tmp_path / "m.off"
    p.write_text(text)
    try:
        want = rs.load_off(p)
    except rs.ParseError as e:
        with pytest.raises(ParseError) as got:
            load_off(p)
        assert str(got.value) == str(e)
        return
    got = load_off(p)  # valid: same vertices, zero-area faces dropped
    assert np.array_equal(got.vertices, want.vertices) and np.array_equal(got.faces, want.faces)


@pytest.mark.parametrize("text", [
    "", "0 0 0\n", "1 2\n", "1 2 3 4\n", "1 x 3\n", "# only a comment\n",
    "1 2 3 # trailing\n\n4 5 6\n", "1e400 0 0\n", "nan inf -inf\n", "0 0 0\n1 2 three\n",
])
def test_xyz_parse_matches_reference(tmp_path, text):
    from paper_1503_08294_b200 import ParseError, load_xyz

    rs = _reference()
    p = tmp_path / "c.xyz"
    p.write_text(text)
    try:
        want = rs.load_xyz(p)
    except rs.ParseError as e:
        with pytest.raises(ParseError) as got:
            load_xyz(p)
        assert str(got.value) == str(e)
        return
    got = load_xyz(p)
    assert got.shape == want.shape and np.array_equal(got.view(np.int64), want.view(np.int64))


def test_stats_csv_byte_identical_to_reference(tmp_path):
    """write_stats_csv (metrics.py:130-136): same header, field formatting
    (repr floats, lowercase booleans) and line endings as the reference."""
    from paper_1503_08294_b200 import RunStats, write_stats_csv

    _reference()
    import growsurf.metrics as rm

    rows = [
        dict(variant="multi-b200", dataset="double-torus-1M", seed=7, iterations=6468,
             signals=26_492_928, discarded=15_654_514, units=1958, connections=5880,
             total_s=0.5307, sample_s=0.0, find_s=0.0873, update_s=0.4431, converged=True),
        dict(variant='we"ird,name', dataset="a\nb", seed=0, iterations=0, signals=0,
             discarded=0, units=2, connections=0, total_s=1e-300, sample_s=float("inf"),
             find_s=0.1 + 0.2, update_s=-0.0, converged=False),
    ]
    write_stats_csv(tmp_path / "a.csv", [RunStats(**r) for r in rows])
    rm.write_stats_csv(tmp_path / "b.csv", [rm.RunStats(**r) for r in rows])
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()


def test_run_state_fields_match_reference():
    """RunState has the reference's fields and fresh values (engine.py:101-119)."""
    from paper_1503_08294_b200.multi import RunState

    _reference()
    from growsurf.engine import RunState as RefRunState

    a, b = RunState(), RefRunState()
    assert set(a.__slots__) == set(b.__slots__)
    assert (a.tick, a.next_sweep, dict(a.patience), a.last_active) == (
        b.tick, b.next_sweep, b.patience, b.last_active)
    assert a.patience[12345] == 0 and 12345 not in a.patience


def test_executor_signatures_match_reference():
    """sequential_executor(backend=None, tile=None) and friends keep the
    reference's parameter names and order (multi.py:81-96, parallel.py:91-114)."""
    import inspect

    import paper_1503_08294_b200 as P

    _reference()
    import growsurf as R

    for name in ("sequential_executor", "parallel_executor", "batch_find_winners",
                 "parallel_batch_find_winners", "timed_find", "resolve_and_update",
                 "update_single", "find_winners_exhaustive", "run", "run_multi"):
        want = list(inspect.signature(getattr(R, name)).parameters)
        got = list(inspect.signature(getattr(P, name)).parameters)
        assert got[:len(want)] == want, (name, got, want)


def test_exec_config_validation():
    from paper_1503_08294_b200 import ExecConfig

    assert ExecConfig(workers=3).effective_workers(2) == 2
    with pytest.raises(ValueError):
        ExecConfig(workers=-1)
    with pytest.raises(ValueError):
        ExecConfig(tile=0)


@pytest.mark.gpu
def test_single_signal_run_matches_reference():
    from paper_1503_08294_b200 import EngineParams, SphereSource, run

    gold = load_golden("single")
    if not same_numpy(gold):
        pytest.skip("golden made with another numpy")
    net, st = run(SphereSource(1.0), EngineParams(theta0=0.35, max_signals=20_000), 3,
                  checkpoints=(10, 40))
    for k in ("iterations", "signals", "discarded", "units", "connections", "converged"):
        assert int(getattr(st, k)) == int(gold[f"stat_{k}"]), k
    assert [c[0] for c in st.checkpoints] == list(gold["checkpoint_units"])
    assert [c[1] for c in st.checkpoints] == list(gold["checkpoint_signals"])
    got = net.export()
    assert np.array_equal(got["ids"], gold["ids"]) and np.array_equal(got["edges"], gold["edges"])
    for k in ("pos", "hab", "theta"):
        assert np.array_equal(got[k].view(np.int64), gold[k].view(np.int64)), k


@pytest.mark.gpu
def test_indexed_run_equals_exhaustive_reference_run():
    """run(use_grid=True), the "indexed" variant (engine.py:396-426): the
    winner search goes through the device's exact grid, so the run equals
    the reference's exhaustive single-signal run bit for bit (the
    reference's own HashGrid is approximate)."""
    from paper_1503_08294_b200 import EngineParams, SphereSource, run

    gold = load_golden("single")
    if not same_numpy(gold):
        pytest.skip("golden made with another numpy")
    net, st = run(SphereSource(1.0), EngineParams(theta0=0.35, max_signals=20_000), 3,
                  use_grid=True, checkpoints=(10, 40))
    assert st.variant == "indexed"
    for k in ("iterations", "signals", "units", "connections", "converged"):
        assert int(getattr(st, k)) == int(gold[f"stat_{k}"]), k
    assert [c[1] for c in st.checkpoints] == list(gold["checkpoint_signals"])
    got = net.export()
    assert np.array_equal(got["ids"], gold["ids"]) and np.array_equal(got["edges"], gold["edges"])
    for k in ("pos", "hab", "theta"):
        assert np.array_equal(got[k].view(np.int64), gold[k].view(np.int64)), k


@pytest.mark.gpu
def test_quantization_error_and_parallel_find():
    from paper_1503_08294_b200 import (EngineParams, ExecConfig, Network, batch_find_winners,
                                       parallel_batch_find_winners, quantization_error, timed_find)

    rng = np.random.default_rng(8)
    net = Network(EngineParams())
    pts = rng.random((300, 3))
    for p in pts:
        net.add_unit(p, 0.2)
    probes = rng.random((5000, 3))
    d2 = ((probes[:, None, :] - pts[None, :, :]) ** 2).sum(-1).min(axis=1)
    assert np.isclose(quantization_error(net, probes), d2.mean(), rtol=1e-12)
    snap = net.snapshot()
    a = batch_find_winners(snap, probes[:700])
    b = parallel_batch_find_winners(snap, probes[:700], ExecConfig(workers=4, tile=33))
    c, secs = timed_find(snap, probes[:700])
    assert a == b == c and secs >= 0.0
