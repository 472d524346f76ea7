"""Mesh extraction and validation on the device
against the UNMODIFIED reference's metrics (oracle/_ref growsurf.metrics,
metrics.py:148-240).

* extract_mesh: the reference's own extract_mesh runs on this package's
  Network (duck-typed: snapshot / unit_ids / neighbors read the device
  state) and must produce the identical face array and boundary count as
  the device enumeration, on golden networks of every kind (closed genus 0,
  genus 2, open surface, non-manifold, V > 4096).
* manifold_check / genus: the device face-edge counts against the
  reference's dict loops on those meshes and on synthetic face lists
  (tetrahedra, disconnected parts, fins, bow-ties, strips, a torus grid,
  unused vertices, bad indices, empty).
"""

import os
import sys

import numpy as np
import pytest

from cases import CASES, load_golden, make_source, run_device_trace, same_numpy

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        import growsurf.metrics as rm
    except ImportError:
        pytest.skip("reference package not built (oracle/build_ref.sh)")
    return rm


def _same_verdicts(mesh, rmesh):
    from paper_1503_08294_b200 import StateError, genus, manifold_check

    rm = _ref()
    assert manifold_check(mesh) == rm.manifold_check(rmesh)
    try:
        want = rm.genus(rmesh)
    except Exception as e:  # noqa: BLE001 - the reference's StateError
        with pytest.raises(StateError) as got:
            genus(mesh)
        assert str(got.value) == str(e)
        return
    assert genus(mesh) == want


@pytest.mark.parametrize("name", ["cfg1", "boundary", "stress", "paper_rule", "v8k"])
def test_extract_mesh_matches_reference_on_golden_networks(name):
    from paper_1503_08294_b200 import extract_mesh

    rm = _ref()
    gold = load_golden(name)
    if not same_numpy(gold):
        pytest.skip("golden made with another numpy")
    net, _, _, _ = run_device_trace(name)
    mesh = extract_mesh(net)
    rmesh = rm.extract_mesh(net)  # the reference's loops over the same network
    assert mesh.faces.dtype == np.int64 and np.array_equal(mesh.faces, rmesh.faces)
    assert mesh.boundary_edge_count == rmesh.boundary_edge_count
    assert np.array_equal(mesh.vertices.view(np.int64), rmesh.vertices.view(np.int64))
    _same_verdicts(mesh, rmesh)


def test_cfg3_mesh_is_a_closed_genus_2_surface():
    from paper_1503_08294_b200 import extract_mesh, genus, manifold_check, run_multi, workloads

    rm = _ref()
    gold = load_golden("cfg3_final")
    if not same_numpy(gold):
        pytest.skip("golden made with another numpy")
    src, params, seed, _ = workloads.make("cfg3")
    net, st = run_multi(src, params, seed, capacity=8192)
    mesh = extract_mesh(net)
    rmesh = rm.extract_mesh(net)
    assert np.array_equal(mesh.faces, rmesh.faces)
    assert manifold_check(mesh) == "closed" and genus(mesh) == 2 == rm.genus(rmesh)
    # V - E + F = 2 - 2g with E = 3F / 2 on a closed triangulation
    assert len(mesh.faces) == 2 * (st.units - 2 + 2 * 2)


def _tet(off=0):
    return [(off + 0, off + 1, off + 2), (off + 0, off + 1, off + 3), (off + 0, off + 2, off + 3),
            (off + 1, off + 2, off + 3)]


def _torus_grid(n):
    faces = []
    for i in range(n):
        for j in range(n):
            a, b = i * n + j, i * n + (j + 1) % n
            c, d = ((i + 1) % n) * n + j, ((i + 1) % n) * n + (j + 1) % n
            faces += [(a, b, d), (a, d, c)]
    return n * n, faces


SYNTHETIC = {
    "tetrahedron": (4, _tet()),
    "two_tetrahedra": (8, _tet() + _tet(4)),
    "unused_vertex": (5, _tet()),
    "fin": (5, [(0, 1, 2), (0, 1, 3), (0, 1, 4)]),
    "strip": (4, [(0, 1, 2), (1, 2, 3)]),
    "bowtie": (5, [(0, 1, 2), (0, 3, 4)]),
    "open_fan": (5, [(0, 1, 2), (0, 2, 3), (0, 3, 4)]),
    "torus_grid": _torus_grid(12),
    "degenerate": (3, [(0, 0, 1), (0, 1, 2)]),
    "empty": (3, []),
}


@pytest.mark.parametrize("name", sorted(SYNTHETIC))
def test_manifold_and_genus_match_reference(name):
    from paper_1503_08294_b200 import TriMesh

    rm = _ref()
    nv, faces = SYNTHETIC[name]
    verts = np.zeros((nv, 3))
    f = np.array(faces, np.int64).reshape(-1, 3)
    _same_verdicts(TriMesh(verts, f), rm.TriMesh(verts, f))


def test_large_torus_grid_genus_one():
    """1M vertices, 2M faces: the device counts at the scale the Python
    dict loops struggle with."""
    from paper_1503_08294_b200 import TriMesh, genus, manifold_check

    nv, faces = _torus_grid(1000)
    mesh = TriMesh(np.zeros((nv, 3)), np.array(faces, np.int64))
    assert manifold_check(mesh) == "closed" and genus(mesh) == 1


def test_bad_face_index_raises():
    from paper_1503_08294_b200 import TriMesh, manifold_check

    with pytest.raises(ValueError):
        manifold_check(TriMesh(np.zeros((3, 3)), np.array([[0, 1, 3]], np.int64)))
