"""OFF / XYZ files (on-disk formats).

Same formats and error behaviour as the reference's readers and writers
(pkg/src/growsurf/sampling.py:183-305): '#' starts a comment, blank lines
are skipped, OFF needs the 'OFF' header, a "V F [E]" counts line, V vertex
lines of three floats and F triangle lines '3 i j k' with indices in range;
zero-area faces are dropped on read; writers use 17 significant digits so a
round trip is exact, which makes files written from a B200 run
byte-identical to the reference's for the same network.
"""

from __future__ import annotations

import numpy as np

__all__ = ["ParseError", "load_off", "load_xyz", "save_off", "save_xyz"]


class ParseError(ValueError):
    """Malformed input file: carries the path and 1-based line number."""

    def __init__(self, path, line: int, message: str):
        super().__init__(f"{path}:{line}: {message}")
        self.path = str(path)
        self.line = line


def _lines(path):
    """(line number, text without comment) for every non-blank line."""
    with open(path) as fh:
        for no, raw in enumerate(fh, 1):
            text = raw.partition("#")[0].strip()
            if text:
                yield no, text


def _floats(path, no, text, what):
    fields = text.split()
    if len(fields) != 3:
        raise ParseError(path, no, f"{what} line needs 3 coordinates: {text!r}")
    try:
        return [float(f) for f in fields]
    except ValueError:
        # sampling.py:243 (OFF vertices) / :283 (XYZ points)
        bad = "bad vertex coordinates" if what == "vertex" else "bad coordinates"
        raise ParseError(path, no, f"{bad}: {text!r}") from None


def load_off(path):
    """ASCII OFF triangle mesh -> TriMeshInput (vertices (V,3), faces (F,3))."""
    from .sampling import TriMeshInput

    it = _lines(path)
    no, head = next(it, (1, None))
    if head is None:
        raise ParseError(path, 1, "empty file, expected OFF header")
    if head != "OFF":
        raise ParseError(path, no, f"expected 'OFF' header, got {head!r}")
    no, counts = next(it, (no, None))
    if counts is None:
        raise ParseError(path, no, "missing counts line")
    fields = counts.split()
    if len(fields) < 2:
        raise ParseError(path, no, f"counts line needs vertex and face counts: {counts!r}")
    try:
        nv, nf = int(fields[0]), int(fields[1])
    except ValueError:
        raise ParseError(path, no, f"bad counts line: {counts!r}") from None
    if nv < 0 or nf < 0:
        raise ParseError(path, no, "counts must be non-negative")
    verts = np.empty((nv, 3), np.float64)
    for i in range(nv):
        no, text = next(it, (no, None))
        if text is None:
            raise ParseError(path, no, f"expected {nv} vertices, file ended at {i}")
        verts[i] = _floats(path, no, text, "vertex")
    if nv and not np.isfinite(verts).all():
        raise ParseError(path, no, "non-finite vertex coordinates")
    faces = np.empty((nf, 3), np.int64)
    for i in range(nf):
        no, text = next(it, (no, None))
        if text is None:
            raise ParseError(path, no, f"expected {nf} faces, file ended at {i}")
        fields = text.split()
        if len(fields) != 4 or fields[0] != "3":
            raise ParseError(path, no, f"face line must be '3 i j k': {text!r}")
        try:
            tri = [int(f) for f in fields[1:]]
        except ValueError:
            raise ParseError(path, no, f"bad face indices: {text!r}") from None
        bad = [k for k in tri if not 0 <= k < nv]
        if bad:
            raise ParseError(path, no, f"face index {bad[0]} out of range [0, {nv})")
        faces[i] = tri
    if nf:  # drop zero-area triangles
        a, b, c = verts[faces[:, 0]], verts[faces[:, 1]], verts[faces[:, 2]]
        n = np.cross(b - a, c - a)
        faces = faces[(n * n).sum(axis=1) > 0.0]
    return TriMeshInput(verts, faces)


def load_xyz(path) -> np.ndarray:
    """Point cloud, one 'x y z' per line -> (n, 3) float64."""
    pts = [_floats(path, no, text, "point") for no, text in _lines(path)]
    return np.asarray(pts, dtype=np.float64).reshape(-1, 3)


def _fmt(v) -> str:
    return format(float(v), ".17g")


def save_off(path, mesh) -> None:
    """mesh.vertices / mesh.faces as ASCII OFF (exact round trip)."""
    verts = np.asarray(mesh.vertices, dtype=np.float64).reshape(-1, 3)
    faces = np.asarray(mesh.faces, dtype=np.int64).reshape(-1, 3)
    out = ["OFF", f"{len(verts)} {len(faces)} 0"]
    out += [" ".join(_fmt(v) for v in row) for row in verts]
    out += ["3 " + " ".join(str(int(k)) for k in row) for row in faces]
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")


def save_xyz(path, points) -> None:
    """Points one 'x y z' per line (exact round trip)."""
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    with open(path, "w") as fh:
        fh.write("".join(" ".join(_fmt(v) for v in row) + "\n" for row in pts))
