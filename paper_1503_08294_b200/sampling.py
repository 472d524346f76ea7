"""Signal sources: the host-side input boundary of the multi-signal path.

The reference draws every batch on the host from a caller-owned
``numpy.random.Generator(Philox(seed))`` (pkg/src/growsurf/multi.py:151,170).
These sources reproduce its streams value for value, so a seeded B200 run
consumes exactly the signals the reference consumes:

  SphereSource  sampling.py:51-74   (normalised Gaussian triples)
  TorusSource   sampling.py:77-124  (rejection-corrected poloidal angle)
  MeshSource    sampling.py:127-160 (area-weighted barycentric draws)
  CloudSource   sampling.py:163-180 (uniform index draws over a point set)

``DoubleTorusSource`` is new: the reference ships no genus-2 generator, and
BASELINE config 3 needs one.  It is only used to materialise point clouds
that both the reference and this package then read through ``CloudSource``.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = [
    "SphereSource",
    "TorusSource",
    "MeshSource",
    "CloudSource",
    "DoubleTorusSource",
    "TriMeshInput",
]


class TriMeshInput:
    """Triangle mesh: (n, 3) float64 vertices and (f, 3) int64 faces."""

    def __init__(self, vertices, faces):
        self.vertices = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
        self.faces = np.asarray(faces, dtype=np.int64).reshape(-1, 3)


class SphereSource:
    """Uniform on a sphere: Gaussian triples scaled to the radius.

    Stream contract (sampling.py:63-70): one ``standard_normal((n, 3))`` draw,
    zero-norm rows redrawn, then ``center + radius * (g / |g|)``.
    """

    def __init__(self, radius: float, center=(0.0, 0.0, 0.0)):
        if not (radius > 0.0 and math.isfinite(radius)):
            raise ValueError(f"radius must be positive and finite, got {radius}")
        self.radius = float(radius)
        self.center = np.asarray(center, dtype=np.float64).reshape(3)
        if not np.all(np.isfinite(self.center)):
            raise ValueError("center must be finite")
        self.label = f"sphere:{radius:g}"

    def sample(self, rng: np.random.Generator, n: int) -> np.ndarray:
        gauss = rng.standard_normal((n, 3))
        length = np.sqrt(np.sum(gauss * gauss, axis=1))
        while np.any(length == 0.0):
            redo = length == 0.0
            gauss[redo] = rng.standard_normal((int(np.sum(redo)), 3))
            length = np.sqrt(np.sum(gauss * gauss, axis=1))
        return self.center + self.radius * (gauss / length[:, None])

    def bounds(self):
        return self.center - self.radius, self.center + self.radius


class TorusSource:
    """Area-uniform on a torus of radii (major, minor).

    Stream contract (sampling.py:87-117): the poloidal angle is drawn by
    rejection against ``major + minor*cos(v)`` in rounds over the still-open
    slots; then one uniform toroidal angle per point.  ``n == 1`` uses the
    scalar draw order of the reference.
    """

    def __init__(self, major: float, minor: float):
        if not (major > minor > 0.0 and math.isfinite(major)):
            raise ValueError(f"need major > minor > 0, got {major}, {minor}")
        self.major = float(major)
        self.minor = float(minor)
        self.label = f"torus:{major:g},{minor:g}"

    def sample(self, rng: np.random.Generator, n: int) -> np.ndarray:
        big, small = self.major, self.minor
        two_pi = 2.0 * math.pi
        if n == 1:
            while True:
                v = rng.random() * two_pi
                if rng.random() * (big + small) <= big + small * math.cos(v):
                    break
            u = rng.random() * two_pi
            ring = big + small * math.cos(v)
            return np.array([[ring * math.cos(u), ring * math.sin(u), small * math.sin(v)]])
        poloidal = np.empty(n, dtype=np.float64)
        open_slots = np.arange(n)
        while open_slots.size:
            cand = rng.random(open_slots.size) * two_pi
            gate = rng.random(open_slots.size) * (big + small)
            keep = gate <= big + small * np.cos(cand)
            poloidal[open_slots[keep]] = cand[keep]
            open_slots = open_slots[~keep]
        toroidal = rng.random(n) * two_pi
        ring = big + small * np.cos(poloidal)
        out = np.empty((n, 3), dtype=np.float64)
        out[:, 0] = ring * np.cos(toroidal)
        out[:, 1] = ring * np.sin(toroidal)
        out[:, 2] = small * np.sin(poloidal)
        return out

    def bounds(self):
        reach = self.major + self.minor
        return (np.array([-reach, -reach, -self.minor]), np.array([reach, reach, self.minor]))


class MeshSource:
    """Area-weighted uniform draws on a triangle mesh (sampling.py:127-160)."""

    def __init__(self, mesh, label: str = "mesh"):
        if len(mesh.faces) == 0:
            raise ValueError("mesh has no usable faces")
        self.mesh = mesh
        self.label = label
        corners = mesh.vertices[mesh.faces]
        normal = np.cross(corners[:, 1] - corners[:, 0], corners[:, 2] - corners[:, 0])
        area = 0.5 * np.sqrt(np.sum(normal * normal, axis=1))
        self._cum = np.cumsum(area)
        self._total = float(self._cum[-1])
        if self._total <= 0.0:
            raise ValueError("mesh has zero total area")

    def sample(self, rng: np.random.Generator, n: int) -> np.ndarray:
        target = rng.random(n) * self._total
        face = np.minimum(np.searchsorted(self._cum, target, side="right"), len(self._cum) - 1)
        a = rng.random(n)
        b = rng.random(n)
        fold = a + b > 1.0
        a[fold] = 1.0 - a[fold]
        b[fold] = 1.0 - b[fold]
        corners = self.mesh.vertices[self.mesh.faces[face]]
        return (
            corners[:, 0]
            + a[:, None] * (corners[:, 1] - corners[:, 0])
            + b[:, None] * (corners[:, 2] - corners[:, 0])
        )

    def bounds(self):
        return self.mesh.vertices.min(axis=0), self.mesh.vertices.max(axis=0)


class CloudSource:
    """Uniform draws over a fixed point set (sampling.py:163-180).

    ``sample(rng, n)`` is one ``rng.integers(0, N, size=n)`` followed by a
    gather.  numpy's bounded-int path draws 32-bit halves from the bit
    generator's own buffer, so consecutive calls concatenate: the stream of
    K batches equals one draw of the summed size (checked in tests).
    """

    def __init__(self, points, label: str = "cloud"):
        pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        if pts.shape[0] == 0:
            raise ValueError("point cloud is empty")
        if not np.all(np.isfinite(pts)):
            raise ValueError("point cloud must be finite")
        self.points = np.ascontiguousarray(pts)
        self.label = label

    def sample_indices(self, rng: np.random.Generator, n: int) -> np.ndarray:
        return rng.integers(0, self.points.shape[0], size=n)

    def sample(self, rng: np.random.Generator, n: int) -> np.ndarray:
        return self.points[self.sample_indices(rng, n)]

    def bounds(self):
        return self.points.min(axis=0), self.points.max(axis=0)


class DoubleTorusSource:
    """Genus-2 surface: smooth union of two overlapping tori (an "eight").

    Signed distance to torus i: T_i = |(rho_i - R, z)| - r with
    rho_i = |(x -/+ c, y)|; blended union F = T1 + T2 - sqrt(T1^2 + T2^2 + d^2)
    (an R-function union whose crease along the intersection is rounded over
    a width ~d).  The tori overlap (c < R + r), so the union's boundary is one
    closed surface with two handles.  Points are drawn uniformly in the
    bounding box, kept near F = 0 and Newton-projected onto it.  Not exactly
    area-uniform; used only to materialise deterministic benchmark clouds
    that both the reference and this package read through CloudSource.
    """

    def __init__(self, major: float = 1.0, minor: float = 0.4, offset: float = 1.1,
                 blend: float = 0.1):
        if not (major > minor > 0.0 and 0.0 < offset < major + minor and blend > 0.0):
            raise ValueError("need major > minor > 0, 0 < offset < major + minor, blend > 0")
        self.major, self.minor, self.offset, self.blend = map(float, (major, minor, offset, blend))
        self.label = f"double-torus:{major:g},{minor:g},{offset:g}"

    def _field(self, p):
        x, y, z = p[:, 0], p[:, 1], p[:, 2]
        vals, grads = [], []
        for sgn in (-1.0, 1.0):
            dx = x + sgn * self.offset
            rho = np.sqrt(dx * dx + y * y)
            rho = np.maximum(rho, 1e-12)
            q = rho - self.major
            dist = np.sqrt(q * q + z * z)
            dist = np.maximum(dist, 1e-12)
            vals.append(dist - self.minor)
            grads.append(np.stack([q / dist * dx / rho, q / dist * y / rho, z / dist], axis=1))
        t1, t2 = vals
        root = np.sqrt(t1 * t1 + t2 * t2 + self.blend * self.blend)
        f = t1 + t2 - root
        grad = grads[0] * (1.0 - t1 / root)[:, None] + grads[1] * (1.0 - t2 / root)[:, None]
        return f, grad

    def sample(self, rng: np.random.Generator, n: int) -> np.ndarray:
        lo, hi = self.bounds()
        chunks, have = [], 0
        while have < n:
            p = lo + (hi - lo) * rng.random((2 * n + 1024, 3))
            f, _ = self._field(p)
            p = p[np.abs(f) < 0.25 * self.minor]
            for _ in range(12):
                f, grad = self._field(p)
                gg = np.maximum(np.sum(grad * grad, axis=1), 1e-300)
                p = p - (f / gg)[:, None] * grad
            f, _ = self._field(p)
            p = p[np.abs(f) < 1e-9]
            chunks.append(p)
            have += p.shape[0]
        return np.concatenate(chunks)[:n]

    def bounds(self):
        reach = self.offset + self.major + self.minor + self.blend
        side = self.major + self.minor + self.blend
        h = self.minor + self.blend
        return np.array([-reach, -side, -h]), np.array([reach, side, h])
