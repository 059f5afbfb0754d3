"""Geodesic icosphere generator for the BASELINE scenarios.

Same construction as the reference's `icosphere(frequency, radius, centre)`
(reference: pkg/src/tdwavebem/shapes.py:30-67): every icosahedron face is cut
into a frequency x frequency barycentric grid whose points are projected once
onto the sphere; vertices are de-duplicated on a 12-digit rounded key in first-
seen order.  The vertex order matters (config 2's radial jitter draws one
number per vertex in that order), so the enumeration order is reproduced and
checked against the reference's own mesh in tests/test_host.py.
"""
from __future__ import annotations

import numpy as np

from .mesh import TriMesh

__all__ = ["icosphere"]

_G = (1.0 + 5.0 ** 0.5) / 2.0
# the 12 icosahedron corners and 20 outward-wound faces
_CORNERS = np.array([[-1, _G, 0], [1, _G, 0], [-1, -_G, 0], [1, -_G, 0],
                     [0, -1, _G], [0, 1, _G], [0, -1, -_G], [0, 1, -_G],
                     [_G, 0, -1], [_G, 0, 1], [-_G, 0, -1], [-_G, 0, 1]], dtype=float)
_FACES = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
          (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
          (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
          (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]


def icosphere(frequency: int, radius: float = 0.5, centre=(0.5, 0.0, 0.0)) -> TriMesh:
    if frequency < 1:
        raise ValueError("subdivision frequency must be >= 1")
    n = int(frequency)
    seen: dict = {}
    pts: list = []
    tris: list = []

    def vertex(p):
        key = tuple(np.round(p, 12))
        k = seen.get(key)
        if k is None:
            k = seen[key] = len(pts)
            pts.append(p)
        return k

    for fa, fb, fc in _FACES:
        a, b, c = _CORNERS[fa], _CORNERS[fb], _CORNERS[fc]
        ids = {}
        for i in range(n + 1):
            for j in range(n + 1 - i):
                p = (a * (n - i - j) + b * i + c * j) / n
                ids[i, j] = vertex(p / np.linalg.norm(p))
        for i in range(n):
            for j in range(n - i):
                tris.append((ids[i, j], ids[i + 1, j], ids[i, j + 1]))
                if i + j < n - 1:
                    tris.append((ids[i + 1, j], ids[i + 1, j + 1], ids[i, j + 1]))
    v = np.asarray(centre, dtype=float) + radius * np.array(pts)
    return TriMesh(v, np.array(tris, dtype=np.int64))
