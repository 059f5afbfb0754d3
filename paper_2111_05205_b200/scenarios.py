"""The BASELINE.json scenarios as concrete ProblemSpecs.

Unit icosphere(s) (the reference's single-projection geodesic construction),
c = 1, c*dt = 0.5 * mean edge, incident Gaussian plane pulse along z with
sigma = 4 dt, t0 = 6 sigma; Neumann data q = -du_in/dn, Dirichlet data
u = -u_in at the centroids (collocation points).  Synthetic, seeded: there is
no external dataset in this benchmark.
"""
from __future__ import annotations

import warnings

import numpy as np

from .marching import ProblemSpec
from .mesh import TriMesh
from .shapes import icosphere
from .tbasis import BSplineBasis

# cfg -> (frequency, bie, d, phi, nt, jitter seed, two spheres)
CONFIGS = {
    0: dict(f=4, bie="obie", d=1, phi=1.0, nt=64, seed=None, two=False),
    1: dict(f=8, bie="bmbie", d=2, phi=1.0, nt=128, seed=None, two=False),
    2: dict(f=16, bie="bmbie", d=1, phi=0.0, nt=256, seed=12345, two=False),
    3: dict(f=32, bie="bmbie", d=2, phi=1.0, nt=512, seed=None, two=False),
    4: dict(f=32, bie="bmbie", d=2, phi=1.0, nt=1024, seed=None, two=True),
}

DESCRIPTION = {
    0: "config0: 320-element unit icosphere, OBIE d=1, Neumann, Nt=64",
    1: "config1: 1280-element unit icosphere, BMBIE d=2, Neumann, Nt=128",
    2: "config2: 5120-element unit icosphere (+-2% radial jitter, seed 12345), BMBIE d=1, Dirichlet, Nt=256",
    3: "config3: 20480-element unit icosphere, BMBIE d=2, Neumann, Nt=512",
    4: "config4: two 20480-element unit spheres 3 apart, BMBIE d=2, Neumann, Nt=1024",
}


def build_mesh(cfg: int, frequency: int | None = None) -> TriMesh:
    p = CONFIGS[cfg]
    f = frequency or p["f"]
    if p["two"]:
        a = icosphere(f, radius=1.0, centre=(-1.5, 0.0, 0.0))
        b = icosphere(f, radius=1.0, centre=(1.5, 0.0, 0.0))
        return TriMesh(np.vstack([a.vertices, b.vertices]),
                       np.vstack([a.triangles, b.triangles + len(a.vertices)]))
    m = icosphere(f, radius=1.0, centre=(0.0, 0.0, 0.0))
    if p["seed"] is None:
        return m
    rng = np.random.default_rng(p["seed"])
    v = m.vertices * (1.0 + rng.uniform(-0.02, 0.02, size=(len(m.vertices), 1)))
    return TriMesh(v, m.triangles)


def time_step(mesh) -> float:
    a, b, c = mesh.element_vertices()
    e = np.concatenate([np.linalg.norm(b - a, axis=1), np.linalg.norm(c - b, axis=1),
                        np.linalg.norm(a - c, axis=1)])
    return 0.5 * float(e.mean())


def build_spec(cfg: int, nt: int | None = None, frequency: int | None = None,
               dt: float | None = None) -> ProblemSpec:
    p = CONFIGS[cfg]
    mesh = build_mesh(cfg, frequency)
    if dt is None:
        dt = time_step(mesh) if not p["two"] else time_step(build_mesh(3, frequency))
    sig = 4.0 * dt
    t0 = 6.0 * sig
    zc = mesh.centroids[:, 2].copy()
    nz = mesh.normals[:, 2].copy()

    def q_data(t):
        a = (t - zc - t0) / sig
        return -(nz * 2.0 * a / sig * np.exp(-a * a))

    def u_data(t):
        a = (t - zc - t0) / sig
        return -np.exp(-a * a)

    phi = np.full(mesh.n_elements, p["phi"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")   # edge/(c dt) ~ 2.2 trips the reference's guideline
        return ProblemSpec(mesh, phi, p["bie"], BSplineBasis(p["d"], dt), 1.0, nt or p["nt"],
                           u_data=u_data if p["phi"] == 0.0 else None,
                           q_data=q_data if p["phi"] == 1.0 else None)


def known_data(spec):
    """Greville samples of the data, vectorised (same values as greville_samples)."""
    from .marching import greville_samples
    return greville_samples(spec)
