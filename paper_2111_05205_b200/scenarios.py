"""The BASELINE.json scenarios as concrete ProblemSpecs.

Unit icosphere(s) (the reference's single-projection geodesic construction),
c = 1, c*dt = 0.5 * mean edge, incident Gaussian plane pulse along z with
sigma = 4 dt, t0 = 6 sigma; Neumann data q = -du_in/dn, Dirichlet data
u = -u_in at the centroids (collocation points).  Synthetic, seeded: there is
no external dataset in this benchmark.
"""
from __future__ import annotations

import os
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


_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        n = int(os.environ.get("TDW_SAMPLE_THREADS", "0")) or min(16, os.cpu_count() or 1)
        _POOL = ThreadPoolExecutor(max_workers=max(1, n))
    return _POOL


class PlanePulseData:
    """Boundary data of the incident Gaussian plane pulse along +z,
    u_in(x, t) = exp(-((t - z - t0) / sig)^2), at the centroids: kind "u" is the
    Dirichlet datum -u_in, kind "q" the Neumann datum -du_in/dn.

    Callable per time like the reference's data callables (marching.py:33-64);
    `sample_many(times, out)` evaluates every Greville time at once (numpy,
    chunks of steps on a thread pool), element for element the same values."""

    def __init__(self, kind: str, zc, nz, t0: float, sig: float):
        self.kind, self.zc, self.nz, self.t0, self.sig = kind, zc, nz, float(t0), float(sig)

    def device_form(self):
        """(zc, nz, t0, sig) for the device-side sampler (tdw_known_plane_pulse)."""
        return (np.ascontiguousarray(self.zc, dtype=np.float64), np.ascontiguousarray(self.nz, dtype=np.float64),
                self.t0, self.sig)

    def __call__(self, t):
        a = (t - self.zc - self.t0) / self.sig
        if self.kind == "u":
            return -np.exp(-a * a)
        return -(self.nz * 2.0 * a / self.sig * np.exp(-a * a))

    def sample_many(self, times, out, on_chunk=None):
        """out[k] = self(times[k]) for every k; on_chunk(k0, k1), if given, is
        called (from a pool thread) as soon as rows k0..k1-1 are written."""
        times = np.asarray(times, dtype=np.float64)
        n = len(times)
        step = max(1, -(-n // 16))

        def chunk(k0):  # the operations of __call__, in place on the output rows
            k1 = min(n, k0 + step)
            o = out[k0:k1]
            a = np.subtract(times[k0:k1, None], self.zc)
            a -= self.t0
            a /= self.sig
            np.multiply(a, a, out=o)
            np.negative(o, out=o)
            np.exp(o, out=o)
            if self.kind == "u":
                np.negative(o, out=o)
            else:  # -(nz * 2 a / sig * e)
                a *= 2.0
                np.multiply(self.nz, a, out=a)
                a /= self.sig
                np.multiply(a, o, out=o)
                np.negative(o, out=o)
            if on_chunk is not None:
                on_chunk(k0, k1)
        list(_pool().map(chunk, range(0, n, step)))
        return out


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
    u_data = PlanePulseData("u", zc, nz, t0, sig)
    q_data = PlanePulseData("q", zc, nz, t0, sig)

    phi = np.full(mesh.n_elements, p["phi"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")   # edge/(c dt) ~ 2.2 trips the reference's guideline
        return ProblemSpec(mesh, phi, p["bie"], BSplineBasis(p["d"], dt), 1.0, nt or p["nt"],
                           u_data=u_data if p["phi"] == 0.0 else None,
                           q_data=q_data if p["phi"] == 1.0 else None)


def known_data(spec):
    """Greville samples of the data (vectorised through PlanePulseData.sample_many)."""
    from .marching import greville_samples
    return greville_samples(spec)
