"""Generate the committed golden fixtures by running the REFERENCE itself.

This script is the only place that imports the upstream `tdwavebem` package
(from /root/reference/pkg/src, present only in the build container).  Its
outputs are small .npz fixtures under tests/golden/ that travel to the GPU box;
the reference itself never does.

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py coeff
    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py march 0
    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py march 1
    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py march 2   # ~1 h, ~15 GB RAM
    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py tree 3
    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py tree 4   # two spheres, ~1 min
    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py fmm_ref  # patched reference fast_march
    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py march_pairs  # pairs= restriction
    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py physics      # sphere series validation

Scenario recipe: SURVEY.md section 8(c)/(d) (icosphere f=4/8/16, c=1,
c*dt = 0.5 * mean edge, Gaussian plane pulse along z, sigma=4dt, t0=6 sigma).
Versions of numpy/scipy/numba are recorded in every fixture.
"""
from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")

import scipy  # noqa: E402
import numba  # noqa: E402
from tdwavebem import elemint, marching, shapes  # noqa: E402
from tdwavebem.mesh import TriMesh  # noqa: E402
from tdwavebem.tbasis import BSplineBasis  # noqa: E402

OUT = Path(__file__).resolve().parent
VERSIONS = f"numpy {np.__version__}; scipy {scipy.__version__}; numba {numba.__version__}; reference tdwavebem 0.1.0"

# (f, bie, d, phi, nt, jitter_seed)
CONFIGS = {
    0: (4, "obie", 1, 1.0, 64, None),
    1: (8, "bmbie", 2, 1.0, 128, None),
    2: (16, "bmbie", 1, 0.0, 256, 12345),
    3: (32, "bmbie", 2, 1.0, 512, None),
    4: (32, "bmbie", 2, 1.0, 1024, None),   # two spheres, centres (+-1.5, 0, 0); dt of one sphere
}


def build_mesh(cfg):
    f, _, _, _, _, seed = CONFIGS[cfg]
    if cfg == 4:
        a = shapes.icosphere(f, radius=1.0, centre=(-1.5, 0.0, 0.0))
        b = shapes.icosphere(f, radius=1.0, centre=(1.5, 0.0, 0.0))
        return TriMesh(np.vstack([a.vertices, b.vertices]),
                       np.vstack([a.triangles, b.triangles + len(a.vertices)]))
    m = shapes.icosphere(f, radius=1.0, centre=(0.0, 0.0, 0.0))
    if seed is None:
        return m
    rng = np.random.default_rng(seed)
    v = m.vertices * (1.0 + rng.uniform(-0.02, 0.02, size=(len(m.vertices), 1)))
    return TriMesh(v, m.triangles)


def build_spec(cfg):
    f, bie, d, phival, nt, _ = CONFIGS[cfg]
    mesh = build_mesh(cfg)
    v0, v1, v2 = (build_mesh(3) if cfg == 4 else mesh).element_vertices()
    edges = np.concatenate([np.linalg.norm(v1 - v0, axis=1),
                            np.linalg.norm(v2 - v1, axis=1),
                            np.linalg.norm(v0 - v2, axis=1)])
    dt = 0.5 * float(edges.mean())
    sig = 4.0 * dt
    t0 = 6.0 * sig
    zc = mesh.centroids[:, 2]
    nz = mesh.normals[:, 2]

    def q_data(t):
        a = (t - zc - t0) / sig
        return -(nz * 2.0 * a / sig * np.exp(-a * a))

    def u_data(t):
        a = (t - zc - t0) / sig
        return -np.exp(-a * a)

    phi = np.full(mesh.n_elements, phival)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        spec = marching.ProblemSpec(
            mesh, phi, bie, BSplineBasis(d, dt), 1.0, nt,
            u_data=u_data if phival == 0.0 else None,
            q_data=q_data if phival == 1.0 else None)
    return spec


# ---------------------------------------------------------------------------
def _structured_cases(rng):
    """Hand-picked configurations: self, coplanar, near-singular, clipped,
    not-yet-arrived, fully passed (SURVEY 8(c) golden list)."""
    P, A, B, C, s = [], [], [], [], []
    E0 = np.array([[0.0, 0, 0], [0.4, 0, 0], [0.1, 0.5, 0]])
    cen = E0.mean(axis=0)
    for g in (0.03, 0.1, 0.2, 0.35, 0.6, 1.5, 4.0):
        P.append(cen); A.append(E0[0]); B.append(E0[1]); C.append(E0[2]); s.append(g)   # self
        P.append(np.array([2.0, 1.0, 0.0])); A.append(E0[0]); B.append(E0[1]); C.append(E0[2]); s.append(g * 2 + 1.5)  # coplanar
        P.append(cen + np.array([0, 0, 2e-3])); A.append(E0[0]); B.append(E0[1]); C.append(E0[2]); s.append(g)  # near-singular +
        P.append(cen - np.array([0, 0, 2e-3])); A.append(E0[0]); B.append(E0[1]); C.append(E0[2]); s.append(g)  # near-singular -
        P.append(np.array([0.2, 0.1, 0.3])); A.append(E0[0]); B.append(E0[1]); C.append(E0[2]); s.append(g)    # partially clipped
        P.append(np.array([0.0, 0.0, 10.0])); A.append(E0[0]); B.append(E0[1]); C.append(E0[2]); s.append(g)   # not arrived
        P.append(np.array([0.4, 0.0, 0.0])); A.append(E0[0]); B.append(E0[1]); C.append(E0[2]); s.append(g)    # at a vertex
        P.append(np.array([0.2, 0.0, 0.0])); A.append(E0[0]); B.append(E0[1]); C.append(E0[2]); s.append(g)    # on an edge
        P.append(np.array([0.2, -0.3, 0.0])); A.append(E0[0]); B.append(E0[1]); C.append(E0[2]); s.append(g)   # edge line, outside
    for _ in range(40):   # fully passed, random orientation
        E = rng.uniform(-0.5, 0.5, (3, 3))
        p = rng.uniform(-1, 1, 3)
        rmax = max(np.linalg.norm(p - E[k]) for k in range(3))
        P.append(p); A.append(E[0]); B.append(E[1]); C.append(E[2]); s.append(rmax * rng.uniform(1.01, 3.0))
    return [np.array(v) for v in (P, A, B, C)] + [np.array(s)]


def _random_cases(rng, n):
    P = rng.uniform(-1, 1, (n, 3))
    A = rng.uniform(-0.5, 0.5, (n, 3))
    B = rng.uniform(-0.5, 0.5, (n, 3))
    C = rng.uniform(-0.5, 0.5, (n, 3))
    s = rng.uniform(0.01, 2.5, n)
    # push a share of the points into the element plane (coplanar family)
    k = n // 8
    nrm = np.cross(B[:k] - A[:k], C[:k] - A[:k])
    nrm /= np.linalg.norm(nrm, axis=1)[:, None]
    P[:k] -= np.einsum("ij,ij->i", P[:k] - A[:k], nrm)[:, None] * nrm
    return P, A, B, C, s


def make_coeff():
    rng = np.random.default_rng(20240817)
    sets = [_structured_cases(rng), _random_cases(rng, 3000)]
    P, A, B, C, s = (np.concatenate([st[k] for st in sets]) for k in range(5))
    ez = np.cross(B - A, C - A)
    dbl = np.linalg.norm(ez, axis=1)
    keep = dbl > 1e-3
    P, A, B, C, s, ez = P[keep], A[keep], B[keep], C[keep], s[keep], ez[keep] / dbl[keep][:, None]
    nx = rng.normal(size=P.shape)
    nx /= np.linalg.norm(nx, axis=1)[:, None]
    out = dict(P=P, A=A, B=B, C=C, ez=ez, s=s, nx=nx, c=1.0, dt=0.05, versions=VERSIONS)
    for d in (1, 2, 3):
        U, W = elemint.retarded_coeff_table(P, A, B, C, ez, s, d, 1.0, 0.05)
        BU, BW = elemint.retarded_coeff_table(P, A, B, C, ez, s, d, 1.0, 0.05, which="bm", nx=nx)
        out[f"U{d}"], out[f"W{d}"], out[f"BU{d}"], out[f"BW{d}"] = U, W, BU, BW
    np.savez_compressed(OUT / "coeff_table.npz", **out)
    print("coeff_table.npz:", len(P), "triples")


def make_march(cfg):
    spec = build_spec(cfg)
    mesh = spec.mesh
    stats = marching.mesh_stats(mesh)
    gstar = marching.compute_gamma_star(stats, spec.basis, spec.c)
    n_lags = min(gstar, spec.nt - 1)
    t0 = time.perf_counter()
    mats = marching.build_retarded_matrices(spec, n_lags)
    t_asm = time.perf_counter() - t0
    nnz = sum(m.nnz for m in mats.U)
    trace = []
    t0 = time.perf_counter()
    hist = marching.march(spec, mats=mats, rhs_trace=trace)
    t_march = time.perf_counter() - t0
    unknown = hist.u if spec.phi[0] == 1.0 else hist.q
    rhs = np.array(trace)
    ns = mesh.n_elements
    rng = np.random.default_rng(7)
    sub = np.sort(rng.choice(ns, size=min(ns, 256), replace=False))
    full_steps = np.unique(np.linspace(0, spec.nt - 2, 6).astype(int))
    out = dict(
        cfg=cfg, vertices=mesh.vertices, triangles=mesh.triangles, dt=spec.basis.dt,
        gamma_star=gstar, n_lags=n_lags, nnz_lagcsr=nnz, status=hist.status,
        n_steps=hist.n_steps, t_assembly=t_asm, t_march=t_march,
        unknown_norm=np.linalg.norm(unknown, axis=1), rhs_norm=np.linalg.norm(rhs, axis=1),
        sub=sub, unknown_sub=unknown[:, sub], rhs_sub=rhs[:, sub],
        full_steps=full_steps, unknown_full=unknown[full_steps],
        versions=VERSIONS)
    if cfg == 0:   # small enough to keep everything
        out.update(u=hist.u, q=hist.q, tau=hist.tau, sigma=hist.sigma, rhs=rhs)
    np.savez_compressed(OUT / f"march_cfg{cfg}.npz", **out)
    print(f"cfg{cfg}: ns={ns} gstar={gstar} nnz={nnz} asm={t_asm:.1f}s march={t_march:.1f}s "
          f"status={hist.status} n_steps={hist.n_steps} max|x|={np.abs(unknown).max():.4g}")


def pair_subset(mesh, radius=1.2):
    """The pair restriction of the pairs= fixture: centroid distance < radius."""
    c = mesh.centroids
    dist = np.linalg.norm(c[:, None, :] - c[None, :, :], axis=2)
    ii, jj = np.nonzero(dist < radius)
    return ii.astype(np.int64), jj.astype(np.int64)


def make_march_pairs():
    """build_retarded_matrices(spec, n_lags, pairs=...) + march(mats=...) of the
    reference on config 0 with the pairs restricted to centroid distance < 1.2."""
    spec = build_spec(0)
    stats = marching.mesh_stats(spec.mesh)
    n_lags = min(marching.compute_gamma_star(stats, spec.basis, spec.c), spec.nt - 1)
    ii, jj = pair_subset(spec.mesh)
    mats = marching.build_retarded_matrices(spec, n_lags, pairs=(ii, jj))
    trace = []
    hist = marching.march(spec, mats=mats, rhs_trace=trace)
    np.savez_compressed(OUT / "march_pairs_cfg0.npz", radius=1.2, n_pairs=len(ii), u=hist.u, rhs=np.array(trace),
                        status=hist.status, n_steps=hist.n_steps, versions=VERSIONS)
    print("march_pairs_cfg0:", len(ii), "pairs", hist.status, hist.n_steps, np.abs(hist.u).max())


def physics_spec(bc, bie, d, frequency=4, nt=64):
    """The reference's own sphere scenario (reference.py:23-93): icosphere of
    radius 0.5 at (0.5, 0, 0), plane cosine pulse of length 0.5 along +x1, the
    scattered field solved with the incident field's data (Neumann: q = -du_in/dn;
    Dirichlet: u = -u_in), c dt = 0.5 mean edge."""
    from tdwavebem.reference import IncidentPulse
    mesh = shapes.icosphere(frequency, radius=0.5, centre=(0.5, 0.0, 0.0))
    v0, v1, v2 = mesh.element_vertices()
    dt = 0.5 * float(np.concatenate([np.linalg.norm(v1 - v0, axis=1), np.linalg.norm(v2 - v1, axis=1),
                                     np.linalg.norm(v0 - v2, axis=1)]).mean())
    pulse = IncidentPulse(0.5, 1.0)
    cen, nrm = mesh.centroids, mesh.normals
    phi = np.full(mesh.n_elements, 1.0 if bc == "neumann" else 0.0)
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return marching.ProblemSpec(mesh, phi, bie, BSplineBasis(d, dt), 1.0, nt,
                                    u_data=(lambda t: -pulse.value(cen, t)) if bc == "dirichlet" else None,
                                    q_data=(lambda t: -pulse.normal_derivative(cen, nrm, t)) if bc == "neumann" else None)


def make_physics():
    """Physics validation fixture: the reference's march on its
    sphere scenario, the total field on the arc x2 = 0, x3 >= 0 at the knots, the
    reference's semi-analytic series there (reference_solution) and the relative
    L2 error between the two, for Neumann (OBIE d=1, BMBIE d=2) and Dirichlet
    (BMBIE d=1)."""
    from tdwavebem import reference as R
    out = dict(versions=VERSIONS)
    for bc, bie, d in (("neumann", "obie", 1), ("neumann", "bmbie", 2), ("dirichlet", "bmbie", 1)):
        spec = physics_spec(bc, bie, d)
        scen = R.SphereScenario(0.5, (0.5, 0.0, 0.0), bc, 0.5, 1.0)
        idx = R.arc_evaluation_indices(spec.mesh, scen)
        hist = marching.march(spec)
        pulse = R.IncidentPulse(0.5, 1.0)
        cen, nrm = spec.mesh.centroids[idx], spec.mesh.normals[idx]
        times = np.arange(spec.nt) * spec.basis.dt
        if bc == "neumann":
            num = hist.knot_values("u")[:, idx] + np.array([pulse.value(cen, t) for t in times])
        else:
            num = hist.knot_values("q")[:, idx] + np.array([pulse.normal_derivative(cen, nrm, t) for t in times])
        ref = R.reference_solution(scen, cen, spec.nt, spec.basis.dt)
        key = f"{bc}_{bie}{d}"
        out[f"{key}_idx"] = idx
        out[f"{key}_numerical"] = num
        out[f"{key}_reference"] = ref
        out[f"{key}_error"] = R.rel_l2_error(num, ref)
        out[f"{key}_status"] = hist.status
        print(key, hist.status, "rel L2 error vs the sphere series", out[f"{key}_error"])
    np.savez_compressed(OUT / "physics_sphere.npz", **out)


def make_tree(cfg, leaf_capacity=20):
    """Octree + interaction lists from the reference build_tree (bit-exact target)."""
    from tdwavebem.fmm_tree import build_tree
    spec = build_spec(cfg)
    t0 = time.perf_counter()
    tree = build_tree(spec.mesh, spec.c, spec.basis.dt, leaf_capacity, 8)
    out = dict(cfg=cfg, leaf_capacity=leaf_capacity, leaf_level=tree.leaf_level,
               root_centre=tree.root_centre, root_half=tree.root_half,
               near_i=tree.near_pairs[0].astype(np.int32), near_j=tree.near_pairs[1].astype(np.int32),
               t_build=time.perf_counter() - t0, versions=VERSIONS)
    for L, lev in enumerate(tree.levels):
        out[f"L{L}_coords"] = lev.coords.astype(np.int32)
        if lev.il_obs is not None:
            out[f"L{L}_il_obs"] = lev.il_obs.astype(np.int32)
            out[f"L{L}_il_src"] = lev.il_src.astype(np.int32)
            out[f"L{L}_il_off"] = lev.il_offsets.astype(np.int8)
    for L, (ei, ej) in tree.extra_pairs.items():
        out[f"extra{L}_i"] = ei.astype(np.int32)
        out[f"extra{L}_j"] = ej.astype(np.int32)
    np.savez_compressed(OUT / f"tree_cfg{cfg}.npz", **out)
    print(f"tree cfg{cfg}: leaf={tree.leaf_level} near={len(tree.near_pairs[0])}")


def make_fmm_setup():
    """Setup math of the FMM from the reference: interpolation rows, transfer
    matrices, the triangle rule, cmp_coeff, Toeplitz kernel tensors and the
    materialised M2L matrix (fmm_interp.py, fmm.py:44-162).  The node-offset sign
    of _KernelCache._positions is corrected by
    substituting a positions function written here; everything else is the
    reference's own code path."""
    from tdwavebem import fmm, fmm_interp
    from tdwavebem.fmm_tree import build_tree

    def positions_fixed(self, level, offset):
        h = self.tree.levels[level].half_width
        off = np.asarray(offset, float) * 2.0 * h
        g = -h * self._node_diff
        d = [off[k] + g for k in range(3)]
        return np.sqrt(d[0][:, None, None] ** 2 + d[1][None, :, None] ** 2 + d[2][None, None, :] ** 2)

    fmm._KernelCache._positions = positions_fixed
    rng = np.random.default_rng(11)
    out = dict(versions=VERSIONS)
    for p in (4, 5, 6):
        sch = fmm_interp.InterpScheme(p)
        xi = rng.uniform(-1.0, 1.0, 200)
        xe = rng.uniform(-1.9, 1.9, 200)
        out[f"interp{p}_xi"], out[f"interp{p}_xe"] = xi, xe
        out[f"interp{p}_w"], out[f"interp{p}_dw"] = sch.weights(xi), sch.dweights(xi)
        out[f"interp{p}_we"], out[f"interp{p}_dwe"] = sch.weights(xe, 1.0), sch.dweights(xe, 1.0)
        out[f"interp{p}_t0"], out[f"interp{p}_t1"] = sch.transfer(0), sch.transfer(1)
    E = rng.uniform(-1, 1, (3, 3))
    out["tri_E"] = E
    out["tri_pts"], out["tri_w"] = fmm_interp.triangle_gauss_rule(E)
    out["cmp"] = np.array([[p, m, k, fmm.cmp_coeff(p, m, k)] for p in (2, 3) for m in range(p - 1)
                           for k in range(0, 9)], dtype=float)
    spec = build_spec(1)
    tree = build_tree(spec.mesh, spec.c, spec.basis.dt, 20, 8)
    for d in (1, 2):
        cache = fmm._KernelCache(tree, d, 4, 4)
        lev = tree.leaf_level
        offs = tree.levels[lev].il_offsets[[0, len(tree.levels[lev].il_offsets) // 2, -1]]
        out[f"kc{d}_level"] = lev
        out[f"kc{d}_offsets"] = offs
        for k, off in enumerate(offs):
            for pp in range(0, d + 1):
                out[f"kc{d}_{k}_{pp}"] = cache.get(lev, off, pp)
            out[f"kc{d}_{k}_dark"] = np.array([cache.lag_is_dark(lev, off, l) for l in range(1, 10)])
        out[f"m2l{d}"] = fmm.dense_m2l_matrix(tree, d, 4, 4, lev, offs[1], 3, 0)
        if d == 2:
            out["m2l2_p1"] = fmm.dense_m2l_matrix(tree, d, 4, 4, lev, offs[1], tree.mu + 1, 1)
    np.savez_compressed(OUT / "fmm_setup.npz", **out)
    print("fmm_setup.npz")


# the seven line-level corrections of the reference's fast solver,
# applied to the reference SOURCE text in memory (the tree stays read-only and no
# reference source is copied into this repo).  Each (file, old, new) must match once.
FMM_PATCHES = [
    # 1. P2M contraction: tau[elems] @ p2m_tau[ci] (fmm.py:517-518)
    ("fmm.py", "spat = (self.p2m_tau[ci] @ hist.tau[beta0][elems]\n"
               "                        - self.p2m_sig[ci] @ hist.sigma[beta0][elems])",
               "spat = (hist.tau[beta0][elems] @ self.p2m_tau[ci]\n"
               "                        - hist.sigma[beta0][elems] @ self.p2m_sig[ci])"),
    # 2. node-offset sign of the kernel samples (fmm.py:87)
    ("fmm.py", "g = h_s * self._node_diff", "g = -h_s * self._node_diff"),
    # 3. source interval: the one containing t_{beta+1} (fmm.py:512)
    ("fmm.py", "k_src = int(np.floor(t_src / interval + 1e-12))",
               "k_src = int(np.floor((t_src + self.dt) / interval + 1e-12))"),
    # 4. its temporal weights may extrapolate by 2 dt / I (fmm.py:514)
    ("fmm.py", "wts = self.scheme_t.weights([eta_s])[0]",
               "wts = self.scheme_t.weights([eta_s], 2.0 * self.dt / interval)[0]"),
    # 5. extra-list break test on the corrected source interval (fmm.py:464)
    ("fmm.py", "if int(np.floor(t_src / int_L + 1e-12)) != k_now:",
               "if int(np.floor((t_src + self.dt) / int_L + 1e-12)) != k_now:"),
    # 6. extra-list lag count (fmm.py:226)
    ("fmm.py", "lags = int(np.floor(tree.interval(L) / self.dt)) + 1",
               "lags = int(np.floor(tree.interval(L) / self.dt)) + 2"),
    # 7. marginal margin c I_L and reach c (I_L + dt) + 2 rho (fmm_tree.py:202, 206)
    ("fmm_tree.py", "margin = c * (interval - dt)", "margin = c * interval"),
    ("fmm_tree.py", "reach = c * interval + 2 * rho", "reach = c * (interval + dt) + 2 * rho"),
    # not a correction: numba cannot cache functions of an in-memory module
    ("fmm.py", "@numba.njit(cache=True, fastmath=True)", "@numba.njit(cache=False, fastmath=True)"),
]


def patched_fmm():
    """The reference's fmm / fmm_tree modules with FMM_PATCHES applied (in memory)."""
    import types
    mods = {}
    for name in ("fmm_tree", "fmm"):
        src = (REF / "tdwavebem" / f"{name}.py").read_text()
        for f, old, new in FMM_PATCHES:
            if f == f"{name}.py":
                assert src.count(old) == 1, (f, old)
                src = src.replace(old, new)
        mod = types.ModuleType(f"tdwavebem.{name}")
        mod.__package__ = "tdwavebem"
        mod.__file__ = f"<patched {name}.py>"
        sys.modules[f"tdwavebem.{name}"] = mod
        exec(compile(src, mod.__file__, "exec"), mod.__dict__)
        mods[name] = mod
    return mods["fmm"]


FMM_REF_SUB = np.sort(np.random.default_rng(5).choice(1280, size=256, replace=False))


def make_fmm_ref():
    """fast_march of the runtime-corrected reference on the 1280-element sphere
    (OBIE d=1 and BMBIE d=2, Neumann, ps = pt = 4, Nt = 128, leaf capacity 100
    and 20): per-step rhs and unknown density, the pin of oracle/fmm_oracle.py."""
    fmm = patched_fmm()
    base = build_spec(1)
    out = dict(versions=VERSIONS, patches=np.array([f"{f}: {o!r} -> {n!r}" for f, o, n in FMM_PATCHES]),
               sub=FMM_REF_SUB)
    import warnings
    for bie, d in (("obie", 1), ("bmbie", 2)):
        for Z in (100, 20):
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                spec = marching.ProblemSpec(base.mesh, np.ones(base.mesh.n_elements), bie,
                                            BSplineBasis(d, base.basis.dt), 1.0, 128, q_data=base.q_data)
            trace = []
            t0 = time.perf_counter()
            hist = fmm.fast_march(spec, fmm.FmmConfig(ps=4, pt=4, leaf_capacity=Z, mu=8), rhs_trace=trace)
            key = f"{bie}{d}_Z{Z}"
            rhs = np.array(trace)
            out[f"{key}_u_sub"] = hist.u[:, FMM_REF_SUB]
            out[f"{key}_rhs_sub"] = rhs[:, FMM_REF_SUB]
            out[f"{key}_u_norm"] = np.linalg.norm(hist.u, axis=1)
            out[f"{key}_rhs_norm"] = np.linalg.norm(rhs, axis=1)
            out[f"{key}_status"] = hist.status
            out[f"{key}_n_steps"] = hist.n_steps
            print(f"{key}: {hist.status} {hist.n_steps} steps, {time.perf_counter() - t0:.1f} s")
    np.savez_compressed(OUT / "fmm_ref.npz", **out)


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "coeff":
        make_coeff()
    elif what == "march":
        make_march(int(sys.argv[2]))
    elif what == "tree":
        make_tree(int(sys.argv[2]))
    elif what == "physics":
        make_physics()
    elif what == "march_pairs":
        make_march_pairs()
    elif what == "fmm_ref":
        make_fmm_ref()
    elif what == "fmm_setup":
        make_fmm_setup()
    else:
        raise SystemExit(__doc__)
