"""Host-side operator data of the interpolation space-time FMM.

Builds, once per problem, everything the time loop needs, as flat numpy
arrays consumed by the GPU loop (libtdw `tdw_fmm_*`) and by the CPU
restatement (oracle/fmm_oracle.py):

  * the space-time octree (fmm_tree.build_tree, corrected extra pairs),
  * interpolation schemes in space (ps) and time (pt) (fmm_interp),
  * P2M rows per element -- 7-point rule x cardinal weights, value and normal
    derivative (reference fmm.py:238-275), L2P rows per element -- value and
    the Burton-Miller operator n.grad with n = -n_i (fmm.py:276-292),
  * Toeplitz kernel tensors per (level, offset, order p) with the corrected
    node-offset sign (fmm.py:72-122; SURVEY.md 8(c) correction 2) and the dark-
    lag masks (fmm.py:124-131),
  * interaction lists of every level regrouped by observation cell,
  * child octants / parent links for M2M and L2L (fmm.py:314-326, 371-419),
  * the extra (same-interval) pair lists and their lag counts (corrected rule,
    fmm.py:223-234 with SURVEY correction 6).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from math import comb

import numpy as np

from .fmm_interp import TRI7_BARY, TRI7_W, InterpScheme, triangle_gauss_rule
from .fmm_tree import build_tree
from .tbasis import trunc_pow


@dataclass
class FmmConfig:
    """Reference FmmConfig (fmm.py:35-41), with the reference's defaults (ps = pt = 8,
    leaf capacity 100, mu = 8).  The GPU fast solver implements ps = pt = 4 and
    mu <= 8 (the BASELINE configuration, with leaf capacity 20 as SURVEY 8(d) pins):
    `check_gpu()` raises ValueError naming that limit for anything else."""
    ps: int = 8
    pt: int = 8
    leaf_capacity: int = 100
    mu: int = 8
    element_extrapolation: float = 1.0

    GPU_PS = 4
    GPU_PT = 4
    GPU_MU_MAX = 8

    def check_gpu(self):
        if self.ps != self.GPU_PS or self.pt != self.GPU_PT:
            raise ValueError(f"the GPU fast solver supports ps = pt = {self.GPU_PS} interpolation "
                             f"orders (BASELINE configs 3-4); got ps={self.ps}, pt={self.pt}")
        if not 1 <= self.mu <= self.GPU_MU_MAX:
            raise ValueError(f"the GPU fast solver supports 1 <= mu <= {self.GPU_MU_MAX}; got mu={self.mu}")
        return self


def baseline_config() -> FmmConfig:
    """BASELINE configs 3-4: 4 x 4 x 4 spatial nodes, temporal order 4, leaf capacity
    20 (leaf edge 3.3-4.2 c dt: the smallest the mu = 8 causality check admits), mu = 8."""
    return FmmConfig(ps=4, pt=4, leaf_capacity=20, mu=8)


def cmp_coeff(p: int, m: int, k: int) -> float:
    """Auxiliary recurrence coefficients c_m^p(k) (fmm.py:44-49, PAPER Algorithm 1)."""
    if not 0 <= m <= p - 2:
        raise ValueError(f"m must lie in [0, {p - 2}], got {m}")
    return float(comb(p, m) * ((k - 1) ** (p - m) - 2 * k ** (p - m) + (k + 1) ** (p - m)) * (-1) ** m)


def kernel_tensor(tree, level: int, offset, p: int, d: int, ps: int, pt: int) -> np.ndarray:
    """Toeplitz tensor K[da1, da2, da3, tau] of the M2L operator (corrected sign)."""
    lev = tree.levels[level]
    h = lev.half_width
    node_diff = 2.0 * np.arange(-(ps - 1), ps) / (ps - 1)
    off = np.asarray(offset, float) * 2.0 * h
    g = -h * node_diff
    dx, dy, dz = off[0] + g, off[1] + g, off[2] + g
    r = np.sqrt(dx[:, None, None] ** 2 + dy[None, :, None] ** 2 + dz[None, None, :] ** 2)
    interval = tree.interval(level)
    tick = interval / (pt - 1)
    if p == 0:
        T = tree.c * tick * np.arange(0, (tree.mu + 2) * (pt - 1) + 1)
        return np.ascontiguousarray(trunc_pow(T[None, None, None, :] - r[..., None], d) / r[..., None])
    base = tree.mu * (pt - 1)
    T = tree.c * tick * np.arange(base, base + 2 * (pt - 1) + 1)
    diff = T[None, None, None, :] - r[..., None]
    if np.any(diff <= 0.0):
        raise RuntimeError("distant-future kernel sampled inside the causality cone")
    return np.ascontiguousarray(comb(d, p) * diff ** (d - p) / r[..., None])


def lag_is_dark(tree, level: int, offset, lag: int) -> bool:
    h = tree.levels[level].half_width
    gap = np.maximum(np.abs(np.asarray(offset, float)) - 1.0, 0.0) * 2.0 * h
    return tree.c * (lag + 1) * tree.interval(level) <= float(np.linalg.norm(gap))


def dense_operator(K: np.ndarray, ps: int, pt: int, toff: int) -> np.ndarray:
    """Materialise the (ps^3 pt) x (ps^3 pt) matrix of a Toeplitz tensor
    (row ((a1 ps + a2) ps + a3) pt + m, fmm.py:134-162)."""
    P = ps - 1
    a = np.arange(ps)
    da = a[:, None] - a[None, :] + P                    # (ps, ps)
    dm = np.arange(pt)[:, None] - np.arange(pt)[None, :] + toff
    M = K[da[:, None, None, :, None, None], da[None, :, None, None, :, None],
          da[None, None, :, None, None, :]]             # (a1,a2,a3,b1,b2,b3, tau)
    M = M[..., dm]                                      # (..., m, n)
    M = M.transpose(0, 1, 2, 6, 3, 4, 5, 7)
    n = ps ** 3 * pt
    return np.ascontiguousarray(M.reshape(n, n))


@dataclass
class LevelOps:
    level: int
    n_cells: int
    interval: float
    parent: np.ndarray            # (n,) index into level-1 (M2M/L2L), -1 at level 2
    octant: np.ndarray            # (n, 3) child position inside the parent
    offsets: np.ndarray           # (n_off, 3) distinct interaction offsets
    il_obs: np.ndarray            # interaction pairs sorted by (obs, original order)
    il_src: np.ndarray
    il_off: np.ndarray            # offset index per pair
    obs_ptr: np.ndarray           # (n+1,) CSR over observation cells
    K0: np.ndarray                # (n_off, (2ps-1)^3, ntau0) near-future tensors
    Kp: np.ndarray                # (d, n_off, (2ps-1)^3, ntaup) derivative tensors
    dark: np.ndarray              # (n_off, mu+1) lag l=1..mu+1 dark


@dataclass
class FmmPlan:
    cfg: FmmConfig
    tree: object
    d: int
    c: float
    dt: float
    bie: str
    ps: int
    pt: int
    mu: int
    leaf: int
    levels: dict = field(default_factory=dict)     # level -> LevelOps (2..leaf)
    elem_cell: np.ndarray | None = None            # (ns,) leaf cell of each element
    cell_ptr: np.ndarray | None = None             # (ncell+1,) CSR of leaf cells -> elements
    cell_elems: np.ndarray | None = None
    p2m_tau: np.ndarray | None = None              # (ns, ps^3) rows, element order
    p2m_sig: np.ndarray | None = None
    l2p_val: np.ndarray | None = None              # (ns, ps^3)
    l2p_bm: np.ndarray | None = None
    t_space: np.ndarray | None = None              # (2, ps, ps) transfer (half 0, 1)
    t_time: np.ndarray | None = None               # (2, pt, pt)
    gamma_near: int = 0
    near_i: np.ndarray | None = None
    near_j: np.ndarray | None = None
    extra: dict = field(default_factory=dict)      # level -> (ii, jj, lags)
    scheme_s: object = None
    scheme_t: object = None


def _gpu_visible() -> bool:
    try:
        from . import _lib
        return _lib.load().tdw_device_count() > 0
    except Exception:
        return False


def build_plan(spec, config: FmmConfig | None = None, tree: str = "auto") -> FmmPlan:
    """tree: "device" (csrc/tree.cu, the GPU fast solver's default), "host"
    (fmm_tree.build_tree, numpy; the CPU oracle's), or "auto" (device when a GPU
    is visible).  Both builders give the same tree bit for bit."""
    cfg = config or FmmConfig()
    mesh = spec.mesh
    d, c, dt = spec.basis.d, spec.c, spec.basis.dt
    ps, pt, mu = cfg.ps, cfg.pt, cfg.mu
    if tree not in ("auto", "device", "host"):
        raise ValueError(f"unknown tree builder {tree!r}")
    if tree == "device" or (tree == "auto" and _gpu_visible()):
        from .fmm_tree import build_tree_device
        tree = build_tree_device(mesh, c, dt, cfg.leaf_capacity, mu, corrected=True)
    else:
        tree = build_tree(mesh, c, dt, cfg.leaf_capacity, mu, corrected=True)
    sch_s, sch_t = InterpScheme(ps), InterpScheme(pt)
    plan = FmmPlan(cfg, tree, d, c, dt, spec.bie, ps, pt, mu, tree.leaf_level,
                   scheme_s=sch_s, scheme_t=sch_t)
    leaf = tree.levels[tree.leaf_level]
    ns = mesh.n_elements
    plan.elem_cell = tree.elem_cell[tree.leaf_level].astype(np.int64)
    counts = np.array([len(e) for e in leaf.cell_elems])
    plan.cell_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    plan.cell_elems = np.concatenate(leaf.cell_elems).astype(np.int64)

    # P2M / L2P rows (element order)
    prefactor = 1.0 / (4.0 * np.pi * (c * dt) ** d)
    v0, v1, v2 = mesh.element_vertices()
    ex = cfg.element_extrapolation
    h = leaf.half_width
    n3 = ps ** 3
    # all elements at once: 7-point rule points (ns, 7, 3) and weights (ns, 7)
    E = np.stack([v0, v1, v2], axis=1)
    pts = np.einsum("gk,ekc->egc", TRI7_BARY, E)
    area = 0.5 * np.linalg.norm(np.cross(E[:, 1] - E[:, 0], E[:, 2] - E[:, 0]), axis=1)
    wts = TRI7_W[None, :] * area[:, None]
    xi = (pts - leaf.centres[plan.elem_cell][:, None, :]) / h
    ng = xi.shape[1]
    w = [sch_s.weights(xi[:, :, k].reshape(-1), ex).reshape(ns, ng, ps) for k in range(3)]
    dw = [(sch_s.dweights(xi[:, :, k].reshape(-1), ex) / h).reshape(ns, ng, ps) for k in range(3)]
    n = mesh.normals
    p2m_tau = np.einsum("eg,ega,egb,egc->eabc", wts, w[0], w[1], w[2]).reshape(ns, n3)
    p2m_sig = (np.einsum("eg,ega,egb,egc->eabc", wts, n[:, 0, None, None] * dw[0], w[1], w[2])
               + np.einsum("eg,ega,egb,egc->eabc", wts, w[0], n[:, 1, None, None] * dw[1], w[2])
               + np.einsum("eg,ega,egb,egc->eabc", wts, w[0], w[1], n[:, 2, None, None] * dw[2])
               ).reshape(ns, n3)
    plan.p2m_tau = prefactor * p2m_tau
    plan.p2m_sig = prefactor * p2m_sig
    xi = (mesh.centroids - leaf.centres[plan.elem_cell]) / h
    w = [sch_s.weights(xi[:, k]) for k in range(3)]
    plan.l2p_val = np.einsum("ga,gb,gc->gabc", w[0], w[1], w[2]).reshape(ns, n3)
    if spec.bie == "bmbie":
        dw = [sch_s.dweights(xi[:, k]) / h for k in range(3)]
        nrm = -mesh.normals
        plan.l2p_bm = (np.einsum("g,ga,gb,gc->gabc", nrm[:, 0], dw[0], w[1], w[2])
                       + np.einsum("g,ga,gb,gc->gabc", nrm[:, 1], w[0], dw[1], w[2])
                       + np.einsum("g,ga,gb,gc->gabc", nrm[:, 2], w[0], w[1], dw[2])).reshape(ns, n3)
    plan.t_space = np.stack([sch_s.transfer(0), sch_s.transfer(1)])
    plan.t_time = np.stack([sch_t.transfer(0), sch_t.transfer(1)])

    # per level operators
    for L in range(2, tree.leaf_level + 1):
        lev = tree.levels[L]
        if L >= 3:
            par = tree.levels[L - 1]
            parent = lev.parent.astype(np.int64)
            octant = lev.coords - (par.coords[parent] << 1)
        else:
            parent = np.full(lev.n_cells, -1, np.int64)
            octant = np.zeros((lev.n_cells, 3), np.int64)
        if lev.il_obs is not None and len(lev.il_obs):
            offs, inv = np.unique(lev.il_offsets, axis=0, return_inverse=True)
            inv = inv.reshape(-1)
            order = np.argsort(lev.il_obs, kind="stable")
            il_obs, il_src, il_off = lev.il_obs[order], lev.il_src[order], inv[order]
        else:
            offs = np.zeros((0, 3), np.int64)
            il_obs = il_src = il_off = np.zeros(0, np.int64)
        obs_ptr = np.searchsorted(il_obs, np.arange(lev.n_cells + 1)).astype(np.int64)
        K0 = np.stack([kernel_tensor(tree, L, o, 0, d, ps, pt).reshape((2 * ps - 1) ** 3, -1)
                       for o in offs]) if len(offs) else np.zeros((0, (2 * ps - 1) ** 3, 1))
        Kp = np.stack([np.stack([kernel_tensor(tree, L, o, p, d, ps, pt).reshape((2 * ps - 1) ** 3, -1)
                                 for o in offs]) for p in range(1, d + 1)]) if len(offs) else \
            np.zeros((d, 0, (2 * ps - 1) ** 3, 1))
        dark = np.array([[lag_is_dark(tree, L, o, l) for l in range(1, mu + 2)] for o in offs],
                        dtype=bool).reshape(len(offs), mu + 1)
        plan.levels[L] = LevelOps(L, lev.n_cells, tree.interval(L), parent, octant, offs,
                                  il_obs, il_src, il_off, obs_ptr, K0, Kp, dark)

    # near field and extra (same-interval) pairs
    cent = mesh.centroids
    radii = mesh.element_radii()
    ii, jj = tree.near_pairs
    dist = np.linalg.norm(cent[ii] - cent[jj], axis=1) + radii[jj]
    plan.gamma_near = int(np.ceil(dist.max() / (c * dt))) + d + 1
    plan.near_i, plan.near_j = ii, jj
    for L, (ei, ej) in tree.extra_pairs.items():
        lags = int(np.floor(tree.interval(L) / dt)) + 2          # corrected lag count
        plan.extra[L] = (ei, ej, lags)
    return plan


def step_schedule(plan: FmmPlan, nt: int):
    """Per step alpha = 1..nt-1 the host-side time bookkeeping of the loop
    (fmm.py:438-520 with SURVEY corrections 3-5): ticks to run before the step,
    the observation interval / L2P weights, the extra-list lag limits and the
    P2M interval / weights of the step's source.  Returned as arrays."""
    tree, dt = plan.tree, plan.dt
    interval = tree.interval(plan.leaf)
    sch_t = plan.scheme_t
    ticks_before = np.zeros(nt, np.int64)
    k_obs = np.zeros(nt, np.int64)
    wt = np.zeros((nt, plan.pt))
    dwt = np.zeros((nt, plan.pt))
    k_src = np.zeros(nt, np.int64)
    wts = np.zeros((nt, plan.pt))
    extra_gmax = {L: np.zeros(nt, np.int64) for L in plan.extra}
    last_tick = -1
    for alpha in range(1, nt):
        t_alpha = alpha * dt
        while (last_tick + 2) * interval <= t_alpha + 1e-12:
            last_tick += 1
        ticks_before[alpha] = last_tick                  # ticks 0..last_tick done before the step
        ko = int(np.floor(t_alpha / interval + 1e-12))
        k_obs[alpha] = ko
        eta = (t_alpha - (ko + 0.5) * interval) / (0.5 * interval)
        wt[alpha] = sch_t.weights([eta])[0]
        dwt[alpha] = sch_t.dweights([eta])[0] / (0.5 * interval * plan.c)
        for L, (_, _, lags) in plan.extra.items():
            int_L = tree.interval(L)
            k_now = int(np.floor(t_alpha / int_L + 1e-12))
            g_ok = 0
            for g in range(1, min(alpha, lags) + 1):
                t_src = (alpha - g) * dt
                if int(np.floor((t_src + dt) / int_L + 1e-12)) != k_now:
                    break
                g_ok = g
            extra_gmax[L][alpha] = g_ok
        t_src = (alpha - 1) * dt
        ks = int(np.floor((t_src + dt) / interval + 1e-12))
        k_src[alpha] = ks
        eta_s = (t_src - (ks + 0.5) * interval) / (0.5 * interval)
        wts[alpha] = sch_t.weights([eta_s], extrapolate=2.0 * dt / interval)[0]
    return dict(ticks_before=ticks_before, k_obs=k_obs, wt=wt, dwt=dwt, k_src=k_src, wts=wts,
                extra_gmax=extra_gmax)
