"""Interpolation space-time FMM on the B200 (drop-in for tdwavebem.fmm.fast_march).

Same entry point as the reference (pkg/src/tdwavebem/fmm.py:534-544):
`fast_march(spec, config=None, window=True, blowup_factor=1e6, rhs_trace=None,
return_solver=False)`, returning the reference's `TimeHistory`.  The reference
ships this solver broken; this is the corrected algorithm
(SURVEY.md 8(c) corrections 1-7), restated for the GPU:
  host   fmm_plan.build_plan   -- octree, interpolation, P2M/L2P rows, Toeplitz kernels
  device tdw_fmm_setup + tdw_assemble (near field) + tdw_march (csrc/fmm.cu)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .fmm_plan import FmmConfig, build_plan, step_schedule
from .marching import BandStore, TimeHistory, greville_samples

__all__ = ["FmmConfig", "fast_march", "FmmStore", "fmm_desc_arrays"]


class FmmDesc(C.Structure):
    _p64 = C.POINTER(C.c_int64)
    _pd = C.POINTER(C.c_double)
    _pi = C.POINTER(C.c_int32)
    _fields_ = [("ps", C.c_int32), ("pt", C.c_int32), ("mu", C.c_int32), ("leaf", C.c_int32),
                ("gamma_near", C.c_int32), ("n_leaf_cells", C.c_int32),
                ("leaf_coords", _p64), ("elem_cell", _p64), ("p2m_tau", _pd), ("p2m_sig", _pd),
                ("l2p_val", _pd), ("l2p_bm", _pd), ("t_space", _pd), ("t_time", _pd),
                ("n_levels", C.c_int32), ("lev_ncell", _pi), ("lev_interval", _pd),
                ("lev_parent", _p64), ("lev_octant", _p64), ("lev_noff", _pi),
                ("lev_dark", C.POINTER(C.c_uint8)), ("lev_K0", _pd), ("lev_Kp", _pd),
                ("lev_nil", _p64), ("lev_obs_ptr", _p64), ("lev_il_src", _p64), ("lev_il_off", _p64),
                ("n_extra", C.c_int32), ("extra_lags", _pi), ("extra_npair", _p64),
                ("extra_i", _p64), ("extra_j", _p64), ("ticks_before", _p64), ("k_obs", _p64),
                ("wt", _pd), ("dwt", _pd), ("wts", _pd), ("extra_gmax", _p64)]


def fmm_desc_arrays(plan, nt):
    """Flatten the plan into the arrays of tdw_fmm_desc (kept alive by the caller)."""
    tree = plan.tree
    leaf = tree.levels[plan.leaf]
    levels = [plan.levels[L] for L in range(2, plan.leaf + 1)]
    sch = step_schedule(plan, nt)
    xs = sorted(plan.extra)
    A = dict(
        leaf_coords=np.ascontiguousarray(leaf.coords[plan.elem_cell], dtype=np.int64),
        elem_cell=np.ascontiguousarray(plan.elem_cell, dtype=np.int64),
        p2m_tau=np.ascontiguousarray(plan.p2m_tau), p2m_sig=np.ascontiguousarray(plan.p2m_sig),
        l2p_val=np.ascontiguousarray(plan.l2p_val),
        l2p_bm=np.ascontiguousarray(plan.l2p_bm) if plan.l2p_bm is not None else None,
        t_space=np.ascontiguousarray(plan.t_space), t_time=np.ascontiguousarray(plan.t_time),
        lev_ncell=np.array([o.n_cells for o in levels], np.int32),
        lev_interval=np.array([o.interval for o in levels], np.float64),
        lev_parent=np.concatenate([o.parent for o in levels]).astype(np.int64) if levels else np.zeros(1, np.int64),
        lev_octant=np.ascontiguousarray(np.concatenate([o.octant for o in levels]).astype(np.int64)) if levels else np.zeros(3, np.int64),
        lev_noff=np.array([len(o.offsets) for o in levels], np.int32),
        lev_dark=np.ascontiguousarray(np.concatenate([o.dark.reshape(-1) for o in levels]).astype(np.uint8)) if levels else np.zeros(1, np.uint8),
        lev_K0=np.ascontiguousarray(np.concatenate([o.K0.reshape(-1) for o in levels])) if levels else np.zeros(1),
        lev_Kp=np.ascontiguousarray(np.concatenate([o.Kp.reshape(-1) for o in levels])) if levels else np.zeros(1),
        lev_nil=np.array([len(o.il_obs) for o in levels], np.int64),
        lev_obs_ptr=np.concatenate([o.obs_ptr for o in levels]).astype(np.int64) if levels else np.zeros(1, np.int64),
        lev_il_src=np.concatenate([o.il_src for o in levels] + [np.zeros(0)]).astype(np.int64),
        lev_il_off=np.concatenate([o.il_off for o in levels] + [np.zeros(0)]).astype(np.int64),
        extra_lags=np.array([plan.extra[L][2] for L in xs], np.int32),
        extra_npair=np.array([len(plan.extra[L][0]) for L in xs], np.int64),
        extra_i=np.concatenate([plan.extra[L][0] for L in xs] + [np.zeros(0)]).astype(np.int64),
        extra_j=np.concatenate([plan.extra[L][1] for L in xs] + [np.zeros(0)]).astype(np.int64),
        ticks_before=sch["ticks_before"].astype(np.int64), k_obs=sch["k_obs"].astype(np.int64),
        wt=np.ascontiguousarray(sch["wt"]), dwt=np.ascontiguousarray(sch["dwt"]),
        wts=np.ascontiguousarray(sch["wts"]),
        extra_gmax=np.ascontiguousarray(np.stack([sch["extra_gmax"][L] for L in xs]).astype(np.int64))
        if xs else np.zeros(1, np.int64),
    )
    return A


def _ptr(a, ct):
    return None if a is None else a.ctypes.data_as(C.POINTER(ct))


class FmmStore(BandStore):
    """Device state of the fast solver: near-field banded store + far-field operators."""

    _streamable = False  # the fast solver's loop takes its known data up front

    def __init__(self, spec, config: FmmConfig | None = None, ctx=None, plan=None,
                 nranks: int = 1, rank: int = 0, shard_only: bool = False):
        # nranks > 1: this rank's rows of the near field, M2L into the target
        # leaf cells of those rows (and their ancestors) only; b is all-gathered
        # every step (csrc/fmm.cu, tdw_fmm_loop / tdw_fmm_march_emulated)
        if plan is None:
            (config or FmmConfig()).check_gpu()
        super().__init__(spec, window=True, ctx=ctx, nranks=nranks, rank=rank, shard_only=shard_only)
        self.plan = plan or build_plan(spec, config, tree="device")
        A = fmm_desc_arrays(self.plan, spec.nt)
        self._arrays = A
        p = self.plan
        desc = FmmDesc(ps=p.ps, pt=p.pt, mu=p.mu, leaf=p.leaf, gamma_near=p.gamma_near,
                       n_leaf_cells=p.tree.levels[p.leaf].n_cells,
                       n_levels=len(A["lev_ncell"]), n_extra=len(A["extra_lags"]))
        for k, ct in (("leaf_coords", C.c_int64), ("elem_cell", C.c_int64), ("p2m_tau", C.c_double),
                      ("p2m_sig", C.c_double), ("l2p_val", C.c_double), ("l2p_bm", C.c_double),
                      ("t_space", C.c_double), ("t_time", C.c_double), ("lev_ncell", C.c_int32),
                      ("lev_interval", C.c_double), ("lev_parent", C.c_int64), ("lev_octant", C.c_int64),
                      ("lev_noff", C.c_int32), ("lev_dark", C.c_uint8), ("lev_K0", C.c_double),
                      ("lev_Kp", C.c_double), ("lev_nil", C.c_int64), ("lev_obs_ptr", C.c_int64),
                      ("lev_il_src", C.c_int64), ("lev_il_off", C.c_int64), ("extra_lags", C.c_int32),
                      ("extra_npair", C.c_int64), ("extra_i", C.c_int64), ("extra_j", C.c_int64),
                      ("ticks_before", C.c_int64), ("k_obs", C.c_int64), ("wt", C.c_double),
                      ("dwt", C.c_double), ("wts", C.c_double), ("extra_gmax", C.c_int64)):
            setattr(desc, k, _ptr(A[k], ct))
        _lib.check(_lib.load().tdw_fmm_setup(self.h, C.byref(desc)), self.ctx.h, "tdw_fmm_setup")


def fast_march(spec, config: FmmConfig | None = None, window: bool = True, blowup_factor: float = 1e6,
               rhs_trace: list | None = None, return_solver: bool = False, ctx=None,
               nranks: int = 1, rank: int = 0):
    """Run the fast solver on the GPU (fmm.py:534-544).  `window` is accepted for
    signature compatibility: the near field always uses the gamma_near window.
    `config=None` means the reference's FmmConfig() (ps = pt = 8), which the GPU
    solver rejects with ValueError; pass fmm_plan.baseline_config() (ps = pt = 4).
    Multi-GPU (one process per GPU): pass the rank's context (with its
    communicator, distributed.init_comm) and nranks / rank."""
    store = FmmStore(spec, config, ctx=ctx, nranks=nranks, rank=rank).assemble()
    hist = TimeHistory(spec.basis, spec.nt, spec.mesh.n_elements)
    uk, qk = greville_samples(spec)
    uk, qk = np.ascontiguousarray(uk), np.ascontiguousarray(qk)
    threshold = blowup_factor * max(spec.blowup_reference, 1e-30)
    rhs = np.zeros((spec.nt - 1, spec.mesh.n_elements)) if rhs_trace is not None else None
    n_steps, status = C.c_int32(0), C.c_int32(0)
    rc = _lib.load().tdw_march(store.h, _lib.dptr(uk), _lib.dptr(qk), float(threshold),
                               _lib.dptr(hist.u), _lib.dptr(hist.q), _lib.dptr(hist.tau),
                               _lib.dptr(hist.sigma), _lib.dptr(rhs) if rhs is not None else None,
                               C.byref(n_steps), C.byref(status))
    _lib.check(rc, store.ctx.h, "fast_march")
    hist.n_steps = int(n_steps.value)
    hist.status = "unstable" if status.value else "stable"
    if rhs_trace is not None:
        rhs_trace.extend(rhs[k].copy() for k in range(hist.n_steps))
    if return_solver:
        return hist, store
    return hist
