"""Retarded element coefficients on the B200 (drop-in for tdwavebem.elemint).

Same names, arguments, return values and errors as the reference
(pkg/src/tdwavebem/elemint.py:89-228); the arithmetic runs in
`tdw_coeff_table` (csrc/coeff_table.cu) -- there is no CPU path.
"""
from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["retarded_coeff_table", "single_layer_coeff", "double_layer_coeff", "bm_coeffs"]

_SUPPORTED_D = (1, 2, 3)


def retarded_coeff_table(P, A, B, C, ez, s, d, c, dt, which="uw", nx=None):
    """(U, W) or the Burton-Miller pair for a batch of (point, triangle, s).

    elemint.py:89-186: P, A, B, C, ez are (n, 3); s is (n,); `which` is "uw" or
    "bm" (the latter needs the collocation normals nx).
    """
    P, A, B, C, ez = (np.ascontiguousarray(np.atleast_2d(np.asarray(v, float))) for v in (P, A, B, C, ez))
    s = np.ascontiguousarray(np.atleast_1d(np.asarray(s, float)))
    if d not in _SUPPORTED_D:
        raise ValueError(f"basis order d={d} not supported by the closed forms (d in 1..3)")
    if which == "bm":
        if nx is None:
            raise ValueError("bm coefficients need the collocation normal nx")
        nx = np.ascontiguousarray(np.atleast_2d(np.asarray(nx, float)))
    elif which != "uw":
        raise ValueError(f"unknown coefficient kind {which!r}")
    n = len(s)
    # broadcast single rows the way numpy does in the reference
    P, A, B, C, ez = (np.ascontiguousarray(np.broadcast_to(v, (n, 3))) for v in (P, A, B, C, ez))
    if nx is not None:
        nx = np.ascontiguousarray(np.broadcast_to(nx, (n, 3)))
    out0, out1 = np.empty(n), np.empty(n)
    if n == 0:
        return out0, out1
    ctx = _lib.default_context()
    rc = _lib.load().tdw_coeff_table(
        ctx.h, n, _lib.dptr(P), _lib.dptr(A), _lib.dptr(B), _lib.dptr(C), _lib.dptr(ez),
        _lib.dptr(s), int(d), float(c), float(dt), 1 if which == "bm" else 0,
        _lib.dptr(nx) if nx is not None else None, _lib.dptr(out0), _lib.dptr(out1))
    _lib.check(rc, ctx.h, "tdw_coeff_table")
    return out0, out1


def _triangle(E):
    E = np.asarray(E, float)
    if E.shape != (3, 3):
        raise ValueError("triangle must be given as 3 vertices of 3 coordinates")
    n = np.cross(E[1] - E[0], E[2] - E[0])
    nn = np.linalg.norm(n)
    if nn == 0.0:
        raise ValueError("degenerate triangle")
    return E[0], E[1], E[2], n / nn


def single_layer_coeff(xi, E, gamma: int, basis, c: float) -> float:
    """U_ij^(gamma) (0 for gamma <= 0), elemint.py:200-207."""
    if gamma <= 0:
        return 0.0
    a, b, cc, n = _triangle(E)
    U, _ = retarded_coeff_table(xi, a, b, cc, n, [c * gamma * basis.dt], basis.d, c, basis.dt)
    return float(U[0])


def double_layer_coeff(xi, E, gamma: int, basis, c: float) -> float:
    """W_ij^(gamma) (0 for gamma <= 0), elemint.py:210-217."""
    if gamma <= 0:
        return 0.0
    a, b, cc, n = _triangle(E)
    _, W = retarded_coeff_table(xi, a, b, cc, n, [c * gamma * basis.dt], basis.d, c, basis.dt)
    return float(W[0])


def bm_coeffs(xi, nx, E, gamma: int, basis, c: float):
    """Burton-Miller pair (Ubar, Wbar) (zeros for gamma <= 0), elemint.py:220-228."""
    if gamma <= 0:
        return 0.0, 0.0
    a, b, cc, n = _triangle(E)
    ub, wb = retarded_coeff_table(xi, a, b, cc, n, [c * gamma * basis.dt], basis.d, c, basis.dt,
                                  which="bm", nx=[nx])
    return float(ub[0]), float(wb[0])
