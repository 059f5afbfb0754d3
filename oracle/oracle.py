"""ctypes front of the CPU oracle (oracle/libtdw_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.
See tdw_oracle.c for the reference file:line map.  Parity of this oracle is
pinned by tests/test_oracle_golden.py against vectors produced by the
reference itself (tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libtdw_oracle.so"

_lib = None
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i64p = C.POINTER(C.c_int64)


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        L = C.CDLL(str(LIB))
        L.oracle_coeff_table.argtypes = [C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int,
                                         C.c_double, C.c_double, C.c_int, _dp, _dp, _dp]
        L.oracle_coeff_table.restype = C.c_int
        L.oracle_gamma_star.argtypes = [C.c_int, _dp, C.c_int, _i64p, C.c_int, C.c_double, C.c_double]
        L.oracle_gamma_star.restype = C.c_int
        L.oracle_max_diameter.argtypes = [C.c_int, _dp, C.c_int, _i64p]
        L.oracle_max_diameter.restype = C.c_double
        L.oracle_march.argtypes = [C.c_int, _dp, C.c_int, _i64p, _dp, C.c_int, C.c_int, C.c_double,
                                   C.c_double, C.c_int, C.c_int, C.c_double, _dp, _dp, _dp, _dp,
                                   _dp, _dp, _dp, _ip, _ip, _dp]
        L.oracle_march.restype = C.c_int
        L.oracle_sample.argtypes = [C.c_int, _dp, C.c_int, _i64p, C.c_int, C.c_int, C.c_double,
                                    C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _i64p]
        L.oracle_sample.restype = C.c_int
        L.oracle_num_threads.restype = C.c_int
        L.oracle_marcher_create.argtypes = [C.c_int, _dp, C.c_int, _i64p, _dp, C.c_int, C.c_int,
                                            C.c_double, C.c_double, C.c_int, C.c_int, C.c_double,
                                            _dp, _dp, C.c_int, C.POINTER(C.c_void_p), _dp]
        L.oracle_marcher_create.restype = C.c_int
        L.oracle_marcher_run.argtypes = [C.c_void_p, C.c_int, _ip, _dp]
        L.oracle_marcher_run.restype = C.c_int
        L.oracle_marcher_reset.argtypes = [C.c_void_p]
        L.oracle_marcher_reset.restype = None
        L.oracle_marcher_get.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _ip, _ip]
        L.oracle_marcher_get.restype = C.c_int
        L.oracle_marcher_destroy.argtypes = [C.c_void_p]
        L.oracle_marcher_destroy.restype = None
        L.oracle_rhs_rows.argtypes = [C.c_int, _dp, C.c_int, _i64p, _dp, C.c_int, C.c_int, C.c_double,
                                      C.c_double, C.c_int, C.c_int, C.c_int, _ip, C.c_int, _ip,
                                      _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        L.oracle_rhs_rows.restype = C.c_int
        _lib = L
    return _lib


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t)


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def coeff_table(P, A, B, Cc, ez, s, d, c, dt, which="uw", nx=None):
    """Oracle of elemint.retarded_coeff_table (elemint.py:89)."""
    P, A, B, Cc, ez = (_d(np.atleast_2d(v)) for v in (P, A, B, Cc, ez))
    s = _d(np.atleast_1d(s))
    n = len(s)
    kind = {"uw": 0, "bm": 1}.get(which, -1)
    if kind == 1 and nx is None:
        raise ValueError("bm coefficients need the collocation normal nx")
    nxa = _d(np.atleast_2d(nx)) if nx is not None else None
    o0, o1 = np.empty(n), np.empty(n)
    rc = lib().oracle_coeff_table(n, _ptr(P), _ptr(A), _ptr(B), _ptr(Cc), _ptr(ez), _ptr(s), int(d),
                                  float(c), float(dt), kind,
                                  _ptr(nxa) if nxa is not None else None, _ptr(o0), _ptr(o1))
    if rc:
        raise ValueError(f"oracle_coeff_table rc={rc} (d={d}, which={which!r})")
    return o0, o1


def gamma_star(vertices, triangles, d, c, dt) -> int:
    v = _d(vertices)
    t = np.ascontiguousarray(triangles, dtype=np.int64)
    return int(lib().oracle_gamma_star(len(v), _ptr(v), len(t), _ptr(t, _i64p), int(d), float(c), float(dt)))


def march(vertices, triangles, phi, bie, d, c, dt, nt, u_known, q_known, window=True,
          threshold=1e6, want_rhs=False):
    """Oracle of marching.march (marching.py:292).  Returns a dict with
    u, q, tau, sigma (nt-1, ns), n_steps, status, rhs (optional), t_asm."""
    v = _d(vertices)
    t = np.ascontiguousarray(triangles, dtype=np.int64)
    ns = len(t)
    phi = _d(phi)
    uk, qk = _d(u_known), _d(q_known)
    u, q, tau, sig = (np.zeros((nt - 1, ns)) for _ in range(4))
    rhs = np.zeros((nt - 1, ns)) if want_rhs else None
    n_steps, status = C.c_int(0), C.c_int(0)
    t_asm = C.c_double(0.0)
    rc = lib().oracle_march(len(v), _ptr(v), ns, _ptr(t, _i64p), _ptr(phi), 1 if bie == "bmbie" else 0,
                            int(d), float(c), float(dt), int(nt), int(bool(window)), float(threshold),
                            _ptr(uk), _ptr(qk), _ptr(u), _ptr(q), _ptr(tau), _ptr(sig),
                            _ptr(rhs) if rhs is not None else None, C.byref(n_steps),
                            C.byref(status), C.byref(t_asm))
    if rc == 2:
        raise RuntimeError("step matrix is singular")
    if rc == 3:
        raise RuntimeError("solve residual too large")
    if rc:
        raise RuntimeError(f"oracle_march rc={rc}")
    return dict(u=u, q=q, tau=tau, sigma=sig, rhs=rhs, n_steps=n_steps.value,
                status="unstable" if status.value else "stable", t_asm=t_asm.value)


def sample(vertices, triangles, bie, d, c, dt, nt, row_lo, row_hi, n_steps):
    """Bounded CPU-baseline sample: (t_asm, t_loop, n_triples) for rows [lo, hi)."""
    v = _d(vertices)
    t = np.ascontiguousarray(triangles, dtype=np.int64)
    ta, tl, nn = C.c_double(0), C.c_double(0), C.c_int64(0)
    rc = lib().oracle_sample(len(v), _ptr(v), len(t), _ptr(t, _i64p), 1 if bie == "bmbie" else 0,
                             int(d), float(c), float(dt), int(nt), int(row_lo), int(row_hi),
                             int(n_steps), C.byref(ta), C.byref(tl), C.byref(nn))
    if rc:
        raise RuntimeError(f"oracle_sample rc={rc}")
    return ta.value, tl.value, nn.value


class Marcher:
    """Stateful form of `march` (oracle_marcher_*): the lag CSR of the whole
    problem is assembled once, then the time loop advances in bounded chunks
    (bench.py's CPU baseline and --impl reference time chunks of the real loop)."""

    def __init__(self, vertices, triangles, phi, bie, d, c, dt, nt, u_known, q_known, window=True,
                 threshold=1e6, want_rhs=False):
        self._v = _d(vertices)
        self._t = np.ascontiguousarray(triangles, dtype=np.int64)
        self._phi = _d(phi)
        self._uk, self._qk = _d(u_known), _d(q_known)
        self.ns, self.nt = len(self._t), int(nt)
        self.want_rhs = bool(want_rhs)
        self.h = C.c_void_p()
        t_asm = C.c_double(0.0)
        rc = lib().oracle_marcher_create(len(self._v), _ptr(self._v), self.ns, _ptr(self._t, _i64p),
                                         _ptr(self._phi), 1 if bie == "bmbie" else 0, int(d), float(c),
                                         float(dt), self.nt, int(bool(window)), float(threshold),
                                         _ptr(self._uk), _ptr(self._qk), int(self.want_rhs),
                                         C.byref(self.h), C.byref(t_asm))
        if rc == 2:
            raise RuntimeError("step matrix is singular")
        if rc:
            raise RuntimeError(f"oracle_marcher_create rc={rc}")
        self.t_asm = t_asm.value

    def run(self, n_steps: int):
        """Advance up to n_steps MOT steps; returns (steps advanced, wall s, done)."""
        before = self.n_steps
        done, t = C.c_int(0), C.c_double(0.0)
        rc = lib().oracle_marcher_run(self.h, int(n_steps), C.byref(done), C.byref(t))
        if rc == 3:
            raise RuntimeError("solve residual too large")
        if rc:
            raise RuntimeError(f"oracle_marcher_run rc={rc}")
        return self.n_steps - before, t.value, bool(done.value)

    def reset(self):
        lib().oracle_marcher_reset(self.h)

    @property
    def n_steps(self) -> int:
        n, st = C.c_int(0), C.c_int(0)
        lib().oracle_marcher_get(self.h, None, None, None, None, None, C.byref(n), C.byref(st))
        return n.value

    def result(self) -> dict:
        u, q, tau, sig = (np.zeros((self.nt - 1, self.ns)) for _ in range(4))
        rhs = np.zeros((self.nt - 1, self.ns)) if self.want_rhs else None
        n, st = C.c_int(0), C.c_int(0)
        lib().oracle_marcher_get(self.h, _ptr(u), _ptr(q), _ptr(tau), _ptr(sig),
                                 _ptr(rhs) if rhs is not None else None, C.byref(n), C.byref(st))
        return dict(u=u, q=q, tau=tau, sigma=sig, rhs=rhs, n_steps=n.value,
                    status="unstable" if st.value else "stable")

    def close(self):
        if self.h.value:
            lib().oracle_marcher_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def rhs_rows(vertices, triangles, phi, bie, d, c, dt, nt, rows, alphas, u_known, q_known, u, q, tau,
             sigma, window=True):
    """The reference's right-hand side b_row^alpha (marching.py:315-327, sigma/tau
    lag-CSR form restricted to `rows`) recomputed from a GIVEN history, and the
    lag-1 residual (A x^{alpha-1})_row - b.  Returns (b, res), each (len(rows), len(alphas))."""
    v = _d(vertices)
    t = np.ascontiguousarray(triangles, dtype=np.int64)
    ns = len(t)
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    alphas = np.ascontiguousarray(alphas, dtype=np.int32)
    if alphas.size and (alphas.min() < 1 or alphas.max() > nt - 1):
        raise ValueError("alpha out of range")
    b = np.zeros((len(rows), len(alphas)))
    res = np.zeros_like(b)
    arrs = [_d(a) for a in (phi, u_known, q_known, u, q, tau, sigma)]
    rc = lib().oracle_rhs_rows(len(v), _ptr(v), ns, _ptr(t, _i64p), _ptr(arrs[0]), 1 if bie == "bmbie" else 0,
                               int(d), float(c), float(dt), int(nt), int(bool(window)), len(rows),
                               _ptr(rows, _ip), len(alphas), _ptr(alphas, _ip), *(_ptr(a) for a in arrs[1:]),
                               _ptr(b), _ptr(res))
    if rc:
        raise RuntimeError(f"oracle_rhs_rows rc={rc}")
    return b, res
