"""Marching-on-in-time on the B200 (drop-in for tdwavebem.marching).

Keeps the reference's public surface (pkg/src/tdwavebem/marching.py):
`ProblemSpec`, `TimeHistory`, `compute_gamma_star`, `greville_samples`,
`build_retarded_matrices`, `march`.  Differences, all behind the same calls:

* `build_retarded_matrices` returns a `BandStore`: an opaque handle to the
  device-resident kappa-combined banded coefficient store (csrc/assemble.cu)
  instead of per-lag scipy CSR matrices.  Like the reference's
  `RetardedMatrixSet` it can be passed back through `march(spec, mats=...)`.
* `march` runs the whole time loop on the GPU (csrc/march.cu): history
  convolution, Jacobi solve of the lag-1 system, residual test, blow-up
  detector.  Only the Greville sampling of the user's data callables stays on
  the host, exactly where the reference does it (marching.py:312).
"""
from __future__ import annotations

import os

import ctypes as C
import warnings
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

from . import _lib
from .mesh import mesh_stats
from .tbasis import decomposition_weights, eval_basis

__all__ = ["ProblemSpec", "TimeHistory", "BandStore", "StepSolver", "compute_gamma_star", "greville_samples",
           "greville_times", "build_retarded_matrices", "build_step_matrix", "march"]


@dataclass
class ProblemSpec:
    """Exterior scattering problem (marching.py:33-64).

    phi[j] = 1: u unknown on element j (q given); 0: q unknown (u given).
    """

    mesh: object
    phi: np.ndarray
    bie: str
    basis: object
    c: float
    nt: int
    u_data: Callable[[float], np.ndarray] | None = None
    q_data: Callable[[float], np.ndarray] | None = None
    blowup_reference: float = 1.0

    def __post_init__(self):
        self.phi = np.asarray(self.phi, dtype=float)
        if self.phi.shape != (self.mesh.n_elements,):
            raise ValueError("phi must have one flag per element")
        if self.bie not in ("obie", "bmbie"):
            raise ValueError(f"unknown integral equation {self.bie!r}")
        if self.nt < 2:
            raise ValueError("need at least two time steps")
        ratio = mesh_stats(self.mesh).max_edge / (self.c * self.basis.dt)
        if ratio > 1.5:
            warnings.warn(f"mesh edge / (c dt) = {ratio:.2f} exceeds the usual "
                          "stability guideline (~1)", stacklevel=2)


def compute_gamma_star(stats, basis, c: float) -> int:
    """gamma* = ceil(diam / (c dt)) + d + 1 (marching.py:67-69)."""
    return int(np.ceil(stats.max_diameter / (c * basis.dt))) + basis.d + 1


@dataclass
class TimeHistory:
    """Coefficient histories and kappa sums per step (marching.py:184-255)."""

    basis: object
    nt: int
    n_elements: int
    u: np.ndarray = field(init=False)
    q: np.ndarray = field(init=False)
    tau: np.ndarray = field(init=False)
    sigma: np.ndarray = field(init=False)
    n_steps: int = 0
    status: str = "stable"

    def __post_init__(self):
        shape = (self.nt - 1, self.n_elements)
        self.u = np.zeros(shape)
        self.q = np.zeros(shape)
        self.tau = np.zeros(shape)
        self.sigma = np.zeros(shape)

    def stock_sums(self, beta: int):
        """Full kappa sums tau/sigma at step beta, zero-padded history (marching.py:205-214)."""
        w = self.basis.weights
        tau = np.zeros(self.n_elements)
        sig = np.zeros(self.n_elements)
        for k in range(min(self.basis.d + 1, beta) + 1):
            tau += w[k] * self.q[beta - k]
            sig += w[k] * self.u[beta - k]
        return tau, sig

    def windowed_sums(self, beta: int, beta_star: int):
        """kappa sums truncated at the sliding-window bottom beta_star (marching.py:216-225)."""
        w = self.basis.weights
        kmax = min(self.basis.d + 1, beta - beta_star, beta)
        tau = np.zeros(self.n_elements)
        sig = np.zeros(self.n_elements)
        for k in range(kmax + 1):
            tau += w[k] * self.q[beta - k]
            sig += w[k] * self.u[beta - k]
        return tau, sig

    def tilde_sums(self, beta: int, phi, u_known, q_known):
        """Current-step sums with the unknown w0 component dropped (marching.py:227-237)."""
        w = self.basis.weights
        tau = w[0] * q_known * phi
        sig = w[0] * u_known * (1.0 - phi)
        for k in range(1, min(self.basis.d + 1, beta) + 1):
            tau += w[k] * self.q[beta - k]
            sig += w[k] * self.u[beta - k]
        return tau, sig

    def finalize_step(self, beta: int, phi, u_known, q_known, solved):
        """Promote the solved density by phi and refresh tau/sigma (marching.py:239-242)."""
        self.u[beta] = np.where(phi == 1.0, solved, u_known)
        self.q[beta] = np.where(phi == 1.0, q_known, solved)
        self.tau[beta], self.sigma[beta] = self.stock_sums(beta)

    def knot_values(self, kind: str = "u") -> np.ndarray:
        coef = self.u if kind == "u" else self.q
        d = self.basis.d
        bv = [eval_basis(self.basis, 0, g * self.basis.dt) for g in range(d + 1)]
        out = np.zeros((self.nt, self.n_elements))
        for alpha in range(self.nt):
            for g in range(1, d + 1):
                beta = alpha - g
                if 0 <= beta < self.nt - 1:
                    out[alpha] += bv[g] * coef[beta]
        return out


def greville_times(spec) -> np.ndarray:
    """The Greville abscissae t_beta = beta dt + (d+1) dt / 2, beta = 0..nt-2 (marching.py:264-266)."""
    basis = spec.basis
    return np.arange(spec.nt - 1) * basis.dt + 0.5 * (basis.d + 1) * basis.dt


def sample_data(fn, times, out: np.ndarray, on_chunk=None) -> np.ndarray:
    """out[k] = fn(times[k]).  A data callable may also expose the vectorised
    form `fn.sample_many(times, out[, on_chunk])` (same values, all steps at
    once; on_chunk(k0, k1) as rows become ready); plain callables are called
    once per step, as the reference does.  on_chunk always covers every row."""
    many = getattr(fn, "sample_many", None)
    if many is not None:
        try:
            many(times, out, on_chunk=on_chunk)
            return out
        except TypeError:
            many(times, out)
    else:
        for k, t in enumerate(times):
            out[k] = fn(float(t))
    if on_chunk is not None:
        on_chunk(0, len(times))
    return out


def greville_samples(spec):
    """Known data at the Greville abscissae t = beta dt + (d+1) dt / 2 (marching.py:258-276)."""
    nt, ns = spec.nt, spec.mesh.n_elements
    uk = np.zeros((nt - 1, ns))
    qk = np.zeros((nt - 1, ns))
    times = greville_times(spec)
    if spec.u_data is not None:
        sample_data(spec.u_data, times, uk)
    if spec.q_data is not None:
        sample_data(spec.q_data, times, qk)
    return uk, qk


class BandStore:
    """Device-resident banded coefficient store + lag-1 step matrix (tdw_problem)."""

    def __init__(self, spec, window: bool = True, ctx: _lib.Context | None = None,
                 nranks: int = 1, rank: int = 0, shard_only: bool = False, pairs=None,
                 gamma_max: int | None = None, mode: str = "auto"):
        self.ctx = ctx or _lib.default_context()
        lib = _lib.load()
        mesh = spec.mesh
        self._v = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
        self._t = np.ascontiguousarray(mesh.triangles, dtype=np.int64)
        self._phi = np.ascontiguousarray(spec.phi, dtype=np.float64)
        self.ns = mesh.n_elements
        self.nt = int(spec.nt)
        self._spec_basis = spec.basis
        self.window = bool(window)
        desc = _lib.ProblemDesc(
            ns=self.ns, nv=len(self._v), vertices=_lib.dptr(self._v),
            triangles=self._t.ctypes.data_as(C.POINTER(C.c_int64)), phi=_lib.dptr(self._phi),
            bie=1 if spec.bie == "bmbie" else 0, d=int(spec.basis.d), c=float(spec.c),
            dt=float(spec.basis.dt), nt=self.nt, window=int(self.window), nranks=int(nranks),
            rank=int(rank), mode=_mode(mode))
        self.h = C.c_void_p()
        create = lib.tdw_problem_create_shard if shard_only else lib.tdw_problem_create
        _lib.check(create(self.ctx.h, C.byref(desc), C.byref(self.h)), self.ctx.h,
                   "tdw_problem_create")
        self.nranks, self.rank = int(nranks), int(rank)
        self.assembled = False
        # what the device store was built from: march(spec, mats=store) refuses a
        # spec that differs (the split-lag store and the step matrix depend on phi,
        # the coefficients on bie, d, c, dt and the geometry)
        self.key = problem_key(spec)
        self.gamma_max = None if gamma_max is None else int(gamma_max)
        self.pairs = None
        if pairs is not None:
            ii = np.ascontiguousarray(np.asarray(pairs[0]).reshape(-1), dtype=np.int64)
            jj = np.ascontiguousarray(np.asarray(pairs[1]).reshape(-1), dtype=np.int64)
            if ii.shape != jj.shape:
                raise ValueError("pairs: row and column index arrays differ in length")
            _lib.check(lib.tdw_restrict_pairs(self.h, len(ii), ii.ctypes.data_as(C.POINTER(C.c_int64)),
                                              jj.ctypes.data_as(C.POINTER(C.c_int64))),
                       self.ctx.h, "tdw_restrict_pairs")
            self.pairs = len(ii)

    def assemble(self):
        if not self.assembled:
            _lib.check(_lib.load().tdw_assemble(self.h), self.ctx.h, "tdw_assemble")
            self.assembled = True
        return self

    def info(self) -> dict:
        inf = _lib.Info()
        _lib.check(_lib.load().tdw_problem_info(self.h, C.byref(inf)), self.ctx.h, "tdw_problem_info")
        return inf.asdict()

    @property
    def gamma_star(self) -> int:
        return self.info()["gamma_star"]

    @property
    def n_lags(self) -> int:
        return self.info()["n_lags"]

    _streamable = True  # the direct path runs the streamed march (FmmStore: False)

    def pinned_flag(self) -> np.ndarray:
        """Page-locked int32 counter of the streamed march (chunks ready), from the
        process-wide page-locked pool (a cold store allocates nothing)."""
        if not hasattr(self, "_flag"):
            self._flag = _lib.pinned_empty((1,)).view(np.int32)
        return self._flag

    def pinned_known(self, which: int) -> np.ndarray:
        """Page-locked (nt-1, ns) host buffer for the u (0) / q (1) samples, owned by the store."""
        if not hasattr(self, "_pinned"):
            self._pinned = [None, None]
        if self._pinned[which] is None:  # from the page-locked pool (cold stores skip cudaHostAlloc)
            self._pinned[which] = _lib.pinned_empty((self.nt - 1, self.ns))
        return self._pinned[which]

    # benchmark helpers (device-resident inputs/outputs)
    def upload_known(self, u_known, q_known):
        self._uk = np.ascontiguousarray(u_known, dtype=np.float64)
        self._qk = np.ascontiguousarray(q_known, dtype=np.float64)
        _lib.check(_lib.load().tdw_upload_known(self.h, _lib.dptr(self._uk), _lib.dptr(self._qk)),
                   self.ctx.h, "tdw_upload_known")

    def run_resident(self, threshold: float, n_repeat: int = 1, time_kernels: bool = False) -> dict:
        t = _lib.Timing()
        _lib.check(_lib.load().tdw_march_resident(self.h, float(threshold), int(n_repeat),
                                                  int(time_kernels), C.byref(t)),
                   self.ctx.h, "tdw_march_resident")
        return t.asdict()

    def download(self) -> "TimeHistory":
        """Device history -> TimeHistory (after run_resident / an emulated march)."""
        hist = TimeHistory(self._spec_basis, self.nt, self.ns)
        n_steps, status = C.c_int32(0), C.c_int32(0)
        _lib.check(_lib.load().tdw_download(self.h, _lib.dptr(hist.u), _lib.dptr(hist.q),
                                            _lib.dptr(hist.tau), _lib.dptr(hist.sigma),
                                            C.byref(n_steps), C.byref(status)), self.ctx.h,
                   "tdw_download")
        hist.n_steps = int(n_steps.value)
        hist.status = "unstable" if status.value else "stable"
        return hist

    def time_conv(self, n: int = 20) -> float:
        """Average device ms of one history-convolution launch (inputs resident)."""
        ms = C.c_float(0.0)
        _lib.check(_lib.load().tdw_time_conv(self.h, int(n), C.byref(ms)), self.ctx.h, "tdw_time_conv")
        return float(ms.value)

    def set_graph(self, enable: bool):
        _lib.check(_lib.load().tdw_set_graph(self.h, int(bool(enable))), self.ctx.h, "tdw_set_graph")

    def close(self):
        if self.h.value:
            _lib.load().tdw_problem_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _mode(mode: str) -> int:
    """Coefficient mode: "auto" (the banded store when it fits in
    device memory, else on the fly), "stored", "on_the_fly"."""
    if mode not in _lib.MODES:
        raise ValueError(f"unknown coefficient mode {mode!r} (expected one of {sorted(_lib.MODES)})")
    return _lib.MODES[mode]


def problem_key(spec) -> tuple:
    """Everything a device store depends on: geometry, phi, bie, d, c, dt."""
    import hashlib
    h = hashlib.sha1()
    for a in (spec.mesh.vertices, spec.mesh.triangles, spec.phi):
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return (h.hexdigest(), spec.bie, int(spec.basis.d), float(spec.c), float(spec.basis.dt))


def _check_store(mats, spec, window):
    if mats.window != window or mats.nt < spec.nt or mats.ns != spec.mesh.n_elements:
        raise ValueError("matrix set does not cover the required lags")
    if mats.gamma_max is not None and mats.gamma_max < mats.n_lags:
        raise ValueError("matrix set does not cover the required lags")
    if mats.nt != spec.nt:
        raise ValueError(f"store built for nt={mats.nt}, spec has nt={spec.nt}: rebuild it "
                         "(the device history is sized at assembly)")
    key = problem_key(spec)
    if key != mats.key:
        names = ("geometry/phi", "bie", "d", "c", "dt")
        diff = [n for n, a, b in zip(names, key, mats.key) if a != b]
        raise ValueError(f"store was assembled for a different problem ({', '.join(diff)} differ): "
                         "build it from this spec")


def build_retarded_matrices(spec, gamma_max: int | None = None, pairs=None, slab: int = 2_000_000,
                            window: bool = True, mode: str = "auto") -> BandStore:
    """Assemble the device banded store (replaces marching.py:132-181).

    `pairs=(ii, jj)` restricts the store -- and the lag-1 step matrix built from
    it -- to those element pairs (marching.py:132-133, 149; tdw_restrict_pairs).
    `gamma_max` is recorded: like the reference's matrix set, a store asked for
    fewer lags than march needs makes march raise ValueError.  The store itself
    always holds the lags of its window (min(gamma*, nt-1), or nt-1 without
    window).  `slab` (the reference's memory chunking) has no meaning here.
    `mode`: "auto" keeps the coefficients in the banded store when it fits in
    device memory and otherwise recomputes them in every convolution pass;
    "stored" / "on_the_fly" force one of the two."""
    return BandStore(spec, window=window, pairs=pairs, gamma_max=gamma_max, mode=mode).assemble()


class StepSolver:
    """The factorisation object of build_step_matrix: `solve(b)` = A^{-1} b on the
    device (tdw_step_solve, BiCGSTAB to round-off), with the reference's
    residual test (marching.py:330-333)."""

    def __init__(self, store: BandStore):
        self.store = store
        self.last_stats = None

    def solve(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        if b.shape != (self.store.ns,):
            raise ValueError(f"b must have shape ({self.store.ns},)")
        x = np.empty_like(b)
        st = np.zeros(3)
        _lib.check(_lib.load().tdw_step_solve(self.store.h, _lib.dptr(b), _lib.dptr(x), _lib.dptr(st)),
                   self.store.ctx.h, "tdw_step_solve")
        self.last_stats = st
        if st[0] > 1e-10 * max(st[1], 1e-300):
            raise RuntimeError(f"step solve residual {st[0]:.3e} too large")
        return x


def build_step_matrix(spec, mats):
    """A = w0 (W1 phi - U1 (1 - phi)) and its solver (marching.py:279-289): A as a
    scipy CSC matrix in the caller's element order, downloaded from the device
    store, and a StepSolver whose solve(b) runs on the GPU."""
    import scipy.sparse as sp
    if not isinstance(mats, BandStore):
        raise TypeError("mats must come from build_retarded_matrices of this package")
    _check_store(mats, spec, mats.window)
    mats.assemble()
    lib = _lib.load()
    nnz = C.c_int64(0)
    _lib.check(lib.tdw_step_matrix(mats.h, C.byref(nnz), None, None, None), mats.ctx.h, "tdw_step_matrix")
    rows = np.empty(nnz.value, np.int64)
    cols = np.empty(nnz.value, np.int64)
    vals = np.empty(nnz.value)
    p64 = C.POINTER(C.c_int64)
    _lib.check(lib.tdw_step_matrix(mats.h, C.byref(nnz), rows.ctypes.data_as(p64), cols.ctypes.data_as(p64),
                                   _lib.dptr(vals)), mats.ctx.h, "tdw_step_matrix")
    ns = spec.mesh.n_elements
    A = sp.csc_matrix((vals, (rows, cols)), shape=(ns, ns))
    return A, StepSolver(mats)

STREAM_CHUNK = 16  # steps per chunk of the streamed march


def _march_streamed(mats, spec, times, threshold, rhs, hist, n_steps, status) -> int:
    """march()'s streamed form: launch, sample chunk by chunk, publish, finish."""
    lib = _lib.load()
    nk = len(times)
    bufs = {w: (mats.pinned_known(w) if fn is not None else None)
            for w, fn in ((0, spec.u_data), (1, spec.q_data))}
    flag = mats.pinned_flag()
    flag[0] = 0
    # the history arrays are page-locked: the loop writes each chunk's rows into
    # them while it runs (tdw_march_stream_outputs), nothing is copied at the end
    if os.environ.get("TDW_STREAM_OUT", "1") != "0":   # 0: A/B, everything copied at the end
        _lib.check(lib.tdw_march_stream_outputs(mats.h, _lib.dptr(hist.u), _lib.dptr(hist.q), _lib.dptr(hist.tau),
                                                _lib.dptr(hist.sigma)), mats.ctx.h, "tdw_march_stream_outputs")
    _lib.check(lib.tdw_march_stream_begin(
        mats.h, threshold, int(rhs is not None),
        bufs[0].ctypes.data if bufs[0] is not None else None,
        bufs[1].ctypes.data if bufs[1] is not None else None,
        STREAM_CHUNK, flag.ctypes.data), mats.ctx.h, "tdw_march_stream_begin")
    try:
        fns = [(bufs[w], fn) for w, fn in ((0, spec.u_data), (1, spec.q_data)) if fn is not None]
        if all(getattr(fn, "sample_many", None) is None for _, fn in fns):
            # plain callables: the reference's order (u then q per step, marching.py:268-275)
            for k, t in enumerate(times):
                for buf, fn in fns:
                    buf[k] = fn(float(t))
                if (k + 1) % STREAM_CHUNK == 0 or k + 1 == nk:
                    flag[0] = -(-(k + 1) // STREAM_CHUNK)
        else:
            # vectorised sources fill rows out of order (thread pool): publish the
            # longest prefix every source has completed
            import threading
            done = np.zeros((len(fns), nk), dtype=bool)
            lock = threading.Lock()

            def progress(i, k0, k1):
                with lock:
                    done[i, k0:k1] = True
                    full = done.all(axis=0)
                    pre = nk if full.all() else int(np.argmin(full))
                    c = nk if pre == nk else pre // STREAM_CHUNK * STREAM_CHUNK
                    flag[0] = max(int(flag[0]), -(-c // STREAM_CHUNK))
            for i, (buf, fn) in enumerate(fns):
                sample_data(fn, times, buf, on_chunk=lambda k0, k1, i=i: progress(i, k0, k1))
    except BaseException:
        flag[0] = -1  # the device loop stops at the next chunk boundary
        lib.tdw_march_stream_finish(mats.h, None, None, None, None, None, None, None)
        raise
    return lib.tdw_march_stream_finish(mats.h, _lib.dptr(hist.u), _lib.dptr(hist.q), _lib.dptr(hist.tau),
                                       _lib.dptr(hist.sigma), _lib.dptr(rhs) if rhs is not None else None,
                                       C.byref(n_steps), C.byref(status))


def march(spec, window: bool = True, blowup_factor: float = 1e6, mats=None,
          rhs_trace: list | None = None, device_data: bool = False, mode: str = "auto") -> TimeHistory:
    """Run the conventional time marching on the GPU (marching.py:292-338).

    gamma* and the lag count are computed by the library from the mesh
    (tdw_problem_create), so a supplied store is validated against its own
    record of them."""
    if mats is None:
        mats = BandStore(spec, window=window, mode=mode)
    elif not isinstance(mats, BandStore):
        raise TypeError("mats must come from build_retarded_matrices of this package")
    else:
        _check_store(mats, spec, window)
    # outputs in page-locked memory (a pool: blocks come back when the arrays die);
    # the library writes every entry, so the history gets no zero-filled arrays first
    out = _lib.pinned_empty((4, spec.nt - 1, spec.mesh.n_elements))
    hist = TimeHistory.__new__(TimeHistory)
    hist.basis, hist.nt, hist.n_elements = spec.basis, spec.nt, spec.mesh.n_elements
    hist.u, hist.q, hist.tau, hist.sigma = out[0], out[1], out[2], out[3]
    hist.n_steps, hist.status = 0, "stable"
    # Greville samples straight into the store's page-locked buffers, each chunk
    # of steps copied to the device as soon as it is written (the copies overlap
    # the sampling); a data callable that is None gives zero samples on the device
    lib = _lib.load()
    times = greville_times(spec)
    nk = len(times)
    # device_data: data callables that describe themselves (the incident plane
    # pulse, scenarios.PlanePulseData.device_form) are sampled on the device
    dev = {}
    if device_data:
        for which, fn in ((0, spec.u_data), (1, spec.q_data)):
            form = getattr(fn, "device_form", None)
            if fn is not None and form is not None and getattr(fn, "kind", None) == ("u", "q")[which]:
                dev[which] = form()
    for which, (zc, nz, t0, sig) in dev.items():
        _lib.check(lib.tdw_known_plane_pulse(mats.h, which, _lib.dptr(zc), _lib.dptr(nz), float(t0), float(sig)),
                   mats.ctx.h, "tdw_known_plane_pulse")
    threshold = blowup_factor * max(spec.blowup_reference, 1e-30)
    ns, nt = spec.mesh.n_elements, spec.nt
    rhs = np.zeros((nt - 1, ns)) if rhs_trace is not None else None
    n_steps, status = C.c_int32(0), C.c_int32(0)
    host = [(w, fn) for w, fn in ((0, spec.u_data), (1, spec.q_data)) if fn is not None and w not in dev]
    if host and not dev and mats._streamable:
        # streamed: the loop starts at once and takes each chunk of steps as soon as
        # the host has sampled it (tdw_march_stream_begin): the Greville sampling of
        # the data callables (marching.py:258-276) overlaps the device loop
        rc = _march_streamed(mats, spec, times, float(threshold), rhs, hist, n_steps, status)
    else:
        for which, fn in ((0, spec.u_data), (1, spec.q_data)):
            if which in dev:
                continue
            _lib.check(lib.tdw_upload_known_rows(mats.h, which, 0, 0 if fn is not None else nk, None),
                       mats.ctx.h, "tdw_upload_known_rows")
            if fn is None:
                continue
            buf = mats.pinned_known(which)

            def on_chunk(k0, k1, which=which, buf=buf):
                if k1 > k0:
                    _lib.check(lib.tdw_upload_known_rows(mats.h, which, k0, k1 - k0, _lib.dptr(buf[k0:k1])),
                               mats.ctx.h, "tdw_upload_known_rows")
            sample_data(fn, times, buf, on_chunk=on_chunk)
        rc = lib.tdw_march_device_known(mats.h, float(threshold),
                                        _lib.dptr(hist.u), _lib.dptr(hist.q), _lib.dptr(hist.tau),
                                        _lib.dptr(hist.sigma), _lib.dptr(rhs) if rhs is not None else None,
                                        C.byref(n_steps), C.byref(status))
    _lib.check(rc, mats.ctx.h, "march")
    mats.assembled = True
    hist.n_steps = int(n_steps.value)
    hist.status = "unstable" if status.value else "stable"
    if rhs_trace is not None:
        rhs_trace.extend(rhs[k].copy() for k in range(hist.n_steps))
    return hist
