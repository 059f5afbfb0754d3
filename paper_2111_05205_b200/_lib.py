"""ctypes binding of libtdw.so (the C ABI declared in include/tdw.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is visible, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("TDW_LIB_PATH") or Path(__file__).resolve().parent / "libtdw.so")

TDW_OK = 0
MODES = {"auto": 0, "stored": 1, "on_the_fly": 2}
_ERRORS = {1: ValueError, 2: ValueError, 3: RuntimeError, 4: RuntimeError, 5: RuntimeError,
           6: RuntimeError, 7: RuntimeError, 8: RuntimeError}

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)


class ProblemDesc(C.Structure):
    _fields_ = [("ns", C.c_int32), ("nv", C.c_int32), ("vertices", _dp), ("triangles", _i64p),
                ("phi", _dp), ("bie", C.c_int32), ("d", C.c_int32), ("c", C.c_double),
                ("dt", C.c_double), ("nt", C.c_int32), ("window", C.c_int32),
                ("nranks", C.c_int32), ("rank", C.c_int32), ("mode", C.c_int32)]


class Info(C.Structure):
    _fields_ = [("gamma_star", C.c_int32), ("n_lags", C.c_int32), ("row_lo", C.c_int32),
                ("row_hi", C.c_int32), ("n_band", C.c_int64), ("n_pairs", C.c_int64),
                ("n_evals", C.c_int64), ("store_bytes", C.c_int64), ("step_nnz", C.c_int32),
                ("jacobi_iters", C.c_int32), ("jacobi_bound", C.c_double),
                ("t_assemble_ms", C.c_double), ("t_fill_ms", C.c_double),
                ("max_unit_bytes", C.c_int64), ("max_lag_span", C.c_int32), ("conv_grid", C.c_int32),
                ("conv_splits", C.c_int32), ("solve_cluster", C.c_int32),
                ("n_units", C.c_int64), ("units_hdr32", C.c_int64),
                ("steps_per_pass", C.c_int32), ("near_width", C.c_int32), ("pass_overlap", C.c_int32),
                ("solve_halo", C.c_int32), ("fmm_m2l_pairs", C.c_int64),
                ("conv_rpw", C.c_int32), ("coeff_mode", C.c_int32)]

    def asdict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Timing(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("conv_ms", C.c_double), ("solve_ms", C.c_double),
                ("comm_ms", C.c_double), ("conv_launches", C.c_int32), ("steps", C.c_int32)]

    def asdict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


EXPORTS = {
    "tdw_init": ([C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "tdw_finalize": ([C.c_void_p], C.c_int),
    "tdw_last_error": ([C.c_void_p], C.c_char_p),
    "tdw_device_count": ([], C.c_int),
    "tdw_host_alloc": ([C.c_int64, C.POINTER(C.c_void_p)], C.c_int),
    "tdw_fp64_peak": ([C.c_void_p, C.POINTER(C.c_double)], C.c_int),
    "tdw_host_free": ([C.c_void_p], C.c_int),
    "tdw_coeff_table": ([C.c_void_p, C.c_int64, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int, C.c_double,
                         C.c_double, C.c_int, _dp, _dp, _dp], C.c_int),
    "tdw_coeff_table_device": ([C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double,
                                C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.POINTER(C.c_float)], C.c_int),
    "tdw_problem_create": ([C.c_void_p, C.POINTER(ProblemDesc), C.POINTER(C.c_void_p)], C.c_int),
    "tdw_assemble": ([C.c_void_p], C.c_int),
    "tdw_restrict_pairs": ([C.c_void_p, C.c_int64, _i64p, _i64p], C.c_int),
    "tdw_step_matrix": ([C.c_void_p, _i64p, _i64p, _i64p, _dp], C.c_int),
    "tdw_step_solve": ([C.c_void_p, _dp, _dp, _dp], C.c_int),
    "tdw_problem_info": ([C.c_void_p, C.POINTER(Info)], C.c_int),
    "tdw_march": ([C.c_void_p, _dp, _dp, C.c_double, _dp, _dp, _dp, _dp, _dp, _i32p, _i32p],
                  C.c_int),
    "tdw_upload_known": ([C.c_void_p, _dp, _dp], C.c_int),
    "tdw_upload_known_rows": ([C.c_void_p, C.c_int, C.c_int, C.c_int, _dp], C.c_int),
    "tdw_known_plane_pulse": ([C.c_void_p, C.c_int, _dp, _dp, C.c_double, C.c_double], C.c_int),
    "tdw_march_stream_begin": ([C.c_void_p, C.c_double, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p],
                               C.c_int),
    "tdw_march_stream_finish": ([C.c_void_p, _dp, _dp, _dp, _dp, _dp, _i32p, _i32p], C.c_int),
    "tdw_march_stream_outputs": ([C.c_void_p, _dp, _dp, _dp, _dp], C.c_int),
    "tdw_march_device_known": ([C.c_void_p, C.c_double, _dp, _dp, _dp, _dp, _dp, _i32p, _i32p], C.c_int),
    "tdw_march_resident": ([C.c_void_p, C.c_double, C.c_int, C.c_int, C.POINTER(Timing)], C.c_int),
    "tdw_download": ([C.c_void_p, _dp, _dp, _dp, _dp, _i32p, _i32p], C.c_int),
    "tdw_time_conv": ([C.c_void_p, C.c_int, C.POINTER(C.c_float)], C.c_int),
    "tdw_fmm_time_m2l": ([C.c_void_p, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_float)], C.c_int),
    "tdw_set_graph": ([C.c_void_p, C.c_int], C.c_int),
    "tdw_problem_destroy": ([C.c_void_p], C.c_int),
    "tdw_fmm_setup": ([C.c_void_p, C.c_void_p], C.c_int),
    "tdw_problem_create_shard": ([C.c_void_p, C.POINTER(ProblemDesc), C.POINTER(C.c_void_p)], C.c_int),
    "tdw_march_emulated": ([C.POINTER(C.c_void_p), C.c_int, C.c_double], C.c_int),
    "tdw_tree_build": ([C.c_void_p, C.c_int, _dp, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int,
                        C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "tdw_tree_info": ([C.c_void_p, _i32p, _dp, _dp, _i64p, _i64p, _i64p, _i32p], C.c_int),
    "tdw_tree_level": ([C.c_void_p, C.c_int, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p], C.c_int),
    "tdw_tree_near": ([C.c_void_p, _i64p, _i64p], C.c_int),
    "tdw_tree_extra": ([C.c_void_p, C.c_int, _i32p, _i64p, _i64p, _i64p], C.c_int),
    "tdw_tree_destroy": ([C.c_void_p], C.c_int),
    "tdw_nccl_unique_id": ([C.c_char_p], C.c_int),
    "tdw_comm_init": ([C.c_void_p, C.c_char_p, C.c_int, C.c_int], C.c_int),
}

_lib = None


def load():
    """Load libtdw.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(the CUDA path has no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (args, res) in EXPORTS.items():
            fn = getattr(lib, name, None)
            if fn is None and os.environ.get("TDW_LIB_PATH"):
                continue  # an older library under A/B (tools/lib_ab.sh)
            if fn is None:
                raise RuntimeError(f"{LIB_PATH} does not export {name}: rebuild it")
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


class PinnedArray:
    """A float64 numpy view of page-locked host memory (tdw_host_alloc); freed with the object."""

    def __init__(self, shape):
        self.shape = tuple(int(x) for x in shape)
        n = int(np.prod(self.shape))
        self._p = C.c_void_p()
        check(load().tdw_host_alloc(max(8, 8 * n), C.byref(self._p)), None, "tdw_host_alloc")
        self.array = np.ctypeslib.as_array(C.cast(self._p, _dp), shape=(max(1, n),))[:n].reshape(self.shape)

    def __del__(self):
        try:
            if self._p.value:
                load().tdw_host_free(self._p)
                self._p = C.c_void_p()
        except Exception:
            pass


_PINNED_POOL: dict[int, list[int]] = {}
_PINNED_KEEP = 4  # idle blocks kept per size


class _PinnedBlock:
    """Owner of one page-locked block; it goes back to the pool (still pinned)
    when the last numpy view of it is gone."""

    def __init__(self, ptr: int, nbytes: int):
        self.ptr, self.nbytes = ptr, nbytes

    def __del__(self):
        try:
            idle = _PINNED_POOL.setdefault(self.nbytes, [])
            if len(idle) < _PINNED_KEEP:
                idle.append(self.ptr)
            else:
                load().tdw_host_free(C.c_void_p(self.ptr))
        except Exception:
            pass


def pinned_empty(shape) -> np.ndarray:
    """Uninitialised float64 array in page-locked host memory, from a pool (the
    time loop's outputs are copied into such arrays at full link rate).  The
    array owns its block through `base`; nothing else aliases it."""
    shape = tuple(int(x) for x in shape)
    n = int(np.prod(shape))
    nbytes = max(8, 8 * n)
    idle = _PINNED_POOL.get(nbytes)
    if idle:
        ptr = idle.pop()
    else:
        p = C.c_void_p()
        check(load().tdw_host_alloc(nbytes, C.byref(p)), None, "tdw_host_alloc")
        ptr = p.value
    carr = (C.c_double * max(1, n)).from_address(ptr)
    carr._owner = _PinnedBlock(ptr, nbytes)
    return np.frombuffer(carr, dtype=np.float64)[:n].reshape(shape)


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def check(rc: int, ctx=None, what: str = ""):
    if rc == TDW_OK:
        return
    msg = ""
    if ctx is not None and ctx.value:
        raw = load().tdw_last_error(ctx)
        msg = raw.decode() if raw else ""
    exc = _ERRORS.get(rc, RuntimeError)
    raise exc(f"{what}: {msg or f'libtdw error {rc}'}")


class Context:
    """One CUDA device, one stream (tdw_ctx)."""

    def __init__(self, device: int | None = None):
        lib = load()
        if device is None:
            device = int(os.environ.get("LOCAL_RANK", "0"))
        if lib.tdw_device_count() <= device:
            raise RuntimeError("no CUDA device visible: the MOT path runs on the GPU only")
        self.h = C.c_void_p()
        check(lib.tdw_init(int(device), C.byref(self.h)), None, "tdw_init")
        self.device = device

    def close(self):
        if self.h.value:
            load().tdw_finalize(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Context | None = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context()
    return _default_ctx


def set_default_context(ctx: Context):
    global _default_ctx
    _default_ctx = ctx
