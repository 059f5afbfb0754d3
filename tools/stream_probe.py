"""Does host activity slow the streamed device loop?  Every chunk is published before the
launch; the host then idles / spins in Python / runs numpy until the loop ends (TDW_TRACE_MARCH=1)."""
import sys, time, ctypes as C
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2111_05205_b200 import marching, scenarios, _lib
spec = scenarios.build_spec(2)
st = marching.BandStore(spec).assemble()
uk, qk = marching.greville_samples(spec)
lib = _lib.load()
bu, bq = st.pinned_known(0), st.pinned_known(1)
bu[:] = uk; bq[:] = qk
flag = st.pinned_flag()
out = _lib.pinned_empty((4, spec.nt - 1, spec.mesh.n_elements))
n, s = C.c_int32(0), C.c_int32(0)
chunk = marching.STREAM_CHUNK
nch = -(-(spec.nt - 1) // chunk)
x = np.linspace(0, 1, 5120)
for mode in ("idle", "idle", "idle", "python-spin", "numpy", "numpy-write-pinned", "idle", "late-last-chunk", "late-last-chunk", "idle"):
    flag[0] = nch - 1 if mode.startswith("late") else nch
    _lib.check(lib.tdw_march_stream_outputs(st.h, *[_lib.dptr(out[k]) for k in range(4)]), st.ctx.h, "o")
    print(mode, flush=True)
    t0 = time.perf_counter()
    _lib.check(lib.tdw_march_stream_begin(st.h, 1e6, 0, bu.ctypes.data, bq.ctypes.data, chunk, flag.ctypes.data), st.ctx.h, "b")
    k = 0
    while time.perf_counter() - t0 < 0.015 and mode != "idle":
        if mode == "python-spin":
            k += 1
        elif mode == "numpy":
            y = np.exp(-x * x) * np.sin(x)
        else:
            bu[k % 255] = np.exp(-x * x) * np.sin(x) * 0 + uk[k % 255]
            k += 1
    if mode.startswith("late"):
        while time.perf_counter() - t0 < 0.012:
            pass
        flag[0] = nch
    _lib.check(lib.tdw_march_stream_finish(st.h, *[_lib.dptr(out[k]) for k in range(4)], None, C.byref(n), C.byref(s)), st.ctx.h, "f")
    print("   call ms", (time.perf_counter() - t0) * 1e3)
