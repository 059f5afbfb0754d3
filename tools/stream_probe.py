"""Device time of the streamed loop when every chunk is published before the launch
(TDW_TRACE_MARCH=1 prints it): separates the loop's own cost from the host's pacing."""
import sys, ctypes as C
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
for mode in ("prepublished", "prepublished", "prepublished+outputs", "prepublished+outputs"):
    flag[0] = nch
    if "outputs" in mode:
        _lib.check(lib.tdw_march_stream_outputs(st.h, *[_lib.dptr(out[k]) for k in range(4)]), st.ctx.h, "o")
    print(mode, flush=True)
    _lib.check(lib.tdw_march_stream_begin(st.h, 1e6, 0, bu.ctypes.data, bq.ctypes.data, chunk, flag.ctypes.data), st.ctx.h, "b")
    _lib.check(lib.tdw_march_stream_finish(st.h, *[_lib.dptr(out[k]) for k in range(4)], None, C.byref(n), C.byref(s)), st.ctx.h, "f")
tm = st.run_resident(1e6, 3)
print("resident loop ms", tm["total_ms"] / 3)
