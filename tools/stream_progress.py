"""Device progress against host publishing in a streamed march: after every published chunk
the host notes how many output chunks the loop has already written back (NaN-prefilled rows)."""
import sys, time, ctypes as C
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import bench
from paper_2111_05205_b200 import marching, scenarios, _lib
spec = bench.per_step_spec(scenarios.build_spec(2))
st = marching.BandStore(spec).assemble()
for _ in range(3):
    marching.march(spec, mats=st)
lib = _lib.load()
times = marching.greville_times(spec)
nk = len(times)
bu, bq = st.pinned_known(0), st.pinned_known(1)
flag = st.pinned_flag()
out = _lib.pinned_empty((4, spec.nt - 1, spec.mesh.n_elements))
n, s = C.c_int32(0), C.c_int32(0)
CH = marching.STREAM_CHUNK
for rep in range(2):
    out[0][:] = np.nan
    flag[0] = 0
    log = []
    t0 = time.perf_counter()
    _lib.check(lib.tdw_march_stream_outputs(st.h, *[_lib.dptr(out[k]) for k in range(4)]), st.ctx.h, "o")
    _lib.check(lib.tdw_march_stream_begin(st.h, 1e6, 0, bu.ctypes.data if spec.u_data else None,
                                          bq.ctypes.data if spec.q_data else None, CH, flag.ctypes.data), st.ctx.h, "b")
    def arrived():
        return sum(1 for c in range(-(-nk // CH)) if not np.isnan(out[0][min(nk, (c + 1) * CH) - 1, 0]))
    for k, t in enumerate(times):
        if spec.u_data: bu[k] = spec.u_data(float(t))
        if spec.q_data: bq[k] = spec.q_data(float(t))
        if (k + 1) % CH == 0 or k + 1 == nk:
            flag[0] = -(-(k + 1) // CH)
            log.append(((time.perf_counter() - t0) * 1e3, int(flag[0]), arrived()))
    while arrived() < -(-nk // CH):
        log.append(((time.perf_counter() - t0) * 1e3, int(flag[0]), arrived()))
        time.sleep(0.0005)
    _lib.check(lib.tdw_march_stream_finish(st.h, *[_lib.dptr(out[k]) for k in range(4)], None, C.byref(n), C.byref(s)), st.ctx.h, "f")
    print("total ms", (time.perf_counter() - t0) * 1e3)
    print(" ".join(f"{t:.1f}:{p}/{a}" for t, p, a in log))
