import sys, time, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_2111_05205_b200 import _lib, marching, scenarios
spec = scenarios.build_spec(2)
st = marching.BandStore(spec)
lib = _lib.load()
times = marching.greville_times(spec)
pu = st.pinned_known(0)
res = []
for k in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    spec.u_data.sample_many(times, pu)
    t1 = time.perf_counter()
    _lib.check(lib.tdw_upload_known(st.h, _lib.dptr(pu), None), st.ctx.h, "u")
    torch.cuda.synchronize(); t2 = time.perf_counter()
    res.append((1e3*(t1-t0), 1e3*(t2-t1)))
print(os.environ.get("TDW_SAMPLE_THREADS"), "sample %.2f ms upload %.2f ms" % min(res, key=lambda r: r[0]+r[1]), flush=True)
