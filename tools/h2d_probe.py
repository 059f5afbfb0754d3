"""H2D rate of tdw_upload_known from page-locked vs pageable buffers (config 2 sizes),
right after the host wrote the buffer (as march() does) and after a pause."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2111_05205_b200 import _lib, marching, scenarios
spec = scenarios.build_spec(2)
st = marching.BandStore(spec)
lib = _lib.load()
times = marching.greville_times(spec)
pu = st.pinned_known(0)
def up(a):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _lib.check(lib.tdw_upload_known(st.h, _lib.dptr(a), None), st.ctx.h, "u")
    torch.cuda.synchronize(); return 1e3 * (time.perf_counter() - t0)
for k in range(4):
    spec.u_data.sample_many(times, pu)
    a = up(pu)
    time.sleep(0.05)
    b = up(pu)
    pu[:] = 1.0
    c = up(pu)
    print(f"after sample_many {a:.2f} ms, after a pause {b:.2f} ms, after a single-thread write {c:.2f} ms", flush=True)
