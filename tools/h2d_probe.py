"""H2D rate of tdw_upload_known from page-locked vs pageable buffers (config 2 sizes)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from paper_2111_05205_b200 import _lib, marching, scenarios
spec = scenarios.build_spec(2)
st = marching.BandStore(spec)
uk, qk = marching.greville_samples(spec)
pu = st.pinned_known(0); pu[:] = uk
pq = st.pinned_known(1); pq[:] = qk
for label, a, b in (("pageable", uk, qk), ("pinned", pu, pq), ("pinned u, NULL q", pu, None)):
    for k in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lib = _lib.load()
        _lib.check(lib.tdw_upload_known(st.h, _lib.dptr(a), _lib.dptr(b) if b is not None else None), st.ctx.h, "u")
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{label}: {1e3*dt:.2f} ms", flush=True)
x = torch.empty(255 * 5120, dtype=torch.float64, pin_memory=True)
y = torch.empty_like(x, device="cuda")
for k in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize()
print(f"torch pinned H2D 10.4 MB: {1e3*(time.perf_counter()-t0):.2f} ms")
