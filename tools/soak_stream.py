"""Soak test of the streamed march: repeated march(spec, mats=store) calls must be bit-identical."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import bench
from paper_2111_05205_b200 import marching, scenarios
for cfg, n in ((0, 300), (2, 60), (1, 100)):
    spec = bench.per_step_spec(scenarios.build_spec(cfg))
    st = marching.BandStore(spec).assemble()
    ref = marching.march(spec, mats=st)
    t0 = time.perf_counter()
    for k in range(n):
        h = marching.march(spec, mats=st)
        assert h.status == ref.status and h.n_steps == ref.n_steps
        for name in ("u", "q", "tau", "sigma"):
            if not np.array_equal(getattr(h, name), getattr(ref, name)):
                raise SystemExit(f"cfg{cfg} call {k}: {name} differs")
    print(f"cfg{cfg}: {n} streamed marches bit-identical, {(time.perf_counter()-t0)/n*1e3:.2f} ms per call", flush=True)
    st.close()
