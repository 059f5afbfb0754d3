"""Where the end-to-end march(spec, mats=store) time goes (config from argv, default 2).
Run with TDW_TRACE_MARCH=1 for the library's own upload / loop / download split."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2111_05205_b200 import marching, scenarios
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec = scenarios.build_spec(cfg)
st = marching.BandStore(spec).assemble()
for k in range(4):
    t0 = time.perf_counter(); uk, qk = marching.greville_samples(spec); t1 = time.perf_counter()
    h = marching.march(spec, mats=st); t2 = time.perf_counter()
    print(f'greville {1e3*(t1-t0):.2f} ms  march (incl. its own sampling) {1e3*(t2-t1):.2f} ms', flush=True)
st.upload_known(uk, qk)
tm = st.run_resident(1e6, 3)
print('resident per loop ms', tm['total_ms'] / 3)
st.close()
