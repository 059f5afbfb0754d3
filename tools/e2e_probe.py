import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2111_05205_b200 import marching, scenarios
spec = scenarios.build_spec(2)
st = marching.BandStore(spec).assemble()
for k in range(3):
    t0 = time.perf_counter(); uk, qk = marching.greville_samples(spec); t1 = time.perf_counter()
    h = marching.march(spec, mats=st); t2 = time.perf_counter()
    print(f'greville {1e3*(t1-t0):.1f} ms  march {1e3*(t2-t1):.1f} ms', flush=True)
st.upload_known(uk, qk)
tm = st.run_resident(1e6, 3)
print('resident per loop ms', tm['total_ms'] / 3)
