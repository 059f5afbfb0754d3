"""e2e of march(spec, mats=store) with per-step callables for several stream chunk sizes."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench
from paper_2111_05205_b200 import marching, scenarios
spec = bench.per_step_spec(scenarios.build_spec(2))
st = marching.BandStore(spec).assemble()
for ch in [16, 8, 4, 2, 32, 16]:
    marching.STREAM_CHUNK = ch
    for _ in range(4):
        h = marching.march(spec, mats=st)
    t0 = time.perf_counter()
    for _ in range(10):
        h = marching.march(spec, mats=st)
    dt = (time.perf_counter() - t0) / 10
    print(f"chunk {ch}: {dt*1e3:.2f} ms per call, {(spec.nt-1)/dt:.0f} steps/s", flush=True)
