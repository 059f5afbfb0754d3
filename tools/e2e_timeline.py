"""Host timeline of one warm streamed march(spec, mats=store) (config 2, per-step callables):
when tdw_march_stream_begin returns, when the sampling ends, when finish returns."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench
from paper_2111_05205_b200 import marching, scenarios, _lib
spec = bench.per_step_spec(scenarios.build_spec(2))
st = marching.BandStore(spec).assemble()
for _ in range(4):
    marching.march(spec, mats=st)
lib = _lib.load()
stamps = {}
class Wrap:
    def __init__(self, fn, name):
        self.fn, self.name = fn, name
    def __call__(self, *a):
        stamps[self.name + "_in"] = time.perf_counter()
        r = self.fn(*a)
        stamps[self.name + "_out"] = time.perf_counter()
        return r
class LibProxy:
    def __getattr__(self, k):
        f = getattr(lib, k)
        return Wrap(f, k) if k.startswith("tdw_march_stream") else f
marching._lib.load = lambda: LibProxy()
tm = st.run_resident(1e6, 2)
print("device loop ms", tm["total_ms"] / 2)
for rep in range(3):
    t0 = time.perf_counter()
    h = marching.march(spec, mats=st)
    t1 = time.perf_counter()
    f = lambda k: (stamps.get(k, t0) - t0) * 1e3
    print(f"call {(t1 - t0) * 1e3:.2f} ms: outputs {f('tdw_march_stream_outputs_in'):.2f}, begin in {f('tdw_march_stream_begin_in'):.2f} "
          f"out {f('tdw_march_stream_begin_out'):.2f}, sampling done / finish in {f('tdw_march_stream_finish_in'):.2f}, "
          f"finish out {f('tdw_march_stream_finish_out'):.2f}")
