"""Where one warm march(spec, mats=store) call spends its host time (config 2, per-step callables)."""
import cProfile, pstats, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench
from paper_2111_05205_b200 import marching, scenarios
spec = bench.per_step_spec(scenarios.build_spec(2))
st = marching.BandStore(spec).assemble()
for _ in range(4):
    h = marching.march(spec, mats=st)
t0 = time.perf_counter()
for _ in range(10):
    h = marching.march(spec, mats=st)
print("per call ms", (time.perf_counter() - t0) * 100)
pr = cProfile.Profile(); pr.enable()
for _ in range(10):
    h = marching.march(spec, mats=st)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
