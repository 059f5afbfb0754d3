"""Cold march(spec) split with per-step callables: store create, assemble, first march (streamed)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench
from paper_2111_05205_b200 import marching, scenarios
spec = bench.per_step_spec(scenarios.build_spec(2))
marching.march(spec)
for rep in range(3):
    t0 = time.perf_counter(); st = marching.BandStore(spec); t1 = time.perf_counter()
    st.assemble(); t2 = time.perf_counter()
    h = marching.march(spec, mats=st); t3 = time.perf_counter()
    h = marching.march(spec, mats=st); t4 = time.perf_counter()
    h = marching.march(spec, mats=st); t5 = time.perf_counter()
    st.close(); t6 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} assemble {1e3*(t2-t1):.1f} march1 {1e3*(t3-t2):.1f} march2 {1e3*(t4-t3):.1f} "
          f"march3 {1e3*(t5-t4):.1f} close {1e3*(t6-t5):.1f} ms", flush=True)
