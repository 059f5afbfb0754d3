"""Where a cold march(spec) spends its time (config <cfg>): problem create, assembly, loop."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2111_05205_b200 import marching, scenarios, _lib
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec = scenarios.build_spec(cfg)
marching.march(spec)  # warm (context, modules, pinned pool)
for rep in range(3):
    t0 = time.perf_counter(); st = marching.BandStore(spec); t1 = time.perf_counter()
    st.assemble(); t2 = time.perf_counter()
    h = marching.march(spec, mats=st); t3 = time.perf_counter()
    inf = st.info(); st.close(); t4 = time.perf_counter()
    st2 = marching.BandStore(spec).assemble(); st2.set_graph(False); st2.upload_known(*marching.greville_samples(spec))
    tg = st2.run_resident(1e6, 1)["total_ms"]; st2.close()
    print(f"direct-launch loop {tg:.1f} ms; create {1e3*(t1-t0):.1f} ms, assemble {1e3*(t2-t1):.1f} ms (device {inf['t_assemble_ms']:.1f}, fill {inf['t_fill_ms']:.1f}), "
          f"march {1e3*(t3-t2):.1f} ms, close {1e3*(t4-t3):.1f} ms", flush=True)
