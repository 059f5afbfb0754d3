"""Quick perf probe: per-config assembly, resident loop (graph / no graph), conv-only timing."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2111_05205_b200 import marching, scenarios

cfgs = [int(a) for a in sys.argv[1:]] or [0, 1, 2]
for cfg in cfgs:
    spec = scenarios.build_spec(cfg)
    t0 = time.time()
    st = marching.BandStore(spec).assemble()
    inf = st.info()
    print(f'cfg{cfg} host-wall assemble {time.time()-t0:.3f}s', inf, flush=True)
    st.upload_known(*marching.greville_samples(spec))
    for graph in (True,):
        st.set_graph(graph)
        st.run_resident(1e6, 1)
        tm = st.run_resident(1e6, n_repeat=2)
        print(f'cfg{cfg} graph={graph} steps/s {tm["steps"]/tm["total_ms"]*1e3:.1f} ms/step {tm["total_ms"]/tm["steps"]*1e3:.2f}us', tm, flush=True)
    st.set_graph(True)
    tm = st.run_resident(1e6, n_repeat=1, time_kernels=True)
    print(f'cfg{cfg} timed: conv avg {tm["conv_ms"]/max(tm["conv_launches"],1)*1e3:.2f}us total/step {tm["total_ms"]/tm["steps"]*1e3:.2f}us', tm, flush=True)
    ms = st.time_conv(20)
    gbs = inf['n_band'] * 16 / (ms * 1e-3) / 1e9
    print(f'cfg{cfg} conv-only {ms*1e3:.2f}us  algorithmic {gbs:.0f} GB/s  (store bytes/step {inf["store_bytes"]/1e6:.1f} MB)', flush=True)
    print(f'cfg{cfg} fill: {inf["n_evals"]/(inf["t_fill_ms"]*1e-3):.3e} evals/s', flush=True)
    st.close()
