"""Assembly fill-kernel rate (evals/s) of a config: python tools/fill_probe.py <cfg> <label>"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2111_05205_b200 import marching, scenarios
cfg = int(sys.argv[1])
spec = scenarios.build_spec(cfg)
best = None
for _ in range(2):
    st = marching.BandStore(spec).assemble()
    i = st.info()
    r = i["n_evals"] / (i["t_fill_ms"] * 1e-3)
    best = max(best or 0, r)
    st.close()
print(f"{sys.argv[2]}: cfg{cfg} fill {i['t_fill_ms']:.1f} ms, {best:.3e} evals/s", flush=True)
