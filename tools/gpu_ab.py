"""A/B of assembly-time environment switches on one box, interleaved:
python tools/gpu_ab.py <cfg> VAR=a,b [rounds]  (e.g. TDW_SCHED=rr,bytes)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2111_05205_b200 import marching, scenarios

cfg = int(sys.argv[1])
var, vals = sys.argv[2].split("=")
vals = vals.split(",")
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
spec = scenarios.build_spec(cfg)
known = marching.greville_samples(spec)
res = {v: [] for v in vals}
for r in range(rounds):
    for v in vals:
        os.environ[var] = v
        st = marching.BandStore(spec).assemble()
        inf = st.info()
        st.upload_known(*known)
        st.run_resident(1e6, 1)
        tm = st.run_resident(1e6, n_repeat=4)
        sps = tm["steps"] / tm["total_ms"] * 1e3
        conv = st.time_conv(20)
        res[v].append((sps, conv * 1e3))
        print(f"cfg{cfg} {var}={v} round {r}: steps/s {sps:.1f}  conv-only {conv*1e3:.2f}us "
              f"grid {inf['conv_grid']} S {inf['conv_splits']}", flush=True)
        st.close()
for v in vals:
    print(f"{var}={v}: best steps/s {max(s for s, _ in res[v]):.1f}  best conv {min(c for _, c in res[v]):.2f}us")
