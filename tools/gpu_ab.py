"""A/B of assembly-time environment switches on one box, interleaved:
python tools/gpu_ab.py <cfg> <variant> <variant> ... [--rounds R]
a variant is 'default' or VAR=val[+VAR=val...], e.g. TDW_SCHED=rr or
TDW_SOLVER=smem+TDW_SOLVE_CL=8."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2111_05205_b200 import marching, scenarios

args = sys.argv[1:]
rounds = 2
if "--rounds" in args:
    i = args.index("--rounds")
    rounds = int(args[i + 1])
    args = args[:i] + args[i + 2:]
cfg = int(args[0])
variants = args[1:]
spec = scenarios.build_spec(cfg)
known = marching.greville_samples(spec)
base_env = dict(os.environ)
res = {v: [] for v in variants}
for r in range(rounds):
    for v in variants:
        os.environ.clear()
        os.environ.update(base_env)
        if v != "default":
            for kv in v.split("+"):
                k, val = kv.split("=")
                os.environ[k] = val
        st = marching.BandStore(spec).assemble()
        inf = st.info()
        st.upload_known(*known)
        st.run_resident(1e6, 1)
        tm = st.run_resident(1e6, n_repeat=4)
        sps = tm["steps"] / tm["total_ms"] * 1e3
        conv = st.time_conv(20)
        res[v].append((sps, conv * 1e3))
        print(f"cfg{cfg} {v} round {r}: steps/s {sps:.1f}  conv-only {conv*1e3:.2f}us "
              f"grid {inf['conv_grid']} S {inf['conv_splits']} solve_cluster {inf['solve_cluster']} kb {inf['steps_per_pass']} near_w {inf['near_width']} halo {inf['solve_halo']}", flush=True)
        st.close()
for v in variants:
    print(f"{v}: best steps/s {max(s for s, _ in res[v]):.1f}  best conv {min(c for _, c in res[v]):.2f}us")
