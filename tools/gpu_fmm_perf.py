import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_2111_05205_b200 import fmm, fmm_plan, marching, scenarios
cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 3
nt = int(sys.argv[2]) if len(sys.argv) > 2 else None
spec = scenarios.build_spec(cfgn, nt=nt)
t0 = time.time()
plan = fmm_plan.build_plan(spec, fmm_plan.FmmConfig(ps=4, pt=4, leaf_capacity=20))
t1 = time.time()
print(f"cfg{cfgn} plan {t1-t0:.1f}s leaf {plan.leaf} gamma_near {plan.gamma_near} near {len(plan.near_i)} IL "
      f"{ {L: len(o.il_obs) for L, o in plan.levels.items()} } extra { {L: (len(v[0]), v[2]) for L, v in plan.extra.items()} }", flush=True)
store = fmm.FmmStore(spec, plan=plan)
t2 = time.time()
store.assemble()
t3 = time.time()
print("setup", t2 - t1, "assemble", t3 - t2, store.info(), flush=True)
store.upload_known(*marching.greville_samples(spec))
for r in range(2):
    tm = store.run_resident(1e6, 1)
    print(f"loop {tm['total_ms']:.1f} ms  -> {tm['steps']/tm['total_ms']*1e3:.1f} MOT steps/s", flush=True)
h = store.download()
print("status", h.status, h.n_steps, "max|u|", np.abs(h.u).max())
