import sys, time, warnings
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from oracle import fmm_oracle
from paper_2111_05205_b200 import fmm, fmm_plan, marching, scenarios
base = scenarios.build_spec(1, nt=40)
for bie, d, Z in (("bmbie", 2, 20), ("obie", 1, 100)):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        spec = marching.ProblemSpec(base.mesh, np.ones(1280), bie, type(base.basis)(d, base.basis.dt), 1.0, 40, q_data=base.q_data)
    cfg = fmm_plan.FmmConfig(ps=4, pt=4, leaf_capacity=Z)
    h = fmm.fast_march(spec, cfg)
    plan = fmm_plan.build_plan(spec, cfg)
    uk, qk = marching.greville_samples(spec)
    r = fmm_oracle.FmmOracle(spec, plan).run(uk, qk)
    e = np.linalg.norm(h.u - r["u"], axis=1) / np.maximum(np.linalg.norm(r["u"], axis=1), 1e-300)
    print(bie, d, Z, "worst step vs oracle", e.max(), flush=True)
