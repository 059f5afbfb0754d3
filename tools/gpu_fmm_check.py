import sys, time, warnings
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from oracle import fmm_oracle, oracle
from paper_2111_05205_b200 import fmm, fmm_plan, marching, scenarios

def spec1280(bie, d, nt=128):
    base = scenarios.build_spec(1, nt=nt)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return marching.ProblemSpec(base.mesh, np.ones(1280), bie, type(base.basis)(d, base.basis.dt), 1.0, nt, q_data=base.q_data)

for bie, d, Z in (("obie", 1, 100), ("bmbie", 2, 100), ("bmbie", 2, 20), ("obie", 1, 20)):
    spec = spec1280(bie, d)
    cfg = fmm_plan.FmmConfig(ps=4, pt=4, leaf_capacity=Z)
    plan = fmm_plan.build_plan(spec, cfg)
    t0 = time.time()
    h, store = fmm.fast_march(spec, cfg, return_solver=True)
    t1 = time.time()
    uk, qk = marching.greville_samples(spec)
    r = fmm_oracle.FmmOracle(spec, plan).run(uk, qk)
    t2 = time.time()
    e = np.linalg.norm(h.u - r["u"], axis=1) / np.maximum(np.linalg.norm(r["u"], axis=1), 1e-300)
    d_ = oracle.march(spec.mesh.vertices, spec.mesh.triangles, spec.phi, bie, d, 1.0, spec.basis.dt, spec.nt, uk, qk)
    print(f"{bie} d={d} Z={Z} leaf={plan.leaf} gpu {t1-t0:.2f}s oracle {t2-t1:.1f}s status {h.status}/{r['status']} "
          f"worst-step vs oracle {e.max():.3e} whole {np.linalg.norm(h.u-r['u'])/np.linalg.norm(r['u']):.3e} "
          f"| vs direct {np.linalg.norm(h.u-d_['u'])/np.linalg.norm(d_['u']):.4f}", flush=True)
