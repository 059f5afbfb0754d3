"""Full-size FMM fixtures for configs 3 and 4 from the CPU restatement.

oracle/fmm_oracle.py is the corrected restatement of the reference's fast
solver; it is pinned to the runtime-patched reference itself at 1280 elements
(tests/golden/fmm_ref.npz, make_golden.py fmm_ref).  This script runs it at the
BASELINE sizes (config 3: 20480 elements, Nt = 512; config 4: two spheres,
40960 elements, Nt = 1024; ps = pt = 4, leaf capacity 20, mu = 8), which takes
minutes to an hour on the build container's cores, and keeps a row subsample of
every step plus a few complete steps:

    python tests/golden/make_fmm_golden.py 3
    python tests/golden/make_fmm_golden.py 4
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import fmm_oracle  # noqa: E402
from paper_2111_05205_b200 import fmm_plan, marching, scenarios  # noqa: E402

OUT = Path(__file__).resolve().parent


def main(cfg: int):
    spec = scenarios.build_spec(cfg)
    t0 = time.perf_counter()
    plan = fmm_plan.build_plan(spec, fmm_plan.baseline_config())
    t_plan = time.perf_counter() - t0
    uk, qk = marching.greville_samples(spec)
    t0 = time.perf_counter()
    orc = fmm_oracle.FmmOracle(spec, plan)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    r = orc.run(uk, qk)
    t_run = time.perf_counter() - t0
    x = r["u"] if spec.phi[0] == 1.0 else r["q"]
    ns, nt = spec.mesh.n_elements, spec.nt
    rng = np.random.default_rng(7)
    sub = np.sort(rng.choice(ns, size=256, replace=False))
    full_steps = np.unique(np.linspace(0, r["n_steps"] - 1, 6).astype(int))
    np.savez_compressed(
        OUT / f"fmm_cfg{cfg}.npz", cfg=cfg, status=r["status"], n_steps=r["n_steps"],
        unknown_norm=np.linalg.norm(x, axis=1), rhs_norm=np.linalg.norm(r["rhs"], axis=1),
        sub=sub, unknown_sub=x[:, sub], full_steps=full_steps,
        unknown_full=x[full_steps], t_plan=t_plan, t_setup=t_setup, t_run=t_run,
        note="oracle/fmm_oracle.py (corrected restatement), ps=pt=4, Z=20, mu=8")
    print(f"cfg{cfg}: {r['status']} {r['n_steps']} steps, plan {t_plan:.1f} s, setup {t_setup:.1f} s, "
          f"run {t_run:.1f} s, max|x| {np.abs(x).max():.4g}")


if __name__ == "__main__":
    main(int(sys.argv[1]))
