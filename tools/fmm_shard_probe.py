"""Target-cell sharding of the FMM: per-shard near-field band and M2L pairs
(python tools/fmm_shard_probe.py <cfg> <nranks> [--run])."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2111_05205_b200 import distributed, fmm, fmm_plan, scenarios

cfg, n = int(sys.argv[1]), int(sys.argv[2])
spec = scenarios.build_spec(cfg)
conf = fmm_plan.FmmConfig(ps=4, pt=4, leaf_capacity=20)
plan = fmm_plan.build_plan(spec, conf)
one = fmm.FmmStore(spec, conf, plan=plan).assemble()
i1 = one.info()
one.close()
print(f"cfg{cfg} 1 rank: n_band {i1['n_band']} m2l_pairs {i1['fmm_m2l_pairs']}", flush=True)
for r in range(n):
    sh = fmm.FmmStore(spec, conf, plan=plan, nranks=n, rank=r, shard_only=True).assemble()
    i = sh.info()
    print(f"  rank {r}/{n}: rows [{i['row_lo']},{i['row_hi']}) n_band {i['n_band']} "
          f"({i['n_band'] / i1['n_band']:.3f}) m2l_pairs {i['fmm_m2l_pairs']} ({i['fmm_m2l_pairs'] / i1['fmm_m2l_pairs']:.3f})",
          flush=True)
    sh.close()
if "--run" in sys.argv:
    t0 = time.time()
    hs, infos = distributed.fast_march_emulated(spec, n, conf, plan=plan)
    print(f"emulated {n} shards: {time.time() - t0:.1f} s wall, status {hs[0].status}", flush=True)
