"""Short FMM run for ncu launch lists: python tools/fmm_prof.py <cfg> <nt>"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2111_05205_b200 import fmm, fmm_plan, marching, scenarios
cfg, nt = int(sys.argv[1]), int(sys.argv[2])
spec = scenarios.build_spec(cfg, nt=nt)
st = fmm.FmmStore(spec, fmm_plan.FmmConfig(ps=4, pt=4, leaf_capacity=20)).assemble()
st.upload_known(*marching.greville_samples(spec))
tm = st.run_resident(1e6, 1)
print(tm, flush=True)
