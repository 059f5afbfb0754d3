"""Solve phase trace and loop timeline (TDW_TRACE_SOLVE=1), march host trace (TDW_TRACE_MARCH=1)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("TDW_TRACE_SOLVE", "1")
os.environ.setdefault("TDW_TRACE_MARCH", "1")
from paper_2111_05205_b200 import marching, scenarios

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec = scenarios.build_spec(cfg)
st = marching.BandStore(spec).assemble()
print(st.info(), flush=True)
st.upload_known(*marching.greville_samples(spec))
st.run_resident(1e6, 1)
st.run_resident(1e6, 1)
