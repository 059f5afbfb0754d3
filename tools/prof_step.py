"""Small driver for ncu: assemble config <cfg> and run a short resident march (nt steps)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2111_05205_b200 import marching, scenarios

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 8
spec = scenarios.build_spec(cfg, nt=nt)
st = marching.BandStore(spec).assemble()
st.upload_known(*marching.greville_samples(spec))
st.set_graph(False)
tm = st.run_resident(1e6, 1)
print(st.info(), tm)
