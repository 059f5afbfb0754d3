"""One resident loop of config <cfg> with nt steps under the current environment: prints ok / the error."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2111_05205_b200 import marching, scenarios
cfg, nt = int(sys.argv[1]), int(sys.argv[2])
spec = scenarios.build_spec(cfg, nt=nt)
try:
    st = marching.BandStore(spec).assemble()
    inf = st.info()
    st.upload_known(*marching.greville_samples(spec))
    if len(sys.argv) > 3:
        st.set_graph(False)
    st.run_resident(1e6, 1)
    print("ok", inf["steps_per_pass"], inf["pass_overlap"], inf["solve_halo"], flush=True)
except Exception as e:
    print("FAIL", str(e)[:120], flush=True)
