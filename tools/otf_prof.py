"""One on-the-fly convolution pass of config <cfg> (for ncu): python tools/otf_prof.py <cfg>"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2111_05205_b200 import marching, scenarios
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec = scenarios.build_spec(cfg)
st = marching.BandStore(spec, mode="on_the_fly").assemble()
st.upload_known(*marching.greville_samples(spec))
print(st.info(), st.time_conv(1), flush=True)
