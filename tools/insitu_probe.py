"""In-situ timing of the loop: total per pass vs the convolution launches inside it
(CUDA-event nodes around every K2 launch): python tools/insitu_probe.py <cfg> <label>"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2111_05205_b200 import marching, scenarios
cfg = int(sys.argv[1])
spec = scenarios.build_spec(cfg)
st = marching.BandStore(spec).assemble()
inf = st.info()
st.upload_known(*marching.greville_samples(spec))
st.run_resident(1e6, 2)
tm = st.run_resident(1e6, 3)
tk = st.run_resident(1e6, 3, time_kernels=True)
npass = tk["conv_launches"]
print(f"{sys.argv[2] if len(sys.argv) > 2 else ''}: cfg{cfg} kb {inf['steps_per_pass']} steps/s {tm['steps'] / tm['total_ms'] * 1e3:.0f} "
      f"per-pass {tm['total_ms'] / (npass):.1f} us-equiv "
      f"conv in situ {tk['conv_ms'] / npass * 1e3:.1f} us, timed-loop per pass {tk['total_ms'] / npass * 1e3:.1f} us, "
      f"isolated conv {st.time_conv(10) * 1e3:.1f} us", flush=True)
