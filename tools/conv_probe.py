"""time_conv of one config under the current environment (A/B knobs: TDW_KB, TDW_RPW,
TDW_CONV_DRY, TDW_CONV_RESERVE, ...): python tools/conv_probe.py <cfg> <label>"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2111_05205_b200 import marching, scenarios
cfg = int(sys.argv[1])
spec = scenarios.build_spec(cfg)
st = marching.BandStore(spec).assemble()
inf = st.info()
st.time_conv(3)
us = min(st.time_conv(10) for _ in range(3)) * 1e3
print(f"{sys.argv[2] if len(sys.argv) > 2 else ''}: cfg{cfg} conv {us:.1f} us grid {inf['conv_grid']} kb {inf['steps_per_pass']} "
      f"store {inf['store_bytes']/1e9:.3f} GB -> {inf['store_bytes']/us/1e3:.0f} GB/s", flush=True)
