"""Per-rank convolution pass of the row-sharded direct path, measured on one GPU:
shard r of N assembles only its rows; tdw_time_conv times its pass alone.  The loop
at N GPUs adds the (redundant) solves and one all-gather per step, so this is the
per-rank work, not a multi-GPU measurement.  python tools/shard_conv_probe.py <cfg>"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2111_05205_b200 import marching, scenarios
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec = scenarios.build_spec(cfg)
for n in (1, 2, 4, 8):
    worst = 0.0
    for r in range(n):
        st = marching.BandStore(spec, nranks=n, rank=r, shard_only=n > 1).assemble()
        i = st.info()
        st.upload_known(*marching.greville_samples(spec))
        us = min(st.time_conv(10) for _ in range(2)) * 1e3
        worst = max(worst, us)
        st.close()
        if r == 0:
            kb = i["steps_per_pass"]
            print(f"cfg{cfg} N={n} rank 0: rows {i['row_hi'] - i['row_lo']} band {i['n_band']} kb {kb} m {i['pass_overlap']} "
                  f"conv {us:.1f} us", flush=True)
    print(f"cfg{cfg} N={n}: slowest rank's pass {worst:.1f} us = {worst / kb:.1f} us per step", flush=True)
