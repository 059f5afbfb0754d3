timeout 900 python tools/fmm_shard_probe.py 4 8 2>&1 | tail -12
timeout 900 python tools/fmm_shard_probe.py 3 4 --run 2>&1 | tail -8
