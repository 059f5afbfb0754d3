timeout 900 python -m pytest tests/test_gpu_fmm.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -2
timeout 600 python tools/gpu_fmm_perf.py 3 2>&1 | tail -3
