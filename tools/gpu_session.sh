timeout 900 python -m pytest tests/test_gpu_fmm.py tests/test_gpu_sharded.py -x -q 2>&1 | tail -2
