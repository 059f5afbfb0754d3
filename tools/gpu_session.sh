for c in 0 1 2 3; do timeout 200 python tools/fill_probe.py $c new; done
timeout 900 python -m pytest tests/test_gpu_coeff.py tests/test_gpu_march.py -x -q 2>&1 | tail -2
