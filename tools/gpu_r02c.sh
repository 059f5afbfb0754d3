timeout 600 python -m pytest -x -q tests/test_gpu_fmm.py 2>&1 | grep -E "Error|error|assert|passed|failed" | head -20
timeout 900 python -m pytest -x -q -s tests/test_gpu_march.py -k "rhs_matches_reference_form" 2>&1 | grep -E "cfg|passed|failed|Error|assert" | head -20
timeout 900 python -m pytest -x -q tests/test_gpu_sharded.py 2>&1 | tail -3
