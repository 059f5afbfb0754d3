timeout 600 python -m pytest tests/test_gpu_march.py -q -x 2>&1 | tail -1
for i in 1 2; do timeout 100 python tools/insitu_probe.py 2 "tail4" 2>&1 | tail -1; done
timeout 100 python tools/trace_solve.py 2 2>&1 | grep "phases\|timeline" | tail -2
timeout 100 python tools/insitu_probe.py 1 "cfg1" 2>&1 | tail -1
