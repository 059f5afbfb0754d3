timeout 600 python -m pytest tests/test_gpu_march.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -1
for i in 1 2; do timeout 100 python tools/insitu_probe.py 2 "tail tasks" 2>&1 | tail -1; TDW_KB=6 timeout 100 python tools/insitu_probe.py 2 "tail tasks kb6" 2>&1 | tail -1; done
timeout 100 python tools/trace_solve.py 2 2>&1 | grep "phases\|timeline" | tail -2
for c in 0 1; do timeout 100 python tools/insitu_probe.py $c "tail tasks" 2>&1 | tail -1; done
