timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -1
for i in 1 2; do for pk in 1 0; do TDW_NEAR_PACKED=$pk timeout 100 python tools/insitu_probe.py 2 "packed$pk" 2>&1 | tail -1; done; done
TDW_NEAR_PACKED=1 timeout 100 python tools/trace_solve.py 2 2>&1 | grep "timeline\|near structure" | tail -2
for c in 0 1; do TDW_NEAR_PACKED=1 timeout 100 python tools/insitu_probe.py $c "packed" 2>&1 | tail -1; done
