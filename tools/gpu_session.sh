timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for i in 1 2; do timeout 100 python tools/insitu_probe.py 2 "default" 2>&1 | tail -1; TDW_NEAR_IN_SOLVE=2 TDW_OVERLAP=5 timeout 100 python tools/insitu_probe.py 2 "m5 tail2" 2>&1 | tail -1; done
timeout 100 python tools/trace_solve.py 2 2>&1 | grep "pass_overlap" | python -c "
import sys
for l in sys.stdin:
    d=eval(l); print('m', d['pass_overlap'], 'near_w', d['near_width'], 'kb', d['steps_per_pass'], 'halo', d['solve_halo'])"
