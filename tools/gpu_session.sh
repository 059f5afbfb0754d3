for t in 2 3 4; do TDW_LIB_PATH=ab/libtdw_nm384.so TDW_NEAR_IN_SOLVE=$t timeout 100 python tools/insitu_probe.py 2 "nm384 tail$t" 2>&1 | tail -1; done
TDW_LIB_PATH=ab/libtdw_nm384.so TDW_NEAR_IN_SOLVE=3 timeout 100 python tools/trace_solve.py 2 2>&1 | grep "timeline\|pass_overlap" | python -c "
import sys
for l in sys.stdin:
    if l.startswith('{'):
        d=eval(l); print('m', d['pass_overlap'], 'near_w', d['near_width'])
    else: print(l.strip())"
timeout 100 python tools/insitu_probe.py 2 "current" 2>&1 | tail -1
