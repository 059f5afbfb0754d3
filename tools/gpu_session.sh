timeout 900 python -m pytest tests/test_gpu_march.py -x -q -k "device_side" 2>&1 | tail -2
timeout 200 python -c "
import sys, time; sys.path.insert(0,'.')
from paper_2111_05205_b200 import marching, scenarios
spec=scenarios.build_spec(2); st=marching.BandStore(spec).assemble()
for dd in (False, True, False, True):
    for _ in range(2): marching.march(spec, mats=st, device_data=dd)
    t0=time.perf_counter()
    for _ in range(5): h=marching.march(spec, mats=st, device_data=dd)
    print('device_data', dd, 255*5/(time.perf_counter()-t0), 'steps/s', flush=True)
"
