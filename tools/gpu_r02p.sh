for rep in 1 2 3; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value']), round(d['e2e']['value']), round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],3))"
done
python -c "
import sys; sys.path.insert(0,'.')
from paper_2111_05205_b200 import marching, scenarios
spec = scenarios.build_spec(2); st = marching.BandStore(spec).assemble(); st.upload_known(*marching.greville_samples(spec))
print('conv alone ms', st.time_conv(20))"
timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_sharded.py tests/test_gpu_fmm.py -q -x 2>&1 | tail -2
