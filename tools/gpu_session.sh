timeout 900 python -m pytest tests/test_gpu_fmm.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -1
timeout 600 python bench.py --config 3 --fmm --steps 2 --warmup 1 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['value'], d['roofline']['frac'])"
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', d['value'], d['roofline']['frac'], d['config']['plan_host_s'])"
