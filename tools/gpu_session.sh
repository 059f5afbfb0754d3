timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x 2>&1 | tail -1
timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu 2>&1 | tail -1 > gpurun_out/bench_cfg4.json; python -c "import json; d=json.load(open('gpurun_out/bench_cfg4.json')); print('cfg4', d['value'], d['e2e']['value'], d['roofline']['frac'])"
