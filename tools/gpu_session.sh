timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -1
for c in 0 1 2 3; do timeout 200 python tools/insitu_probe.py $c "new default" 2>&1 | tail -1; done
timeout 600 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['e2e_device_boundary_data']['value'], d['roofline']['frac'], d['config']['steps_per_conv_pass'])"
