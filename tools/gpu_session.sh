timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do timeout 300 python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['graph'])"; done
TDW_TRACE_MARCH=1 timeout 120 python tools/e2e_probe.py 2 2>&1 | tail -4
