for ch in 1 0; do
  echo "== TDW_CHEB=$ch"
  TDW_CHEB=$ch TDW_TRACE_SOLVE=1 timeout 300 python tools/trace_solve.py 2 2>&1 | grep -E "solve phases|timeline" | tail -2
  TDW_CHEB=$ch timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value']), round(d['e2e']['value']), d['roofline']['avg_launch_ms'])"
done
timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -3
