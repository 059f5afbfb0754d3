for tol in 1e-15 1e-14 1e-13; do
  echo "== tol $tol"
  TDW_SOLVE_TOL=$tol TDW_TRACE_SOLVE=1 timeout 300 python tools/trace_solve.py 2 2>&1 | grep -E "solve phases|timeline" | tail -2
  TDW_SOLVE_TOL=$tol timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['avg_launch_ms'])"
done
