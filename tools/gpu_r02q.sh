run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value']), round(d['roofline']['avg_launch_ms'],4))"; }
run TDW_X=0
run TDW_DIAG_NO_NEAR=1
run TDW_NEAR_IN_SOLVE=0
