run() { echo "== $*"; env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value']), round(d['e2e']['value']), round(d['roofline']['avg_launch_ms'],4), d['config']['conv_grid'], d['config']['steps_per_conv_pass'])"; }
run TDW_X=0
run TDW_CONV_RESERVE=0
run TDW_KB=6
run TDW_KB=6 TDW_NEAR_IN_SOLVE=3
run TDW_KB=6 TDW_CONV_RESERVE=0
run TDW_NEAR_IN_SOLVE=2
run TDW_NEAR_IN_SOLVE=4
