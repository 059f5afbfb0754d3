timeout 900 python bench.py --config 4 --steps 2 --warmup 1 --no-cpu 2>&1 | tail -1
timeout 600 python bench.py --config 3 --fmm --steps 2 --warmup 1 --no-cpu 2>&1 | tail -1
