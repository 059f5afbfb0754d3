timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python bench.py --no-cpu 2>&1 | tail -1
timeout 100 python tools/insitu_probe.py 3 "default"
