timeout 400 python bench.py 2>&1 | tail -1
