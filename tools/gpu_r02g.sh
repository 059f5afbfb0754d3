for gt in 0 80 160; do
  if [ $gt = 0 ]; then unset TDW_GROUP_TILES; else export TDW_GROUP_TILES=$gt; fi
  for rep in 1 2; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gt $gt', round(d['value']), round(d['e2e']['value']), round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],3))"
  done
done
