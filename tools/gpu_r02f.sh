for gt in 4 8 16 40; do
  echo "== group tiles $gt"
  TDW_GROUP_TILES=$gt timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['roofline']['avg_launch_ms'], d['config']['conv_grid'])"
done
