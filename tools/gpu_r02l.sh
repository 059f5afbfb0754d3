for m in 5 6 4; do
  python -c "from paper_2111_05205_b200 import build as b; b.build(extra=['-DTDW_FILL_MINB(D)=$m'])" > /dev/null 2>&1 || echo build failed
  echo "== minb $m"; python tools/cold_probe.py 2 2>&1 | tail -1; python tools/cold_probe.py 3 2>&1 | tail -1
done
