for v in "TDW_GUESS=0" "TDW_GUESS=1" "TDW_GUESS=1 TDW_CHECK_EVERY=2"; do echo "== $v"; env $v python tools/trace_solve.py 2 2>&1 | grep "solve phases"; done
python tools/gpu_ab.py 2 TDW_GUESS=0 TDW_GUESS=1 TDW_GUESS=1+TDW_CHECK_EVERY=2 TDW_GUESS=1+TDW_OVERLAP=3 --rounds 1
