for v in "" "TDW_L2HINT=0" "TDW_HROWS=0" "TDW_SCHED=rr"; do
for i in 1 2; do env $v timeout 100 python tools/insitu_probe.py 2 "[$v]" 2>&1 | tail -1; done; done
