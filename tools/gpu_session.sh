for v in "TDW_RPW=4" "TDW_RPW=2" "TDW_RPW=3" "TDW_OVERLAP=4"; do env $v timeout 100 python tools/insitu_probe.py 2 "[$v]" 2>&1 | tail -1; done
