timeout 300 python -m pytest tests/test_gpu_march.py -x -q 2>&1 | tail -2
timeout 100 python tools/insitu_probe.py 2 "default"
TDW_KB=3 timeout 100 python tools/insitu_probe.py 2 "kb3"
TDW_KB=5 TDW_RPW=2 timeout 100 python tools/insitu_probe.py 2 "kb5 rpw2"
TDW_KB=4 TDW_RPW=4 timeout 100 python tools/insitu_probe.py 2 "kb4 rpw4"
timeout 100 python tools/insitu_probe.py 3 "default"
