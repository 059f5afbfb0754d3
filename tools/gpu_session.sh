for i in 1 2; do
TDW_LIB_PATH=ab/libtdw_near16.so TDW_RPW=3 timeout 100 python tools/insitu_probe.py 2 "near32regs rpw3 kb6" 2>&1 | tail -1
TDW_LIB_PATH=ab/libtdw_near16.so timeout 100 python tools/insitu_probe.py 2 "near32regs rpw4 kb6" 2>&1 | tail -1
timeout 100 python tools/insitu_probe.py 2 "current" 2>&1 | tail -1
done
