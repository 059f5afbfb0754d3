for r in 1 2; do for lib in ab/libtdw_near16.so ab/libtdw_near12.so; do TDW_LIB_PATH=$lib timeout 100 python tools/insitu_probe.py 2 $lib; done; done
