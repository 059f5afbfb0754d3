for nt in 16 32 64; do echo -n "cfg2 nt$nt: "; timeout 60 python tools/bisect_short.py 2 $nt; done
echo -n "cfg1 nt16: "; timeout 60 python tools/bisect_short.py 1 16
timeout 600 python -m pytest tests/test_gpu_march.py -x -q 2>&1 | tail -2
