# A/B of library builds on one box: bash tools/lib_ab.sh <cfg> <rounds> lib1.so lib2.so ...
cfg=$1; rounds=$2; shift 2
for r in $(seq $rounds); do for lib in "$@"; do
  echo "== $lib round $r"; TDW_LIB_PATH=$lib python tools/gpu_ab.py $cfg default --rounds 1 2>&1 | grep "round 0"
done; done
