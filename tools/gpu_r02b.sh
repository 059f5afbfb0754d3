set -x
timeout 900 python -m pytest -x -q tests/test_gpu_fmm.py tests/test_gpu_sharded.py 2>&1 | tail -5
timeout 900 python -m pytest -x -q -s tests/test_gpu_march.py -k "rhs_matches_reference_form" 2>&1 | grep -E "cfg|passed|failed|Error" | tail -8
for impl in cublas own; do
  if [ $impl = cublas ]; then export TDW_M2L=cublas; else unset TDW_M2L; fi
  timeout 600 python bench.py --config 3 --fmm --steps 3 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/fmm3_$impl.json
  python -c "import json; d=json.load(open('gpurun_out/fmm3_$impl.json')); print('$impl cfg3', d['value'], d['roofline']['achieved'])"
done
unset TDW_M2L
timeout 600 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu 2>&1 | tail -1 > gpurun_out/fmm4_own.json
python -c "import json; d=json.load(open('gpurun_out/fmm4_own.json')); print('own cfg4', d['value'], d['roofline']['achieved'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_fmm3_own.csv python tools/fmm_prof.py 3 48 > /dev/null 2>&1
TDW_M2L=cublas timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_fmm3_cublas.csv python tools/fmm_prof.py 3 48 > /dev/null 2>&1
ls gpurun_out | tail
