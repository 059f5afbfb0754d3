for impl in cublas own; do
  if [ $impl = cublas ]; then export TDW_M2L=cublas; else unset TDW_M2L; fi
  timeout 600 python bench.py --config 3 --fmm --steps 3 --warmup 3 --no-cpu > gpurun_out/fmm3_$impl.log 2>&1
  tail -1 gpurun_out/fmm3_$impl.log > gpurun_out/fmm3_$impl.json
  python -c "import json; d=json.load(open('gpurun_out/fmm3_$impl.json')); print('$impl cfg3', d['value'], d['e2e']['value'], d['roofline']['achieved'])"
done
unset TDW_M2L
timeout 600 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu > gpurun_out/fmm4_own.log 2>&1; tail -1 gpurun_out/fmm4_own.log > gpurun_out/fmm4_own.json
python -c "import json; d=json.load(open('gpurun_out/fmm4_own.json')); print('own cfg4', d['value'], d['e2e']['value'], d['roofline']['achieved'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_fmm3_own.csv python tools/fmm_prof.py 3 48 > /dev/null 2>&1
TDW_M2L=cublas timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_fmm3_cublas.csv python tools/fmm_prof.py 3 48 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:m2l_dmma -s 3 -c 1 -o gpurun_out/full_r02d_m2l python tools/fmm_prof.py 3 48 > /dev/null 2>&1
ncu -i gpurun_out/full_r02d_m2l.ncu-rep --page details --csv > gpurun_out/r02d_ncu_full_m2l_details.csv 2>/dev/null
ncu -i gpurun_out/full_r02d_m2l.ncu-rep --page raw --csv > gpurun_out/r02d_ncu_full_m2l_raw.csv 2>/dev/null
ls gpurun_out
