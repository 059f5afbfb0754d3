timeout 900 python -m pytest tests/test_gpu_march.py -q -s -k "cfg0_matches or cfg1_d2 or cfg2_full_size_matches or rhs_matches" 2>&1 | grep -E "vs reference|passed|failed"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:otf_conv -s 1 -c 1 -o gpurun_out/full_r02h_otf python tools/otf_prof.py 2 > gpurun_out/ncu_otf.log 2>&1
ncu -i gpurun_out/full_r02h_otf.ncu-rep --page details --csv > gpurun_out/r02h_ncu_full_otf_details.csv 2>/dev/null
ncu -i gpurun_out/full_r02h_otf.ncu-rep --page raw --csv > gpurun_out/r02h_ncu_full_otf_raw.csv 2>/dev/null
tail -2 gpurun_out/ncu_otf.log
