timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
python tools/prof_step.py 2 16 > gpurun_out/pp.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:fill_kernel -c 1 -o gpurun_out/full_r01e_fill_kernel python tools/prof_step.py 2 16 > gpurun_out/ncu_r01e_fill.log 2>&1; tail -1 gpurun_out/ncu_r01e_fill.log
timeout 600 python bench.py > gpurun_out/bench_final.log 2>&1; tail -1 gpurun_out/bench_final.log | cut -c1-300
