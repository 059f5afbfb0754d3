# Round-2 ncu evidence (config 2): bench line, launch list, full captures of K2 and K1
# at the bench configuration.  usage: bash tools/profile_r02.sh <tag>
tag=${1:-r02a}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$tag.log 2>&1; tail -1 gpurun_out/bench_$tag.log > gpurun_out/bench_$tag.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_$tag.log 2>&1
for ks in conv_kernel:4 fill_kernel:0 solve_halo_kernel:40 near_step_kernel:40; do
  k=${ks%%:*}; skip=${ks##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s $skip -c 1 -o gpurun_out/full_${tag}_$k \
      python tools/prof_step.py 2 256 > gpurun_out/ncu_${tag}_$k.log 2>&1 || true
  ncu -i gpurun_out/full_${tag}_$k.ncu-rep --page details --csv > gpurun_out/${tag}_ncu_full_${k}_details.csv 2>/dev/null || true
  ncu -i gpurun_out/full_${tag}_$k.ncu-rep --page raw --csv > gpurun_out/${tag}_ncu_full_${k}_raw.csv 2>/dev/null || true
done
ls -la gpurun_out
