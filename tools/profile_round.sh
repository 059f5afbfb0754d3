# ncu evidence for profiles/: launch list of the bench, full captures of the hot kernels (config 2)
# usage: bash tools/profile_round.sh <tag>
tag=${1:-r01c}
set -e
python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_plain_$tag.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_$tag.log 2>&1
python tools/prof_step.py 2 64 > gpurun_out/prof_plain_$tag.log 2>&1
for k in conv_kernel solve_halo_kernel near_step_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -o gpurun_out/full_${tag}_$k \
      python tools/prof_step.py 2 64 > gpurun_out/ncu_${tag}_$k.log 2>&1 || true
done
ls -la gpurun_out
