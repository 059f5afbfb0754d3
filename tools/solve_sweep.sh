for v in "TDW_SOLVER=smem TDW_SOLVE_CL=2" "TDW_SOLVER=smem TDW_SOLVE_CL=4" "TDW_SOLVER=smem TDW_SOLVE_CL=8" "TDW_SOLVER=smem" "TDW_SOLVER=reg"; do
  env $v python tools/prof_step.py 2 64 > gpurun_out/p.log 2>&1 || { echo "$v failed"; tail -3 gpurun_out/p.log; continue; }
  env $v ncu --metrics gpu__time_duration.sum --clock-control none -k regex:solve --csv python tools/prof_step.py 2 64 2>/dev/null | grep solve | awk -F'","' '{print $NF}' | tr -d '"' | sort -n | awk -v v="$v" '{a[NR]=$1} END {print v, "n", NR, "median", a[int(NR/2)], "max", a[NR]}'
done
