#!/bin/bash
# Kernel time split of one FGMRES+MG solve per mode (ncu launch list; never a timing number).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for m in fp64 fp16_ec; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/solve_launches_$m.csv python tools/bench_solve.py --degree 7 --level 6 --modes $m --reps 1 > gpurun_out/solve_ncu_$m.log 2>&1
done
timeout 600 python tools/bench_solve.py --degree 7 --level 6 --modes fp64,fp16_ec > gpurun_out/solve_q7l6.jsonl 2>&1
