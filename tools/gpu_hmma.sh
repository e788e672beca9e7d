#!/bin/bash
# FP16 / FP16-EC kernel iteration: parity tests of the binary16 paths, bench extras, EC / FP64 solves,
# per-kernel durations of the EC solve kernels.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_vmult.py tests/test_gpu_multigrid.py tests/test_gpu_solve_histories.py \
  tests/test_gpu_fuzz.py -x -q > gpurun_out/h_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/h_pytest.log
timeout 600 python bench.py --no-cpu > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
timeout 600 python tools/bench_solve.py --degree 7 --level 6 --modes fp64,fp16_ec,fp16 > gpurun_out/h_solve_q7.jsonl 2>&1
timeout 600 python tools/bench_solve.py --degree 3 --level 7 --modes fp64,fp16_ec > gpurun_out/h_solve_q3.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:"k_colour_h8|k_vmult_h8|k_resid_restrict_h8" -c 6 --csv --log-file gpurun_out/h_ncu.csv \
  python tools/profile_vmult.py --degree 7 --level 6 --mode fp16_ec --what colour --reps 1 > /dev/null 2>&1
echo done
