#!/bin/bash
# Round-end verification on one B200: full GPU tests, smoke, bench (+ reference arm), launch list of the bench
# command, DRAM traffic of the headline kernel, the CPU baseline cases, solve timings.  Outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r_smoke.log
timeout 1500 python bench.py > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r_bench_ref.json 2> gpurun_out/r_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu --no-extras > gpurun_out/r_bench_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:k_vmult_dmma8 -c 2 --csv --log-file gpurun_out/r_traffic.csv \
  python tools/profile_vmult.py --degree 7 --level 7 --reps 2 > /dev/null 2>&1
timeout 1200 python -m oracle.cpu_timing --out gpurun_out/r_cpu_baseline.json > gpurun_out/r_cpu_baseline.log 2>&1
timeout 900 python tools/bench_solve.py --degree 7 --level 6 --modes fp64,fp16_ec > gpurun_out/r_solve_q7l6.jsonl 2>&1
timeout 900 python tools/bench_solve.py --degree 3 --level 7 --modes fp64,fp16_ec > gpurun_out/r_solve_q3l7.jsonl 2>&1
echo done
