#!/bin/bash
# Quick GPU iteration: vmult tests, bench headline (no extras), dram bytes of the vmult.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_vmult.py ${QUICK_TESTS} -x -q > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 600 python bench.py --no-cpu --no-extras ${BENCH_ARGS} > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_vmult -c 2 --csv --log-file gpurun_out/q_ncu.csv python tools/profile_vmult.py --degree 7 --level 7 --reps 2 > /dev/null 2>&1
echo done
