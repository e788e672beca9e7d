#!/bin/bash
# One targeted-metrics ncu pass per hot kernel (never timed): duration, tensor pipe %, DRAM bytes.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"
run() { timeout 600 ncu --metrics $M --clock-control none -k "regex:$1" -c 1 --csv --log-file gpurun_out/pa_$2.csv python tools/profile_vmult.py $3 > /dev/null 2>&1; }
run k_vmult_dmma8 vmult_q7_fp64 "--degree 7 --level 7 --reps 1"
run k_vmult_dmma_line vmult_q3_fp64 "--degree 3 --level 8 --reps 1"
run k_vmult_h8 vmult_q7_ec "--degree 7 --level 7 --mode fp16_ec --reps 1"
run k_vmult_h8 vmult_q7_fp16 "--degree 7 --level 7 --mode fp16 --reps 1"
run k_vmult_h8 vmult_q3_ec "--degree 3 --level 8 --mode fp16_ec --reps 1"
run k_colour_dmma colour_q7_fp64 "--degree 7 --level 6 --mode fp64 --what colour --reps 1"
run k_colour_dmma colour_q3_fp64 "--degree 3 --level 7 --mode fp64 --what colour --reps 1"
run k_colour_h8 colour_q7_ec "--degree 7 --level 6 --mode fp16_ec --what colour --reps 1"
run k_colour_h8 colour_q3_ec "--degree 3 --level 7 --mode fp16_ec --what colour --reps 1"
run k_resid_restrict vcycle_restrict_q7_fp64 "--degree 7 --level 6 --mode fp64 --what vcycle --reps 1"
run k_prolong_add vcycle_prolong_q7_fp64 "--degree 7 --level 6 --mode fp64 --what vcycle --reps 1"
run k_vmult_dmma8 vmult_q7_fp32 "--degree 7 --level 7 --mode fp32 --reps 1"
run k_vmult_dmma_line vmult_q3_fp32 "--degree 3 --level 8 --mode fp32 --reps 1"
run k_colour_dmma colour_q7_fp32 "--degree 7 --level 6 --mode fp32 --what colour --reps 1"
echo done
