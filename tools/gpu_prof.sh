#!/bin/bash
# ncu captures of the top kernels (one GPU, never timed) + the bench with extras.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
P="ncu --set full --clock-control none --import-source on -c 1 -f"
timeout 600 $P -k regex:k_vmult_dmma8 -o gpurun_out/vmult_fp64 python tools/profile_vmult.py --degree 7 --level 7 --reps 1 > /dev/null 2>&1
timeout 600 $P -k regex:k_vmult_h8 -o gpurun_out/vmult_h8_ec python tools/profile_vmult.py --degree 7 --level 7 --mode fp16_ec --reps 1 > /dev/null 2>&1
timeout 600 $P -k regex:k_colour_h8 -o gpurun_out/colour_h8_ec python tools/profile_vmult.py --degree 7 --level 6 --mode fp16_ec --what colour --reps 1 > /dev/null 2>&1
timeout 600 $P -k regex:k_colour_dmma8 -o gpurun_out/colour_fp64 python tools/profile_vmult.py --degree 7 --level 6 --mode fp64 --what colour --reps 1 > /dev/null 2>&1
echo done
