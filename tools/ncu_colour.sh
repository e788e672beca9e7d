#!/bin/bash
# one ncu --set full capture of the EC (or given mode) colour pass at Q7 L6 -> gpurun_out/$1.ncu-rep
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -c 1 -f -k regex:${KREGEX:-k_colour_h8} -o gpurun_out/$1 \
  python tools/profile_vmult.py --degree ${DEG:-7} --level ${LVL:-6} --mode ${MODE:-fp16_ec} --what ${WHAT:-colour} --reps 1 > gpurun_out/$1.log 2>&1
