#!/bin/bash
# compute-sanitizer over every hot kernel at small sizes (tools/sanitize_cases.py); logs -> gpurun_out/sanitize_*.log
# usage: bash tools/sanitize.sh [tool ...]   (default: memcheck racecheck synccheck initcheck)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
TOOLS=${*:-memcheck racecheck synccheck initcheck}
for t in $TOOLS; do
  extra=""
  [ "$t" = racecheck ] && extra="--racecheck-report all"
  [ "$t" = memcheck ] && extra="--leak-check no"
  args=""
  [ "$t" != memcheck ] && args="--quick"
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $t $extra --print-limit 50 \
    python tools/sanitize_cases.py $args > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/sanitize_$t.log
done
