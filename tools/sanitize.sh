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
  # racecheck / synccheck: this library's kernels only (the coarse setup's cuSOLVER / cuBLAS factorisation
  # kernels are not ours, and racecheck instruments their large trsm far too slowly).  Not for initcheck: it
  # would stop tracking the writes of unchecked kernels (torch.randn) and report their output as uninitialised.
  case $t in racecheck|synccheck) extra="$extra --kernel-name regex=_ZN2sf --kernel-name regex=_sf_[a-z]+_cu_";; esac
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $t $extra --print-limit 50 \
    python tools/sanitize_cases.py $args > gpurun_out/sanitize_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/sanitize_$t.log
done
