#!/bin/bash
# A/B the FP64 vmult variants (env-selected) with the bench's CUDA-event timing.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
: > gpurun_out/ab.txt
for v in ${AB_VARIANTS:-"X=0" "SUMFACT_B200_DMMA_PIPE=1"}; do
  r=$(env $v python bench.py --no-cpu --no-extras --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'])")
  echo "[$v] $r" >> gpurun_out/ab.txt
done
[ -n "$AB_TESTS" ] && timeout 900 python -m pytest $AB_TESTS -q -x >> gpurun_out/ab.txt 2>&1
true
