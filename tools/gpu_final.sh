#!/bin/bash
# Final round check: full GPU tests, smoke, bench (one JSON line), ncu full capture of the FP16-EC vmult.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/f_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f_smoke.log
timeout 1500 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
KREGEX=k_vmult_h8 WHAT=vmult LVL=7 bash tools/ncu_colour.sh vmult_h8_ec_l7
echo done
