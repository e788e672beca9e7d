#!/bin/bash
# A/B of the FP64 vmult headline and the FP64 colour pass: abtest/old.so (baseline) vs the in-tree library, 2 rounds
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p /tmp/A && cp -r paper_2407_09621_b200 tools bench.py oracle /tmp/A/ 2>/dev/null
cp abtest/old.so /tmp/A/paper_2407_09621_b200/libsumfact_b200.so
pb='import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], "vmult", round(d["value"],2), "GDoF/s", round(d["ms_per_step"],3), "ms")'
pc='import json,sys; d=json.load(sys.stdin); print(sys.argv[1], d["k"], "fp64 step", round(d["smooth_step_fp64_ms"],3), "ec step", round(d["smooth_step_fp16_ec_ms"],3))'
for r in 1 2; do
  (cd /tmp/A && python bench.py --no-cpu --no-extras --steps 20 2>/dev/null | python -c "$pb" old)
  python bench.py --no-cpu --no-extras --steps 20 2>/dev/null | python -c "$pb" new
done
(cd /tmp/A && python tools/time_q3.py 7 6 | python -c "$pc" old)
python tools/time_q3.py 7 6 | python -c "$pc" new
