#!/bin/bash
# A/B of the binary16 colour passes: abtest/old.so (baseline) vs the in-tree library, Q3 L7 and Q7 L6, 2 rounds
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p /tmp/A && cp -r paper_2407_09621_b200 tools /tmp/A/ && cp abtest/old.so /tmp/A/paper_2407_09621_b200/libsumfact_b200.so
pr='import json,sys; d=json.load(sys.stdin); print(sys.argv[1], d["k"], "ec step", round(d["smooth_step_fp16_ec_ms"],3), "ec 111", round(d["colour_fp16_ec_111_ms"],4), "fp64 step", round(d["smooth_step_fp64_ms"],3))'
for r in 1 2; do for kl in "3 7" "7 6"; do
  (cd /tmp/A && python tools/time_q3.py $kl | python -c "$pr" old)
  python tools/time_q3.py $kl | python -c "$pr" new
done; done
