#!/bin/bash
# Quick A/B of the FP64 vmult headline: abtest/old.so vs the in-tree library, 3 rounds interleaved
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p /tmp/A && cp -r paper_2407_09621_b200 tools bench.py oracle /tmp/A/ 2>/dev/null
cp abtest/old.so /tmp/A/paper_2407_09621_b200/libsumfact_b200.so
pb='import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], round(d["value"],2))'
for r in 1 2 3; do
  (cd /tmp/A && python bench.py --no-cpu --no-extras --steps 20 2>/dev/null | python -c "$pb" old)
  python bench.py --no-cpu --no-extras --steps 20 2>/dev/null | python -c "$pb" new
done
