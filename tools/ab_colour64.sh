cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p /tmp/A && cp -r paper_2407_09621_b200 tools /tmp/A/ && cp abtest/old.so /tmp/A/paper_2407_09621_b200/libsumfact_b200.so
pc='import json,sys; d=json.load(sys.stdin); print(sys.argv[1], "fp64 step", round(d["smooth_step_fp64_ms"],3), "colour000", round(d["colour_fp64_000_ms"],4))'
for r in 1 2; do (cd /tmp/A && python tools/time_q3.py 7 6 | python -c "$pc" old); python tools/time_q3.py 7 6 | python -c "$pc" new; done
