cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p /tmp/A && cp -r paper_2407_09621_b200 tools bench.py oracle /tmp/A/ 2>/dev/null
cp abtest/old.so /tmp/A/paper_2407_09621_b200/libsumfact_b200.so
pc='import json,sys; d=json.load(sys.stdin); print(sys.argv[1], d["k"], "fp64 step", round(d["smooth_step_fp64_ms"],3), "ec step", round(d["smooth_step_fp16_ec_ms"],3), "vmult64", round(d["vmult_fp64_ms"],3), "vmultec", round(d["vmult_fp16_ec_ms"],3))'
for kl in "7 6" "3 7"; do for r in 1 2; do
  (cd /tmp/A && python tools/time_q3.py $kl | python -c "$pc" old)
  python tools/time_q3.py $kl | python -c "$pc" new
done; done
