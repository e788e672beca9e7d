"""Hottest SASS lines of a kernel by warp-stall samples (ncu --page source): python tools/ncu_hot.py rep [N] [phase]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
want = int(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS, iE = hdr.index("Source"), hdr.index("Instructions Executed")
iW = hdr.index("Warp Stall Sampling (All Samples)")
iA = hdr.index("Address") if "Address" in hdr else 0
seg, lines = 0, []
for r in rows[2:]:
    s = r[iS].strip()
    try:
        w = int(r[iW] or 0)
    except ValueError:
        continue
    lines.append((w, seg, r[iA], s, r[iE]))
    if "BAR.SYNC" in s:
        seg += 1
sel = [l for l in lines if want is None or l[1] == want]
tot = sum(l[0] for l in lines)
for w, sg, a, s, e in sorted(sel, key=lambda l: -l[0])[:N]:
    print(f"{w:7d} {100 * w / tot:5.1f}% ph{sg} {a:>6s} {s[:80]:80s} x{e}")
