"""SASS lines with the most excess shared-memory wavefronts (bank conflicts): python tools/ncu_conflicts.py rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS = hdr.index("Source")
iX = hdr.index("L1 Wavefronts Shared Excessive")
iW = hdr.index("L1 Wavefronts Shared")
iE = hdr.index("Instructions Executed")
seg, lines = 0, []
for r in rows[2:]:
    try:
        x = int(r[iX] or 0)
    except ValueError:
        continue
    s = r[iS].strip()
    lines.append((x, seg, s, r[iW], r[iE]))
    if "BAR.SYNC" in s:
        seg += 1
tot = sum(l[0] for l in lines)
print("total excess", tot)
for x, sg, s, w, e in sorted(lines, key=lambda l: -l[0])[:N]:
    print(f"{x:12d} ph{sg} {s[:70]:70s} wf={w} x{e}")
