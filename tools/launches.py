"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: time per kernel."""
import collections
import csv
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    i_name, i_val, i_unit = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[1:]:
        try:
            v = float(r[i_val].replace(",", ""))
        except ValueError:
            continue
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                 "second": 1e3, "s": 1e3}[r[i_unit]]
        out.append((r[i_name], v * scale))
    return out


def summary(path, top=14):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, ms in load(path):
        short = name.replace("void ", "").split("(")[0][:70]
        agg[short][0] += 1
        agg[short][1] += ms
    tot = sum(v[1] for v in agg.values())
    lines = [f"total {tot:.3f} ms over {sum(v[0] for v in agg.values())} launches"]
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        lines.append(f"  {v:9.3f} ms {100 * v / tot:5.1f}%  x{c:<5d} {k}")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        print(summary(p))
