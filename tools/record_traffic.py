"""Record roofline.traffic for bench.py: dram__bytes_read.sum + dram__bytes_write.sum of one k_vmult_dmma8
launch from an ncu capture, stamped with the hash of the kernel sources it was measured on (bench.py
reports it only while the sources are unchanged; otherwise traffic is null).
python tools/record_traffic.py gpurun_out/q_ncu.csv   (the --metrics CSV of tools/gpu_quick.sh)"""
import csv
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SOURCES = ["paper_2407_09621_b200/csrc/sf_dmma.cu", "paper_2407_09621_b200/csrc/sf_dmma.cuh",
           "paper_2407_09621_b200/csrc/sf_common.cuh"]


def source_hash():
    h = hashlib.sha256()
    for p in SOURCES:
        h.update(open(os.path.join(ROOT, p), "rb").read())
    return h.hexdigest()[:16]


def main(path):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    hdr = rows[0]
    iK, iM, iV, iU = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    for r in rows[1:]:
        if "k_vmult_dmma8" in r[iK] and r[iM] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            per.setdefault(r[iM], []).append(float(r[iV].replace(",", "")) * scale[r[iU]])
    traffic = int(sum(v[-1] for v in per.values()))
    out = {"_comment": "dram__bytes_read.sum + dram__bytes_write.sum per launch of k_vmult_dmma8 (Q7 level 7, "
                       "1.07e9 DoF) from " + os.path.basename(path) + "; valid while source_hash matches",
           "source_hash": source_hash(), "k7_l7_fp64": traffic}
    json.dump(out, open(os.path.join(ROOT, "profiles", "vmult_traffic.json"), "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main(sys.argv[1])
