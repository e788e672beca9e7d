"""SASS instruction census of libsumfact_b200.so per hot kernel (cuobjdump -sass): static counts of the tensor /
memory instructions that prove which hardware paths the kernels use.  python tools/sass_census.py > profiles/..."""
import collections
import os
import re
import subprocess

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2407_09621_b200",
                   "libsumfact_b200.so")
KEYS = ["DMMA", "HMMA", "UTCHMMA", "UTCBAR", "LDTM", "LDSM", "STSM", "LDGSTS", "UTMALDG", "FFMA2", "FMUL2", "FHFMA",
        "REDUX", "CREDUX", "DFMA"]
WANT = ["k_vmult_dmma8", "k_colour_dmma", "k_resid_restrict_dmma", "k_prolong_dmma", "k_vmult_h8", "k_colour_h8",
        "k_resid_restrict_h8", "k_prolong_h8", "k_vmult_u8", "k_vmult_dmma_line", "k_axpy_dot_partial", "k_dense_apply"]
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", sass)[1:]
print(f"# SASS census of {os.path.basename(LIB)} (static instruction counts per kernel instantiation)\n")
print("| kernel | instructions | " + " | ".join(KEYS) + " |")
print("|---|---|" + "---|" * len(KEYS))
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    short = re.sub(r"\(.*", "", dem).replace("sf::", "").replace("(anonymous namespace)::", "")
    if not any(w in short for w in WANT):
        continue
    ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", f)
    c = collections.Counter(ops)
    print(f"| `{short[:60]}` | {len(ops)} | " + " | ".join(str(c.get(k, 0)) for k in KEYS) + " |")
