"""The tcgen05 (UMMA) binary16 vmult (SUMFACT_UMMA=1: TMEM accumulators, canonical shared-memory operand
layouts written by the producing stage) against the mma.sync kernels and the fp64 vmult, in a child
process (the path is chosen once per process)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_tcgen05_vmult_matches_mma_sync_and_fp64():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "umma_check.py")], capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr
    rows = [l.split() for l in r.stdout.splitlines() if l.startswith("k7_")]
    assert len(rows) == 8, r.stdout
    for row in rows:
        mode = row[0].split("_", 2)[2]
        vs64, ab = float(row[8]), float(row[12])
        # same operand semantics: fp16 bitwise-level, EC to the accumulation-order level
        assert ab <= (1e-9 if mode == "fp16" else 1e-8), row
        assert vs64 <= (6e-4 if mode == "fp16" else 3e-7), row
