"""Build ``oracle/_ref/``: the reference's own native kernel, compiled from its sources in place.

TEST INFRASTRUCTURE ONLY.  The reference package's single native component is the
Cython-generated C batched contraction ``src/sumfact/_core/_contract.c``
(``/root/reference/pkg/src/sumfact/_core/_contract.pyx:14-45``, built by
``pkg/setup.py:5-13`` with ``-O3``).  This recipe compiles that file where it lies
with gcc (same flags as the reference's setup.py; no copy of the source enters the
repo) into ``oracle/_ref/_contract<EXT_SUFFIX>``.  ``tests/test_oracle_ref.py`` pins
``oracle.port.contract`` to it.  ``oracle/_ref/`` is git-ignored but travels to the
GPU box with the snapshot; ``/root/reference`` itself exists only in the build
container, so this is a no-op there when the .so is already built.

    python oracle/build_ref.py
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
SRC = "/root/reference/pkg/src/sumfact/_core/_contract.c"
SO = os.path.join(OUT, "_contract" + sysconfig.get_config_var("EXT_SUFFIX"))


def build(force: bool = False) -> str | None:
    """Compile the reference kernel; returns the .so path, or None when the reference is absent."""
    if not os.path.exists(SRC):
        return SO if os.path.exists(SO) else None
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= os.path.getmtime(SRC):
        return SO
    import numpy as np

    os.makedirs(OUT, exist_ok=True)
    cmd = ["gcc", "-O3", "-shared", "-fPIC", f"-I{sysconfig.get_paths()['include']}", f"-I{np.get_include()}",
           "-DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION", SRC, "-o", SO + ".tmp"]
    subprocess.run(cmd, check=True, capture_output=True)
    os.replace(SO + ".tmp", SO)
    return SO


def load():
    """Import the compiled reference kernel module (``contract_f8``/``contract_f4``), or None."""
    if not os.path.exists(SO):
        return None
    import importlib.util

    spec = importlib.util.spec_from_file_location("_contract", SO)
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


if __name__ == "__main__":
    print(build(force="-f" in sys.argv))
