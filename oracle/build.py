"""Build recipe for the oracle's C restatement (TEST INFRASTRUCTURE ONLY).

``python -m oracle.build`` compiles oracle/csrc/chol.c with gcc into
oracle/_build/liboracle_chol.so.  ``__graft_entry__.build()`` calls
``build()``: building the checker is not using it.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "liboracle_chol.so")
SRC = os.path.join(HERE, "csrc", "chol.c")


def build(force: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        # -fno-fast-math / -ffp-contract=off: keep IEEE evaluation order like numba
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", LIB, SRC, "-lm"])
    return LIB


if __name__ == "__main__":
    print(build(force=True))
