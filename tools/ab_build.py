#!/usr/bin/env python
"""Builds variants of libcachegram_b200.so with extra preprocessor flags, for same-box
A/B timing of kernel experiments (select one with CG_LIB=<path> in the environment).

  python tools/ab_build.py NAME -DCG_EXP=1 [...]   ->  _ab/NAME/libcachegram_b200.so
"""
from __future__ import annotations

import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1606_07822_b200 import build as B  # noqa: E402


def main():
    name, flags = sys.argv[1], sys.argv[2:]
    out = ROOT / "_ab" / name / "libcachegram_b200.so"
    out.parent.mkdir(parents=True, exist_ok=True)
    cmd = [B.nvcc(), *B.NVCC_FLAGS, *flags, f"-I{ROOT / 'include'}", f"-I{B.CSRC}",
           *[str(B.CSRC / s) for s in B.SOURCES], "-o", str(out)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        sys.exit(1)
    print(out)


if __name__ == "__main__":
    main()
