"""The C++ drop-in: a program written against include/cachegram/*.hpp (the
reference's header names and signatures) linked with libcachegram_b200.so."""
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_1606_07822_b200 import build

ROOT = Path(__file__).resolve().parents[1]
GOLD = ROOT / "tests" / "golden"


def test_cpp_dropin_builds():
    exe = build.build_cpp_dropin_test()
    assert exe.exists()


@pytest.mark.gpu
def test_cpp_dropin_runs_and_matches_golden(tmp_path):
    exe = build.build_cpp_dropin_test()
    r = subprocess.run([str(exe), str(tmp_path)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    # the deterministic C++ train() of the g1 fixture (K=15) equals the reference's bits
    z = np.load(GOLD / "g1_small.npz")
    s0 = np.fromfile(tmp_path / "g1_syn0.bin", dtype=np.float32)
    s1 = np.fromfile(tmp_path / "g1_syn1.bin", dtype=np.float32)
    assert np.array_equal(s0.view(np.uint32), z["syn0"].ravel().view(np.uint32))
    assert np.array_equal(s1.view(np.uint32), z["syn1"].ravel().view(np.uint32))
