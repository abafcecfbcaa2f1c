"""The reference's own unit-test sources (trainer_test.cpp, huffman_test.cpp,
corpus_test.cpp), compiled unmodified against this repo's drop-in headers and linked
with libcachegram_b200.so by tests/cpp/build_reftests.sh (GTest replaced by the shim in
tests/cpp/gtest_shim). They are built where /root/reference exists and travel prebuilt."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "_reftests"


def run(name):
    exe = BIN / name
    if not exe.exists():
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=900, cwd="/tmp")
    tail = "\n".join(r.stdout.splitlines()[-40:])
    assert r.returncode == 0, tail + r.stderr
    assert " 0 failed" in r.stdout, tail
    return r.stdout


def test_reference_huffman_suite_on_dropin():
    out = run("huffman_test")
    assert "[==========] 14 tests" in out


def test_reference_corpus_suite_on_dropin():
    out = run("corpus_test")
    assert "[==========] 19 tests" in out


@pytest.mark.gpu
def test_reference_trainer_suite_on_dropin():
    """trainer_test.cpp: train_center known answers (device kernels; arbitrary sigmoid
    functors via the host callback), NodeCache, schedule helpers, and train() runs
    (workers = 1 -> deterministic device mode, workers = 3 -> Hogwild)."""
    out = run("trainer_test")
    assert "[==========] 20 tests" in out


def test_reference_model_suite_on_dropin():
    """model_test.cpp: init bits, sigmoid table, and the model files (text/binary round
    trips, auto-detection, malformed/truncated/mismatched inputs) -- host code."""
    out = run("model_test")
    assert "[==========] 14 tests" in out


@pytest.mark.gpu
def test_reference_eval_suite_on_dropin():
    """eval_test.cpp: question parsing, 3CosAdd answers (exact ties, exclusions,
    restrict_top), evaluate() reports, and a train -> save -> load -> answer pipeline."""
    out = run("eval_test")
    assert "[==========] 15 tests" in out


@pytest.mark.gpu
def test_reference_bench_suite_on_dropin():
    """bench_test.cpp: run_bench grid order, words/s consistency, accuracy column, failing
    cells, CSV schema."""
    out = run("bench_test")
    assert "[==========] 6 tests" in out
