"""In-tree build of libcachegram_b200.so for sm_100a (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "libcachegram_b200.so"
SOURCES = ["cg_capi.cu", "cg_det.cu", "cg_hogwild.cu", "cg_hog8.cu", "cg_eval.cu", "cg_ingest.cu", "cg_modelio.cpp"]
HEADERS = ["cg_device.cuh", "cg_kernels.h", "cg_host.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++20",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
    "-Xcompiler", "-fvisibility=hidden,-fvisibility-inlines-hidden",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + list((ROOT / "include").rglob("*.h*"))
    return any(d.stat().st_mtime > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, f"-I{ROOT / 'include'}", f"-I{CSRC}",
           *[str(CSRC / s) for s in SOURCES], "-o", str(OUT)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = PKG / "build.log"
    log.write_text(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode}); see {log}")
    if verbose:
        sys.stdout.write(res.stderr)
    return OUT


def build_oracle() -> None:
    """Test infrastructure: the C restatement and (when /root/reference exists) the
    reference headers compiled unchanged into oracle/_ref."""
    res = subprocess.run(["make", "-C", str(ROOT / "oracle")], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("oracle build failed")


def build_cpp_dropin_test() -> Path:
    """A C++ program written against include/cachegram/*.hpp exactly like the
    reference's own tests, linked with the library (tests/cpp/dropin_test.cpp)."""
    src = ROOT / "tests" / "cpp" / "dropin_test.cpp"
    out = ROOT / "tests" / "cpp" / "dropin_test"
    if not src.exists():
        return out
    if out.exists() and out.stat().st_mtime > max(src.stat().st_mtime, OUT.stat().st_mtime) and not any(
            h.stat().st_mtime > out.stat().st_mtime for h in (ROOT / "include").rglob("*.h*")):
        return out
    cxx = os.environ.get("CXX", "g++")
    cmd = [cxx, "-std=gnu++20", "-O2", f"-I{ROOT / 'include'}", str(src), "-o", str(out),
           f"-L{PKG}", "-lcachegram_b200", f"-Wl,-rpath,{PKG}", f"-Wl,-rpath,$ORIGIN/../../paper_1606_07822_b200"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("C++ drop-in test build failed")
    return out


def build_reference_suites() -> None:
    """The reference's own unit tests against the drop-in headers (needs /root/reference)."""
    script = ROOT / "tests" / "cpp" / "build_reftests.sh"
    if not Path("/root/reference/proj/tests").exists():
        return
    out = ROOT / "tests" / "cpp" / "_reftests" / "trainer_test"
    deps = [OUT, ROOT / "tests" / "cpp" / "gtest_shim" / "gtest" / "gtest.h", *(ROOT / "include").rglob("*.h*")]
    if out.exists() and all(d.stat().st_mtime < out.stat().st_mtime for d in deps):
        return
    res = subprocess.run(["sh", str(script)], capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("reference test suites failed to build against the drop-in headers")


def build_all(force: bool = False) -> None:
    build_library(force=force)
    build_oracle()
    build_cpp_dropin_test()
    build_reference_suites()


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print(OUT)
