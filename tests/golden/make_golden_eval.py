#!/usr/bin/env python
"""Regenerates tests/golden/eval_analogy.npz and tests/golden/model_small.{txt,bin} from
the reference itself (oracle/_ref/libcgref.so: the reference headers compiled
unchanged). Runs in the build container only.

eval_analogy.npz: for each case, seeded embeddings with planted hazards (duplicated
rows -> exact ties, zero rows, NaN rows; tests/oracle_lib.eval_case), random questions,
restrict_top, and the answers of the reference's AnalogySolver::answer (eval.hpp:117-136).

model_small.*: the reference's save_text / save_binary (model.hpp:119-144) of a small
model whose values cover signs, -0, tiny, large and denormal floats and whose words
vary in length; the drop-in must write these bytes exactly.
"""
import sys
import tempfile
from pathlib import Path

import ctypes as C
import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import oracle_lib as O  # noqa: E402

CASES = [  # seed, rows, dim, questions, dup, zero, nan, restrict_top
    (11, 50, 4, 200, 5, 2, 0, 0),
    (12, 300, 7, 300, 20, 3, 2, 0),
    (13, 500, 33, 200, 10, 0, 0, 120),
    (14, 4, 3, 8, 0, 0, 0, 0),
    (15, 1000, 24, 150, 30, 5, 3, 700),
]


def model_values():
    rng = np.random.default_rng(77)
    v = ((rng.random((20, 6), dtype=np.float32) - 0.5) * 3).astype(np.float32)
    v[0] = [0.0, -0.0, 1e-7, -1e-7, 123456.789, -0.0000005]
    v[1] = [np.float32(1.4e-45), 3.4e38, -3.4e38, 0.5, 0.0000005, 1.0]
    return v


def model_words():
    return [f"w{i}" * (1 + i % 3) for i in range(19)] + ["longer-word_x"]


def main():
    assert O.ref_available(), "needs oracle/_ref/libcgref.so (make -C oracle)"
    out = {"n_cases": np.array(len(CASES))}
    for i, (seed, rows, dim, nq, dup, zero, nan, top) in enumerate(CASES):
        v, abc = O.eval_case(seed, rows, dim, nq, dup, zero, nan)
        size = min(rows, top) if top > 0 else rows
        abc = (abc % size).astype(np.int32)
        out[f"v{i}"], out[f"abc{i}"], out[f"top{i}"] = v, abc, np.array(top)
        out[f"ans{i}"] = O.ref_analogy(v, top, abc)
    np.savez_compressed(HERE / "eval_analogy.npz", **out)
    v = model_values()
    words = b"".join(w.encode() + b"\0" for w in model_words())
    for binary, name in ((0, "model_small.txt"), (1, "model_small.bin")):
        rc = O.ref().ref_model_save(str(HERE / name).encode(), binary, words, O._p(v, C.c_float), 20, 6)
        assert rc == 0
    np.save(HERE / "model_small_values.npy", v)
    print("eval_analogy:", len(CASES), "cases; model_small.{txt,bin}")


if __name__ == "__main__":
    main()
