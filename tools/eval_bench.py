#!/usr/bin/env python
"""Evaluation kernels (cg_eval.cu) timed against the reference's CPU AnalogySolver.

* 3CosAdd analogies: Q questions over a restricted table of R rows x D dims (the shape of
  the reference's default evaluation: restrict_top 30000, D 300, ~20k questions), device
  time of one batched cg_analogy_answer vs the reference's AnalogySolver::answer loop
  (oracle/_ref, headers compiled unchanged) on a bounded sample of the questions, and
  answers checked equal on that sample.
* Exact cosine top-10 over a C3-shaped table (50k x 128), the recall@10 metric.

  python tools/eval_bench.py [--rows 30000 --dim 300 --questions 20000]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_lib as O  # noqa: E402  (checker / CPU baseline)
from paper_1606_07822_b200 import api  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", type=int, default=30000)
    p.add_argument("--dim", type=int, default=300)
    p.add_argument("--questions", type=int, default=20000)
    p.add_argument("--ref-questions", type=int, default=400)
    p.add_argument("--knn-rows", type=int, default=50000)
    p.add_argument("--knn-dim", type=int, default=128)
    a = p.parse_args()
    rng = np.random.default_rng(11)
    v = (rng.random((a.rows, a.dim), dtype=np.float32) - 0.5)
    abc = rng.integers(0, a.rows, size=(a.questions, 3)).astype(np.int32)
    emb = api.Embeddings(v)
    emb.analogy(abc[:64])  # warm-up
    t0 = time.perf_counter()
    got = emb.analogy(abc)
    t_gpu = time.perf_counter() - t0
    out = {"analogy": {"rows": a.rows, "dim": a.dim, "questions": a.questions, "gpu_s": t_gpu,
                       "gpu_questions_per_s": a.questions / t_gpu,
                       "gpu_score_tflops": 2.0 * a.questions * a.rows * a.dim / t_gpu / 1e12}}
    if O.ref_available():
        n = a.ref_questions
        t0 = time.perf_counter()
        want = O.ref_analogy(v, 0, abc[:n])
        t_ref = time.perf_counter() - t0
        out["analogy"].update(ref_questions=n, ref_s=t_ref, ref_questions_per_s=n / t_ref, ref_threads=1,
                              answers_equal_on_ref_sample=bool(np.array_equal(want, got[:n])))
    nv = (rng.random((a.knn_rows, a.knn_dim), dtype=np.float32) - 0.5)
    e2 = api.Embeddings(nv)
    e2.nearest(np.arange(64, dtype=np.int32), 10)
    t0 = time.perf_counter()
    ids, _ = e2.nearest(np.arange(a.knn_rows, dtype=np.int32), 10)
    t_knn = time.perf_counter() - t0
    sample = np.arange(0, a.knn_rows, max(1, a.knn_rows // 200), dtype=np.int32)
    wid, _ = O.orc_topk(O.orc_normalize(nv), sample, 10)
    out["topk"] = {"rows": a.knn_rows, "dim": a.knn_dim, "k": 10, "gpu_s": t_knn,
                   "gpu_score_tflops": 2.0 * a.knn_rows * a.knn_rows * a.knn_dim / t_knn / 1e12,
                   "oracle_sample": int(sample.size), "equal_on_sample": bool(np.array_equal(ids[sample], wid))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
