#!/usr/bin/env python
"""North-star quality gates for the Hogwild (throughput) mode.

* HS log-loss: mean over a fixed set of 2^20 evaluation pairs (harness seed, the
  reference's pair rules; formula of tests/acceptance.cpp:100-110) of the GPU model vs
  the reference's own model -- cachegram::train() compiled unchanged (oracle/_ref), run
  multithreaded on this host's cores, i.e. its Hogwild mode. Gate: within 2%. The gate
  alone is loose (an untrained model is ~2.7% off at C1), so the learning ratio -- the
  share of the reference's loss reduction (init -> trained) the GPU model achieves -- is
  reported and gated too (>= 0.95).
* C3 planted-cluster recall@10 (cosine over unit syn0, self excluded): GPU vs the
  reference model. Gate: within 0.02.

Both sides train the same id stream (a prefix of the configuration's corpus when
`tokens` is given, with the full corpus's vocabulary and tree) for `epochs` passes.

  python tools/quality_gates.py --configs c1 c2 c3 [--tokens c4=20000000 c5=50000000] [--out f.json]
"""
from __future__ import annotations

import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import bench  # noqa: E402  (workload + reference-sample helpers)
import oracle_lib as O  # noqa: E402  (checker side)
from paper_1606_07822_b200 import api  # noqa: E402
from paper_1606_07822_b200.corpus_gen import CONFIGS, cluster_raw_ids, vocab_from_raw  # noqa: E402


def recall_at_10(syn0: np.ndarray, cluster: np.ndarray, sample: np.ndarray) -> float:
    """Share of the 10 exact cosine nearest neighbours (self excluded, ties to the lower
    id) that share the query's planted cluster -- through the product's own evaluation
    kernel (cg_nearest, cg_eval.cu), for the GPU model and the reference model alike."""
    emb = api.Embeddings(syn0)
    hits = 0
    for a in range(0, len(sample), 8192):
        q = np.ascontiguousarray(sample[a:a + 8192], dtype=np.int32)
        ids, _ = emb.nearest(q, 10)
        hits += int((cluster[ids] == cluster[q][:, None]).sum())
    return hits / (10 * len(sample))


def gate(name: str, tokens: int | None = None, epochs: int | None = None, k: int = 31, pairs: int = 1 << 20,
         threads: int | None = None) -> dict:
    c = CONFIGS[name]
    t0 = time.time()
    cluster = None
    if c.clusters:
        raw, cluster_of = cluster_raw_ids(c)
        vocab, ids = vocab_from_raw(raw, c.min_count, c.clusters * c.cluster_size)
        cluster = cluster_of[vocab.raw_of_id]
    else:
        _, vocab, ids = bench.workload(name, 0, 1, device=name in ("c4", "c5"))
    n = min(tokens or len(ids), len(ids))
    ids = bench.host_ids(ids, n)
    epochs = epochs or c.iterations
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, k)
    cfg = dict(dim=c.dim, window=c.window, min_count=1, sample=c.sample, iterations=epochs, cache_nodes=k,
               flush_interval=10, seed=c.seed)
    t1 = time.time()
    gpu = api.train(ids, vocab, tree, sel, api.TrainConfig(**cfg, mode="hogwild"))
    gpu_s = time.time() - t1
    threads = threads or bench.cpu_threads()
    with tempfile.TemporaryDirectory() as d:
        Oref, h, path, _ = bench.reference_sample(c, vocab, ids, n, d)
        r0, r1, words, wall = Oref.ref_train(h, path, cfg, workers=threads)
        Oref.ref().ref_close(h)
    t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
    cen, ctx = O.sample_pairs(ids, vocab.counts, vocab.total_tokens(), c.sample, c.window, 20240917, pairs)
    init = api.init_model(vocab.size(), c.dim, c.seed)
    loss = {key: O.hs_loss(cen, ctx, m0, m1, t) for key, (m0, m1) in
            {"gpu": (gpu.syn0, gpu.syn1), "reference": (r0, r1), "init": (init.syn0, init.syn1)}.items()}
    row = {"config": name, "tokens": int(n), "k": k, "epochs": epochs, "eval_pairs": int(cen.size), "loss": loss,
           "loss_rel_diff": abs(loss["gpu"] - loss["reference"]) / loss["reference"],
           "loss_gate_2pct": abs(loss["gpu"] - loss["reference"]) / loss["reference"] < 0.02,
           # share of the reference's loss reduction (init -> trained) the GPU model achieves
           "learning_ratio": (loss["init"] - loss["gpu"]) / (loss["init"] - loss["reference"]),
           "reference_threads": threads, "reference_words_per_s": words / wall, "gpu_train_s": gpu_s}
    if cluster is not None:
        sample = np.arange(vocab.size())
        rg, rr = recall_at_10(gpu.syn0, cluster, sample), recall_at_10(r0, cluster, sample)
        row.update(recall_gpu=rg, recall_reference=rr, recall_gate_0p02=abs(rg - rr) <= 0.02)
    row["seconds"] = time.time() - t0
    return row


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", nargs="+", default=["c1", "c2", "c3"])
    p.add_argument("--tokens", nargs="*", default=[], help="per-config prefixes, e.g. c4=20000000")
    p.add_argument("--epochs", nargs="*", default=[], help="per-config pass counts, e.g. c3=1")
    p.add_argument("--k", type=int, default=31)
    p.add_argument("--pairs", type=int, default=1 << 20)
    p.add_argument("--out", default="")
    a = p.parse_args()
    tok = {k: int(v) for k, v in (x.split("=") for x in a.tokens)}
    ep = {k: int(v) for k, v in (x.split("=") for x in a.epochs)}
    results = []
    for name in a.configs:
        row = gate(name, tok.get(name), ep.get(name), a.k, a.pairs)
        print(json.dumps(row), flush=True)
        results.append(row)
    if a.out:
        Path(a.out).write_text(json.dumps(results, indent=1))


if __name__ == "__main__":
    main()
