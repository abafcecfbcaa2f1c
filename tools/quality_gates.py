#!/usr/bin/env python
"""North-star quality gates for the Hogwild (throughput) mode, at full config size.

* HS log-loss: mean over a fixed set of 2^20 evaluation pairs (harness seed, the
  reference's pair rules; formula of tests/acceptance.cpp:100-110) of the GPU model vs
  the reference's own model -- cachegram::train() compiled unchanged (oracle/_ref),
  run multithreaded on this host's cores, i.e. its Hogwild mode. Gate: within 2%.
* C3 planted-cluster recall@10 (cosine over unit syn0, self excluded): GPU vs the
  reference model. Gate: within 0.02.

  python tools/quality_gates.py --configs c1 c2 c3 [--out gpurun_out/quality.json]
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


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--configs", nargs="+", default=["c1", "c2", "c3"])
    p.add_argument("--k", type=int, default=31)
    p.add_argument("--pairs", type=int, default=1 << 20)
    p.add_argument("--out", default="")
    p.add_argument("--kernel", type=int, default=0, help="K1 version (0 = default)")
    a = p.parse_args()
    results = []
    threads = bench.cpu_threads()
    for name in a.configs:
        c = CONFIGS[name]
        t0 = time.time()
        cluster = None
        if c.clusters:
            raw, cluster_of = cluster_raw_ids(c)
            vocab, ids = vocab_from_raw(raw, c.min_count, c.clusters * c.cluster_size)
            cluster = cluster_of[vocab.raw_of_id]
        else:
            _, vocab, ids = bench.workload(name, 0, 1, device=name in ("c4", "c5"))
            ids = bench.host_ids(ids)
        tree = api.build_huffman_tree(vocab)
        sel = api.select_cached_nodes(tree, a.k)
        cfg = dict(dim=c.dim, window=c.window, min_count=1, sample=c.sample, iterations=c.iterations,
                   cache_nodes=a.k, flush_interval=10, seed=c.seed)
        tcfg = api.TrainConfig(**cfg, mode="hogwild")
        if a.kernel:
            sess = api.Session(vocab, tree, sel, tcfg)
            sess.tune(kernel=a.kernel)
            sess.upload_ids(ids)
            sess.train()
            gpu = sess.download()
            sess.close()
        else:
            gpu = api.train(ids, vocab, tree, sel, tcfg)
        with tempfile.TemporaryDirectory() as d:
            Oref, h, path, n = bench.reference_sample(c, vocab, ids, len(ids), d)
            r0, r1, words, wall = Oref.ref_train(h, path, cfg, workers=threads)
            Oref.ref().ref_close(h)
        t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
        cen, ctx = O.sample_pairs(ids, vocab.counts, vocab.total_tokens(), c.sample, c.window, 20240917, a.pairs)
        init = api.init_model(vocab.size(), c.dim, c.seed)
        loss = {k: O.hs_loss(cen, ctx, m0, m1, t) for k, (m0, m1) in
                {"gpu": (gpu.syn0, gpu.syn1), "reference": (r0, r1), "init": (init.syn0, init.syn1)}.items()}
        row = {"config": name, "k": a.k, "epochs": c.iterations, "eval_pairs": int(cen.size), "loss": loss,
               "loss_rel_diff": abs(loss["gpu"] - loss["reference"]) / loss["reference"],
               "loss_gate_2pct": abs(loss["gpu"] - loss["reference"]) / loss["reference"] < 0.02,
               # share of the reference's loss reduction (init -> trained) the GPU model achieves
               "learning_ratio": (loss["init"] - loss["gpu"]) / (loss["init"] - loss["reference"]),
               "kernel": a.kernel or 4,
               "reference_threads": threads, "reference_words_per_s": words / wall}
        if cluster is not None:
            sample = np.arange(vocab.size())
            rg, rr = recall_at_10(gpu.syn0, cluster, sample), recall_at_10(r0, cluster, sample)
            row.update(recall_gpu=rg, recall_reference=rr, recall_gate_0p02=abs(rg - rr) <= 0.02)
        row["seconds"] = time.time() - t0
        print(json.dumps(row), flush=True)
        results.append(row)
    if a.out:
        Path(a.out).write_text(json.dumps(results, indent=1))


if __name__ == "__main__":
    main()
