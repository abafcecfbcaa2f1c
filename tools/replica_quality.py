#!/usr/bin/env python
"""Learning of N in-process replicas (cg_train_replicas, replicas sharing the visible GPU)
on a corpus split N ways, against one replica on the whole corpus: HS loss on 2^20
evaluation pairs (the quality gates' seed) and the learning ratio (init - replicas) /
(init - single).  python tools/replica_quality.py --config c1 --n 2 4 --sync 50000 200000"""
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

import bench  # noqa: E402
import oracle_lib as O  # noqa: E402  (checker side: HS loss)
from paper_1606_07822_b200 import api  # noqa: E402
from paper_1606_07822_b200.corpus_gen import CONFIGS  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c1")
    p.add_argument("--n", type=int, nargs="+", default=[2, 4])
    p.add_argument("--sync", type=int, nargs="+", default=[100_000])
    p.add_argument("--pairs", type=int, default=1 << 20)
    p.add_argument("--kernel", type=int, default=0)
    p.add_argument("--tokens", type=int, default=0, help="train on this prefix of the corpus (0 = all of it)")
    p.add_argument("--out", default="")
    a = p.parse_args()
    c = CONFIGS[a.config]
    _, vocab, ids = bench.workload(a.config, 0, 1, device=a.config in ("c4", "c5"))
    ids = bench.host_ids(ids, a.tokens or None)
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, 31)
    cfg = api.TrainConfig(dim=c.dim, window=c.window, min_count=1, sample=c.sample, iterations=c.iterations,
                          cache_nodes=31, seed=c.seed, mode="hogwild")
    t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
    cen, ctx = O.sample_pairs(ids, vocab.counts, vocab.total_tokens(), c.sample, c.window, 20240917, a.pairs)
    loss = lambda m: O.hs_loss(cen, ctx, m.syn0, m.syn1, t)  # noqa: E731
    li = loss(api.init_model(vocab.size(), c.dim, c.seed))
    t0 = time.time()
    ls = loss(api.train(ids, vocab, tree, sel, cfg))
    rows = []
    for n in a.n:
        for sw in a.sync:
            st = api.TrainStats()
            t1 = time.time()
            m = api.train(ids, vocab, tree, sel, cfg, st, devices=[0] * n, sync_words=sw)
            lr = loss(m)
            row = {"config": a.config, "n": n, "sync_words": sw, "loss": lr, "loss_single": ls, "loss_init": li,
                   "learning_ratio": (li - lr) / (li - ls), "loss_rel_diff": abs(lr - ls) / ls,
                   "words": st.words_processed, "seconds": time.time() - t1, "finite": bool(np.isfinite(lr))}
            print(json.dumps(row), flush=True)
            rows.append(row)
    if a.out:
        Path(a.out).write_text("".join(json.dumps(r) + "\n" for r in rows))


if __name__ == "__main__":
    main()
