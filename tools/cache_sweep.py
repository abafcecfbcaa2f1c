#!/usr/bin/env python
"""Per-CTA cache sweep on one session: cached rows K (both tiers), shared-memory rows,
stability floor, flush period and flush-scale rule; per setting the K1 time per pass and
the HS loss of the trained model (2^20 evaluation pairs, the quality gates' seed) with
its learning ratio against the initial model and a reference loss when one is given.

  python tools/cache_sweep.py --config c2 --grid k [--ref-loss 9.4629] [--out f.jsonl]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import bench  # noqa: E402
import oracle_lib as O  # noqa: E402  (checker side: HS loss)
from paper_1606_07822_b200 import api  # noqa: E402
from paper_1606_07822_b200.corpus_gen import CONFIGS, CorpusConfig, generate, vocab_from_raw  # noqa: E402

GRIDS = {
    # (K, smem_rows, min_cache_rows, flush_interval u, scale rule)
    "k": [(0, -1, -1, 10, 0), (0, -1, 0, 10, 0), (8, -1, -1, 10, 0), (31, -1, 0, 10, 0), (31, -1, 0, 10, 1),
          (31, 31, 0, 10, 0), (64, -1, 0, 10, 0), (256, -1, 0, 10, 0), (1024, -1, 0, 10, 0)],
    "rule": [(31, -1, 0, 10, 0), (31, -1, 0, 10, 1), (64, -1, 0, 10, 1), (256, -1, 0, 10, 1), (0, -1, 0, 10, 1),
             (8, -1, -1, 10, 0)],
    "rule2": [(31, -1, 0, 10, 2, 256), (64, -1, 0, 10, 2, 256), (256, -1, 0, 10, 2, 256), (1024, -1, 0, 10, 2, 256),
              (0, -1, 0, 10, 0, 512), (31, -1, 0, 10, 2, 512), (0, -1, 0, 10, 0, 1024), (31, -1, 0, 10, 2, 1024)],
    "rule3": [(31, -1, 0, 10, 3, 256, 256), (64, -1, 0, 10, 3, 256, 256), (256, -1, 0, 10, 3, 256, 256),
              (1024, -1, 0, 10, 3, 256, 256), (0, -1, 0, 10, 3, 256, 256), (31, -1, 0, 10, 3, 256, 128),
              (256, -1, 0, 10, 3, 256, 128), (0, -1, 0, 10, 3, 256, 128), (31, -1, 0, 10, 3, 512, 256),
              (31, -1, 0, 10, 3, 256, 512)],
    "rule3b": [(0, -1, 0, 10, 3, 256, 64), (31, -1, 0, 10, 3, 256, 64), (256, -1, 0, 10, 3, 256, 64),
               (0, -1, 0, 10, 3, 256, 32), (31, -1, 0, 10, 3, 256, 32), (256, -1, 0, 10, 3, 256, 32),
               (8, -1, -1, 10, 0, 256, 64)],
    "flush": [(31, -1, 0, 10, 3, 256, h, f) for h in (32, 64) for f in (10, 20, 40, 80, 0)],
    "v6": [(31, -1, 0, 10, 3, 256, 32, 0, 0), (31, -1, 0, 10, 3, 256, 32, 0, 5), (8, -1, -1, 10, 0, 256, 64, 0, 0),
           (8, -1, -1, 10, 0, 256, 64, 0, 5)],
    "h": [(31, -1, 0, 10, 3, 256, 32, 0, 0), (8, -1, -1, 10, 0, 256, 64, 0, 0), (0, -1, 0, 10, 3, 256, 32, 0, 0)],
    "ab": [(31, -1, 0, 10, 3), (8, -1, -1, 10, 0)],
    "final": [(31, -1, 0, 10, 3), (31, -1, 0, 10, 3, 256, 32, 1), (256, -1, 0, 10, 3), (0, -1, 0, 10, 3),
              (8, -1, -1, 10, 3)],
    "stab": [(31, -1, 0, 10, 3, 256, 32), (31, -1, 0, 10, 3, 256, 32), (31, -1, 0, 10, 3, 256, 16),
             (31, -1, 0, 10, 3, 256, 16), (31, -1, 0, 10, 3, 256, 8), (31, -1, 0, 10, 3, 256, 1),
             (31, -1, 0, 10, 3, 256, 16, 1), (31, -1, 0, 10, 3, 256, 1, 1), (256, -1, 0, 10, 3, 256, 16)],
    "v8": [(31, -1, 0, 10, 3, 256, 32, 0, 5), (31, -1, 0, 10, 3, 256, 32, 0, 8), (8, -1, -1, 10, 3, 256, 32, 0, 8)],
    "k8": [(31, -1, 0, 10, 3, 256, 32, 0, 5), (31, -1, 0, 10, 3, 256, 32, 0, 8)],
    "sweep": [(0, -1, 0, 10, 0), (64, -1, 0, 10, 0), (256, -1, 0, 10, 0), (1024, -1, 0, 10, 0), (31, -1, 0, 10, 0)],
}


def workload(name):
    small = {"variants": CorpusConfig("variants", 300_000, 5000, 1.0, 100, 5, 1e-3, 1, 11),
             # heavy tail: the top word holds ~41% of the tokens
             "heavy": CorpusConfig("heavy", 1_000_000, 10000, 1.6, 100, 5, 1e-3, 1, 17),
             # C1 without subsampling: the top words sit in thousands of concurrent windows
             "c1ns": CorpusConfig("c1ns", 1_000_000, 10000, 1.0, 100, 5, 0.0, 1, 1)}
    if name in small:
        c = small[name]
        vocab, ids = vocab_from_raw(generate(c), 1, c.vocab)
        return c, vocab, ids
    c, vocab, ids = bench.workload(name, 0, 1, device=name in ("c4", "c5"))
    return CONFIGS[name], vocab, ids


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c2")
    p.add_argument("--grid", default="k")
    p.add_argument("--passes", type=int, default=2)
    p.add_argument("--pairs", type=int, default=1 << 20)
    p.add_argument("--ref-loss", type=float, default=0.0)
    p.add_argument("--out", default="")
    a = p.parse_args()

    c, vocab, ids = workload(a.config)
    T = int(len(ids))
    tree = api.build_huffman_tree(vocab)
    t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
    hids = bench.host_ids(ids, min(T, 50_000_000))
    cen, ctx = O.sample_pairs(hids, vocab.counts, vocab.total_tokens(), c.sample, c.window, 20240917, a.pairs)
    init = api.init_model(vocab.size(), c.dim, c.seed)
    li = O.hs_loss(cen, ctx, init.syn0, init.syn1, t)
    if a.config in ("variants", "c1", "heavy", "c1ns") and not a.ref_loss:  # the reference's single-stream training (oracle)
        r0, r1, _ = O.orc_train(hids, vocab.counts, vocab.total_tokens(),
                                dict(dim=c.dim, window=c.window, min_count=1, sample=c.sample, iterations=1,
                                     cache_nodes=31, flush_interval=10, seed=c.seed))
        a.ref_loss = O.hs_loss(cen, ctx, r0, r1, t)
    out = []
    for k, srows, floor, u, rule, *hot in GRIDS[a.grid]:
        os.environ["CG_SCALE_RULE"] = str(rule)
        os.environ["CG_HOT_UPDATERS"] = str(hot[0] if hot else 256)
        os.environ["CG_SCALE_H"] = str(hot[1] if len(hot) > 1 else 256)
        sel = api.select_cached_nodes(tree, k)
        cfg = api.TrainConfig(dim=c.dim, window=c.window, min_count=c.min_count, sample=c.sample, iterations=1,
                              cache_nodes=k, flush_interval=u, seed=c.seed, mode="hogwild")
        sess = api.Session(vocab, tree, sel, cfg)
        kern = hot[3] if len(hot) > 3 else 0
        sess.tune(smem_rows=srows, min_cache_rows=floor, flush_centers=hot[2] if len(hot) > 2 else 0, kernel=kern)
        if isinstance(ids, np.ndarray):
            sess.upload_ids(ids)
        else:
            sess.upload_ids_device(ids)
        sess.train_range(900, 0, T)  # warm-up
        kms, e = [], None
        for i in range(a.passes):
            sess.reset_model()
            e = sess.train_range(i, 0, T)
            kms.append(e.train_ms)
        m = sess.download()
        sess.close()
        lg = O.hs_loss(cen, ctx, m.syn0, m.syn1, t)
        row = {"config": a.config, "k": k, "smem_rows_req": srows, "min_cache_rows": floor, "u": u, "scale_rule": rule, "hot_updaters": hot[0] if hot else 256, "scale_h": hot[1] if len(hot) > 1 else 256, "kernel": kern,
               "cached_rows_per_cta": e.cached_rows, "smem_rows": e.smem_rows, "floor_rows": e.floor_rows,
               "flush_centers": e.flush_centers, "worker_warps": e.worker_warps, "ctx_batch": e.ctx_batch,
               "k1_ms": float(np.median(kms)), "k1_ms_all": kms, "words_per_s_k1": T / (float(np.median(kms)) / 1e3),
               "loss": lg, "loss_init": li, "finite": bool(np.isfinite(lg))}
        if a.ref_loss:
            row["loss_ref"] = a.ref_loss
            row["learning_ratio"] = (li - lg) / (li - a.ref_loss)
        print(json.dumps(row), flush=True)
        out.append(row)
    if a.out:
        Path(a.out).write_text("".join(json.dumps(r) + "\n" for r in out))


if __name__ == "__main__":
    main()
