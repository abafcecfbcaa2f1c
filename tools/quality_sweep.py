#!/usr/bin/env python
"""Hogwild quality/throughput sweep (development tool).

Trains one config with several kernel geometries / update modes and reports the
mean HS log-loss on a fixed evaluation pair set next to the reference's
single-worker loss (the oracle restatement, bit-identical to the reference) and the
initial-model loss. One JSON line per setting.

  python tools/quality_sweep.py --config c1 [--grid default|wide]
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

import oracle_lib as O  # noqa: E402  (checker side)
from paper_1606_07822_b200 import api  # noqa: E402
from paper_1606_07822_b200.corpus_gen import CONFIGS, generate, vocab_from_raw  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c1")
    p.add_argument("--tokens", type=int, default=0)
    p.add_argument("--k", type=int, default=31)
    p.add_argument("--iterations", type=int, default=1)
    p.add_argument("--grid", default="default")
    p.add_argument("--no-ref", action="store_true")
    a = p.parse_args()
    c = CONFIGS[a.config]
    raw = generate(c, a.tokens or None)
    vocab, ids = vocab_from_raw(raw, c.min_count, c.vocab)
    tree = api.build_huffman_tree(vocab)
    t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
    cen, ctx = O.sample_pairs(ids, vocab.counts, vocab.total_tokens(), c.sample, c.window, 12345, 1 << 16)

    def loss(m0, m1):
        return O.hs_loss(cen, ctx, m0, m1, t)

    init = api.init_model(vocab.size(), c.dim, c.seed)
    print(json.dumps({"what": "init", "loss": loss(init.syn0, init.syn1)}), flush=True)
    cfgd = dict(dim=c.dim, window=c.window, min_count=c.min_count, sample=c.sample, iterations=a.iterations,
                cache_nodes=a.k, flush_interval=10, seed=c.seed)
    if not a.no_ref:
        t0 = time.time()
        r0, r1, _ = O.orc_train(ids, vocab.counts, vocab.total_tokens(), cfgd)
        print(json.dumps({"what": "reference(single worker)", "loss": loss(r0, r1), "s": time.time() - t0}),
              flush=True)

    grids = {}
    grids["kscale"] = [dict(k=0), dict(k=0, minrows=-1), dict(k=31), dict(k=64), dict(k=255), dict(k=1024),
                       dict(k=31, scale=1 / 148), dict(k=255, scale=1 / 148)]
    grids["scales"] = [dict(k=0)] + [dict(k=k, scale=sc) for k in (31, 255) for sc in (1 / 148, 1 / 64, 1 / 32, 1 / 16, 1 / 8)]
    grids["probe"] = [dict(), dict(probe=1), dict(probe=2), dict(probe=3), dict(probe=4), dict(probe=7),
                      dict(k=0, probe=1), dict(cold=1)]
    grids["probe34"] = [dict(kernel=kn, probe=pb) for kn in (4, 3) for pb in (0, 1, 2, 4, 7)] + \
        [dict(kernel=4, cpw=1), dict(kernel=4, cpw=16), dict(kernel=4, warps=8), dict(kernel=4, k=0)]
    grids["perf4"] = [dict(), dict(cpw=8), dict(cpw=16), dict(flush=32), dict(flush=128), dict(flush=256),
                      dict(warps=9), dict(warps=11), dict(cpw=16, flush=128)]
    grids["warps"] = [dict(), dict(warps=4), dict(warps=5), dict(warps=6), dict(k=64), dict(k=255)]
    grids["probe8"] = [dict(), dict(probe=8), dict(probe=4), dict(probe=12)]
    grids["perf"] = [dict(), dict(cpw=1), dict(cpw=8), dict(cpw=16), dict(flush=16), dict(flush=256), dict(k=0),
                     dict(warps=8), dict(scale=1 / 16), dict(cold=1)]
    grids["default"] = [
        dict(blocks=1, warps=1), dict(blocks=1, warps=1, k=0), dict(blocks=1, warps=12), dict(blocks=148, warps=1),
        dict(blocks=148, warps=1, k=0), dict(blocks=16, warps=12), dict(), dict(k=0), dict(cold=1), dict(k=0, cold=1),
        dict(scale=1 / 148), dict(scale=1 / 16), dict(cpw=1), dict(cpw=1, scale=1 / 148),
    ]
    for g in grids[a.grid]:
        k = g.get("k", a.k)
        sel = api.select_cached_nodes(tree, k)
        cfg = api.TrainConfig(**dict(cfgd, cache_nodes=k), mode="hogwild")
        s = api.Session(vocab, tree, sel, cfg)
        s.tune(g.get("blocks", 0), g.get("warps", 0), g.get("cpw", 0), -1, g.get("cold", 0), g.get("scale", 0.0),
               g.get("flush", 0), g.get("minrows", 0), g.get("probe", 0), g.get("kernel", 0))
        s.upload_ids(ids)
        ms = 0.0
        for it in range(a.iterations):
            e = s.train_range(it, 0, ids.size, it * ids.size, 1)
            ms += e.train_ms + e.subsample_ms
        m = s.download()
        s.close()
        fin = bool(np.isfinite(m.syn0).all() and np.isfinite(m.syn1).all())
        print(json.dumps({"what": g, "k": k, "loss": loss(m.syn0, m.syn1) if fin else None, "finite": fin,
                          "ms": ms, "words_per_s": ids.size * a.iterations / (ms / 1e3)}), flush=True)


if __name__ == "__main__":
    main()
