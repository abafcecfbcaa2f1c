#!/usr/bin/env python
"""K1 launch-geometry sweep on one session: shared-memory cache rows per CTA (and
optionally worker warps), timing K1 per pass and the HS loss of the model it trains.

  python tools/rows_sweep.py --config c2 --rows 0 2 4 8 16 31 [--warps 0 11] [--out f.jsonl]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import bench  # noqa: E402
import oracle_lib as O  # noqa: E402  (checker side: HS loss)
from paper_1606_07822_b200 import api  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c2")
    p.add_argument("--rows", type=int, nargs="+", default=[4, 8, 16, 31])
    p.add_argument("--warps", type=int, nargs="+", default=[0])
    p.add_argument("--k", type=int, default=31)
    p.add_argument("--passes", type=int, default=3)
    p.add_argument("--pairs", type=int, default=1 << 18, help="evaluation pairs for the loss (0 = skip)")
    p.add_argument("--flush", type=int, default=0, help="flush_centers (0 = default)")
    p.add_argument("--probes", type=int, nargs="+", default=[0], help="cg_tuning.probe values to sweep")
    p.add_argument("--out", default="")
    a = p.parse_args()

    c, vocab, ids = bench.workload(a.config, 0, 1, device=a.config in ("c4", "c5"))
    T = int(len(ids))
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, a.k)
    cfg = api.TrainConfig(dim=c.dim, window=c.window, min_count=c.min_count, sample=c.sample, iterations=1,
                          cache_nodes=a.k, seed=c.seed, mode="hogwild")
    sess = api.Session(vocab, tree, sel, cfg)
    if isinstance(ids, np.ndarray):
        sess.upload_ids(ids)
    else:
        sess.upload_ids_device(ids)
    ev = None
    if a.pairs:
        t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
        cen, ctx = O.sample_pairs(bench.host_ids(ids, min(T, 50_000_000)), vocab.counts, vocab.total_tokens(),
                                  c.sample, c.window, 20240917, a.pairs)
        ev = (cen, ctx, t)
    rows_out = []
    for w, r, pr in [(w, r, pr) for w in a.warps for r in a.rows for pr in a.probes]:
        if True:
            sess.tune(warps=w, cache_rows=r, flush_centers=a.flush, min_cache_rows=-1 if r == 0 else 0, probe=pr)
            sess.train_range(900, 0, T)  # warm-up
            kms, e = [], None
            for i in range(a.passes):
                sess.reset_model()
                e = sess.train_range(i, 0, T)
                kms.append(e.train_ms)
            row = {"config": a.config, "rows_req": r, "warps_req": w, "probe": pr, "cached_rows_per_cta": e.cached_rows,
                   "worker_warps": e.worker_warps, "ctx_batch": e.ctx_batch, "k1_ms": float(np.median(kms)),
                   "k1_ms_all": kms, "words_per_s_k1": T / (float(np.median(kms)) / 1e3), "flush": a.flush}
            if ev:
                m = sess.download()
                row["loss"] = O.hs_loss(ev[0], ev[1], m.syn0, m.syn1, ev[2])
            print(json.dumps(row), flush=True)
            rows_out.append(row)
    sess.close()
    if a.out:
        Path(a.out).write_text("".join(json.dumps(r) + "\n" for r in rows_out))


if __name__ == "__main__":
    main()
