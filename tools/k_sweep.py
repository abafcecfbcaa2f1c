#!/usr/bin/env python
"""Hot-node cache sweep (BASELINE config 5: "Hot-node cache swept over K in
{0, 64, 256, 1024} inner nodes").

For each K, on one GPU:
* K1 throughput: trained words/s of one full pass (K3 + K1, ids resident in HBM). K is
  honoured: every CTA caches the K CacheSelection rows (the hottest 8 in shared memory,
  the rest as CTA-private delta rows in L2), plus the stability floor when K is below it
  (`floor_rows`; cg_tuning.min_cache_rows), flushed every u x (worker warps) merged
  centers (cg_capi.cu, hog_plan in cg_hogwild.cu);
* HS log-loss of the trained model on 2^20 evaluation pairs (checker: the C oracle's
  formula of acceptance.cpp:100-110), against the untrained model's;
* the reference's own train() (oracle/_ref, all host threads) with the same K on a
  bounded prefix of the corpus: the paper's effect on CPU.

  python tools/k_sweep.py [--config c5] [--ks 0 64 256 1024] [--out gpurun_out/k_sweep_c5.jsonl]
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

import bench  # noqa: E402  (workload + reference helpers)
import oracle_lib as O  # noqa: E402  (checker side)
from paper_1606_07822_b200 import api  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c5")
    p.add_argument("--ks", type=int, nargs="+", default=[0, 31, 64, 256, 1024])
    p.add_argument("--passes", type=int, default=2, help="timed passes per K (after one warm-up pass)")
    p.add_argument("--pairs", type=int, default=1 << 20)
    p.add_argument("--eval-prefix", type=int, default=100_000_000, help="tokens the evaluation pairs are drawn from")
    p.add_argument("--ref-tokens", type=int, default=20_000_000, help="reference sample per K (0 = skip)")
    p.add_argument("--out", default="")
    p.add_argument("--kernel", type=int, default=0, help="K1 version (cg_tuning.kernel; 0 = default)")
    p.add_argument("--min-cache-rows", type=int, default=0,
                   help="cg_tuning.min_cache_rows: 0 = the stability floor, < 0 = none (K honoured literally)")
    a = p.parse_args()

    import torch

    c, vocab, ids = bench.workload(a.config, 0, 1, device=a.config in ("c4", "c5"))
    T = int(len(ids))
    tree = api.build_huffman_tree(vocab)
    t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
    host_prefix = bench.host_ids(ids, min(T, a.eval_prefix))
    cen, ctx = O.sample_pairs(host_prefix, vocab.counts, vocab.total_tokens(), c.sample, c.window, 20240917, a.pairs)
    init = api.init_model(vocab.size(), c.dim, c.seed)
    loss_init = O.hs_loss(cen, ctx, init.syn0, init.syn1, t)
    del init
    threads = bench.cpu_threads()
    rows = []
    for k in a.ks:
        t0 = time.time()
        sel = api.select_cached_nodes(tree, k)
        cfg = api.TrainConfig(dim=c.dim, window=c.window, min_count=c.min_count, sample=c.sample, iterations=1,
                              cache_nodes=k, seed=c.seed, mode="hogwild")
        sess = api.Session(vocab, tree, sel, cfg)
        if a.kernel or a.min_cache_rows:
            sess.tune(kernel=a.kernel, min_cache_rows=a.min_cache_rows)
        if isinstance(ids, np.ndarray):
            sess.upload_ids(ids)
        else:
            sess.upload_ids_device(ids)
        sess.train_range(900, 0, T)  # warm-up pass
        sess.reset_model()
        ms, kms, e = [], [], None
        for i in range(a.passes):
            if i:
                sess.reset_model()
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            e = sess.train_range(i, 0, T)
            ms.append((time.perf_counter() - w0) * 1e3)
            kms.append(e.train_ms)
        m = sess.download()  # the last pass's model (one pass from init, like every timed pass)
        sess.close()
        loss = O.hs_loss(cen, ctx, m.syn0, m.syn1, t)
        finite = bool(np.isfinite(m.syn0).all() and np.isfinite(m.syn1).all())
        del m
        kmed = float(np.median(kms))
        row = {"config": a.config, "k": k, "cached_rows_per_cta": e.cached_rows, "smem_rows": e.smem_rows,
               "l2_tier_rows": e.cached_rows - e.smem_rows, "floor_rows": e.floor_rows,
               "flush_centers": e.flush_centers, "worker_warps": e.worker_warps,
               "ctx_batch": e.ctx_batch, "blocks": e.blocks, "kernel": e.kernel, "tokens": T, "pairs": int(e.pairs), "steps": int(e.steps),
               "k1_ms": kmed, "pass_ms_wall": float(np.median(ms)), "words_per_s_k1": T / (kmed / 1e3),
               "words_per_s_pass": T / (float(np.median(ms)) / 1e3),
               "algorithmic_gbs": 4.0 * c.dim * (2.0 * e.steps + 2.0 * e.pairs) / (kmed / 1e3) / 1e9,
               "loss": loss, "loss_init": loss_init, "finite": finite, "eval_pairs": int(cen.size)}
        if a.ref_tokens > 0:
            rates, walls, n = bench.run_reference(c, vocab, ids, threads, a.ref_tokens, 1, k)
            row.update(ref_words_per_s=float(rates[0]), ref_threads=threads, ref_sample_tokens=n)
        row["seconds"] = time.time() - t0
        print(json.dumps(row), flush=True)
        rows.append(row)
    if a.out:
        Path(a.out).write_text("".join(json.dumps(r) + "\n" for r in rows))


if __name__ == "__main__":
    main()
