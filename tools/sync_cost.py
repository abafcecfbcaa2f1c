#!/usr/bin/env python
"""Cost of the replicas' delta sync at a configuration, measured on one GPU and projected
to N GPUs of one NVSwitch node (verdict item "syncs affordable at C5").

Trains one sync period (sync_words tokens) on a session, then times the device work of a
sync -- cg_session_sync_delta (delta = model - snapshot) and cg_session_sync_apply
(model = snapshot + scale x delta) -- with CUDA events, counts the rows the period touched
(non-zero delta rows: what a sparse exchange would move), and projects the NCCL
all-reduce of the dense delta with the pool's measured 8-rank all-reduce bus bandwidth
(B200_PROFILING.md: 725 GB/s at 1 GiB; ring bytes per GPU = 2 (N-1)/N x buffer).

  python tools/sync_cost.py --config c5 --sync 1000000 10000000 25000000 [--out f.json]
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

import bench  # noqa: E402
from paper_1606_07822_b200 import api  # noqa: E402
from paper_1606_07822_b200.corpus_gen import CONFIGS  # noqa: E402

BUS_GBS = 725.0  # measured 8-rank all-reduce bus bandwidth at 1 GiB (B200_PROFILING.md)


def main():
    import torch

    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c5")
    p.add_argument("--sync", type=int, nargs="+", default=[1_000_000, 10_000_000, 25_000_000])
    p.add_argument("--out", default="")
    a = p.parse_args()
    c = CONFIGS[a.config]
    _, vocab, ids = bench.workload(a.config, 0, 1, device=a.config in ("c4", "c5"))
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, 31)
    cfg = api.TrainConfig(dim=c.dim, window=c.window, min_count=c.min_count, sample=c.sample, iterations=1,
                          cache_nodes=31, seed=c.seed, mode="hogwild")
    stream = torch.cuda.current_stream()
    s = api.Session(vocab, tree, sel, cfg, stream=stream.cuda_stream)
    if isinstance(ids, np.ndarray):
        s.upload_ids(ids)
    else:
        s.upload_ids_device(ids)
    T = int(len(ids))
    full = s.train_range(0, 0, T)  # one pass: the pass time the sync cost is set against
    pass_ms = full.train_ms + full.subsample_ms
    out = {"config": a.config, "pass_ms_one_gpu": pass_ms, "tokens_per_pass": T, "rows": []}
    for sw in a.sync:
        s.reset_model()
        s.sync_begin()
        # the first apply of an (N, interval) pair builds and uploads the per-row prior table
        # on the host (cached afterwards): do that on an empty delta, outside the timed apply
        s.sync_delta_tensor()
        s.sync_apply(2, sw)
        s.train_range(1, 0, min(sw, T))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record(stream)
        d = s.sync_delta_tensor()
        ev[1].record(stream)
        nbytes = d.numel() * 4
        # the buffer is the model-layout delta followed by the per-row squared norms (the all-reduce moves both)
        n_model = s.model_buffer()[1] // 4
        row = d[:n_model].view(-1, (c.dim + 7) // 8 * 8)
        touched = int((row != 0).any(dim=1).sum().item())
        torch.cuda.synchronize()
        ev[2].record(stream)
        s.sync_apply(2, sw)
        ev[3].record(stream)
        torch.cuda.synchronize()
        t_delta, t_apply = ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])
        syncs = int(np.ceil(T / sw))
        r = {"sync_words": sw, "syncs_per_pass": syncs, "delta_bytes": nbytes, "rows": int(row.shape[0]),
             "touched_rows": touched, "touched_share": touched / row.shape[0], "delta_ms": t_delta,
             "apply_ms": t_apply, "projection": {}}
        for n in (2, 4, 8):
            ar_ms = 2 * (n - 1) / n * nbytes / (BUS_GBS * 1e9) * 1e3
            per_sync = ar_ms + t_delta + t_apply
            r["projection"][f"n{n}"] = {"allreduce_ms": ar_ms, "per_sync_ms": per_sync,
                                        "per_pass_ms": per_sync * syncs,
                                        "share_of_pass": per_sync * syncs / (pass_ms + per_sync * syncs),
                                        "sparse_allreduce_ms": ar_ms * touched / row.shape[0]}
        print(json.dumps(r), flush=True)
        out["rows"].append(r)
    s.close()
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
