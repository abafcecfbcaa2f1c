"""Stability of K1 without subsampling: C1/C2 with sample 0 and with their own sample,
with the hot syn0-row cache (default) and without it (probe bit 6); prints finiteness and
HS loss against the untrained model's.  python tools/stability_probe.py"""
import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle_lib as O, bench
from paper_1606_07822_b200 import api
for name, sample in (("c1", 0.0), ("c1", 1e-3), ("c2", 0.0), ("c2", 1e-4)):
    c, vocab, ids = bench.workload(name, 0, 1)
    tree = api.build_huffman_tree(vocab); sel = api.select_cached_nodes(tree, 31)
    t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
    cen, ctx = O.sample_pairs(ids, vocab.counts, vocab.total_tokens(), sample, c.window, 7, 1 << 16)
    init = api.init_model(vocab.size(), c.dim, c.seed)
    li = O.hs_loss(cen, ctx, init.syn0, init.syn1, t)
    top = vocab.counts[0] / vocab.total_tokens()
    for rows, pr in ((0, 0), (0, 64)):
        s = api.Session(vocab, tree, sel, api.TrainConfig(dim=c.dim, window=c.window, min_count=1, sample=sample, iterations=1, cache_nodes=31, seed=c.seed, mode="hogwild"))
        s.tune(min_cache_rows=rows, probe=pr)
        s.upload_ids(ids); e = s.train_range(0, 0, ids.size); m = s.download(); s.close()
        fin = bool(np.isfinite(m.syn0).all() and np.isfinite(m.syn1).all())
        l = O.hs_loss(cen, ctx, m.syn0, m.syn1, t) if fin else float("nan")
        print(f"{name} sample {sample} top-word share {top:.3f} rows {rows} probe {pr} finite {fin} loss {l:.4f} init {li:.4f} kept {e.kept}", flush=True)
