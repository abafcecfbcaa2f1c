import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle_lib as O
from paper_1606_07822_b200 import api
from paper_1606_07822_b200.corpus_gen import vocab_from_raw
rng = np.random.default_rng(21)
raw = (np.minimum(rng.zipf(1.1, 2_800_000), 20000) - 1).astype(np.int64)
vocab, ids = vocab_from_raw(raw, 1, 20000)
tree = api.build_huffman_tree(vocab); sel = api.select_cached_nodes(tree, 31)
t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
cen, ctx = O.sample_pairs(ids, vocab.counts, vocab.total_tokens(), 1e-3, 5, 7, 1 << 15)
for d in (16, 32, 64, 100):
    init = api.init_model(vocab.size(), d, 5)
    li = O.hs_loss(cen, ctx, init.syn0, init.syn1, t)
    for rows in (0,):
        s = api.Session(vocab, tree, sel, api.TrainConfig(dim=d, window=5, min_count=1, sample=1e-3, iterations=1, cache_nodes=31, seed=5, mode="hogwild"))
        s.tune(min_cache_rows=rows)
        s.upload_ids(ids); e = s.train_range(0, 0, ids.size); m = s.download(); s.close()
        fin = bool(np.isfinite(m.syn0).all() and np.isfinite(m.syn1).all())
        l = O.hs_loss(cen, ctx, m.syn0, m.syn1, t) if fin else float("nan")
        print(f"D {d} rows {rows} (cached {e.cached_rows}, warps {e.worker_warps}) finite {fin} loss {l:.4f} init {li:.4f}", flush=True)
