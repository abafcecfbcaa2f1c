import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle_lib as O
from paper_1606_07822_b200 import api
from paper_1606_07822_b200.corpus_gen import CorpusConfig, generate, vocab_from_raw

def loss(m, tree, vocab, ids, sample, w=5):
    cen, ctx = O.sample_pairs(ids, vocab.counts, vocab.total_tokens(), sample, w, 12345, 1 << 16)
    return O.hs_loss(cen, ctx, m.syn0, m.syn1, O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage))

# small corpus (the variant test): learning ratio vs the deterministic reference stream
c = CorpusConfig("variants", 300_000, 5000, 1.0, 100, 5, 1e-3, 1, 11)
vocab, ids = vocab_from_raw(generate(c), 1, c.vocab)
tree = api.build_huffman_tree(vocab); sel = api.select_cached_nodes(tree, 31)
base = dict(dim=100, window=5, min_count=1, sample=1e-3, iterations=1, cache_nodes=31, seed=11)
det = api.train(ids, vocab, tree, sel, api.TrainConfig(**base, mode="deterministic"))
init = api.init_model(vocab.size(), 100, 11)
li, ld = loss(init, tree, vocab, ids, 1e-3), loss(det, tree, vocab, ids, 1e-3)
for rows in (8, 12, 16):
    s = api.Session(vocab, tree, sel, api.TrainConfig(**base, mode="hogwild")); s.tune(min_cache_rows=rows)
    s.upload_ids(ids); s.train_range(0, 0, ids.size); m = s.download(); s.close()
    lh = loss(m, tree, vocab, ids, 1e-3)
    print(f"small rows {rows}: ratio {(li - lh) / (li - ld):.3f}", flush=True)
# heavy-tail corpus
rng = np.random.default_rng(21)
raw = (np.minimum(rng.zipf(1.1, 2_800_000), 20000) - 1).astype(np.int64)
vocab, ids = vocab_from_raw(raw, 1, 20000)
tree = api.build_huffman_tree(vocab); sel = api.select_cached_nodes(tree, 31)
for rows in (8, 12, 16):
    s = api.Session(vocab, tree, sel, api.TrainConfig(dim=100, window=5, min_count=1, sample=1e-3, iterations=1, cache_nodes=31, seed=5, mode="hogwild"))
    s.tune(min_cache_rows=rows); s.upload_ids(ids); s.train_range(0, 0, ids.size); m = s.download(); s.close()
    fin = bool(np.isfinite(m.syn0).all() and np.isfinite(m.syn1).all())
    print(f"heavy rows {rows}: finite {fin} loss {loss(m, tree, vocab, ids, 1e-3) if fin else float('nan'):.4f}", flush=True)
