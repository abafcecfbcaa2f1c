"""In-process replicas (cg_train_replicas / cg_train_file_replicas / cg_average_buffers):
the peer-memory reduction kernel is exact (fixed summation order, identical bits on every
replica); replicated training covers every token once per pass; and with the delta sync
(the replicas' deltas summed, scaled per row -- cg_session_sync_apply) a corpus split N
ways learns as much as one replica on the whole corpus. The box has one GPU, so the
replicas share device 0 -- the same code paths, with peer pointers that happen to be
local."""
import ctypes as C

import numpy as np
import pytest

import fixtures as F
import oracle_lib as O
from paper_1606_07822_b200 import _lib, api

pytestmark = pytest.mark.gpu

# delta-sync interval per replica for the split-corpus tests (tools/replica_quality.py)
# (C1 is a 1M-token corpus: a replica's hot rows see 1/N of its updates between syncs, so it
# needs short periods; C2 learns like one replica at any period measured, 100k-1M)
SYNC_WORDS = {"c1": 500, "c2": 250_000, "c5": 2_500_000}
# configurations trained on a prefix of their corpus (with the full corpus's vocabulary and tree)
PREFIX = {"c5": 100_000_000}


def test_average_buffers_exact():
    import torch

    rng = np.random.default_rng(3)
    host = [rng.standard_normal(4096 * 3 + 4).astype(np.float32) for _ in range(3)]
    bufs = [torch.from_numpy(h).cuda() for h in host]
    ptrs = (C.c_void_p * 3)(*[b.data_ptr() for b in bufs])
    dev = np.zeros(3, np.int32)
    _lib.check(_lib.load().cg_average_buffers(ptrs, _lib.ptr(dev, C.c_int32), 3, host[0].size))
    want = ((host[0] + host[1]) + host[2]) * np.float32(1.0 / 3.0)
    for b in bufs:
        assert np.array_equal(b.cpu().numpy().view(np.uint32), want.view(np.uint32))
    with pytest.raises(ValueError):
        _lib.check(_lib.load().cg_average_buffers(ptrs, _lib.ptr(dev, C.c_int32), 3, 5))


def _setup(tmp_path):
    path = F.write(tmp_path / "r.txt", F.make_zipf_corpus(600_000, 3000, 5))
    vocab = api.build_vocabulary_file(path, 2)
    ids = api.read_id_stream(path, vocab)
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, 31)
    return path, vocab, ids, tree, sel


def _loss(m, vocab, ids, tree, cfg):
    t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
    cen, ctx = O.sample_pairs(ids, vocab.counts, vocab.total_tokens(), cfg["sample"], cfg["window"], 99, 1 << 16)
    return O.hs_loss(cen, ctx, m.syn0, m.syn1, t)


@pytest.mark.parametrize("n_rep", [1, 2, 3])
def test_replicas_cover_the_stream_and_learn(tmp_path, n_rep):
    """Weak scaling, as in bench.py at N GPUs: every replica trains a full-size shard (here
    n_rep copies of the corpus), so the averaged model must learn as much as one replica
    on one copy. (With a fixed corpus split n ways, model averaging learns roughly 1/n as
    much per pass -- the known cost of synchronous averaging.)"""
    path, vocab, ids, tree, sel = _setup(tmp_path)
    cfg = dict(dim=32, window=5, min_count=2, sample=1e-3, iterations=2, cache_nodes=31, seed=4)
    tc = api.TrainConfig(**cfg, mode="hogwild")
    single = api.train(ids, vocab, tree, sel, tc)
    st = api.TrainStats()
    stream = np.tile(ids, n_rep)
    vocab_n = api.Vocabulary(vocab.counts * n_rep, vocab.words)  # totals of the n-copy stream
    rep = api.train(stream, vocab_n, tree, sel, tc, st, devices=[0] * n_rep, sync_words=20_000)
    assert st.words_processed == stream.size * 2
    assert np.isfinite(rep.syn0).all() and np.isfinite(rep.syn1).all()
    init = api.init_model(vocab.size(), 32, 4)
    l_init, l_one, l_rep = (_loss(m, vocab, ids, tree, cfg) for m in (init, single, rep))
    assert l_one < l_init and l_rep < l_init
    assert (l_init - l_rep) > 0.8 * (l_init - l_one), (l_init, l_one, l_rep)


def test_file_replicas_match_id_replicas_in_coverage(tmp_path):
    path, vocab, ids, tree, sel = _setup(tmp_path)
    tc = api.TrainConfig(dim=16, window=3, min_count=2, sample=1e-3, iterations=1, cache_nodes=31, seed=9,
                         mode="hogwild")
    st = api.TrainStats()
    m = api.train(path, vocab, tree, sel, tc, st, devices=[0, 0], sync_words=50_000)
    assert st.words_processed == ids.size
    assert np.isfinite(m.syn0).all()
    with pytest.raises(ValueError):  # deterministic replicas are refused
        api.train(ids, vocab, tree, sel, api.TrainConfig(dim=16, window=3, min_count=2, iterations=1,
                                                          mode="deterministic", workers=1), devices=[0, 0])


SPLIT_CASES = [("c1", 2), ("c1", 4), ("c2", 2), ("c2", 4), ("c5", 8)]


@pytest.mark.parametrize("name,n_rep", SPLIT_CASES, ids=[f"{c}-n{n}" for c, n in SPLIT_CASES])
def test_replicas_on_a_split_corpus_learn_like_one_replica(name, n_rep):
    """Strong split (the verdict's multi-GPU parity case): BASELINE config 1
    or 2 split N ways over N replicas, the replicas' deltas summed every SYNC_WORDS words per
    replica. The result must be within 2% of one replica's HS loss on the whole corpus and
    reach 95% of its loss reduction from the initial model. (Round 1's whole-model
    averaging reached 38% at N = 2.) The C5 case is the headline configuration's model (V 1M,
    D 300) on a 100M-token prefix split 8 ways: summing the deltas with only the
    update-count prior diverged there (loss 1e9); the norm-ratio rule holds it."""
    import bench
    from paper_1606_07822_b200.corpus_gen import CONFIGS

    c = CONFIGS[name]
    _, vocab, ids = bench.workload(name, 0, 1, device=name in ("c4", "c5"))
    ids = bench.host_ids(ids, PREFIX.get(name))
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, 31)
    cfg = api.TrainConfig(dim=c.dim, window=c.window, min_count=1, sample=c.sample, iterations=1, cache_nodes=31,
                          seed=c.seed, mode="hogwild")
    t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
    cen, ctx = O.sample_pairs(ids, vocab.counts, vocab.total_tokens(), c.sample, c.window, 20240917, 1 << 18)
    loss = lambda m: O.hs_loss(cen, ctx, m.syn0, m.syn1, t)  # noqa: E731
    li = loss(api.init_model(vocab.size(), c.dim, c.seed))
    ls = loss(api.train(ids, vocab, tree, sel, cfg))
    st = api.TrainStats()
    rep = api.train(ids, vocab, tree, sel, cfg, st, devices=[0] * n_rep, sync_words=SYNC_WORDS[name])
    assert st.words_processed == ids.size
    lr = loss(rep)
    assert abs(lr - ls) / ls < 0.02, (lr, ls, li)
    assert (li - lr) >= 0.95 * (li - ls), (lr, ls, li)
