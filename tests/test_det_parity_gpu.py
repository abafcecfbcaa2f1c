"""Deterministic mode (K2) vs the oracle, through the C-ABI: bit-identical syn0/syn1.

North-star gate: "in deterministic single-stream mode on a fixed pair order, the
updated matrices must match the reference to within 1e-5 relative (fp32)". The test
asserts the stronger property, bit equality, and reports the acceptance.cpp:251-263
relative metric alongside."""
import numpy as np
import pytest

import fixtures as F
import oracle_lib as O
from paper_1606_07822_b200 import api
from paper_1606_07822_b200.corpus_gen import CONFIGS, generate, vocab_from_raw

pytestmark = pytest.mark.gpu


def _gpu_det(ids, vocab, cfg):
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, cfg["cache_nodes"])
    tc = api.TrainConfig(dim=cfg["dim"], window=cfg["window"], min_count=cfg["min_count"], sample=cfg["sample"],
                         alpha0=cfg.get("alpha0", 0.025), iterations=cfg["iterations"], workers=1,
                         cache_nodes=cfg["cache_nodes"], flush_interval=cfg["flush_interval"], seed=cfg["seed"],
                         mode="deterministic")
    st = api.TrainStats()
    m = api.train(ids, vocab, tree, sel, tc, st)
    return m, st


FIXTURE_CASES = [
    (200 * 1024, 2000, 4242, dict(dim=100, window=5, min_count=5, sample=1e-3, alpha0=0.001, iterations=1,
                                  cache_nodes=31, flush_interval=10, seed=11)),
    (200 * 1024, 2000, 4242, dict(dim=100, window=5, min_count=5, sample=1e-3, alpha0=0.001, iterations=1,
                                  cache_nodes=0, flush_interval=10, seed=11)),
    (100 * 1024, 1000, 31337, dict(dim=64, window=5, min_count=5, sample=1e-3, iterations=2, cache_nodes=31,
                                   flush_interval=1, seed=7)),
    (30000, 120, 21, dict(dim=16, window=3, min_count=2, sample=1e-3, iterations=2, cache_nodes=15,
                          flush_interval=10, seed=7)),
    (60000, 300, 5, dict(dim=33, window=4, min_count=1, sample=0.0, iterations=2, cache_nodes=1024,
                         flush_interval=7, seed=3)),
    (40000, 50, 8, dict(dim=3, window=7, min_count=1, sample=1e-2, iterations=3, cache_nodes=49,
                        flush_interval=3, seed=99)),
]


@pytest.mark.parametrize("mb,types,seed,cfg", FIXTURE_CASES)
def test_det_fixture_bit_exact(tmp_path, mb, types, seed, cfg):
    path = F.write(tmp_path / "c.txt", F.make_zipf_corpus(mb, types, seed))
    vocab = api.build_vocabulary_file(path, cfg["min_count"])
    ids = api.read_id_stream(path, vocab)
    m, st = _gpu_det(ids, vocab, cfg)
    s0, s1, ost = O.orc_train(ids, vocab.counts, vocab.total_tokens(), cfg)
    assert st.words_processed == ost.words_processed
    assert st.pairs == ost.pairs and st.steps == ost.steps and st.centers == ost.centers
    assert O.max_relative_diff(m.syn0, s0) <= 1e-5 and O.max_relative_diff(m.syn1, s1) <= 1e-5
    assert np.array_equal(m.syn0.view(np.uint32), s0.view(np.uint32))
    assert np.array_equal(m.syn1.view(np.uint32), s1.view(np.uint32))
    if O.ref_available():  # and the reference itself, through its own train()
        h, *_ = O.ref_vocab_file(path, cfg["min_count"])
        r0, r1, words, _ = O.ref_train(h, path, cfg)
        O.ref().ref_close(h)
        assert np.array_equal(m.syn0.view(np.uint32), r0.view(np.uint32))
        assert np.array_equal(m.syn1.view(np.uint32), r1.view(np.uint32))


def test_det_c1_full_size_bit_exact():
    """BASELINE config 1 at full size (1M tokens, V 10k, D 100, W 5, 1e-3), K=31, u=10."""
    c = CONFIGS["c1"]
    vocab, ids = vocab_from_raw(generate(c), c.min_count, c.vocab)
    cfg = dict(dim=c.dim, window=c.window, min_count=c.min_count, sample=c.sample, iterations=1, cache_nodes=31,
               flush_interval=10, seed=c.seed)
    m, st = _gpu_det(ids, vocab, cfg)
    s0, s1, ost = O.orc_train(ids, vocab.counts, vocab.total_tokens(), cfg)
    assert st.pairs == ost.pairs
    assert np.array_equal(m.syn0.view(np.uint32), s0.view(np.uint32))
    assert np.array_equal(m.syn1.view(np.uint32), s1.view(np.uint32))


def test_det_is_reproducible_and_seed_sensitive(tmp_path):
    # trainer_test.cpp:362-400
    path = F.write(tmp_path / "c.txt", F.make_zipf_corpus(30000, 120, 21))
    vocab = api.build_vocabulary_file(path, 2)
    ids = api.read_id_stream(path, vocab)
    cfg = dict(dim=16, window=3, min_count=2, sample=1e-3, iterations=2, cache_nodes=15, flush_interval=10, seed=7)
    a, _ = _gpu_det(ids, vocab, cfg)
    b, _ = _gpu_det(ids, vocab, cfg)
    assert np.array_equal(a.syn0, b.syn0) and np.array_equal(a.syn1, b.syn1)
    c, _ = _gpu_det(ids, vocab, dict(cfg, seed=8))
    assert not np.array_equal(a.syn0, c.syn0)


def test_det_cache_transparency(tmp_path):
    # acceptance.cpp:265-307: K=31,u=10 vs K=0 < 1e-4; u=1 < 1e-6
    path = F.write(tmp_path / "c.txt", F.make_zipf_corpus(200 * 1024, 2000, 4242))
    vocab = api.build_vocabulary_file(path, 5)
    ids = api.read_id_stream(path, vocab)
    cfg = dict(dim=100, window=5, min_count=5, sample=1e-3, alpha0=0.001, iterations=1, seed=11)
    k0, _ = _gpu_det(ids, vocab, dict(cfg, cache_nodes=0, flush_interval=10))
    u10, _ = _gpu_det(ids, vocab, dict(cfg, cache_nodes=31, flush_interval=10))
    u1, _ = _gpu_det(ids, vocab, dict(cfg, cache_nodes=31, flush_interval=1))
    d10 = max(O.max_relative_diff(k0.syn0, u10.syn0), O.max_relative_diff(k0.syn1, u10.syn1))
    d1 = max(O.max_relative_diff(k0.syn0, u1.syn0), O.max_relative_diff(k0.syn1, u1.syn1))
    assert d10 < 1e-4 and d1 < 1e-6


def test_session_range_api_matches_one_shot(tmp_path):
    path = F.write(tmp_path / "c.txt", F.make_zipf_corpus(50000, 300, 4))
    vocab = api.build_vocabulary_file(path, 1)
    ids = api.read_id_stream(path, vocab)
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, 31)
    tc = api.TrainConfig(dim=24, window=4, min_count=1, iterations=2, seed=5, mode="deterministic")
    one = api.train(ids, vocab, tree, sel, tc)
    s = api.Session(vocab, tree, sel, tc)
    s.upload_ids(ids)
    for it in range(2):
        s.train_range(it, 0, ids.size, it * ids.size, 1)
    two = s.download()
    s.close()
    assert np.array_equal(one.syn0, two.syn0) and np.array_equal(one.syn1, two.syn1)
