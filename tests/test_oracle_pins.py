"""Pins the C restatement (oracle/cg_oracle.c) to the reference compiled unchanged
(oracle/_ref/libcgref.so): every function bit for bit, and whole single-worker
training runs byte-identical. CPU only."""
import ctypes as C
import os

import numpy as np
import pytest

import fixtures as F
import oracle_lib as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


def test_rng_streams_and_mix_seed():
    orc, ref = O.oracle(), O.ref()
    for seed in (0, 1, 7, 0xDEADBEEF, (1 << 64) - 1):
        n = 257
        u = np.zeros(n, np.uint64)
        f = np.zeros(n, np.float32)
        b = np.zeros(n, np.uint32)
        ref.ref_rng_stream(seed, n, O._p(u, C.c_uint64), O._p(f, C.c_float), 7, O._p(b, C.c_uint32))
        s = C.c_uint64(seed)
        mine = np.array([orc.orc_splitmix_next(C.byref(s)) for _ in range(n)], np.uint64)
        assert np.array_equal(mine, u)
        assert np.array_equal((u >> np.uint64(40)).astype(np.float32) * np.float32(1 / 16777216), f)
        assert np.array_equal((u % np.uint64(7)).astype(np.uint32), b)
        for stream in (0, 1, 3, 0x1817):
            assert orc.orc_mix_seed(seed, stream) == ref.ref_mix_seed(seed, stream)


def test_keep_probability_and_alpha():
    orc, ref = O.oracle(), O.ref()
    # corpus_test.cpp:120-129 known answers
    assert abs(orc.orc_keep_probability(10, 1000, 0.001) - 0.4162277660) < 1e-9
    assert orc.orc_keep_probability(1, 1000, 0.001) == 1.0
    assert orc.orc_keep_probability(5, 10000, 0.01) == 1.0
    rng = np.random.default_rng(0)
    for c, t, s in zip(rng.integers(1, 10**7, 300), rng.integers(10**6, 10**9, 300), rng.choice([1e-3, 1e-4, 1e-5], 300)):
        assert orc.orc_keep_probability(int(c), int(t), float(s)) == ref.ref_keep_probability(int(c), int(t), float(s))
    for done in (0, 1, 9999, 10000, 500000, 999999, 1000000, 2000000):
        assert orc.orc_update_alpha(done, 1000000, 0.025) == ref.ref_update_alpha(done, 1000000, 0.025)
    # trainer_test.cpp:299-307
    assert orc.orc_update_alpha(1000000, 1000000, 0.025) == np.float32(0.025) * np.float32(1e-4)


def test_sigmoid_table_bits():
    t = np.zeros(1000, np.float32)
    O.oracle().orc_sigmoid_table(O._p(t, C.c_float))
    ref = O.ref()
    # bucket centres, edges, clamps and a dense sweep through ref's value()
    xs = np.concatenate([np.linspace(-7, 7, 20001, dtype=np.float32), np.float32([-6, 6, -5.994, 5.994, 0])])
    scale = np.float32(1000) / np.float32(12.0)
    for x in xs:
        x = np.float32(x)
        if x <= -6:
            mine = t[0]
        elif x >= 6:
            mine = t[999]
        else:
            mine = t[min(int(np.float32(np.float32(x + np.float32(6)) * scale)), 999)]
        assert mine == np.float32(ref.ref_sigmoid_value(float(x))), x


def test_init_model_bits():
    for v, d, seed in ((10, 16, 1), (40, 25, 3), (12, 8, 42), (7, 300, 5)):
        a0, a1 = O.orc_init(v, d, seed)
        b0 = np.zeros((v, d), np.float32)
        b1 = np.zeros((v - 1, d), np.float32)
        O.ref().ref_init_model(v, d, seed, O._p(b0, C.c_float), O._p(b1, C.c_float))
        assert np.array_equal(a0.view(np.uint32), b0.view(np.uint32))
        assert not b1.any() and not a1.any()
        assert (np.abs(a0) < 0.5 / d).all()


def test_huffman_trees_and_selection():
    rng = np.random.default_rng(1)
    cases = [[4, 2, 1, 1], [1, 1], [9, 7, 5, 3, 2, 1, 1], [3, 3, 2, 2, 2, 1], [13, 8, 8, 5, 5, 3, 2, 2, 1, 1]]
    cases += [sorted(rng.integers(1, 50, rng.integers(2, 40)).tolist(), reverse=True) for _ in range(40)]
    cases += [rng.integers(1, 9, 300).tolist()]  # unsorted, many ties
    for counts in cases:
        counts = np.array(counts, np.int64)
        h = O.ref().ref_open_counts(O._p(counts, C.c_int64), counts.size)
        rt, ot = O.ref_tree(h), O.orc_tree(counts)
        for a, b in ((rt.off, ot.off), (rt.nodes, ot.nodes), (rt.turns, ot.turns), (rt.usage, ot.usage)):
            assert np.array_equal(a, b)
        for k in (0, 1, 3, 31, 1000):
            inner = counts.size - 1
            hot_r = np.zeros(max(inner, 1), np.int32)
            slot_r = np.zeros(inner, np.int32)
            n = O.ref().ref_select(h, k, O._p(hot_r, C.c_int32), O._p(slot_r, C.c_int32))
            hot_o, slot_o = O.orc_select(ot.usage, k)
            assert np.array_equal(hot_r[:n], hot_o) and np.array_equal(slot_r, slot_o)
        O.ref().ref_close(h)
    # huffman_test.cpp:46-57: counts 4,2,1,1 -> depths 1,2,3,3
    t = O.orc_tree(np.array([4, 2, 1, 1], np.int64))
    assert np.diff(t.off).tolist() == [1, 2, 3, 3]
    assert t.usage[0] == 2


CASES = [
    # (bytes, types, seed, config) -- acceptance.cpp:265-307 / 544-571, trainer_test.cpp:484-496 fixtures
    (200 * 1024, 2000, 4242, dict(dim=100, window=5, min_count=5, sample=1e-3, alpha0=0.001, iterations=1,
                                  cache_nodes=31, flush_interval=10, seed=11)),
    (200 * 1024, 2000, 4242, dict(dim=100, window=5, min_count=5, sample=1e-3, alpha0=0.001, iterations=1,
                                  cache_nodes=31, flush_interval=1, seed=11)),
    (100 * 1024, 1000, 31337, dict(dim=64, window=5, min_count=5, sample=1e-3, iterations=2, cache_nodes=0,
                                   flush_interval=10, seed=7)),
    (30000, 120, 21, dict(dim=16, window=3, min_count=2, sample=1e-3, iterations=2, cache_nodes=15,
                          flush_interval=10, seed=7)),
    (60000, 300, 5, dict(dim=33, window=4, min_count=1, sample=0.0, iterations=2, cache_nodes=1024,
                         flush_interval=7, seed=3)),
]


@pytest.mark.parametrize("mb,types,seed,cfg", CASES)
def test_train_single_worker_bit_exact(tmp_path, mb, types, seed, cfg):
    path = F.write(tmp_path / "c.txt", F.make_zipf_corpus(mb, types, seed))
    h, counts, raws, total = O.ref_vocab_file(path, cfg["min_count"])
    s0r, s1r, words, _ = O.ref_train(h, path, cfg)
    rank = {f"w{r}": i for i, r in enumerate(raws)}
    ids = np.array([rank[t] for t in open(path).read().split() if t in rank], np.int32)
    s0o, s1o, st = O.orc_train(ids, counts, total, cfg)
    assert st.words_processed == words == cfg["iterations"] * total
    assert np.array_equal(s0r.view(np.uint32), s0o.view(np.uint32))
    assert np.array_equal(s1r.view(np.uint32), s1o.view(np.uint32))
    O.ref().ref_close(h)


def _center_case(counts, dim, syn0, syn1, k, sentence, pos, hw, alpha, mode, const=0.5):
    counts = np.array(counts, np.int64)
    a0, a1 = syn0.copy(), syn1.copy()
    e_ref = O.ref().ref_train_center(O._p(counts, C.c_int64), counts.size, dim, O._p(a0, C.c_float),
                                     O._p(a1, C.c_float), k, 1, sentence[pos], O._p(np.array(sentence, np.int32),
                                                                                    C.c_int32),
                                     len(sentence), pos, hw, alpha, mode, const)
    t = O.orc_tree(counts)
    hot, slot = O.orc_select(t.usage, k)
    b0, b1 = syn0.copy(), syn1.copy()
    kk = max(hot.size, 1)
    work = np.zeros((kk, dim), np.float32)
    snap = np.zeros((kk, dim), np.float32)
    flag = np.zeros(kk, np.uint8)
    acq = np.zeros(kk, np.int32)
    nacq = C.c_int32(0)
    sent = np.array(sentence, np.int32)
    e_orc = O.oracle().orc_train_center(sentence[pos], O._p(sent, C.c_int32), sent.size, pos, hw, dim,
                                        O._p(b0, C.c_float), O._p(b1, C.c_float), O._p(t.off, C.c_int64),
                                        O._p(t.nodes, C.c_int32), O._p(t.turns, C.c_uint8),
                                        O._p(slot, C.c_int32) if k else None, O._p(work, C.c_float),
                                        O._p(snap, C.c_float), O._p(flag, C.c_uint8), O._p(acq, C.c_int32),
                                        C.byref(nacq), alpha, mode, const)
    O.oracle().orc_cache_flush(dim, O._p(b1, C.c_float), O._p(hot, C.c_int32), O._p(work, C.c_float),
                               O._p(snap, C.c_float), O._p(flag, C.c_uint8), O._p(acq, C.c_int32), C.byref(nacq))
    return (a0, a1, e_ref), (b0, b1, e_orc)


def test_train_center_matches_reference():
    rng = np.random.default_rng(2)
    for inst in range(60):
        v = int(rng.integers(2, 17))
        dim = int(rng.integers(2, 9))
        counts = sorted(rng.integers(1, 11, v).tolist(), reverse=True)
        syn0 = rng.uniform(-0.5, 0.5, (v, dim)).astype(np.float32)
        syn1 = rng.uniform(-0.5, 0.5, (v - 1, dim)).astype(np.float32)
        sentence = rng.integers(0, v, int(rng.integers(1, 12))).tolist()
        pos = int(rng.integers(0, len(sentence)))
        for k in (0, v - 1):
            for mode in (0, 1):
                (a0, a1, ea), (b0, b1, eb) = _center_case(counts, dim, syn0, syn1, k, sentence, pos,
                                                          int(rng.integers(1, 6)), 0.05, mode)
                assert ea == eb
                assert np.array_equal(a0, b0) and np.array_equal(a1, b1)


def test_known_answer_neutral_sigmoid():
    # trainer_test.cpp:35-59: zero node row, f = 0.5, turn 0 -> g = 0.0125
    counts = [2, 1]
    t = O.orc_tree(np.array(counts, np.int64))
    center = 0 if t.turns[t.off[0]] == 0 else 1
    ctx = 1 - center
    syn0 = np.zeros((2, 2), np.float32)
    syn0[ctx] = [0.4, 0.2]
    syn1 = np.zeros((1, 2), np.float32)
    sentence = [ctx, center]
    (_, _, _), (b0, b1, e) = _center_case(counts, 2, syn0, syn1, 0, sentence, 1, 1, 0.025, 1)
    assert e == 1
    np.testing.assert_allclose(b1[0], [0.0125 * 0.4, 0.0125 * 0.2], rtol=4e-7)
    assert np.array_equal(b0[ctx], np.float32([0.4, 0.2]))
