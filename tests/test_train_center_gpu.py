"""Known-answer tests of the reference (trainer_test.cpp:35-293, acceptance.cpp:112-221),
run on the device kernel through the kernel-level C-ABI entry (cg_train_center /
cg_cache_flush)."""
import math

import numpy as np
import pytest

import oracle_lib as O
from paper_1606_07822_b200 import api

pytestmark = pytest.mark.gpu


def vocab_tree(counts):
    v = api.Vocabulary(counts)
    return v, api.build_huffman_tree(v)


def test_gradient_scales_with_alpha_at_neutral_sigmoid():
    vocab, tree = vocab_tree([2, 1])
    m = api.Model(2, 2)
    center = 0 if tree.path(0)[0][1] == 0 else 1
    ctx = 1 - center
    m.syn0[ctx] = [0.4, 0.2]
    sel = api.select_cached_nodes(tree, 0)
    cache = api.NodeCache(sel, 2, 10)
    calls = api.train_center(center, [ctx, center], 1, 1, m, tree, sel, cache, 0.025, "exact")
    assert calls == 1
    np.testing.assert_array_max_ulp(m.syn1[0], np.float32([0.0125 * 0.4, 0.0125 * 0.2]), 4)
    assert m.syn0[ctx].tolist() == np.float32([0.4, 0.2]).tolist()


def test_saturated_sigmoid_is_a_fixed_point():
    vocab, tree = vocab_tree([2, 1])
    m = api.init_model(2, 4, 9)
    rng = np.random.default_rng(17)
    m.syn1[:] = rng.uniform(-0.5, 0.5, m.syn1.shape).astype(np.float32)
    center = 0 if tree.path(0)[0][1] == 0 else 1
    before = m.copy()
    sel = api.select_cached_nodes(tree, 0)
    api.train_center(center, [1 - center, center], 1, 1, m, tree, sel, api.NodeCache(sel, 4, 10), 0.05, 1.0)
    assert np.array_equal(m.syn0, before.syn0) and np.array_equal(m.syn1, before.syn1)


def test_matches_hand_computed_single_step():
    vocab, tree = vocab_tree([3, 2])
    m = api.Model(2, 3)
    v = [0.3, -0.1, 0.2]
    u = [-0.4, 0.25, 0.05]
    m.syn0[1] = v
    m.syn1[0] = u
    turn = tree.path(0)[0][1]
    alpha = 0.1
    f = 1 / (1 + math.exp(-sum(a * b for a, b in zip(v, u))))
    g = (1 - turn - f) * alpha
    sel = api.select_cached_nodes(tree, 0)
    api.train_center(0, [1, 0], 1, 1, m, tree, sel, api.NodeCache(sel, 3, 10), alpha, "exact")
    np.testing.assert_allclose(m.syn1[0], [u[d] + g * v[d] for d in range(3)], atol=1e-6)
    np.testing.assert_allclose(m.syn0[1], [v[d] + g * u[d] for d in range(3)], atol=1e-6)


def test_hot_rows_bypass_shared_memory_until_flush():
    vocab, tree = vocab_tree([4, 3, 2, 1])
    m = api.init_model(4, 4, 2)
    sel = api.select_cached_nodes(tree, 1)
    cache = api.NodeCache(sel, 4, 1000)
    center = 3
    assert len(tree.path(center)) >= 2
    api.train_center(center, [0, center], 1, 1, m, tree, sel, cache, 0.05, "exact")
    root = tree.root_id()
    assert not m.syn1[root].any()
    assert cache.is_cached(0)
    assert any(m.syn1[n].any() for n, _ in tree.path(center) if n != root)
    cache.flush(m)
    assert m.syn1[root].any()
    assert not cache.is_cached(0)


def test_flush_adds_delta_on_top_of_concurrent_moves():
    vocab, tree = vocab_tree([2, 1])
    m = api.Model(2, 2)
    m.syn1[0] = [1.0, 1.0]
    sel = api.select_cached_nodes(tree, 1)
    cache = api.NodeCache(sel, 2, 10)
    w = cache.acquire(0, m.syn1[0])
    w[:] = [1.5, 0.5]
    m.syn1[0] = [1.1, 1.0]
    cache.flush(m)
    np.testing.assert_array_max_ulp(m.syn1[0], np.float32([1.6, 0.5]), 4)


def test_interleaved_flushes_compose():
    vocab, tree = vocab_tree([2, 1])
    m = api.Model(2, 2)
    m.syn1[0] = [0.5, -0.25]
    sel = api.select_cached_nodes(tree, 1)
    a, b = api.NodeCache(sel, 2, 10), api.NodeCache(sel, 2, 10)
    ra, rb = a.acquire(0, m.syn1[0]), b.acquire(0, m.syn1[0])
    ra += [0.125, 0.25]
    rb += [0.125, 0.25]
    a.flush(m)
    assert m.syn1[0].tolist() == [0.625, 0.0]
    b.flush(m)
    assert m.syn1[0].tolist() == [0.75, 0.25]


def test_full_window_trains_at_most_ten_pairs():
    vocab, tree = vocab_tree([2, 1])
    m = api.init_model(2, 4, 1)
    sel = api.select_cached_nodes(tree, 0)
    cache = api.NodeCache(sel, 4, 10)
    sentence = [i % 2 for i in range(11)]
    assert api.train_center(sentence[5], sentence, 5, 5, m, tree, sel, cache, 0.025, 0.5) == 10
    assert api.train_center(sentence[0], sentence, 0, 5, m, tree, sel, cache, 0.025, 0.5) == 5


def test_gradient_oracle_finite_differences():
    """acceptance.cpp:112-221: 50 random instances, uncached and fully cached routes."""
    rng = np.random.default_rng(20260808)
    worst = 0.0
    for _ in range(50):
        v = int(rng.integers(2, 17))
        dim = int(rng.integers(2, 9))
        counts = sorted((1 + rng.integers(0, 10, v)).tolist(), reverse=True)
        vocab, tree = vocab_tree(counts)
        ref = api.Model(v, dim)
        mag = lambda shape: (rng.uniform(0.1, 0.5, shape) * rng.choice([-1, 1], shape)).astype(np.float32)
        ref.syn0[:] = mag(ref.syn0.shape)
        ref.syn1[:] = mag(ref.syn1.shape)
        center, ctx = int(rng.integers(0, v)), int(rng.integers(0, v))
        path = tree.path(center)
        alpha, h = 0.05, 1e-4

        def ll(cv, rows):
            tot = 0.0
            for (n, t), r in zip(path, rows):
                f = 1 / (1 + math.exp(-float(np.dot(cv, r))))
                tot += math.log(f) if t == 0 else math.log(1 - f)
            return tot

        cv = ref.syn0[ctx].astype(np.float64)
        rows = [ref.syn1[n].astype(np.float64) for n, _ in path]
        exp_ctx = np.array([alpha * (ll(cv + h * e, rows) - ll(cv - h * e, rows)) / (2 * h) for e in np.eye(dim)])
        exp_rows = []
        for i in range(len(rows)):
            g = []
            for e in np.eye(dim):
                up = [r + (h * e if j == i else 0) for j, r in enumerate(rows)]
                dn = [r - (h * e if j == i else 0) for j, r in enumerate(rows)]
                g.append(alpha * (ll(cv, up) - ll(cv, dn)) / (2 * h))
            exp_rows.append(np.array(g))
        for k in (0, v - 1):
            m = ref.copy()
            sel = api.select_cached_nodes(tree, k)
            cache = api.NodeCache(sel, dim, 1000)
            api.train_center(center, [ctx, center], 1, 1, m, tree, sel, cache, alpha, "exact")
            cache.flush(m)
            err = lambda a, b, e: np.linalg.norm((a.astype(np.float64) - b) - e) / max(np.linalg.norm(e), 1e-6)
            worst = max(worst, err(m.syn0[ctx], ref.syn0[ctx], exp_ctx))
            for (n, _), e in zip(path, exp_rows):
                worst = max(worst, err(m.syn1[n], ref.syn1[n], e))
            others = [w for w in range(v) if w != ctx]
            assert np.array_equal(m.syn0[others], ref.syn0[others])
    assert worst < 1e-3


def test_train_center_matches_oracle_bitwise():
    rng = np.random.default_rng(5)
    for _ in range(25):
        v = int(rng.integers(2, 40))
        dim = int(rng.integers(1, 70))
        counts = np.sort(rng.integers(1, 30, v))[::-1].copy()
        vocab, tree = vocab_tree(counts)
        m = api.Model(v, dim)
        m.syn0[:] = rng.uniform(-1, 1, m.syn0.shape).astype(np.float32)
        m.syn1[:] = rng.uniform(-1, 1, m.syn1.shape).astype(np.float32)
        sent = rng.integers(0, v, int(rng.integers(1, 15))).tolist()
        pos = int(rng.integers(0, len(sent)))
        hw = int(rng.integers(1, 6))
        k = int(rng.integers(0, v))
        sel = api.select_cached_nodes(tree, k)
        o0, o1 = m.syn0.copy(), m.syn1.copy()
        cache = api.NodeCache(sel, dim, 10)
        calls = api.train_center(sent[pos], sent, pos, hw, m, tree, sel, cache, 0.05, "table")
        cache.flush(m)
        t = O.orc_tree(counts)
        hot, slot = O.orc_select(t.usage, k)
        import ctypes as C
        kk = max(hot.size, 1)
        work = np.zeros((kk, dim), np.float32)
        snap = np.zeros((kk, dim), np.float32)
        flag = np.zeros(kk, np.uint8)
        acq = np.zeros(kk, np.int32)
        na = C.c_int32(0)
        s = np.array(sent, np.int32)
        e = O.oracle().orc_train_center(sent[pos], O._p(s, C.c_int32), s.size, pos, hw, dim, O._p(o0, C.c_float),
                                        O._p(o1, C.c_float), O._p(t.off, C.c_int64), O._p(t.nodes, C.c_int32),
                                        O._p(t.turns, C.c_uint8), O._p(slot, C.c_int32) if k else None,
                                        O._p(work, C.c_float), O._p(snap, C.c_float), O._p(flag, C.c_uint8),
                                        O._p(acq, C.c_int32), C.byref(na), 0.05, 0, 0.0)
        O.oracle().orc_cache_flush(dim, O._p(o1, C.c_float), O._p(hot, C.c_int32), O._p(work, C.c_float),
                                   O._p(snap, C.c_float), O._p(flag, C.c_uint8), O._p(acq, C.c_int32), C.byref(na))
        assert calls == e
        assert np.array_equal(m.syn0.view(np.uint32), o0.view(np.uint32))
        assert np.array_equal(m.syn1.view(np.uint32), o1.view(np.uint32))
