"""CPU checks of the C-ABI library: it loads, exports every entry point declared in
include/cachegram_b200.h, and its host pieces (reference algorithms computed once on
the host before upload) agree with the oracle. No GPU compute is called here except
to verify that the training entry points refuse to run without a device."""
import ctypes as C
import re

import numpy as np
import pytest

import fixtures as F
import oracle_lib as O
from paper_1606_07822_b200 import _lib, api
from paper_1606_07822_b200.corpus_gen import vocab_from_raw, zipf_raw_ids


def _has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False

HEADER = O.ROOT / "include" / "cachegram_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(cg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.exported_symbols())
    assert lib.cg_abi_version() == 3


def test_host_helpers_match_oracle():
    orc = O.oracle()
    for c, t, s in ((10, 1000, 1e-3), (1, 1000, 1e-3), (123456, 17_000_000, 1e-4)):
        assert api.keep_probability(c, t, s) == orc.orc_keep_probability(c, t, s)
    for d in (0, 10000, 123457, 999999):
        assert api.update_alpha(d, 10**6, 0.025) == orc.orc_update_alpha(d, 10**6, 0.025)
    t = np.zeros(1000, np.float32)
    orc.orc_sigmoid_table(O._p(t, C.c_float))
    assert np.array_equal(api.sigmoid_table(), t)
    m = api.init_model(57, 33, 9)
    s0, _ = O.orc_init(57, 33, 9)
    assert np.array_equal(m.syn0.view(np.uint32), s0.view(np.uint32))


def test_huffman_and_selection_match_oracle():
    rng = np.random.default_rng(3)
    for _ in range(30):
        counts = rng.integers(1, 40, int(rng.integers(2, 300)))
        if rng.random() < 0.5:
            counts = np.sort(counts)[::-1].copy()
        tree = api.build_huffman_tree(counts)
        ot = O.orc_tree(counts)
        assert np.array_equal(tree.offsets, ot.off) and np.array_equal(tree.nodes, ot.nodes)
        assert np.array_equal(tree.turns, ot.turns) and np.array_equal(tree.usage, ot.usage)
        for k in (0, 1, 31, 10**6):
            sel = api.select_cached_nodes(tree, k)
            hot, slot = O.orc_select(ot.usage, k)
            assert np.array_equal(sel.hot, hot) and np.array_equal(sel.slot, slot)
            # hot nodes form a prefix of every path (the device relies on it)
            is_hot = np.zeros(tree.inner_count(), bool)
            is_hot[sel.hot] = True
            for w in range(0, len(counts), 7):
                flags = is_hot[tree.nodes[tree.offsets[w]:tree.offsets[w + 1]]]
                assert not np.any(~flags[:-1] & flags[1:])
    with pytest.raises(ValueError):
        api.build_huffman_tree([5])
    with pytest.raises(ValueError):
        api.select_cached_nodes(api.build_huffman_tree([2, 1]), -1)


def test_corpus_vocab_and_id_stream(tmp_path):
    text = F.make_zipf_corpus(60_000, 400, 77) + "\n\tw3  w9\r\nunseen"
    path = F.write(tmp_path / "c.txt", text)
    v = api.build_vocabulary_file(path, 2)
    if O.ref_available():
        h, counts, raws, total = O.ref_vocab_file(path, 2)
        assert np.array_equal(v.counts, counts) and v.total_tokens() == total
        assert [w for w in v.words] == [f"w{r}" for r in raws]
        O.ref().ref_close(h)
    ids = api.read_id_stream(path, v)
    expect = [v.id_of(t) for t in text.split() if v.id_of(t) >= 0]
    assert ids.tolist() == expect
    with pytest.raises(OSError):
        api.build_vocabulary_file(str(tmp_path / "missing.txt"), 1)


def test_vocab_from_raw_matches_oracle_rules():
    raw = zipf_raw_ids(50_000, 3000, 1.0, 9)
    vocab, ids = vocab_from_raw(raw, 3, 3000)
    rank, counts, total = O.orc_vocab(raw, 3, 3000)
    assert np.array_equal(vocab.counts, counts) and vocab.total_tokens() == total
    r = rank[raw]
    assert np.array_equal(ids, r[r >= 0])


def test_config_validation_messages():
    base = api.TrainConfig()
    base.validate()
    for field, bad, msg in (("dim", 0, "dim must be >= 1"), ("workers", 0, "workers must be >= 1"),
                            ("flush_interval", 0, "flush-interval must be >= 1"),
                            ("cache_nodes", -1, "cache-nodes must be >= 0"), ("sample", -1.0, "sample must be >= 0")):
        c = api.TrainConfig(**{field: bad})
        with pytest.raises(ValueError, match=msg):
            c.validate()


def test_training_refuses_without_device_or_bad_args():
    """The C-ABI validates first (same messages as trainer.hpp:37-47, 256-260) and
    then needs a CUDA device: without one it reports CG_ERR_CUDA, never a CPU path."""
    lib = _lib.load()
    counts = np.array([5, 3, 2, 1], np.int64)
    tree = api.build_huffman_tree(counts)
    sel = api.select_cached_nodes(tree, 1)
    keep = []
    desc = api.model_desc(api.Vocabulary(counts), tree, sel, keep)
    cfg = api.TrainConfig(dim=4, workers=0).to_c()
    s = C.c_void_p()
    assert lib.cg_session_create(C.byref(cfg), 0, C.byref(desc), 0, None, C.byref(s)) == _lib.CG_ERR_INVALID_ARGUMENT
    assert b"workers must be >= 1" in lib.cg_last_error()
    cfg = api.TrainConfig(dim=4).to_c()
    rc = lib.cg_session_create(C.byref(cfg), 0, C.byref(desc), 0, None, C.byref(s))
    if lib.cg_device_count() == 0:
        assert rc == _lib.CG_ERR_CUDA and b"no CUDA device" in lib.cg_last_error()
    else:
        assert rc == 0
        lib.cg_session_destroy(s)


@pytest.mark.skipif(_has_cuda(), reason="checks the behaviour without a device")
def test_gpu_entry_points_fail_loudly_without_a_device(tmp_path):
    """No CPU fallback: every device entry point reports CG_ERR_CUDA on a host without a
    GPU (argument errors are still reported first where they are checked first)."""
    lib = _lib.load()
    v = np.ones((4, 3), np.float32)
    h = C.c_void_p()
    assert lib.cg_embeddings_create(_lib.ptr(v, C.c_float), 4, 3, -1, C.byref(h)) == _lib.CG_ERR_CUDA
    p = F.write(tmp_path / "c.txt", "a b a c")
    assert lib.cg_corpus_open_gpu(str(p).encode(), 1, 0, C.byref(h)) == _lib.CG_ERR_CUDA
    dev = np.zeros(2, np.int32)
    st = _lib.CgTrainStats()
    cfg = api.TrainConfig(dim=4, window=2, min_count=1, iterations=1).to_c()
    counts = np.array([3, 2, 1], np.int64)
    tree = api.build_huffman_tree(counts)
    sel = api.select_cached_nodes(tree, 1)
    keep: list = []
    desc = api.model_desc(api.Vocabulary(counts), tree, sel, keep)
    ids = np.array([0, 1, 2, 0], np.int32)
    out0 = np.zeros((3, 4), np.float32)
    out1 = np.zeros((2, 4), np.float32)
    args = (C.byref(cfg), 1, C.byref(desc), _lib.ptr(ids, C.c_int32), 4, _lib.ptr(dev, C.c_int32), 2, 100,
            _lib.ptr(out0, C.c_float), _lib.ptr(out1, C.c_float), C.byref(st))
    assert lib.cg_train_replicas(*args) == _lib.CG_ERR_INVALID_ARGUMENT  # deterministic replicas
    args = (C.byref(cfg), 0) + args[2:]
    assert lib.cg_train_replicas(*args) == _lib.CG_ERR_CUDA
    assert lib.cg_train(C.byref(cfg), 0, C.byref(desc), _lib.ptr(ids, C.c_int32), 4, _lib.ptr(out0, C.c_float),
                        _lib.ptr(out1, C.c_float), C.byref(st)) == _lib.CG_ERR_CUDA
