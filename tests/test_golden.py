"""Golden vectors produced by the reference itself (tests/golden/make_golden.py):
the oracle restatement (CPU) and the device kernels (GPU) must reproduce them bit
for bit. These tests never read /root/reference."""
import ast
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import fixtures as F
import oracle_lib as O
from paper_1606_07822_b200 import api

GOLD = Path(__file__).resolve().parent / "golden"
CASES = sorted(p.stem for p in GOLD.glob("g*.npz"))


def load(name):
    z = np.load(GOLD / f"{name}.npz")
    cfg = ast.literal_eval(str(z["cfg"]))
    mb, types, seed = (int(x) for x in z["corpus"])
    text = F.make_zipf_corpus(mb, types, seed)
    rank = {f"w{int(r)}": i for i, r in enumerate(z["raws"])}
    ids = np.array([rank[t] for t in text.split() if t in rank], np.int32)
    return z, cfg, ids


@pytest.mark.parametrize("name", CASES)
def test_golden_host_pieces(name):
    z, cfg, ids = load(name)
    assert ids.size * cfg["iterations"] == int(z["words"])
    tree = api.build_huffman_tree(z["counts"])
    assert np.array_equal(tree.offsets, z["off"]) and np.array_equal(tree.nodes, z["nodes"])
    assert np.array_equal(tree.turns, z["turns"]) and np.array_equal(tree.usage, z["usage"])
    sel = api.select_cached_nodes(tree, cfg["cache_nodes"])
    assert np.array_equal(sel.hot, z["hot"]) and np.array_equal(sel.slot, z["slot"])


@pytest.mark.parametrize("name", CASES)
def test_golden_oracle_bit_exact(name):
    z, cfg, ids = load(name)
    s0, s1, st = O.orc_train(ids, z["counts"], int(z["total"]), cfg)
    assert st.words_processed == int(z["words"])
    assert np.array_equal(s0.view(np.uint32), z["syn0"].view(np.uint32))
    assert np.array_equal(s1.view(np.uint32), z["syn1"].view(np.uint32))


def test_golden_scalars():
    z = np.load(GOLD / "scalars.npz")
    orc = O.oracle()
    t = np.zeros(1000, np.float32)
    orc.orc_sigmoid_table(O._p(t, C.c_float))
    assert np.array_equal(api.sigmoid_table(), t)
    scale = np.float32(1000) / np.float32(12)
    mine = []
    for x in z["sig_x"]:
        x = np.float32(x)
        mine.append(t[0] if x <= -6 else t[999] if x >= 6 else t[min(int(np.float32(np.float32(x + 6) * scale)), 999)])
    assert np.array_equal(np.array(mine, np.float32), z["sig"])
    s = C.c_uint64(1)
    assert [orc.orc_splitmix_next(C.byref(s)) for _ in range(64)] == [int(x) for x in z["rng_u64"]]
    for (c, tt, smp), k in zip(z["keep_args"], z["keep"]):
        assert api.keep_probability(int(c), int(tt), float(smp)) == k
    for d, a in zip(z["alpha_done"], z["alpha"]):
        assert np.float32(api.update_alpha(int(d), 1000000, 0.025)) == a
    m = api.init_model(13, 9, 42)
    assert np.array_equal(m.syn0.view(np.uint32), z["init_syn0"].view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_golden_device_deterministic_bit_exact(name):
    z, cfg, ids = load(name)
    vocab = api.Vocabulary(z["counts"], total=int(z["total"]))
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, cfg["cache_nodes"])
    tc = api.TrainConfig(**{k: v for k, v in cfg.items()}, workers=1, mode="deterministic")
    st = api.TrainStats()
    m = api.train(ids, vocab, tree, sel, tc, st)
    assert st.words_processed == int(z["words"])
    assert np.array_equal(m.syn0.view(np.uint32), z["syn0"].view(np.uint32))
    assert np.array_equal(m.syn1.view(np.uint32), z["syn1"].view(np.uint32))
