"""Device evaluation kernels (cg_eval.cu) through the C-ABI, against the reference's
AnalogySolver answers (golden vectors) and the pinned C oracle: the normalised table
and every analogy / top-k answer must be bit-identical."""
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
from paper_1606_07822_b200 import api

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden" / "eval_analogy.npz"


def _bits(a):
    """Bit patterns with every NaN canonicalised (x86 and the GPU use different NaN payloads)."""
    a = np.ascontiguousarray(a, dtype=np.float32).copy()
    b = a.view(np.uint32)
    b[np.isnan(a)] = 0x7FC00000
    return b


@pytest.mark.parametrize("rows,dim", [(1, 1), (5, 3), (300, 7), (1000, 100), (129, 300), (4000, 17)])
def test_normalized_table_bit_exact(rows, dim):
    v, _ = O.eval_case(rows + dim, rows, dim, 0, dup=3, zero=2, nan=2)
    e = api.Embeddings(v)
    assert np.array_equal(_bits(e.normalized()), _bits(O.orc_normalize(v)))


def test_analogy_matches_reference_golden():
    g = np.load(GOLDEN)
    for i in range(int(g["n_cases"])):
        v, abc, top, want = g[f"v{i}"], g[f"abc{i}"], int(g[f"top{i}"]), g[f"ans{i}"]
        size = min(v.shape[0], top) if top > 0 else v.shape[0]
        got = api.Embeddings(v[:size]).analogy(abc)
        assert np.array_equal(got, want), i


@pytest.mark.parametrize("seed,rows,dim,nq", [(21, 3000, 300, 400), (22, 777, 33, 1000), (23, 130, 128, 64),
                                              (24, 5, 2, 20)])
def test_analogy_matches_oracle(seed, rows, dim, nq):
    v, abc = O.eval_case(seed, rows, dim, nq, dup=rows // 20, zero=3, nan=2)
    abc %= rows
    got = api.Embeddings(v).analogy(abc)
    assert np.array_equal(got, O.orc_analogy(O.orc_normalize(v), abc))


def test_analogy_exact_ties_and_exhaustion():
    e = api.Embeddings(np.eye(6, dtype=np.float32))
    assert list(e.analogy(np.array([[0, 0, 0], [3, 4, 5], [1, 2, 3]]))) == [1, 0, 0]
    three = api.Embeddings(np.eye(3, dtype=np.float32))
    assert three.analogy(np.array([[0, 1, 2]]))[0] == -1  # nothing left
    with pytest.raises(ValueError):
        three.analogy(np.array([[0, 1, 3]]))


@pytest.mark.parametrize("rows,dim,k", [(2000, 100, 10), (700, 300, 32), (64, 8, 1), (5, 4, 10), (1300, 128, 10)])
def test_topk_matches_oracle(rows, dim, k):
    v, _ = O.eval_case(rows * 3 + k, rows, dim, 0, dup=rows // 10, zero=2, nan=1)
    n = O.orc_normalize(v)
    q = np.arange(0, rows, max(1, rows // 300), dtype=np.int32)
    ids, sc = api.Embeddings(v).nearest(q, k)
    wid, wsc = O.orc_topk(n, q, k)
    assert np.array_equal(ids, wid)
    both_nan = np.isnan(sc) & np.isnan(wsc)
    assert np.array_equal(sc[~both_nan], wsc[~both_nan])


def test_evaluate_report_and_restrict_top(tmp_path):
    rng = np.random.default_rng(4)
    words = [f"w{i}" for i in range(60)]
    vec = (rng.random((60, 8), dtype=np.float32) - 0.5)
    emb = api.LoadedEmbeddings(8, words, vec)
    qs = tmp_path / "q.txt"
    lines = [": first"] + [" ".join(words[j] for j in rng.integers(0, 60, 4)) for _ in range(40)]
    lines += [": second", "w1 W2 w3 w59", "w0 w1 unknown w2"]
    qs.write_text("\n".join(lines) + "\n")
    qset = api.load_questions(str(qs))
    assert qset.sections == ["first", "second"] and qset.questions[40].b == "w2"
    for top in (0, 30):
        rep = api.evaluate(emb, qset, top)
        size = 60 if top == 0 else 30
        norm = O.orc_normalize(vec[:size])
        att = cor = skip = 0
        for q in qset.questions:
            ids = [words.index(x) if x in words[:size] else -1 for x in (q.a, q.b, q.c, q.d)]
            if min(ids) < 0:
                skip += 1
                continue
            att += 1
            cor += int(O.orc_analogy(norm, np.array([ids[:3]]))[0] == ids[3])
        assert (rep.total.attempted, rep.total.correct, rep.total.skipped) == (att, cor, skip)


def test_embeddings_from_session_device_buffer():
    """Zero-copy table over a training session's syn0 (no host round trip)."""
    raw = np.random.default_rng(1).zipf(1.3, 60000) % 200
    counts = np.bincount(raw, minlength=200)
    order = np.argsort(-counts, kind="stable")
    remap = np.empty(200, np.int64)
    remap[order] = np.arange(200)
    ids = remap[raw].astype(np.int32)
    vocab = api.Vocabulary(counts[order].astype(np.int64))
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, 31)
    cfg = api.TrainConfig(dim=20, window=3, min_count=1, sample=0.0, iterations=1, cache_nodes=31, seed=3,
                          mode="hogwild")
    s = api.Session(vocab, tree, sel, cfg)
    s.upload_ids(ids)
    s.train()
    m = s.download()
    p, _, stride = s.model_buffer()
    dev = api.Embeddings(rows=200, dim=20, device_ptr=p, row_stride=stride)
    host = api.Embeddings(m.syn0)
    assert np.array_equal(_bits(dev.normalized()), _bits(host.normalized()))
