"""GPU corpus ingest (cg_ingest.cu) against the host implementation of the drop-in
(build_vocabulary_file / read_id_stream, itself pinned to the reference by the
reference's own corpus suite): the vocabulary (words, counts, order, total) and the
in-vocabulary id stream must be identical, including separators of every kind, ties,
OOV tokens, min_count filtering and multi-chunk files; train(corpus_path) -- which now
tokenises on the GPU -- must stay bit-identical to the reference in deterministic mode."""
from pathlib import Path

import numpy as np
import pytest

import fixtures as F
import oracle_lib as O
from paper_1606_07822_b200 import _lib, api

pytestmark = pytest.mark.gpu


def _vocab_pair(path, min_count):
    host = api.build_vocabulary_file(str(path), min_count)
    gpu = api.build_vocabulary_file(str(path), min_count, device=0)
    return host, gpu


def _same_vocab(a, b):
    assert a.words == b.words
    assert np.array_equal(a.counts, b.counts)
    assert a.total_tokens() == b.total_tokens()


def _raw_corpus(seed, n_tokens, types, seps=(" ", "\n", "\t", "\r\n", "  ", "\x0b", "\x0c")):
    rng = np.random.default_rng(seed)
    ranks = np.minimum(rng.zipf(1.1, n_tokens), types) - 1
    sep = rng.integers(0, len(seps), n_tokens)
    parts = []
    for r, s in zip(ranks, sep):
        parts.append(f"t{r}" if r % 7 else f"longer_token_{r}_xyz")
        parts.append(seps[s])
    return "\t " + "".join(parts) + ("tail" if seed % 2 else "")


CASES = [(1, 20000, 300, 1), (2, 50000, 2000, 2), (3, 3000, 50, 5), (4, 100000, 40000, 1)]


@pytest.mark.parametrize("seed,n,types,min_count", CASES)
def test_gpu_vocabulary_equals_host(tmp_path, seed, n, types, min_count):
    p = tmp_path / "c.txt"
    p.write_text(_raw_corpus(seed, n, types))
    host, gpu = _vocab_pair(p, min_count)
    _same_vocab(host, gpu)


@pytest.mark.parametrize("seed,n,types,min_count", CASES)
def test_gpu_id_stream_equals_host(tmp_path, seed, n, types, min_count):
    p = tmp_path / "c.txt"
    p.write_text(_raw_corpus(seed, n, types))
    vocab = api.build_vocabulary_file(str(p), min_count)
    # a vocabulary from another file: the GPU reader must drop exactly the same OOV tokens
    q = tmp_path / "other.txt"
    q.write_text(_raw_corpus(seed + 100, n // 2, types))
    other = api.build_vocabulary_file(str(q), 1)
    for v in (vocab, other):
        assert np.array_equal(api.read_id_stream(str(p), v), api.read_id_stream(str(p), v, device=0))


def test_reference_fixture_corpora(tmp_path):
    for mb, types, seed in ((200 * 1024, 2000, 4242), (30000, 120, 21)):
        p = F.write(tmp_path / "f.txt", F.make_zipf_corpus(mb, types, seed))
        for mc in (1, 5):
            host, gpu = _vocab_pair(p, mc)
            _same_vocab(host, gpu)
            assert np.array_equal(api.read_id_stream(p, host), api.read_id_stream(p, gpu, device=0))


def test_edge_cases(tmp_path):
    p = tmp_path / "e.txt"
    p.write_text("")
    with pytest.raises(_lib.CgError):  # NoTrainableWords
        api.build_vocabulary_file(str(p), 1, device=0)
    p.write_text(" \n\t  ")
    with pytest.raises(_lib.CgError):
        api.build_vocabulary_file(str(p), 1, device=0)
    p.write_text("a b a c b a " + "x" * 100000 + " a")  # a very long token
    host, gpu = _vocab_pair(p, 1)
    _same_vocab(host, gpu)
    with pytest.raises(OSError):
        api.build_vocabulary_file("/nonexistent/corpus.txt", 1, device=0)


def test_multi_chunk_file(tmp_path):
    """> 2 chunks of the id reader (128 MiB) and of the counter (64 MiB)."""
    rng = np.random.default_rng(7)
    words = np.array([f"w{i}" for i in range(70000)])
    p = tmp_path / "big.txt"
    with open(p, "w") as f:
        for _ in range(12):
            r = np.minimum(rng.zipf(1.05, 4_000_000), 70000) - 1
            f.write(" ".join(words[r]))
            f.write("\n")
    assert p.stat().st_size > 200 << 20
    host, gpu = _vocab_pair(p, 1)
    _same_vocab(host, gpu)
    assert np.array_equal(api.read_id_stream(str(p), host), api.read_id_stream(str(p), host, device=0))


def test_train_from_file_is_bit_exact(tmp_path):
    """train(corpus_path) tokenises on the GPU; deterministic mode must equal the oracle."""
    path = F.write(tmp_path / "t.txt", F.make_zipf_corpus(60_000, 300, 77))
    vocab = api.build_vocabulary_file(path, 2)
    ids = api.read_id_stream(path, vocab)
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, 31)
    cfg = dict(dim=24, window=4, min_count=2, sample=1e-3, iterations=2, cache_nodes=31, flush_interval=10, seed=5)
    m = api.train(path, vocab, tree, sel, api.TrainConfig(**cfg, mode="deterministic"))
    s0, s1, _ = O.orc_train(ids, vocab.counts, vocab.total_tokens(), cfg)
    assert np.array_equal(m.syn0.view(np.uint32), s0.view(np.uint32))
    assert np.array_equal(m.syn1.view(np.uint32), s1.view(np.uint32))


@pytest.mark.parametrize("chunk", [64, 1000, 4097])
def test_tiny_chunks_and_tokens_longer_than_a_chunk(tmp_path, monkeypatch, chunk):
    """Many chunks, and tokens longer than a whole chunk (the reader grows its buffers),
    through both GPU paths; bytes beyond ASCII are ordinary token bytes."""
    monkeypatch.setenv("CG_INGEST_CHUNK", str(chunk))
    rng = np.random.default_rng(chunk)
    toks = [f"t{int(r)}" for r in rng.zipf(1.2, 20000) % 500]
    for pos in (7, 5000, 19000):
        toks[pos] = "L" * 3000 + str(pos)  # longer than the chunk
    toks[11] = "café"
    toks[12] = "über"
    text = "".join(t + (" " if i % 17 else "\n") for i, t in enumerate(toks))
    p = tmp_path / "u.txt"
    p.write_bytes(text.encode("utf-8") + b"\xff\xfe tail")
    host, gpu = _vocab_pair(p, 1)
    _same_vocab(host, gpu)
    assert np.array_equal(api.read_id_stream(str(p), host), api.read_id_stream(str(p), host, device=0))


def test_hogwild_train_from_file_pipelined(tmp_path, monkeypatch):
    """train(corpus_path) in Hogwild mode trains the first pass chunk by chunk while the
    file is still being tokenised: every token is covered once per pass, and the model
    learns as much as training from the id stream. A vocabulary that undercounts the
    file (built from a prefix) falls back to the sequential path and still covers it."""
    monkeypatch.setenv("CG_INGEST_CHUNK", "65536")  # several chunks on a small file
    path = F.write(tmp_path / "h.txt", F.make_zipf_corpus(400_000, 2000, 13))
    vocab = api.build_vocabulary_file(path, 1)
    ids = api.read_id_stream(path, vocab)
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, 31)
    cfg = dict(dim=24, window=5, min_count=1, sample=1e-3, iterations=2, cache_nodes=31, seed=3)
    tc = api.TrainConfig(**cfg, mode="hogwild")
    st = api.TrainStats()
    m_file = api.train(path, vocab, tree, sel, tc, st)
    assert st.words_processed == 2 * ids.size
    m_ids = api.train(ids, vocab, tree, sel, tc)
    t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
    cen, ctx = O.sample_pairs(ids, vocab.counts, vocab.total_tokens(), 1e-3, 5, 7, 1 << 16)
    init = api.init_model(vocab.size(), 24, 3)
    l0, lf, li = (O.hs_loss(cen, ctx, m.syn0, m.syn1, t) for m in (init, m_file, m_ids))
    # Hogwild runs differ run to run; the chunked first pass flushes a little more often
    # (measured: 0.097 vs 0.092 loss reduction), so the band is 10% around the id-stream run
    assert lf < l0 and abs((l0 - lf) - (l0 - li)) < 0.10 * (l0 - li), (l0, lf, li)
    # undercounting vocabulary: counts from the first half of the file only
    half = tmp_path / "half.txt"
    half.write_text(open(path).read()[: 200_000])
    small = api.build_vocabulary_file(str(half), 1)
    ids_small = api.read_id_stream(path, small)
    assert ids_small.size > small.total_tokens()
    tree2 = api.build_huffman_tree(small)
    st2 = api.TrainStats()
    m2 = api.train(path, small, tree2, api.select_cached_nodes(tree2, 31), tc, st2)
    assert st2.words_processed == 2 * ids_small.size
    assert np.isfinite(m2.syn0).all()


def test_hogwild_train_from_file_ramped_chunks(tmp_path):
    """Without the chunk override the pipelined reader ramps its chunks up from 4 MB
    (4, 8, 16, 32 MB ...): a ~14 MB file is trained in several launches while it is
    read, covering every token once, with the same id stream as the host reader."""
    rng = np.random.default_rng(21)
    words = np.array([f"w{i}" for i in range(20000)])
    p = 1.0 / np.arange(1, 20001)
    p /= p.sum()  # Zipf(1.0) truncated to 20k types
    path = str(tmp_path / "r.txt")
    with open(path, "w") as f:
        for _ in range(8):
            f.write(" ".join(words[rng.choice(20000, 400_000, p=p)]) + "\n")
    assert Path(path).stat().st_size > 12 << 20
    vocab = api.build_vocabulary_file(path, 1)
    ids = api.read_id_stream(path, vocab)
    tree = api.build_huffman_tree(vocab)
    sel = api.select_cached_nodes(tree, 31)
    tc = api.TrainConfig(dim=16, window=5, min_count=1, sample=1e-3, iterations=1, cache_nodes=31, seed=5,
                         mode="hogwild")
    st = api.TrainStats()
    m = api.train(path, vocab, tree, sel, tc, st)
    assert st.words_processed == ids.size
    assert np.isfinite(m.syn0).all() and np.isfinite(m.syn1).all()
    t = O.Tree(tree.offsets, tree.nodes, tree.turns, tree.usage)
    cen, ctx = O.sample_pairs(ids, vocab.counts, vocab.total_tokens(), 1e-3, 5, 7, 1 << 15)
    init = api.init_model(vocab.size(), 16, 5)
    assert O.hs_loss(cen, ctx, m.syn0, m.syn1, t) < O.hs_loss(cen, ctx, init.syn0, init.syn1, t)
