"""Model files through the C-ABI (cg_model_save / cg_model_load, cg_modelio.cpp): the
bytes equal the reference's save_text / save_binary (golden files written by the
reference, tests/golden/make_golden_eval.py, and -- when oracle/_ref exists -- fresh
reference writes of random models), loads round-trip, and malformed files raise the
reference's error classes (model.hpp:152-276). Host code only: no GPU needed."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O
from paper_1606_07822_b200 import _lib, api

G = Path(__file__).resolve().parent / "golden"


class _Vocab:
    def __init__(self, words):
        self.words = words

    def word(self, i):
        return self.words[i]

    def size(self):
        return len(self.words)


def _model(values):
    m = api.Model(values.shape[0], values.shape[1])
    m.syn0[:] = values.reshape(m.syn0.shape)
    return m


def _golden_words():
    import golden.make_golden_eval as mg
    return mg.model_words()


@pytest.fixture(scope="module", autouse=True)
def _path():
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parent))


@pytest.mark.parametrize("fmt", ["txt", "bin"])
def test_save_matches_reference_bytes(tmp_path, fmt):
    v = np.load(G / "model_small_values.npy")
    out = tmp_path / f"m.{fmt}"
    (api.save_text if fmt == "txt" else api.save_binary)(_model(v), _Vocab(_golden_words()), str(out))
    assert out.read_bytes() == (G / f"model_small.{fmt}").read_bytes()


@pytest.mark.skipif(not O.ref_available(), reason="needs oracle/_ref")
@pytest.mark.parametrize("binary", [0, 1])
def test_save_matches_reference_random(tmp_path, binary):
    rng = np.random.default_rng(5 + binary)
    v = ((rng.standard_normal((700, 37)) * 10.0 ** rng.integers(-8, 6, (700, 37))).astype(np.float32))
    words = [f"tok{i}" + "x" * (i % 5) for i in range(700)]
    ours, theirs = tmp_path / "ours", tmp_path / "theirs"
    (api.save_binary if binary else api.save_text)(_model(v), _Vocab(words), str(ours))
    wn = b"".join(w.encode() + b"\0" for w in words)
    assert O.ref().ref_model_save(str(theirs).encode(), binary, wn, O._p(v, C.c_float), 700, 37) == 0
    assert ours.read_bytes() == theirs.read_bytes()


def test_round_trips(tmp_path):
    v = np.load(G / "model_small_values.npy")
    words = _golden_words()
    b = api.load_embeddings_binary(str(G / "model_small.bin"))
    assert b.words == words and b.dim == 6
    assert np.array_equal(b.vectors.view(np.uint32), v.view(np.uint32))
    t = api.load_embeddings_text(str(G / "model_small.txt"))
    assert t.words == words
    big = np.abs(v) > 1e30
    assert np.allclose(t.vectors[~big], v[~big], atol=1e-5)
    for f in ("model_small.bin", "model_small.txt"):  # auto-detection
        a = api.load_embeddings(str(G / f))
        assert a.words == words and a.vectors.shape == (20, 6)


@pytest.mark.skipif(not O.ref_available(), reason="needs oracle/_ref")
@pytest.mark.parametrize("fmt", [0, 1, 2])
def test_load_equals_reference(fmt):
    name = "model_small.bin" if fmt == 1 else "model_small.txt"
    path = str(G / name)
    rows, dim = C.c_int32(), C.c_int32()
    buf = np.zeros(20 * 6, np.float32)
    assert O.ref().ref_model_load(path.encode(), fmt, C.byref(rows), C.byref(dim), O._p(buf, C.c_float), buf.size) == 0
    ours = {0: api.load_embeddings_text, 1: api.load_embeddings_binary, 2: api.load_embeddings}[fmt](path)
    assert np.array_equal(ours.vectors.reshape(-1).view(np.uint32), buf.view(np.uint32))


BAD_TEXT = [
    "not a header\nx 1.0\n", "", "3\nx 1.0\n", "0 5\n", "2 -1\n", "2 3 \n",
    "2 3\nalpha 0.5 0.25 0.125\n",            # truncated
    "1 3\nalpha 0.5 0.25\n",                  # too few values
    "1 2\nalpha 0.5 0.25 0.125\n",            # trailing values
    "1 2\n 0.5 0.25\n",                       # empty word
    "1 2\nalpha\n",                           # no values
    "2 1\nalpha 1\n\nbeta 2\n",               # blank row
    "1 2\nalpha 0.5 x\n",
]


@pytest.mark.parametrize("content", BAD_TEXT)
def test_malformed_text_raises_parse_error(tmp_path, content):
    p = tmp_path / "bad.txt"
    p.write_text(content)
    with pytest.raises(_lib.ParseError):
        api.load_embeddings_text(str(p))
    if O.ref_available():
        r, d = C.c_int32(), C.c_int32()
        assert O.ref().ref_model_load(str(p).encode(), 0, C.byref(r), C.byref(d), None, 0) == -2


def test_truncated_binary_and_missing(tmp_path):
    f = np.array([0.5, 0.25, 0.125], np.float32).tobytes()
    p = tmp_path / "t.bin"
    p.write_bytes(b"2 3\nalpha " + f + b"\nbeta " + f[:4])
    with pytest.raises(_lib.ParseError):
        api.load_embeddings_binary(str(p))
    p.write_bytes(b"2 3\nalpha " + f + b"\nbeta")
    with pytest.raises(_lib.ParseError):
        api.load_embeddings_binary(str(p))
    with pytest.raises(OSError):
        api.load_embeddings("/nonexistent/model.bin")
    with pytest.raises(OSError):
        api.save_text(_model(np.zeros((2, 2), np.float32)), _Vocab(["a", "b"]), "/nonexistent/dir/m.txt")


def test_large_text_parallel_matches_sequential(tmp_path):
    """Many row blocks: the parallel formatter keeps row order and bytes."""
    rng = np.random.default_rng(3)
    v = (rng.random((5000, 16), dtype=np.float32) - 0.5)
    words = [f"w{i}" for i in range(5000)]
    p = tmp_path / "big.txt"
    api.save_text(_model(v), _Vocab(words), str(p))
    lines = p.read_text().split("\n")
    assert lines[0] == "5000 16" and len(lines) == 5002
    for i in (0, 1, 255, 256, 4999):
        parts = lines[1 + i].split(" ")
        assert parts[0] == words[i]
        assert parts[1:] == [f"{float(x):.6f}" for x in v[i]]
    back = api.load_embeddings_text(str(p))
    assert back.words == words and np.allclose(back.vectors, v, atol=1e-6)
