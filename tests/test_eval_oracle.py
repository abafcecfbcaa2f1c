"""Evaluation oracle (oracle/cg_oracle.c orc_normalize / orc_analogy / orc_topk) pinned
against the reference's own AnalogySolver (eval.hpp:85-150, compiled unchanged into
oracle/_ref) and against the committed golden vectors made from it. CPU only."""
from pathlib import Path

import numpy as np
import pytest

import oracle_lib as O

GOLDEN = Path(__file__).resolve().parent / "golden" / "eval_analogy.npz"

CASES = [  # seed, rows, dim, questions, dup, zero, nan, restrict_top
    (1, 50, 4, 200, 5, 2, 0, 0),
    (2, 300, 7, 300, 20, 3, 2, 0),
    (3, 500, 33, 200, 10, 0, 0, 120),
    (4, 4, 3, 8, 0, 0, 0, 0),       # only one candidate left per question
    (5, 1000, 100, 100, 30, 5, 3, 700),
]


@pytest.mark.skipif(not O.ref_available(), reason="needs oracle/_ref (reference headers)")
@pytest.mark.parametrize("case", CASES)
def test_oracle_analogy_equals_reference(case):
    seed, rows, dim, nq, dup, zero, nan, top = case
    v, abc = O.eval_case(seed, rows, dim, nq, dup, zero, nan)
    size = min(rows, top) if top > 0 else rows
    abc = abc % size
    want = O.ref_analogy(v, top, abc)
    got = O.orc_analogy(O.orc_normalize(v[:size]), abc)
    assert np.array_equal(got, want)


def test_oracle_analogy_matches_golden():
    g = np.load(GOLDEN)
    for i in range(int(g["n_cases"])):
        v, abc, top, want = g[f"v{i}"], g[f"abc{i}"], int(g[f"top{i}"]), g[f"ans{i}"]
        size = min(v.shape[0], top) if top > 0 else v.shape[0]
        assert np.array_equal(O.orc_analogy(O.orc_normalize(v[:size]), abc), want), i


def test_oracle_known_answers():
    v = np.array([[1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 0], [0, 1, 1]], np.float32)
    n = O.orc_normalize(v)
    assert np.allclose(np.linalg.norm(n, axis=1), 1.0, atol=1e-6)
    # a zero row and a row holding NaN both normalise to zeros (norm > 0 is false)
    z = O.orc_normalize(np.array([[0, 0], [np.nan, 1]], np.float32))
    assert np.all(z == 0)
    # b - a + c = e1 - e0 + e2: rows 3 (e0+e1) and 4 (e1+e2) score 0 and sqrt2 -> 4
    assert O.orc_analogy(n, np.array([[0, 1, 2]]))[0] == 4
    # orthogonal candidates tie at 0 -> the lowest id not in {a, b, c}
    e = O.orc_normalize(np.eye(6, dtype=np.float32))
    assert O.orc_analogy(e, np.array([[0, 0, 0]]))[0] == 1
    assert O.orc_analogy(e, np.array([[3, 4, 5]]))[0] == 0


def test_oracle_topk_against_bruteforce():
    rng = np.random.default_rng(9)
    v = (rng.random((200, 9), dtype=np.float32) - 0.5)
    v[10] = v[11]  # tie
    n = O.orc_normalize(v)
    q = np.arange(0, 200, 7, dtype=np.int32)
    ids, sc = O.orc_topk(n, q, 10)
    for i, qi in enumerate(q):
        s = np.array([np.cumsum(n[qi] * n[w], dtype=np.float32)[-1] for w in range(200)], np.float32)
        s[qi] = -np.inf
        order = sorted(range(200), key=lambda w: (-s[w], w))[:10]
        assert list(ids[i]) == order
        assert np.array_equal(sc[i], s[order])
