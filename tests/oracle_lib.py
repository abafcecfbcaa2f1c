"""TEST INFRASTRUCTURE: ctypes access to the CPU checker libraries.

* oracle/libcgoracle.so   -- the plain-C restatement (oracle/cg_oracle.c), always built.
* oracle/_ref/libcgref.so -- the reference headers compiled unchanged (oracle/Makefile);
                             built where /root/reference exists, travels prebuilt.
Only tests/, __graft_entry__.smoke() and bench.py's CPU legs use these.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "libcgoracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libcgref.so"

P = C.POINTER


def _p(a, t):
    return None if a is None else a.ctypes.data_as(P(t))


class OrcConfig(C.Structure):
    _fields_ = [("dim", C.c_int32), ("window", C.c_int32), ("min_count", C.c_int64), ("sample", C.c_double),
                ("alpha0", C.c_float), ("iterations", C.c_int32), ("workers", C.c_int32),
                ("cache_nodes", C.c_int32), ("flush_interval", C.c_int32), ("seed", C.c_uint64)]


class OrcStats(C.Structure):
    _fields_ = [("words_processed", C.c_uint64), ("centers", C.c_uint64), ("pairs", C.c_uint64),
                ("steps", C.c_uint64), ("flushes", C.c_uint64)]


_orc = None
_ref = None


def oracle() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            import subprocess
            subprocess.run(["make", "-C", str(ROOT / "oracle"), "libcgoracle.so"], check=True, capture_output=True)
        lib = C.CDLL(str(ORACLE_SO))
        lib.orc_splitmix_next.restype = C.c_uint64
        lib.orc_splitmix_next.argtypes = [P(C.c_uint64)]
        lib.orc_mix_seed.restype = C.c_uint64
        lib.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.orc_keep_probability.restype = C.c_double
        lib.orc_keep_probability.argtypes = [C.c_int64, C.c_int64, C.c_double]
        lib.orc_update_alpha.restype = C.c_float
        lib.orc_update_alpha.argtypes = [C.c_uint64, C.c_uint64, C.c_float]
        lib.orc_sigmoid_table.argtypes = [P(C.c_float)]
        lib.orc_init_model.argtypes = [C.c_int32, C.c_int32, C.c_uint64, P(C.c_float), P(C.c_float)]
        lib.orc_build_huffman.argtypes = [P(C.c_int64), C.c_int32, P(C.c_int64), P(C.c_int32), P(C.c_uint8),
                                          P(C.c_int64), P(C.c_int64)]
        lib.orc_select_cached.restype = C.c_int32
        lib.orc_select_cached.argtypes = [P(C.c_int64), C.c_int32, C.c_int32, P(C.c_int32), P(C.c_int32)]
        lib.orc_vocab_from_ids.restype = C.c_int32
        lib.orc_vocab_from_ids.argtypes = [P(C.c_int32), C.c_int64, C.c_int32, C.c_int64, P(C.c_int32),
                                           P(C.c_int64), P(C.c_int64)]
        lib.orc_train_single.argtypes = [P(C.c_int32), C.c_int64, C.c_int32, P(C.c_int64), C.c_int64, P(C.c_int64),
                                         P(C.c_int32), P(C.c_uint8), P(C.c_int32), C.c_int32, P(C.c_int32),
                                         P(OrcConfig), P(C.c_float), P(C.c_float), P(OrcStats)]
        lib.orc_train_center.restype = C.c_int64
        lib.orc_train_center.argtypes = [C.c_int32, P(C.c_int32), C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                         P(C.c_float), P(C.c_float), P(C.c_int64), P(C.c_int32), P(C.c_uint8),
                                         P(C.c_int32), P(C.c_float), P(C.c_float), P(C.c_uint8), P(C.c_int32),
                                         P(C.c_int32), C.c_float, C.c_int32, C.c_float]
        lib.orc_cache_flush.argtypes = [C.c_int32, P(C.c_float), P(C.c_int32), P(C.c_float), P(C.c_float),
                                        P(C.c_uint8), P(C.c_int32), P(C.c_int32)]
        lib.orc_hs_loss.restype = C.c_double
        lib.orc_hs_loss.argtypes = [P(C.c_int32), P(C.c_int32), C.c_int64, C.c_int32, P(C.c_float), P(C.c_float),
                                    P(C.c_int64), P(C.c_int32), P(C.c_uint8)]
        lib.orc_sample_pairs.restype = C.c_int64
        lib.orc_sample_pairs.argtypes = [P(C.c_int32), C.c_int64, P(C.c_float), C.c_int32, C.c_uint64, C.c_int64,
                                         P(C.c_int32), P(C.c_int32)]
        lib.orc_normalize.argtypes = [P(C.c_float), C.c_int64, C.c_int32, P(C.c_float)]
        lib.orc_analogy.argtypes = [P(C.c_float), C.c_int64, C.c_int32, P(C.c_int32), C.c_int64, P(C.c_int32)]
        lib.orc_topk.argtypes = [P(C.c_float), C.c_int64, C.c_int32, P(C.c_int32), C.c_int64, C.c_int32,
                                 P(C.c_int32), P(C.c_float)]
        _orc = lib
    return _orc


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(str(REF_SO))
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_mix_seed.restype = C.c_uint64
        lib.ref_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.ref_rng_stream.argtypes = [C.c_uint64, C.c_int64, P(C.c_uint64), P(C.c_float), C.c_uint32,
                                       P(C.c_uint32)]
        lib.ref_keep_probability.restype = C.c_double
        lib.ref_keep_probability.argtypes = [C.c_int64, C.c_int64, C.c_double]
        lib.ref_update_alpha.restype = C.c_float
        lib.ref_update_alpha.argtypes = [C.c_uint64, C.c_uint64, C.c_float]
        lib.ref_sigmoid_value.restype = C.c_float
        lib.ref_sigmoid_value.argtypes = [C.c_float]
        lib.ref_init_model.argtypes = [C.c_int32, C.c_int32, C.c_uint64, P(C.c_float), P(C.c_float)]
        lib.ref_shrink_window.argtypes = [C.c_int32, C.c_uint64, C.c_int64, P(C.c_int32)]
        lib.ref_open_file.restype = C.c_void_p
        lib.ref_open_file.argtypes = [C.c_char_p, C.c_int64]
        lib.ref_open_counts.restype = C.c_void_p
        lib.ref_open_counts.argtypes = [P(C.c_int64), C.c_int32]
        lib.ref_close.argtypes = [C.c_void_p]
        lib.ref_vocab_size.restype = C.c_int32
        lib.ref_vocab_size.argtypes = [C.c_void_p]
        lib.ref_total_tokens.restype = C.c_int64
        lib.ref_total_tokens.argtypes = [C.c_void_p]
        lib.ref_vocab_export.argtypes = [C.c_void_p, P(C.c_int64), P(C.c_int64)]
        lib.ref_tree_steps.restype = C.c_int64
        lib.ref_tree_steps.argtypes = [C.c_void_p]
        lib.ref_tree_export.argtypes = [C.c_void_p, P(C.c_int64), P(C.c_int32), P(C.c_uint8), P(C.c_int64)]
        lib.ref_select.restype = C.c_int32
        lib.ref_select.argtypes = [C.c_void_p, C.c_int32, P(C.c_int32), P(C.c_int32)]
        lib.ref_train.restype = C.c_int
        lib.ref_train.argtypes = [C.c_void_p, C.c_char_p, C.c_int32, C.c_int32, C.c_int64, C.c_double, C.c_float,
                                  C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_uint64, P(C.c_float),
                                  P(C.c_float), P(C.c_uint64), P(C.c_double)]
        lib.ref_train_center.restype = C.c_int64
        lib.ref_train_center.argtypes = [P(C.c_int64), C.c_int32, C.c_int32, P(C.c_float), P(C.c_float), C.c_int32,
                                         C.c_int32, C.c_int32, P(C.c_int32), C.c_int64, C.c_int64, C.c_int32,
                                         C.c_float, C.c_int32, C.c_float]
        lib.ref_analogy.restype = C.c_int
        lib.ref_analogy.argtypes = [P(C.c_float), C.c_int32, C.c_int32, C.c_int32, P(C.c_int32), C.c_int64,
                                    P(C.c_int32)]
        lib.ref_model_save.restype = C.c_int
        lib.ref_model_save.argtypes = [C.c_char_p, C.c_int32, C.c_char_p, P(C.c_float), C.c_int32, C.c_int32]
        lib.ref_model_load.restype = C.c_int
        lib.ref_model_load.argtypes = [C.c_char_p, C.c_int32, P(C.c_int32), P(C.c_int32), P(C.c_float), C.c_int64]
        _ref = lib
    return _ref


# ---------------------------------------------------------------- oracle helpers
class Tree:
    def __init__(self, off, nodes, turns, usage):
        self.off, self.nodes, self.turns, self.usage = off, nodes, turns, usage


def orc_tree(counts: np.ndarray) -> Tree:
    lib = oracle()
    counts = np.ascontiguousarray(counts, np.int64)
    v = counts.size
    n = C.c_int64()
    lib.orc_build_huffman(_p(counts, C.c_int64), v, None, None, None, None, C.byref(n))
    off = np.zeros(v + 1, np.int64)
    nodes = np.zeros(n.value, np.int32)
    turns = np.zeros(n.value, np.uint8)
    usage = np.zeros(v - 1, np.int64)
    lib.orc_build_huffman(_p(counts, C.c_int64), v, _p(off, C.c_int64), _p(nodes, C.c_int32), _p(turns, C.c_uint8),
                          _p(usage, C.c_int64), C.byref(n))
    return Tree(off, nodes, turns, usage)


def orc_select(usage: np.ndarray, k: int):
    inner = usage.size
    hot = np.zeros(max(min(k, inner), 1), np.int32)
    slot = np.zeros(inner, np.int32)
    n = oracle().orc_select_cached(_p(usage, C.c_int64), inner, k, _p(hot, C.c_int32), _p(slot, C.c_int32))
    return hot[:n].copy(), slot


def orc_init(v: int, d: int, seed: int):
    syn0 = np.zeros((v, d), np.float32)
    syn1 = np.zeros((v - 1, d), np.float32)
    oracle().orc_init_model(v, d, seed, _p(syn0, C.c_float), _p(syn1, C.c_float))
    return syn0, syn1


def orc_train(ids: np.ndarray, counts: np.ndarray, total: int, cfg: dict):
    """Single-worker reference training restated in C. Returns (syn0, syn1, stats)."""
    lib = oracle()
    ids = np.ascontiguousarray(ids, np.int32)
    counts = np.ascontiguousarray(counts, np.int64)
    v = counts.size
    t = orc_tree(counts)
    hot, slot = orc_select(t.usage, cfg.get("cache_nodes", 31))
    syn0, syn1 = orc_init(v, cfg["dim"], cfg.get("seed", 1))
    c = OrcConfig(cfg["dim"], cfg.get("window", 5), cfg.get("min_count", 5), cfg.get("sample", 1e-3),
                  cfg.get("alpha0", 0.025), cfg.get("iterations", 1), 1, cfg.get("cache_nodes", 31),
                  cfg.get("flush_interval", 10), cfg.get("seed", 1))
    st = OrcStats()
    lib.orc_train_single(_p(ids, C.c_int32), ids.size, v, _p(counts, C.c_int64), total, _p(t.off, C.c_int64),
                         _p(t.nodes, C.c_int32), _p(t.turns, C.c_uint8), _p(hot, C.c_int32), hot.size,
                         _p(slot, C.c_int32), C.byref(c), _p(syn0, C.c_float), _p(syn1, C.c_float), C.byref(st))
    return syn0, syn1, st


def orc_vocab(raw: np.ndarray, min_count: int, space: int):
    raw = np.ascontiguousarray(raw, np.int32)
    rank = np.zeros(space, np.int32)
    counts = np.zeros(space, np.int64)
    total = C.c_int64()
    v = oracle().orc_vocab_from_ids(_p(raw, C.c_int32), raw.size, space, min_count, _p(rank, C.c_int32),
                                    _p(counts, C.c_int64), C.byref(total))
    return rank, counts[:v].copy(), total.value


def keep_table(counts: np.ndarray, total: int, sample: float) -> np.ndarray | None:
    if sample <= 0:
        return None
    lib = oracle()
    return np.array([lib.orc_keep_probability(int(c), int(total), sample) for c in counts], dtype=np.float32)


def sample_pairs(ids, counts, total, sample, window, seed, n):
    kp = keep_table(counts, total, sample)
    cen = np.zeros(n, np.int32)
    ctx = np.zeros(n, np.int32)
    ids = np.ascontiguousarray(ids, np.int32)
    got = oracle().orc_sample_pairs(_p(ids, C.c_int32), ids.size, _p(kp, C.c_float) if kp is not None else None,
                                    window, seed, n, _p(cen, C.c_int32), _p(ctx, C.c_int32))
    return cen[:got].copy(), ctx[:got].copy()


def hs_loss(centers, contexts, syn0, syn1, tree: Tree) -> float:
    syn0 = np.ascontiguousarray(syn0, np.float32)
    syn1 = np.ascontiguousarray(syn1, np.float32)
    return oracle().orc_hs_loss(_p(centers, C.c_int32), _p(contexts, C.c_int32), centers.size, syn0.shape[1],
                                _p(syn0, C.c_float), _p(syn1, C.c_float), _p(tree.off, C.c_int64),
                                _p(tree.nodes, C.c_int32), _p(tree.turns, C.c_uint8))


# ---------------------------------------------------------------- reference helpers
def ref_vocab_file(path: str, min_count: int):
    lib = ref()
    h = lib.ref_open_file(str(path).encode(), min_count)
    assert h, lib.ref_last_error()
    v = lib.ref_vocab_size(h)
    counts = np.zeros(v, np.int64)
    raws = np.zeros(v, np.int64)
    lib.ref_vocab_export(h, _p(counts, C.c_int64), _p(raws, C.c_int64))
    return h, counts, raws, lib.ref_total_tokens(h)


def ref_tree(h) -> Tree:
    lib = ref()
    v = lib.ref_vocab_size(h)
    n = lib.ref_tree_steps(h)
    off = np.zeros(v + 1, np.int64)
    nodes = np.zeros(n, np.int32)
    turns = np.zeros(n, np.uint8)
    usage = np.zeros(v - 1, np.int64)
    lib.ref_tree_export(h, _p(off, C.c_int64), _p(nodes, C.c_int32), _p(turns, C.c_uint8), _p(usage, C.c_int64))
    return Tree(off, nodes, turns, usage)


def ref_train(h, path: str, cfg: dict, workers: int = 1):
    lib = ref()
    v = lib.ref_vocab_size(h)
    d = cfg["dim"]
    syn0 = np.zeros((v, d), np.float32)
    syn1 = np.zeros((v - 1, d), np.float32)
    words = C.c_uint64()
    wall = C.c_double()
    rc = lib.ref_train(h, str(path).encode(), d, cfg.get("window", 5), cfg.get("min_count", 5),
                       cfg.get("sample", 1e-3), cfg.get("alpha0", 0.025), cfg.get("iterations", 1), workers,
                       cfg.get("cache_nodes", 31), cfg.get("flush_interval", 10), cfg.get("seed", 1),
                       _p(syn0, C.c_float), _p(syn1, C.c_float), C.byref(words), C.byref(wall))
    if rc != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return syn0, syn1, words.value, wall.value


def max_relative_diff(a: np.ndarray, b: np.ndarray) -> float:
    """tests/acceptance.cpp:251-263: |x-y| / max(|x|, |y|, 1e-2)."""
    a = a.astype(np.float64).ravel()
    b = b.astype(np.float64).ravel()
    if a.size == 0:
        return 0.0
    den = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-2)
    return float(np.max(np.abs(a - b) / den))


# ---------------------------------------------------------------- evaluation oracle
def orc_normalize(vectors: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(vectors, dtype=np.float32)
    out = np.empty_like(v)
    oracle().orc_normalize(_p(v, C.c_float), v.shape[0], v.shape[1], _p(out, C.c_float))
    return out


def orc_analogy(norm: np.ndarray, abc: np.ndarray) -> np.ndarray:
    n = np.ascontiguousarray(norm, dtype=np.float32)
    q = np.ascontiguousarray(abc, dtype=np.int32).reshape(-1, 3)
    out = np.empty(q.shape[0], np.int32)
    oracle().orc_analogy(_p(n, C.c_float), n.shape[0], n.shape[1], _p(q, C.c_int32), q.shape[0], _p(out, C.c_int32))
    return out


def orc_topk(norm: np.ndarray, queries: np.ndarray, k: int):
    n = np.ascontiguousarray(norm, dtype=np.float32)
    q = np.ascontiguousarray(queries, dtype=np.int32)
    ids = np.empty((q.size, k), np.int32)
    sc = np.empty((q.size, k), np.float32)
    oracle().orc_topk(_p(n, C.c_float), n.shape[0], n.shape[1], _p(q, C.c_int32), q.size, k, _p(ids, C.c_int32),
                      _p(sc, C.c_float))
    return ids, sc


def ref_analogy(vectors: np.ndarray, restrict_top: int, abc: np.ndarray) -> np.ndarray:
    v = np.ascontiguousarray(vectors, dtype=np.float32)
    q = np.ascontiguousarray(abc, dtype=np.int32).reshape(-1, 3)
    out = np.empty(q.shape[0], np.int32)
    rc = ref().ref_analogy(_p(v, C.c_float), v.shape[0], v.shape[1], restrict_top, _p(q, C.c_int32), q.shape[0],
                           _p(out, C.c_int32))
    assert rc == 0, ref().ref_last_error()
    return out


def eval_case(seed: int, rows: int, dim: int, nq: int, dup: int = 0, zero: int = 0, nan: int = 0):
    """Seeded embeddings with planted hazards for the analogy/top-k parity cases:
    `dup` duplicated rows (exact score ties), `zero` all-zero rows and `nan` rows holding
    a NaN (both normalise to zero rows, so their scores are exactly 0), plus as many rows
    holding an inf (normalised to a NaN entry: their scores are NaN). Questions are
    random distinct triples, plus a few with repeated words."""
    rng = np.random.default_rng(seed)
    v = (rng.random((rows, dim), dtype=np.float32) - 0.5).astype(np.float32)
    for i in range(dup):
        v[rng.integers(rows)] = v[rng.integers(rows)]
    for i in range(zero):
        v[rng.integers(rows)] = 0.0
    for i in range(nan):
        v[rng.integers(rows), rng.integers(dim)] = np.nan
        v[rng.integers(rows), rng.integers(dim)] = np.inf  # inf / inf -> a NaN entry, NaN scores
    abc = rng.integers(0, rows, size=(nq, 3)).astype(np.int32)
    if nq >= 4:
        abc[0, 1] = abc[0, 0]
        abc[1, 2] = abc[1, 0]
    return v, abc
