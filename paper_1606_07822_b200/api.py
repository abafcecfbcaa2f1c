"""Python mirror of the reference's training interface, over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/cachegram
(corpus.hpp, huffman.hpp, model.hpp, trainer.hpp): ``TrainConfig``, ``Vocabulary``,
``build_vocabulary_file``, ``HuffmanTree``/``build_huffman_tree``, ``CacheSelection``/
``select_cached_nodes``, ``Model``/``init_model``, ``keep_probability``,
``update_alpha``, ``NodeCache``, ``train_center`` and ``train``. C++ ``std::invalid_argument``
surfaces as ``ValueError`` and ``IoError`` as ``OSError``. Every training computation
runs in libcachegram_b200.so on the GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from ._lib import CgConfig, CgEpochStats, CgModelDesc, CgTrainStats, check, load, ptr

MODES = {"hogwild": _lib.CG_MODE_HOGWILD, "deterministic": _lib.CG_MODE_DETERMINISTIC}


def resolve_mode(config: "TrainConfig") -> str:
    """"auto" (default): workers == 1 -> the reference's deterministic single-worker
    semantics (bit-identical), workers > 1 -> Hogwild on every SM."""
    if config.mode != "auto":
        return config.mode
    return "deterministic" if config.workers == 1 else "hogwild"


# --------------------------------------------------------------------------- config
@dataclass
class TrainConfig:
    """trainer.hpp:25-48 (+ ``mode``: "auto" (default), "hogwild" or "deterministic")."""
    dim: int = 100
    window: int = 5
    min_count: int = 5
    sample: float = 1e-3
    alpha0: float = 0.025
    iterations: int = 5
    workers: int = 1
    cache_nodes: int = 31
    flush_interval: int = 10
    seed: int = 1
    mode: str = "auto"

    def validate(self) -> None:
        for ok, msg in (
            (self.dim >= 1, "dim must be >= 1"),
            (self.window >= 1, "window must be >= 1"),
            (self.min_count >= 1, "min-count must be >= 1"),
            (self.sample >= 0.0, "sample must be >= 0"),
            (self.alpha0 > 0.0, "alpha must be > 0"),
            (self.iterations >= 1, "iterations must be >= 1"),
            (self.workers >= 1, "workers must be >= 1"),
            (self.cache_nodes >= 0, "cache-nodes must be >= 0"),
            (self.flush_interval >= 1, "flush-interval must be >= 1"),
        ):
            if not ok:
                raise ValueError(msg)
        if self.mode not in MODES and self.mode != "auto":
            raise ValueError(f"unknown training mode {self.mode!r}")

    def to_c(self) -> CgConfig:
        return CgConfig(self.dim, self.window, self.min_count, self.sample, self.alpha0, self.iterations,
                        self.workers, self.cache_nodes, self.flush_interval, self.seed & 0xFFFFFFFFFFFFFFFF)


@dataclass
class TrainStats:
    words_processed: int = 0
    wall_seconds: float = 0.0
    words_per_second: float = 0.0
    kernel_seconds: float = 0.0
    centers: int = 0
    pairs: int = 0
    steps: int = 0


# --------------------------------------------------------------------------- corpus
class Vocabulary:
    """corpus.hpp:55-83: ids 0..V-1 by descending count, first occurrence on ties."""

    def __init__(self, counts: Sequence[int], words: Sequence[str] | None = None, total: int | None = None,
                 _handle=None):
        self.counts = np.ascontiguousarray(np.asarray(counts, dtype=np.int64))
        self.words = list(words) if words is not None else [f"w{i}" for i in range(len(self.counts))]
        self._index = {w: i for i, w in enumerate(self.words)}
        self.total = int(self.counts.sum()) if total is None else int(total)
        self._handle = _handle

    def size(self) -> int:
        return int(self.counts.shape[0])

    def total_tokens(self) -> int:
        return self.total

    def count(self, i: int) -> int:
        return int(self.counts[i])

    def word(self, i: int) -> str:
        return self.words[i]

    def id_of(self, w: str) -> int:
        return self._index.get(w, -1)

    def words_nul(self) -> bytes:
        """The words in id order, each NUL-terminated (the C-ABI's word list); built once
        (joining ~10^5 words took ~12 ms per train(corpus_path) call)."""
        key = (id(self.words), len(self.words))
        if getattr(self, "_nul_key", None) != key:
            self._nul = b"".join(w.encode("utf-8", "surrogateescape") + b"\0" for w in self.words)
            self._nul_key = key
        return self._nul

    def __del__(self):
        if getattr(self, "_handle", None):
            try:
                load().cg_corpus_close(self._handle)
            except Exception:  # interpreter teardown: the library may already be gone
                pass
            self._handle = None


def build_vocabulary_file(path: str, min_count: int, device: int | None = None) -> Vocabulary:
    """corpus.hpp:144-170. device=None: C++ host code in the library; device=k (or -1 for
    the current device): counted on the GPU (cg_corpus_open_gpu), same result."""
    lib = load()
    h = C.c_void_p()
    if device is None:
        check(lib.cg_corpus_open(str(path).encode(), int(min_count), C.byref(h)))
    else:
        check(lib.cg_corpus_open_gpu(str(path).encode(), int(min_count), int(device), C.byref(h)))
    v = lib.cg_corpus_vocab_size(h)
    counts = np.zeros(v, dtype=np.int64)
    buf = C.create_string_buffer(int(lib.cg_corpus_word_bytes(h)) + 1)
    check(lib.cg_corpus_export_vocab(h, ptr(counts, C.c_int64), buf))
    words = buf.raw[: lib.cg_corpus_word_bytes(h)].split(b"\0")[:v]
    return Vocabulary(counts, [w.decode("utf-8", "surrogateescape") for w in words], int(lib.cg_corpus_total_tokens(h)),
                      _handle=h)


def read_id_stream(path: str, vocab: Vocabulary, device: int | None = None) -> np.ndarray:
    """The in-vocabulary id stream of a corpus file (what ShardReader + id_of yield);
    tokenised on the GPU when `device` is given."""
    if vocab._handle is None:
        raise ValueError("vocabulary was not built from a file")
    lib = load()
    n = C.c_int64()
    if device is not None:
        check(lib.cg_corpus_read_ids_gpu(vocab._handle, str(path).encode(), int(device), None, 0, C.byref(n)))
        ids = np.empty(n.value, dtype=np.int32)
        check(lib.cg_corpus_read_ids_gpu(vocab._handle, str(path).encode(), int(device), ptr(ids, C.c_int32),
                                         n.value, C.byref(n)))
        return ids
    check(lib.cg_corpus_read_ids(vocab._handle, str(path).encode(), None, 0, C.byref(n)))
    ids = np.empty(n.value, dtype=np.int32)
    check(lib.cg_corpus_read_ids(vocab._handle, str(path).encode(), ptr(ids, C.c_int32), n.value, C.byref(n)))
    return ids


def sync_row_scale(q: float, n_replicas: int, centers: float) -> float:
    """cg_sync_row_scale: the per-row scale of the replicas' summed delta at a sync."""
    return float(load().cg_sync_row_scale(float(q), int(n_replicas), float(centers)))


def keep_probability(count: int, total_tokens: int, sample: float) -> float:
    return float(load().cg_keep_probability(int(count), int(total_tokens), float(sample)))


def update_alpha(words_processed: int, total_words: int, alpha0: float) -> float:
    return float(load().cg_update_alpha(int(words_processed), int(total_words), float(alpha0)))


def sigmoid_table() -> np.ndarray:
    t = np.zeros(1000, dtype=np.float32)
    load().cg_sigmoid_table(ptr(t, C.c_float))
    return t


# --------------------------------------------------------------------------- tree
class HuffmanTree:
    """huffman.hpp:30-52: root-first (node, turn) paths as CSR, plus node usage."""

    def __init__(self, offsets: np.ndarray, nodes: np.ndarray, turns: np.ndarray, usage: np.ndarray):
        self.offsets, self.nodes, self.turns, self.usage = offsets, nodes, turns, usage

    def inner_count(self) -> int:
        return int(self.usage.shape[0])

    def leaf_count(self) -> int:
        return int(self.offsets.shape[0]) - 1

    def root_id(self) -> int:
        return self.inner_count() - 1

    def path(self, w: int) -> list[tuple[int, int]]:
        a, b = int(self.offsets[w]), int(self.offsets[w + 1])
        return list(zip(self.nodes[a:b].tolist(), self.turns[a:b].tolist()))

    def node_usage(self, n: int) -> int:
        return int(self.usage[n])

    def depth(self) -> np.ndarray:
        return np.diff(self.offsets)


def build_huffman_tree(vocab: Vocabulary | Sequence[int]) -> HuffmanTree:
    counts = vocab.counts if isinstance(vocab, Vocabulary) else np.ascontiguousarray(np.asarray(vocab, np.int64))
    v = int(counts.shape[0])
    if v == 0:
        raise RuntimeError("no trainable words")
    lib = load()
    steps = C.c_int64()
    check(lib.cg_build_huffman(ptr(counts, C.c_int64), v, None, None, None, None, C.byref(steps)))
    off = np.zeros(v + 1, np.int64)
    nodes = np.zeros(steps.value, np.int32)
    turns = np.zeros(steps.value, np.uint8)
    usage = np.zeros(v - 1, np.int64)
    check(lib.cg_build_huffman(ptr(counts, C.c_int64), v, ptr(off, C.c_int64), ptr(nodes, C.c_int32),
                               ptr(turns, C.c_uint8), ptr(usage, C.c_int64), C.byref(steps)))
    return HuffmanTree(off, nodes, turns, usage)


class CacheSelection:
    """huffman.hpp:116-134."""

    def __init__(self, hot: np.ndarray, slot: np.ndarray):
        self.hot, self.slot = hot, slot

    def size(self) -> int:
        return int(self.hot.shape[0])

    def hot_nodes(self) -> np.ndarray:
        return self.hot

    def node_at(self, s: int) -> int:
        return int(self.hot[s])

    def inner_node_count(self) -> int:
        return int(self.slot.shape[0])

    def slot_of(self, n: int) -> int:
        return int(self.slot[n])


def select_cached_nodes(tree: HuffmanTree, k: int) -> CacheSelection:
    if k < 0:
        raise ValueError("cache node count must be >= 0")
    inner = tree.inner_count()
    hot = np.zeros(min(k, inner), np.int32)
    slot = np.zeros(inner, np.int32)
    n = load().cg_select_cached_nodes(ptr(tree.usage, C.c_int64), inner, int(k), ptr(hot, C.c_int32),
                                      ptr(slot, C.c_int32))
    if n < 0:
        check(_lib.CG_ERR_INVALID_ARGUMENT)
    return CacheSelection(hot[:n].copy(), slot)


# --------------------------------------------------------------------------- model
class Model:
    """model.hpp:25-62: syn0 (V x D) input vectors, syn1 ((V-1) x D) node rows."""

    def __init__(self, vocab_size: int, dim: int, syn0: np.ndarray | None = None, syn1: np.ndarray | None = None):
        if vocab_size < 2:
            raise ValueError("model needs a vocabulary of at least two words")
        if dim < 1:
            raise ValueError("vector dimension must be >= 1")
        self.syn0 = syn0 if syn0 is not None else np.zeros((vocab_size, dim), np.float32)
        self.syn1 = syn1 if syn1 is not None else np.zeros((vocab_size - 1, dim), np.float32)

    def vocab_size(self) -> int:
        return int(self.syn0.shape[0])

    def dim(self) -> int:
        return int(self.syn0.shape[1])

    def input_vector(self, w: int) -> np.ndarray:
        return self.syn0[w]

    def node_weight(self, n: int) -> np.ndarray:
        return self.syn1[n]

    def input_matrix(self) -> np.ndarray:
        return self.syn0.reshape(-1)

    def weight_matrix(self) -> np.ndarray:
        return self.syn1.reshape(-1)

    def copy(self) -> "Model":
        return Model(self.vocab_size(), self.dim(), self.syn0.copy(), self.syn1.copy())


def init_model(vocab_size: int, dim: int, seed: int) -> Model:
    """model.hpp:66-72, bit-identical."""
    m = Model(vocab_size, dim)
    check(load().cg_init_model(vocab_size, dim, seed & 0xFFFFFFFFFFFFFFFF, ptr(m.syn0, C.c_float)))
    return m


def model_desc(vocab: Vocabulary, tree: HuffmanTree, selection: CacheSelection, keep: list) -> CgModelDesc:
    """Builds the C-ABI view; `keep` holds references so the arrays outlive the call."""
    counts = np.ascontiguousarray(vocab.counts, np.int64)
    hot = np.ascontiguousarray(selection.hot, np.int32)
    keep.extend([counts, hot, tree])
    d = CgModelDesc()
    d.vocab_size = vocab.size()
    d.counts = ptr(counts, C.c_int64)
    d.total_tokens = vocab.total_tokens()
    d.path_offsets = ptr(tree.offsets, C.c_int64)
    d.path_nodes = ptr(tree.nodes, C.c_int32)
    d.path_turns = ptr(tree.turns, C.c_uint8)
    d.node_usage = ptr(tree.usage, C.c_int64)
    d.hot_nodes = ptr(hot, C.c_int32) if hot.size else None
    d.hot_count = selection.size()
    return d


def _check_consistency(vocab: Vocabulary, tree: HuffmanTree, selection: CacheSelection) -> None:
    # trainer.hpp:256-260
    if vocab.size() != tree.leaf_count():
        raise ValueError("vocabulary and tree sizes disagree")
    if selection.inner_node_count() != tree.inner_count():
        raise ValueError("cache selection was built from a different tree")


# --------------------------------------------------------------------------- kernel-level API
class NodeCache:
    """trainer.hpp:75-138; state on the host, arithmetic (train_center/flush) on the GPU."""

    def __init__(self, selection: CacheSelection, dim: int, flush_interval: int):
        self.selection, self.dim, self.flush_interval = selection, dim, flush_interval
        k = max(selection.size(), 0)
        self.work = np.zeros((max(k, 1), dim), np.float32)
        self.snap = np.zeros((max(k, 1), dim), np.float32)
        self.flag = np.zeros(max(k, 1), np.uint8)
        self._since = 0

    def is_cached(self, slot: int) -> bool:
        return bool(self.flag[slot])

    def words_since_flush(self) -> int:
        return self._since

    def row(self, slot: int) -> np.ndarray:
        return self.work[slot]

    def original(self, slot: int) -> np.ndarray:
        return self.snap[slot]

    def acquire(self, slot: int, shared_row: np.ndarray) -> np.ndarray:
        if not self.flag[slot]:
            self.work[slot] = shared_row
            self.snap[slot] = shared_row
            self.flag[slot] = 1
        return self.work[slot]

    def flush(self, model: Model) -> None:
        if self.selection.size() > 0:
            check(load().cg_cache_flush(model.vocab_size(), self.dim, ptr(model.syn1, C.c_float),
                                        ptr(self.selection.hot, C.c_int32), self.selection.size(),
                                        ptr(self.work, C.c_float), ptr(self.snap, C.c_float),
                                        ptr(self.flag, C.c_uint8)))
        self._since = 0

    def note_center_trained(self) -> bool:
        self._since += 1
        return self._since >= self.flush_interval


def train_center(center: int, sentence: Sequence[int], center_pos: int, half_window: int, model: Model,
                 tree: HuffmanTree, selection: CacheSelection, cache: NodeCache, alpha: float,
                 sigmoid="table") -> int:
    """trainer.hpp:147-175 on the device. sigmoid: "table", "exact", a constant (all
    evaluated on the device) or any callable float -> float (called on the host once per
    path step, in path order, like the reference's SigmoidFn). Returns the number of
    sigmoid evaluations (= pairs x path length)."""
    if callable(sigmoid):
        sent = np.ascontiguousarray(np.asarray(sentence, np.int32))
        slot = np.ascontiguousarray(selection.slot, np.int32)
        cb = _lib.SIGMOID_FN(lambda x, _ctx: float(sigmoid(x)))
        calls = C.c_int64()
        check(load().cg_train_center_cb(
            int(center), ptr(sent, C.c_int32), sent.size, int(center_pos), int(half_window), model.vocab_size(),
            model.dim(), ptr(model.syn0, C.c_float), ptr(model.syn1, C.c_float), ptr(tree.offsets, C.c_int64),
            ptr(tree.nodes, C.c_int32), ptr(tree.turns, C.c_uint8),
            ptr(slot, C.c_int32) if selection.size() else None, selection.size(), ptr(cache.work, C.c_float),
            ptr(cache.snap, C.c_float), ptr(cache.flag, C.c_uint8), float(alpha), C.cast(cb, C.c_void_p), None,
            C.byref(calls)))
        return calls.value
    if isinstance(sigmoid, str):
        mode, const = {"table": 0, "exact": 1}[sigmoid], 0.0
    else:
        mode, const = 2, float(sigmoid)
    sent = np.ascontiguousarray(np.asarray(sentence, np.int32))
    slot = np.ascontiguousarray(selection.slot, np.int32)
    calls = C.c_int64()
    check(load().cg_train_center(
        int(center), ptr(sent, C.c_int32), sent.size, int(center_pos), int(half_window), model.vocab_size(),
        model.dim(), ptr(model.syn0, C.c_float), ptr(model.syn1, C.c_float), ptr(tree.offsets, C.c_int64),
        ptr(tree.nodes, C.c_int32), ptr(tree.turns, C.c_uint8), ptr(slot, C.c_int32) if selection.size() else None,
        selection.size(), ptr(cache.work, C.c_float), ptr(cache.snap, C.c_float), ptr(cache.flag, C.c_uint8),
        float(alpha), mode, const, C.byref(calls)))
    return calls.value


# --------------------------------------------------------------------------- train()
def train(corpus, vocab: Vocabulary, tree: HuffmanTree, selection: CacheSelection, config: TrainConfig,
          stats: TrainStats | None = None, devices: Sequence[int] | None = None,
          sync_words: int = 1_000_000) -> Model:
    """cachegram::train (trainer.hpp:254-316) on the GPU.

    ``corpus`` is a corpus file path (tokenised on the GPU) or an in-vocabulary int32 id
    stream. ``devices`` (Hogwild mode) trains one model replica per listed GPU of this
    process, averaged over peer memory every ``sync_words`` words per replica."""
    config.validate()
    _check_consistency(vocab, tree, selection)
    mode = resolve_mode(config)
    if mode == "deterministic" and config.workers != 1:
        raise ValueError("deterministic mode replays the single-worker stream: set workers = 1")
    keep: list = []
    desc = model_desc(vocab, tree, selection, keep)
    cfg = config.to_c()
    m = Model(vocab.size(), config.dim)
    st = CgTrainStats()
    is_file = isinstance(corpus, (str, bytes)) or hasattr(corpus, "__fspath__")
    words = vocab.words_nul() \
        if is_file else b""
    ids = None if is_file else np.ascontiguousarray(np.asarray(corpus, np.int32))
    out0, out1 = ptr(m.syn0, C.c_float), ptr(m.syn1, C.c_float)
    if devices is not None:
        dev = np.ascontiguousarray(np.asarray(devices, np.int32))
        if is_file:  # tokenised on devices[0], sharded device to device
            check(load().cg_train_file_replicas(C.byref(cfg), MODES[mode], C.byref(desc), str(corpus).encode(), words,
                                                ptr(dev, C.c_int32), dev.size, int(sync_words), out0, out1,
                                                C.byref(st)))
        else:
            check(load().cg_train_replicas(C.byref(cfg), MODES[mode], C.byref(desc), ptr(ids, C.c_int32), ids.size,
                                           ptr(dev, C.c_int32), dev.size, int(sync_words), out0, out1, C.byref(st)))
    elif is_file:  # tokenised on the GPU, like the drop-in C++ train(corpus_path, ...)
        check(load().cg_train_file(C.byref(cfg), MODES[mode], C.byref(desc), str(corpus).encode(), words, out0, out1,
                                   C.byref(st)))
    else:
        check(load().cg_train(C.byref(cfg), MODES[mode], C.byref(desc), ptr(ids, C.c_int32), ids.size, out0, out1,
                              C.byref(st)))
    if stats is not None:
        stats.words_processed = st.words_processed
        stats.wall_seconds = st.wall_seconds
        stats.words_per_second = st.words_per_second
        stats.kernel_seconds = st.kernel_seconds
        stats.centers, stats.pairs, stats.steps = st.centers, st.pairs, st.steps
    return m


# --------------------------------------------------------------------------- sessions
class Session:
    """Device-resident training state (cg_session_*): tree, keep table, ids and model
    stay in HBM across passes; used by bench.py and the multi-GPU replica driver."""

    def __init__(self, vocab: Vocabulary, tree: HuffmanTree, selection: CacheSelection, config: TrainConfig,
                 device: int = 0, stream: int | None = None):
        config.validate()
        _check_consistency(vocab, tree, selection)
        self._keep: list = []
        self.config = config
        self.vocab_size = vocab.size()
        desc = model_desc(vocab, tree, selection, self._keep)
        cfg = config.to_c()
        self._h = C.c_void_p()
        check(load().cg_session_create(C.byref(cfg), MODES[resolve_mode(config)], C.byref(desc), device,
                                       C.c_void_p(stream) if stream else None, C.byref(self._h)))
        self.n_ids = 0

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            load().cg_session_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter teardown
            pass

    def upload_ids(self, ids: np.ndarray) -> None:
        ids = np.ascontiguousarray(ids, np.int32)
        check(load().cg_session_upload_ids(self._h, ptr(ids, C.c_int32), ids.size))
        self.n_ids = int(ids.size)

    def load_corpus(self, path: str, vocab: Vocabulary) -> int:
        """Tokenise a corpus file on the GPU straight into the session's id buffer."""
        words = vocab.words_nul()
        n = C.c_int64()
        check(load().cg_session_load_corpus(self._h, str(path).encode(), words, C.byref(n)))
        self.n_ids = int(n.value)
        return self.n_ids

    def upload_ids_device(self, ids_tensor) -> None:
        """Device-to-device copy of a CUDA int32 tensor of vocabulary ids."""
        assert ids_tensor.is_cuda and ids_tensor.dtype.itemsize == 4 and ids_tensor.is_contiguous()
        check(load().cg_session_upload_ids_device(self._h, C.c_void_p(ids_tensor.data_ptr()), ids_tensor.numel()))
        self.n_ids = int(ids_tensor.numel())

    def reset_model(self) -> None:
        check(load().cg_session_reset_model(self._h))

    def set_model(self, model: Model) -> None:
        check(load().cg_session_set_model(self._h, ptr(np.ascontiguousarray(model.syn0), C.c_float),
                                          ptr(np.ascontiguousarray(model.syn1), C.c_float)))

    def tune(self, blocks: int = 0, warps: int = 0, centers_per_warp: int = 0, smem_rows: int = -1,
             hot_flush_scale: float = 0.0, flush_centers: int = 0, min_cache_rows: int = 0, kernel: int = 0) -> None:
        """Hogwild kernel knobs (cg_tuning): smem_rows = cached rows held in shared memory
        (-1: 8); min_cache_rows = stability floor (0 auto, > 0 at least, < 0 none)."""
        t = _lib.CgTuning(blocks, warps, centers_per_warp, smem_rows, hot_flush_scale, flush_centers, min_cache_rows,
                          kernel)
        check(load().cg_session_tune(self._h, C.byref(t)))

    def train_range(self, epoch: int, begin: int, end: int, progress_base: int = 0,
                    progress_mult: int = 1) -> CgEpochStats:
        st = CgEpochStats()
        check(load().cg_session_train_range(self._h, epoch, begin, end, progress_base, progress_mult,
                                            C.byref(st)))
        return st

    def train(self) -> TrainStats:
        st = CgTrainStats()
        check(load().cg_session_train(self._h, C.byref(st)))
        return TrainStats(st.words_processed, st.wall_seconds, st.words_per_second, st.kernel_seconds,
                          st.centers, st.pairs, st.steps)

    def download(self, dim: int | None = None) -> Model:
        d = dim or self.config.dim
        m = Model(self.vocab_size, d)
        check(load().cg_session_download(self._h, ptr(m.syn0, C.c_float), ptr(m.syn1, C.c_float)))
        return m

    def model_buffer(self) -> tuple[int, int, int]:
        p, n, s = C.c_void_p(), C.c_size_t(), C.c_int32()
        check(load().cg_session_model_buffer(self._h, C.byref(p), C.byref(n), C.byref(s)))
        return int(p.value or 0), int(n.value), int(s.value)

    # ---- replica sync (cg_session_sync_*): deltas since the last sync, summed over replicas
    def sync_begin(self) -> None:
        check(load().cg_session_sync_begin(self._h))

    def sync_delta_tensor(self):
        """delta = model - snapshot, as a zero-copy torch view of the session's delta buffer
        (all-reduce it with SUM across replicas, then call sync_apply)."""
        import torch

        p, n = C.c_void_p(), C.c_size_t()
        check(load().cg_session_sync_delta(self._h, C.byref(p), C.byref(n)))

        class _Cai:
            __cuda_array_interface__ = {"shape": (int(n.value),), "typestr": "<f4", "data": (int(p.value), False),
                                        "version": 3}

        return torch.as_tensor(_Cai(), device="cuda")

    def sync_apply(self, n_replicas: int, words_per_replica: int) -> None:
        check(load().cg_session_sync_apply(self._h, int(n_replicas), int(words_per_replica)))

    def model_tensor(self):
        """Zero-copy torch view of the device model buffer (for all-reduce)."""
        import torch

        p, n, _ = self.model_buffer()

        class _Cai:
            __cuda_array_interface__ = {"shape": (n // 4,), "typestr": "<f4", "data": (p, False), "version": 3}

        return torch.as_tensor(_Cai(), device="cuda")


# --------------------------------------------------------------------------- model files
@dataclass
class LoadedEmbeddings:
    """model.hpp:147-157: the word list in id order and the input vectors (V x D)."""
    dim: int
    words: list
    vectors: np.ndarray

    def size(self) -> int:
        return len(self.words)

    def vector(self, w: int) -> np.ndarray:
        return self.vectors[w]


def _words_nul(words) -> bytes:
    return b"".join(w.encode() + b"\0" for w in words)


def _save(model: Model, vocab: Vocabulary, path: str, fmt: int) -> None:
    syn0 = np.ascontiguousarray(model.syn0, dtype=np.float32)
    words = _words_nul(vocab.word(w) for w in range(model.vocab_size()))
    check(load().cg_model_save(str(path).encode(), fmt, words, ptr(syn0, C.c_float), model.vocab_size(), model.dim()))


def save_text(model: Model, vocab: Vocabulary, path: str) -> None:
    """model.hpp:119-130 ("V D" header, "word v1 ... vD" rows with %.6f)."""
    _save(model, vocab, path, _lib.CG_FORMAT_TEXT)


def save_binary(model: Model, vocab: Vocabulary, path: str) -> None:
    """model.hpp:132-144 ("word " + D little-endian float32 + newline per row)."""
    _save(model, vocab, path, _lib.CG_FORMAT_BINARY)


def to_embeddings(model: Model, vocab: Vocabulary) -> LoadedEmbeddings:
    """model.hpp:159-168."""
    return LoadedEmbeddings(model.dim(), [vocab.word(w) for w in range(vocab.size())],
                            np.array(model.syn0, dtype=np.float32, copy=True))


def _load(path: str, fmt: int) -> LoadedEmbeddings:
    lib = load()
    h = C.c_void_p()
    check(lib.cg_model_load(str(path).encode(), fmt, C.byref(h)))
    try:
        v, d, nb = C.c_int32(), C.c_int32(), C.c_int64()
        check(lib.cg_model_file_info(h, C.byref(v), C.byref(d), C.byref(nb)))
        buf = C.create_string_buffer(int(nb.value) + 1)
        vec = np.empty((v.value, d.value), dtype=np.float32)
        check(lib.cg_model_file_export(h, buf, ptr(vec, C.c_float)))
        words = [w.decode("utf-8", "surrogateescape") for w in buf.raw[: nb.value].split(b"\0")[: v.value]]
        return LoadedEmbeddings(d.value, words, vec)
    finally:
        lib.cg_model_file_close(h)


def load_embeddings_binary(path: str) -> LoadedEmbeddings:
    return _load(path, _lib.CG_FORMAT_BINARY)


def load_embeddings_text(path: str) -> LoadedEmbeddings:
    return _load(path, _lib.CG_FORMAT_TEXT)


def load_embeddings(path: str) -> LoadedEmbeddings:
    """Either format (model.hpp:249-274 auto-detection)."""
    return _load(path, _lib.CG_FORMAT_AUTO)


# --------------------------------------------------------------------------- evaluation
class Embeddings:
    """Device-resident unit-normalised rows (AnalogySolver's table, eval.hpp:91-103).
    Built from host vectors, or zero-copy from a device pointer (e.g. a session's syn0)."""

    def __init__(self, vectors: np.ndarray | None = None, *, rows: int | None = None, dim: int | None = None,
                 device_ptr: int | None = None, row_stride: int | None = None, device: int = -1):
        lib = load()
        self._h = C.c_void_p()
        if device_ptr is not None:
            check(lib.cg_embeddings_create_device(C.c_void_p(device_ptr), int(rows), int(dim), int(row_stride or dim),
                                                  int(device), C.byref(self._h)))
            self.rows, self.dim = int(rows), int(dim)
        else:
            v = np.ascontiguousarray(vectors, dtype=np.float32)
            r = v.shape[0] if rows is None else int(rows)
            self.rows, self.dim = r, int(v.shape[1] if dim is None else dim)
            check(lib.cg_embeddings_create(ptr(v, C.c_float), r, self.dim, int(device), C.byref(self._h)))

    def normalized(self) -> np.ndarray:
        out = np.empty((self.rows, self.dim), dtype=np.float32)
        check(load().cg_embeddings_normalized(self._h, ptr(out, C.c_float)))
        return out

    def analogy(self, abc: np.ndarray) -> np.ndarray:
        """abc: (n, 3) ids -> (n,) answers (eval.hpp:117-136)."""
        q = np.ascontiguousarray(abc, dtype=np.int32).reshape(-1, 3)
        out = np.full(q.shape[0], -1, dtype=np.int32)
        check(load().cg_analogy_answer(self._h, ptr(q, C.c_int32), q.shape[0], ptr(out, C.c_int32)))
        return out

    def nearest(self, queries: np.ndarray, k: int = 10) -> tuple[np.ndarray, np.ndarray]:
        """Exact cosine top-k (self excluded, ties to the lower id): ids (n, k), scores (n, k)."""
        q = np.ascontiguousarray(queries, dtype=np.int32).reshape(-1)
        ids = np.empty((q.size, k), dtype=np.int32)
        sc = np.empty((q.size, k), dtype=np.float32)
        check(load().cg_nearest(self._h, ptr(q, C.c_int32), q.size, int(k), ptr(ids, C.c_int32), ptr(sc, C.c_float)))
        return ids, sc

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                load().cg_embeddings_destroy(self._h)
            except Exception:  # interpreter teardown
                pass
            self._h = None


@dataclass
class AnalogyQuestion:
    a: str
    b: str
    c: str
    d: str
    section: int = 0


@dataclass
class QuestionSet:
    sections: list = field(default_factory=list)
    questions: list = field(default_factory=list)


def _tokens(line: str) -> list:
    return [t for t in line.replace("\t", " ").replace("\r", " ").replace("\v", " ").replace("\f", " ").split(" ") if t]


def load_questions(path: str) -> QuestionSet:
    """eval.hpp:43-80: ": name" opens a section; other non-blank lines hold 4 words."""
    try:
        f = open(path, "rb")
    except OSError as e:
        raise OSError(f"cannot open question file: {path}") from e
    qs = QuestionSet()
    cur = -1
    with f:
        for no, raw in enumerate(f.read().decode("utf-8", "surrogateescape").split("\n"), start=1):
            tok = _tokens(raw)
            if not tok:
                continue
            if tok[0].startswith(":"):
                parts = [t for t in [tok[0][1:], *tok[1:]] if t]
                qs.sections.append(" ".join(parts) or "(unnamed)")
                cur = len(qs.sections) - 1
                continue
            if len(tok) != 4:
                raise _lib.ParseError(f"{path}:{no}: expected 4 words per question, got {len(tok)}")
            if cur < 0:
                qs.sections.append("(no section)")
                cur = 0
            low = [t.translate(str.maketrans("ABCDEFGHIJKLMNOPQRSTUVWXYZ", "abcdefghijklmnopqrstuvwxyz")) for t in tok]
            qs.questions.append(AnalogyQuestion(*low, section=cur))
    return qs


class AnalogySolver:
    """eval.hpp:85-150: 3CosAdd over the restrict_top most frequent words, on the GPU."""

    def __init__(self, emb: LoadedEmbeddings, restrict_top: int):
        self.size = min(emb.size(), restrict_top) if restrict_top > 0 else emb.size()
        self.table = Embeddings(emb.vectors[: self.size], rows=self.size, dim=emb.dim)
        self._index = {}
        for w in range(self.size):
            self._index.setdefault(emb.words[w], w)

    def vocab_size(self) -> int:
        return self.size

    def id_of(self, word: str) -> int:
        return self._index.get(word, -1)

    def answer(self, a: int, b: int, c: int) -> int:
        return int(self.table.analogy(np.array([[a, b, c]]))[0])


@dataclass
class SectionResult:
    name: str
    attempted: int = 0
    skipped: int = 0
    correct: int = 0

    def accuracy(self):
        return None if self.attempted == 0 else self.correct / self.attempted


@dataclass
class EvalReport:
    sections: list = field(default_factory=list)
    total: SectionResult = field(default_factory=lambda: SectionResult("TOTAL"))


def evaluate(emb: LoadedEmbeddings, questions: QuestionSet, restrict_top: int, threads: int = 1) -> EvalReport:
    """eval.hpp:165-225, every resolvable question answered in one device batch."""
    solver = AnalogySolver(emb, restrict_top)
    rep = EvalReport([SectionResult(n) for n in questions.sections])
    abc, want, sec = [], [], []
    for q in questions.questions:
        ids = [solver.id_of(x) for x in (q.a, q.b, q.c, q.d)]
        if min(ids) < 0:
            rep.sections[q.section].skipped += 1
            rep.total.skipped += 1
            continue
        abc.append(ids[:3])
        want.append(ids[3])
        sec.append(q.section)
    got = solver.table.analogy(np.array(abc, dtype=np.int32).reshape(-1, 3)) if abc else np.empty(0, np.int32)
    for g, w, s in zip(got, want, sec):
        for r in (rep.sections[s], rep.total):
            r.attempted += 1
            r.correct += int(g == w)
    return rep
