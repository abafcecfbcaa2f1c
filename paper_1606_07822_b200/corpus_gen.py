"""Seeded synthetic corpora standing in for the benchmark inputs.

text8 and the analogy questions are not available, so every configuration of
BASELINE.json is generated: tokens ``w<rank>`` with ranks drawn i.i.d. from
p(k) ~ k^-s (k = 1..V), a newline every 1000 tokens (20 for C3; newlines are ordinary
separators to the reference, corpus.hpp:19-21), and for C3 a planted-cluster corpus
with a word -> cluster sidecar. Nothing from any public benchmark is reproduced.

The generator produces *raw* ids (rank - 1). ``vocab_from_raw`` applies the
reference's vocabulary rules (count >= min_count, descending count, first
occurrence on ties; corpus.hpp:97-124) and maps the stream to vocabulary ids.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .api import Vocabulary


@dataclass(frozen=True)
class CorpusConfig:
    name: str
    tokens: int
    vocab: int
    zipf_s: float
    dim: int
    window: int
    sample: float
    iterations: int
    seed: int
    line_every: int = 1000
    min_count: int = 5
    clusters: int = 0          # C3: planted clusters
    cluster_size: int = 0
    in_cluster: float = 0.0


# BASELINE.json "configs", in order (C1..C5). Unstated values take the reference
# defaults (trainer.hpp:25-35): min_count 5, alpha 0.025, sample 1e-3, K 31, u 10.
CONFIGS = {
    "c1": CorpusConfig("c1", 1_000_000, 10_000, 1.0, 100, 5, 1e-3, 1, 1, min_count=1),
    "c2": CorpusConfig("c2", 17_000_000, 71_000, 1.05, 200, 5, 1e-4, 1, 2),
    "c3": CorpusConfig("c3", 20_000_000, 50_000, 1.0, 128, 5, 1e-3, 3, 3, line_every=20, clusters=200,
                       cluster_size=250, in_cluster=0.7),
    "c4": CorpusConfig("c4", 100_000_000, 100_000, 1.0, 300, 10, 1e-4, 1, 4),
    "c5": CorpusConfig("c5", 1_000_000_000, 1_000_000, 1.2, 300, 5, 1e-5, 1, 5),
}


def zipf_cdf(vocab: int, s: float) -> np.ndarray:
    w = np.arange(1, vocab + 1, dtype=np.float64) ** (-s)
    c = np.cumsum(w)
    return c / c[-1]


def zipf_raw_ids(n: int, vocab: int, s: float, seed: int, chunk: int = 1 << 24) -> np.ndarray:
    """n raw ids in [0, vocab) with p(rank k) ~ k^-s, from numpy PCG64(seed)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    cdf = zipf_cdf(vocab, s)
    out = np.empty(n, dtype=np.int32)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        out[a:b] = np.minimum(np.searchsorted(cdf, rng.random(b - a), side="right"), vocab - 1)
    return out


def cluster_raw_ids(cfg: CorpusConfig) -> tuple[np.ndarray, np.ndarray]:
    """C3: each sentence of `line_every` tokens picks one of `clusters` clusters
    uniformly; each token is uniform inside it with prob `in_cluster`, else a global
    Zipf(s) draw over all ids. Returns (raw ids, cluster of every raw id)."""
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    v = cfg.clusters * cfg.cluster_size
    n_sent = cfg.tokens // cfg.line_every
    sent_cluster = rng.integers(0, cfg.clusters, size=n_sent)
    cl = np.repeat(sent_cluster, cfg.line_every)
    inside = rng.random(cl.size) < cfg.in_cluster
    local = rng.integers(0, cfg.cluster_size, size=cl.size)
    glob = np.minimum(np.searchsorted(zipf_cdf(v, cfg.zipf_s), rng.random(cl.size), side="right"), v - 1)
    raw = np.where(inside, cl * cfg.cluster_size + local, glob).astype(np.int32)
    cluster_of = (np.arange(v) // cfg.cluster_size).astype(np.int32)
    return raw, cluster_of


def generate(cfg: CorpusConfig, tokens: int | None = None) -> np.ndarray:
    n = cfg.tokens if tokens is None else tokens
    if cfg.clusters:
        raw, _ = cluster_raw_ids(cfg)
        return raw[:n]
    return zipf_raw_ids(n, cfg.vocab, cfg.zipf_s, cfg.seed)


def vocab_from_raw(raw: np.ndarray, min_count: int, space: int | None = None) -> tuple[Vocabulary, np.ndarray]:
    """Reference vocabulary rules over a raw-id stream. Returns (vocab, id stream)."""
    space = int(raw.max()) + 1 if space is None else space
    counts = np.bincount(raw, minlength=space).astype(np.int64)
    first = np.full(space, np.iinfo(np.int64).max, dtype=np.int64)
    uniq, idx = np.unique(raw, return_index=True)
    first[uniq] = idx
    alive = np.nonzero(counts >= max(min_count, 1))[0]
    order = alive[np.lexsort((first[alive], -counts[alive]))]
    rank = np.full(space, -1, dtype=np.int32)
    rank[order] = np.arange(order.size, dtype=np.int32)
    ids = rank[raw]
    ids = ids[ids >= 0]
    vocab = Vocabulary(counts[order], [f"w{r}" for r in order.tolist()], int(counts[order].sum()))
    vocab.raw_of_id = order.astype(np.int32)
    return vocab, np.ascontiguousarray(ids, dtype=np.int32)


def write_text(path: str, raw: np.ndarray, line_every: int = 1000, space: int | None = None) -> int:
    """Writes ``w<raw>`` tokens, space separated, newline every `line_every` tokens."""
    space = int(raw.max()) + 1 if space is None else space
    words = np.array([b"w%d" % i for i in range(space)], dtype=object)
    written = 0
    with open(path, "wb") as f:
        step = line_every * 1000
        for a in range(0, raw.size, step):
            toks = words[raw[a:a + step]]
            lines = [b" ".join(toks[i:i + line_every].tolist()) for i in range(0, toks.size, line_every)]
            blob = b"\n".join(lines) + b"\n"
            f.write(blob)
            written += len(blob)
    return written


# ---------------------------------------------------------------- device-side generation (C4/C5 scale)
def zipf_raw_ids_device(n: int, vocab: int, s: float, seed: int, device="cuda", chunk: int = 1 << 26):
    """Same distribution as zipf_raw_ids, drawn on the GPU with torch's Philox generator
    (1B tokens in seconds instead of minutes; not bit-identical to the numpy stream)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    cdf = torch.tensor(zipf_cdf(vocab, s), dtype=torch.float64, device=device)
    out = torch.empty(n, dtype=torch.int32, device=device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        u = torch.rand(b - a, generator=g, device=device, dtype=torch.float64)
        out[a:b] = torch.searchsorted(cdf, u, right=True).clamp_max_(vocab - 1).to(torch.int32)
    return out


def vocab_from_raw_device(raw, min_count: int, space: int, chunk: int = 1 << 26):
    """vocab_from_raw on a CUDA tensor; returns (Vocabulary, CUDA int32 id stream)."""
    import torch

    n = raw.numel()
    counts = torch.bincount(raw, minlength=space).to(torch.int64)
    first = torch.full((space,), n, dtype=torch.int64, device=raw.device)
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        idx = torch.arange(a, b, dtype=torch.int64, device=raw.device)
        first.scatter_reduce_(0, raw[a:b].long(), idx, reduce="amin")
    c = counts.cpu().numpy()
    f = first.cpu().numpy()
    alive = np.nonzero(c >= max(min_count, 1))[0]
    order = alive[np.lexsort((f[alive], -c[alive]))]
    rank = np.full(space, -1, dtype=np.int32)
    rank[order] = np.arange(order.size, dtype=np.int32)
    rank_t = torch.from_numpy(rank).to(raw.device)
    ids = rank_t[raw.long()]
    if order.size < space:
        ids = ids[ids >= 0]
    vocab = Vocabulary(c[order], [f"w{r}" for r in order.tolist()], int(c[order].sum()))
    vocab.raw_of_id = order.astype(np.int32)
    return vocab, ids.to(torch.int32).contiguous()
