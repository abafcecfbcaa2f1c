#!/usr/bin/env python
"""Corpus ingest (cg_ingest.cu) timed against the host reader.

Writes a Zipf corpus as text (default: the C2 shape, 17M tokens, 71k types), then times
  * vocabulary: the reference's build_vocabulary_file (oracle/_ref, when present), the
    drop-in's host builder (cg_corpus_open) and the GPU counter (cg_corpus_open_gpu);
  * id stream: the host reader (cg_corpus_read_ids) and the GPU tokeniser
    (cg_corpus_read_ids_gpu),
checking that the GPU results equal the host ones.

  python tools/ingest_bench.py [--tokens 17000000 --types 71000]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_lib as O  # noqa: E402
from paper_1606_07822_b200 import api  # noqa: E402


def timed(f):
    t0 = time.perf_counter()
    r = f()
    return r, time.perf_counter() - t0


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--tokens", type=int, default=17_000_000)
    p.add_argument("--types", type=int, default=71_000)
    p.add_argument("--zipf", type=float, default=1.05)
    a = p.parse_args()
    rng = np.random.default_rng(2)
    ranks = np.minimum(rng.zipf(a.zipf, a.tokens), a.types) - 1
    words = np.array([b"w%d" % i for i in range(a.types)], dtype=object)
    out = {"tokens": a.tokens, "types": a.types}
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "corpus.txt")
        with open(path, "wb") as f:
            for s in range(0, a.tokens, 1_000_000):
                t = words[ranks[s:s + 1_000_000]]
                f.write(b"\n".join(b" ".join(t[i:i + 1000].tolist()) for i in range(0, t.size, 1000)) + b"\n")
        out["bytes"] = os.path.getsize(path)
        api.build_vocabulary_file(path, 1, device=0)  # warm-up (context, pools)
        gv, t_gv = timed(lambda: api.build_vocabulary_file(path, 1, device=0))
        hv, t_hv = timed(lambda: api.build_vocabulary_file(path, 1))
        out["vocab"] = {"gpu_s": t_gv, "host_s": t_hv, "equal": gv.words == hv.words and
                        bool(np.array_equal(gv.counts, hv.counts))}
        if O.ref_available():
            h, t_rv = timed(lambda: O.ref().ref_open_file(path.encode(), 1))  # vocab + Huffman tree
            O.ref().ref_close(h)
            out["vocab"]["reference_vocab_and_tree_s"] = t_rv
        api.read_id_stream(path, hv, device=0)
        gi, t_gi = timed(lambda: api.read_id_stream(path, hv, device=0))
        hi, t_hi = timed(lambda: api.read_id_stream(path, hv))
        out["ids"] = {"gpu_s": t_gi, "host_s": t_hi, "gpu_words_per_s": a.tokens / t_gi,
                      "host_words_per_s": a.tokens / t_hi, "equal": bool(np.array_equal(gi, hi)),
                      "note": "gpu includes file read, H2D, tokenise + lookup, D2H of the id stream"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
