#!/usr/bin/env python
"""Regenerates tests/golden/*.npz from the reference itself.

Runs in the build container only (needs /root/reference via oracle/_ref/libcgref.so,
the reference headers compiled unchanged). For each case: the fixture corpus is
written with the reference test utility's generator (tests/fixtures.py restates
testutil.hpp:78-101), the reference builds the vocabulary and tree from the file and
trains through its own cachegram::train() with workers = 1, and the vocabulary
counts, tree, selection and trained syn0/syn1 bits are stored. Small known-answer
vectors of the reference's scalar functions are stored alongside.
"""
import ctypes as C
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import fixtures as F  # noqa: E402
import oracle_lib as O  # noqa: E402

CASES = {
    "g1_small": (30000, 120, 21, dict(dim=16, window=3, min_count=2, sample=1e-3, iterations=2, cache_nodes=15,
                                      flush_interval=10, seed=7)),
    "g2_nosample": (40000, 200, 5, dict(dim=12, window=4, min_count=1, sample=0.0, iterations=2, cache_nodes=1024,
                                        flush_interval=7, seed=3)),
    "g3_fixture200k": (200 * 1024, 2000, 4242, dict(dim=24, window=5, min_count=5, sample=1e-3, alpha0=0.001,
                                                    iterations=1, cache_nodes=31, flush_interval=10, seed=11)),
    "g4_odd_dim": (50000, 300, 9, dict(dim=7, window=6, min_count=1, sample=1e-2, iterations=3, cache_nodes=1,
                                       flush_interval=1, seed=123)),
}


def main():
    assert O.ref_available(), "needs oracle/_ref/libcgref.so (build with make -C oracle)"
    with tempfile.TemporaryDirectory() as d:
        for name, (mb, types, seed, cfg) in CASES.items():
            path = F.write(Path(d) / "c.txt", F.make_zipf_corpus(mb, types, seed))
            h, counts, raws, total = O.ref_vocab_file(path, cfg["min_count"])
            t = O.ref_tree(h)
            hot = np.zeros(max(t.usage.size, 1), np.int32)
            slot = np.zeros(t.usage.size, np.int32)
            n = O.ref().ref_select(h, cfg["cache_nodes"], O._p(hot, C.c_int32), O._p(slot, C.c_int32))
            syn0, syn1, words, _ = O.ref_train(h, path, cfg)
            O.ref().ref_close(h)
            np.savez_compressed(HERE / f"{name}.npz", counts=counts, raws=raws, total=total, off=t.off, nodes=t.nodes,
                                turns=t.turns, usage=t.usage, hot=hot[:n], slot=slot, syn0=syn0, syn1=syn1,
                                words=words, corpus=np.array([mb, types, seed]),
                                cfg=np.array(repr(cfg)))
            print(name, "V", counts.size, "words", words)
    ref = O.ref()
    xs = np.linspace(-7, 7, 4001, dtype=np.float32)
    sig = np.array([ref.ref_sigmoid_value(float(x)) for x in xs], np.float32)
    u = np.zeros(64, np.uint64)
    f = np.zeros(64, np.float32)
    b = np.zeros(64, np.uint32)
    ref.ref_rng_stream(1, 64, O._p(u, C.c_uint64), O._p(f, C.c_float), 5, O._p(b, C.c_uint32))
    keep_args = np.array([(10, 1000, 1e-3), (1, 1000, 1e-3), (123456, 17000000, 1e-4), (7, 50, 1e-2)])
    keep = np.array([ref.ref_keep_probability(int(c), int(t), s) for c, t, s in keep_args])
    alpha_done = np.array([0, 1, 9999, 10000, 500000, 999999, 1000000, 5000000], np.uint64)
    alpha = np.array([ref.ref_update_alpha(int(x), 1000000, 0.025) for x in alpha_done], np.float32)
    i0 = np.zeros((13, 9), np.float32)
    i1 = np.zeros((12, 9), np.float32)
    ref.ref_init_model(13, 9, 42, O._p(i0, C.c_float), O._p(i1, C.c_float))
    np.savez_compressed(HERE / "scalars.npz", sig_x=xs, sig=sig, rng_u64=u, rng_float=f, rng_below5=b,
                        keep_args=keep_args, keep=keep, alpha_done=alpha_done, alpha=alpha, init_syn0=i0)
    print("scalars")


if __name__ == "__main__":
    main()
