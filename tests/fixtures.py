"""Deterministic fixture corpora for the tests.

``make_zipf_corpus`` restates the reference test utility's generator
(tests/testutil.hpp:78-101: words ``w<i>``, p ~ 1/(rank+3), splitmix64 floats,
lower_bound on the normalised cumulative sum) so the fixtures the reference's own
acceptance and trainer tests use (e.g. 200 KB / 2000 types / seed 4242 for
acceptance.cpp:268) can be regenerated here byte for byte.
"""
from __future__ import annotations

import bisect

import numpy as np

M64 = (1 << 64) - 1


class SplitMix:
    def __init__(self, seed: int):
        self.s = seed & M64

    def next_u64(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_float(self) -> float:
        return float(np.float32(self.next_u64() >> 40) * np.float32(1.0 / 16777216.0))

    def next_below(self, n: int) -> int:
        return self.next_u64() % n


def make_zipf_corpus(min_bytes: int, types: int, seed: int) -> str:
    total = 0.0
    cum = []
    for i in range(types):
        total += 1.0 / float(i + 3)
        cum.append(total)
    cum = [c / total for c in cum]
    rng = SplitMix(seed)
    out = []
    size = 0
    while size < min_bytes:
        u = rng.next_float()
        w = bisect.bisect_left(cum, u)
        if w >= types:
            w = types - 1
        tok = f"w{w} "
        out.append(tok)
        size += len(tok)
    s = "".join(out)
    return s[:-1] if s else s


def write(path, text: str) -> str:
    with open(path, "w") as f:
        f.write(text)
    return str(path)
