"""Synthetic routing traces: gen_routing_trace (core.py:436-479) for T tokens.

The reference draws, per (iteration, block), top_k distinct experts from a
Zipf(skew) distribution P(i) ~ 1/(i+1)^skew with one xoshiro256** stream
seeded derive_seed(seed, 6), ids sorted ascending, weights 1/top_k.  The
batched form draws the T tokens of a block one after another from the same
stream (token-major within a block), so at T = 1 the ids are the
reference's own trace value for value (tests/test_traces.py checks this
against moesim).  The result feeds DeviceModel.decoder_iteration(...,
supplied=...) — the `supplied_decisions` path — e.g. for the skewed-trace
expert-cache study (tools/cache_study.py; cache.py:49-103).
"""

from __future__ import annotations

import bisect

import numpy as np

from ._rng import MASK64, derive_seed
from .errors import ConfigError

TAG_TRACE = 6  # core.py:22-28


class Xoshiro256:
    """rng.py:43-68 xoshiro256** (scalar), seeded through SplitMix64."""

    def __init__(self, seed: int):
        s = seed & MASK64
        st = []
        for _ in range(4):
            s = (s + 0x9E3779B97F4A7C15) & MASK64
            z = s
            z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
            z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
            st.append(z ^ (z >> 31))
        self.s = st

    def next_u64(self) -> int:
        s0, s1, s2, s3 = self.s
        x = (s1 * 5) & MASK64
        out = ((((x << 7) | (x >> 57)) & MASK64) * 9) & MASK64
        t = (s1 << 17) & MASK64
        s2 ^= s0
        s3 ^= s1
        s1 ^= s2
        s0 ^= s3
        s2 ^= t
        s3 = ((s3 << 45) | (s3 >> 19)) & MASK64
        self.s = [s0, s1, s2, s3]
        return out

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * (2.0 ** -53)


def zipf_cdf(num_experts: int, skew: float) -> list:
    """Cumulative Zipf(skew) over experts 0..E-1, last edge forced to 1.0."""
    w = [(i + 1) ** -skew for i in range(num_experts)]
    total = sum(w, 0.0)  # CPython's float sum, as the reference computes it
    cdf, acc = [], 0.0
    for v in w:
        acc += v / total
        cdf.append(acc)
    cdf[-1] = 1.0
    return cdf


def routing_trace(config, iterations: int, skew: float, seed: int, tokens: int = 1):
    """(ids int32 [iterations][nb][T][k], w float32 [same]) of a Zipf(skew)
    synthetic trace; see the module docstring for the batched draw order."""
    if iterations < 1:
        raise ConfigError("iterations must be >= 1")
    if skew < 0:
        raise ConfigError("skew must be >= 0")
    E, k, nb = config.num_experts, config.top_k, config.num_blocks
    rng = Xoshiro256(derive_seed(seed, TAG_TRACE))
    cdf = zipf_cdf(E, skew)

    def draw() -> int:
        # first expert whose cumulative edge exceeds u (the reference's scan)
        return min(bisect.bisect_right(cdf, rng.uniform()), E - 1)

    ids = np.empty((iterations, nb, tokens, k), dtype=np.int32)
    for it in range(iterations):
        for b in range(nb):
            for t in range(tokens):
                if k == E:
                    ids[it, b, t] = np.arange(E)
                    continue
                picked: set = set()
                while len(picked) < k:
                    picked.add(draw())
                ids[it, b, t] = sorted(picked)
    w = np.full(ids.shape, np.float32(1.0 / k), dtype=np.float32)
    return ids, w
