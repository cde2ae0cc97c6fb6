"""The HBM expert cache's index follows the reference's LIFO/LFU/LRU rules
(cache.py:49-103): replayed against outcomes recorded from moesim.ExpertCache
(tests/golden/cache.json, written by gen_golden.py)."""

import ctypes
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "cache.json")


def test_cache_replay_matches_reference():
    from paper_2308_12066_b200 import _lib
    L = _lib.load()
    cases = json.load(open(GOLD))["data"]
    assert len(cases) == 45
    pol = {"lifo": 1, "lfu": 2, "lru": 3}
    for c in cases:
        b = np.array(c["blocks"], dtype=np.int32)
        e = np.array(c["experts"], dtype=np.int32)
        hit = np.zeros(b.size, dtype=np.int32)
        ev = np.zeros(b.size, dtype=np.int32)
        _lib.check(L.pgmoe_cache_replay(pol[c["policy"]], c["capacity_records"], b.ctypes.data, e.ctypes.data,
                                        b.size, hit.ctypes.data, ev.ctypes.data))
        assert hit.tolist() == c["hit"], (c["policy"], c["capacity_records"], c["skew"])
        assert ev.tolist() == c["n_evicted"]


def test_zipf_trace_hits_more_than_uniform():
    cases = json.load(open(GOLD))["data"]
    rate = {(c["skew"], c["policy"], c["capacity_records"]): np.mean(c["hit"]) for c in cases}
    assert rate[(1.4, "lru", 40)] > rate[(0.0, "lru", 40)]
