"""Host-side synthetic token inputs (rng.py:15-93 restated, vectorised over
independent substreams with numpy uint64 arithmetic).  Used to build the
benchmark's synthetic batches; the weights are generated on the device
(csrc/rng.cu)."""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def _mix64(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def derive_seed(base: int, *tags: int) -> int:
    x = base & MASK64
    for t in tags:
        x = _mix64((x + GOLDEN) & MASK64)
        x = _mix64(x ^ (t & MASK64))
    return x


def _rotl(x: np.ndarray, k: int) -> np.ndarray:
    return (x << np.uint64(k)) | (x >> np.uint64(64 - k))


def fill_many(seeds, n: int, lo: float = -0.1, hi: float = 0.1) -> np.ndarray:
    """[len(seeds)][n] fp64: Xoshiro256StarStar(seed).fill(n, lo, hi) per row."""
    seeds = [int(s) & MASK64 for s in seeds]
    st = []
    for s in seeds:
        row = []
        for _ in range(4):
            s = (s + GOLDEN) & MASK64
            row.append(_mix64(s))
        st.append(row)
    S = np.array(st, dtype=np.uint64).T.copy()  # [4][B]
    s0, s1, s2, s3 = S[0], S[1], S[2], S[3]
    out = np.empty((len(seeds), n), dtype=np.float64)
    span = hi - lo
    with np.errstate(over="ignore"):
        for i in range(n):
            r = _rotl(s1 * np.uint64(5), 7) * np.uint64(9)
            t = s1 << np.uint64(17)
            s2 ^= s0
            s3 ^= s1
            s1 ^= s2
            s0 ^= s3
            s2 ^= t
            s3 = _rotl(s3, 45)
            u = (r >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
            out[:, i] = lo + span * u
    return out


def fill_f32(seed: int, n: int) -> np.ndarray:
    return fill_many([seed], n)[0].astype(np.float32)


def token_batch(seed: int, d: int, T: int, offset: int = 0) -> np.ndarray:
    """fp32 [T][d]: token t (global index offset+t) = default_input for 0,
    else Xoshiro(derive_seed(seed, 5, t)).fill(d)."""
    seeds = [derive_seed(seed, 5) if (offset + t) == 0 else derive_seed(seed, 5, offset + t) for t in range(T)]
    if T == 0:
        return np.zeros((0, d), dtype=np.float32)
    return fill_many(seeds, d).astype(np.float32)
