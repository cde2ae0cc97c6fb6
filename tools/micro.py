"""Warm per-kernel timings (CUDA events, 200 back-to-back calls) of K1 / K2 /
K3 at Switch shapes, outside the decoder loop.  Prints one JSON line."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2308_12066_b200 as P  # noqa: E402
from paper_2308_12066_b200._rng import token_batch  # noqa: E402


def timeit(fn, n=200):
    """Device time per call: the call is captured once into a CUDA graph and
    replayed n times, so host launch overhead is excluded."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3  # us


def main():
    out = {}
    d, f, E = 1024, 4096, 128
    G = P.fill_weights(d, E, seed=0, tag=1, block=3, dtype="bf16")
    D = P.fill_weights(d, d, seed=0, tag=4, block=3, dtype="bf16")
    recs = torch.randn((E, 2 * f * d), device="cuda").to(torch.bfloat16) * 0.05
    for T in (1, 8, 64, 256):
        x = torch.from_numpy(token_batch(0, d, T)).cuda()
        r = P.DeviceRouting(T, E, 1)
        out[f"route_T{T}_us"] = timeit(lambda: P.route(x, G, 1, out=r))
        P.route(x, G, 1, out=r)
        torch.cuda.synchronize()
        yw = P.expert_ffn(x, r, recs, f, kernel="tcgen05")
        out[f"ffn_T{T}_us"] = timeit(lambda: P.expert_ffn(x, r, recs, f, kernel="tcgen05"), n=50)
        out[f"dense_T{T}_us"] = timeit(lambda: P.dense(yw, T, 1, D, kernel="tcgen05"))
        out[f"n_act_T{T}"] = r.n_act
    print(json.dumps(out))


if __name__ == "__main__":
    main()
