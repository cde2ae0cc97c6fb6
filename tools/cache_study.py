"""Skewed-trace expert-cache study on the B200 (the paper's caching study,
PAPER.md:607-611; reference harness.py:367-407 + cache.py:49-103).

An offloaded pre-gated model replays a Zipf(skew) synthetic routing trace
(paper_2308_12066_b200.traces, gen_routing_trace batched) through the
`supplied_decisions` path, with the HBM expert cache off or under the
reference's LIFO / LFU / LRU victim rules at several capacities.  Measured
per (skew, T, policy, capacity): PCIe bytes per iteration, cache hit rate,
average block latency (blocks 1..nb-1, scheduler.py:391-397) and tokens/s,
over the trace's iterations after a warm-up iteration (which also warms the
cache).  One JSON line per point.

  python tools/cache_study.py --preset large128 --tokens 1 --skews 0,1.0,1.5
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2308_12066_b200.core import DeviceModel, ModelConfig, token_inputs  # noqa: E402
from paper_2308_12066_b200.strategies import PRESETS, block_latencies  # noqa: E402
from paper_2308_12066_b200.traces import routing_trace  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="large128", choices=sorted(PRESETS))
    ap.add_argument("--tokens", type=int, default=1)
    ap.add_argument("--iterations", type=int, default=3, help="measured iterations (after one warm-up)")
    ap.add_argument("--skews", default="0,1.0,1.5")
    ap.add_argument("--capacities", default="0.1,0.25,0.5")
    ap.add_argument("--policies", default="lru,lfu,lifo")
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    cfg = ModelConfig(top_k=1, activation_level=1, seed=0, **PRESETS[args.preset])
    T, nb = args.tokens, cfg.num_blocks
    rec = (2 * cfg.d_model * cfg.d_ff * 2 + 255) // 256 * 256  # bf16 expert record (W1 + W2)
    model = DeviceModel(cfg, dtype="bf16", placement="offloaded", max_tokens=T)
    x = token_inputs(cfg, T)
    y = torch.empty_like(x)
    points = [("none", 0.0)] + [(p, float(c)) for p in args.policies.split(",") for c in args.capacities.split(",")]
    for skew in (float(s) for s in args.skews.split(",")):
        ids, w = routing_trace(cfg, args.iterations + 1, skew, args.seed, tokens=T)
        ids_d = torch.from_numpy(ids).cuda()
        w_d = torch.from_numpy(w).cuda()
        for policy, cap in points:
            model.set_cache(policy, cap)
            model.decoder_iteration(x, out=y, supplied=(ids_d[0], w_d[0]))  # warm-up (and cache warm-up)
            torch.cuda.synchronize()
            model.reset_stats()
            lats, span = [], 0.0
            model.set_timeline(True)
            for it in range(1, args.iterations + 1):
                model.set_timeline(True)
                model.decoder_iteration(x, out=y, supplied=(ids_d[it], w_d[it]))
                torch.cuda.synchronize()
                bl, sp = block_latencies(model.timeline())
                lats += bl[1:]
                span += sp
            model.set_timeline(False)
            st = model.stats()
            acc = st["cache_hits"] + st["cache_misses"]
            nact = sum(len(set(ids[it, b].reshape(-1).tolist())) for it in range(1, args.iterations + 1)
                       for b in range(nb))
            print(json.dumps({
                "preset": args.preset, "tokens": T, "skew": skew, "policy": policy, "capacity_fraction": cap,
                "cache_gb": round(st["cache_bytes"] / 1e9, 3),
                "pcie_gb_per_iteration": round(st["h2d_bytes"] / args.iterations / 1e9, 4),
                "routed_expert_gb_per_iteration": round(nact * rec / args.iterations / 1e9, 4),
                "hit_rate": round(st["cache_hits"] / acc, 4) if acc else None,
                "avg_block_ms": round(sum(lats) / len(lats) * 1e3, 4),
                "tokens_per_s": round(args.iterations * T / span, 3),
                "iterations": args.iterations}), flush=True)
    model.close()


if __name__ == "__main__":
    main()
