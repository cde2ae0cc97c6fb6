"""Batch-size sweep (BASELINE configs[2], configs[3]): one offloaded model,
T = 1..256 sequences, pre-gated migration.  Per T: tokens/s, per-block
latency and its PCIe roofline fraction, measured H2D rate,
peak HBM (Eq. 1 and event ledger).  One JSON line per T.

    python tools/sweep.py --preset large128 --tokens 1,2,4,8,16,32,64,128,256 --steps 3
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2308_12066_b200 as P  # noqa: E402
from bench import PRESETS, measure_pcie_gbs  # noqa: E402
from paper_2308_12066_b200._rng import token_batch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", choices=sorted(PRESETS), default="large128")
    ap.add_argument("--tokens", default="1,2,4,8,16,32,64,128,256")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--placement", default="offloaded")
    ap.add_argument("--strategy", default="pre_gated")
    args = ap.parse_args()
    Ts = [int(t) for t in args.tokens.split(",")]
    cfg = P.ModelConfig(top_k=1, activation_level=1, seed=0, **PRESETS[args.preset])
    t0 = time.perf_counter()
    m = P.DeviceModel(cfg, dtype="bf16", placement=args.placement, max_tokens=max(Ts))
    if args.placement == "offloaded":
        m.set_strategy(args.strategy)
    setup = time.perf_counter() - t0
    pcie = measure_pcie_gbs(torch)
    rec = 2 * cfg.d_model * cfg.d_ff * 2
    nb = cfg.num_blocks
    for T in Ts:
        x = torch.from_numpy(token_batch(0, cfg.d_model, T)).cuda()
        y = torch.empty_like(x)
        for _ in range(args.warmup):
            m.decoder_iteration(x, out=y)
        torch.cuda.synchronize()
        m.reset_stats()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            m.decoder_iteration(x, out=y)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / args.steps
        st = m.stats()
        h2d_per_step = st["h2d_bytes"] / args.steps
        nact_avg = h2d_per_step / rec / nb if args.placement == "offloaded" else None
        block_ms = ms / nb
        t_pcie = (h2d_per_step / nb) / (pcie * 1e9) * 1e3 if args.placement == "offloaded" else None
        print(json.dumps({
            "preset": args.preset, "placement": args.placement, "strategy": args.strategy, "tokens": T,
            "tokens_per_s": T / (ms * 1e-3), "ms_per_step": ms, "per_block_ms": block_ms,
            "pcie_roofline_ms": t_pcie, "pcie_frac": (t_pcie / block_ms) if t_pcie else None,
            "n_act_avg": nact_avg, "pcie_measured_gbs": pcie,
            "h2d_gbs_while_running": (h2d_per_step / (ms * 1e-3) / 1e9) if args.placement == "offloaded" else None,
            "peak_hbm_eq1": st["eq1_peak_bytes"], "peak_hbm_ledger": st["ledger_peak_bytes"],
            "route_fallbacks": st["route_fallbacks"], "setup_s": setup}), flush=True)
    m.close()


if __name__ == "__main__":
    main()
