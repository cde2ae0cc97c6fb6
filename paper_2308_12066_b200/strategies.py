"""The four placement strategies of the reference, executed on the B200.

The reference's `simulate` (scheduler.py:220-410) compares resident_only,
on_demand, prefetch_all and pre_gated on a virtual clock.  Here the same four
run for real: the math on the sm_100a kernels, the migrations as DMA on a
copy stream, and every number measured from CUDA events.  Results use the
reference's definitions and file formats:

* avg MoE-block latency excludes each iteration's block 0
  (scheduler.py:391-397); a block's latency is the time between the ends
  of consecutive blocks' dense layers (scheduler.py:374-379);
* tokens/sec = iterations * T / total time (scheduler.py:398, times T);
* peak fast-tier bytes = the measured HBM ledger peak (pinned gates+dense
  plus live expert slots), Eq. 1 for pre_gated (tiers.py:68-86);
* the CSV trio block_lats.csv / throughputs.csv / peak_mems.csv
  (harness.py:227-282) and the Timeline JSONL (scheduler.py:147-156).

    python -m paper_2308_12066_b200.strategies --preset base128 --tokens 1 --iterations 4 --out results/
"""

from __future__ import annotations

import argparse
import json
import os
from dataclasses import dataclass

import torch

from .core import DeviceModel, ModelConfig, token_inputs

STRATEGIES = ("resident_only", "on_demand", "prefetch_all", "pre_gated")
PRESETS = {  # presets.py:64-70 full-size dims
    "base8": dict(d_model=768, d_ff=3072, num_blocks=12, num_experts=8),
    "base64": dict(d_model=768, d_ff=3072, num_blocks=12, num_experts=64),
    "base128": dict(d_model=768, d_ff=3072, num_blocks=12, num_experts=128),
    "base256": dict(d_model=768, d_ff=3072, num_blocks=12, num_experts=256),
    "large128": dict(d_model=1024, d_ff=4096, num_blocks=24, num_experts=128),
}


@dataclass
class Metrics:
    """scheduler.py:159-167, measured."""

    avg_moe_block_latency_s: float
    tokens_per_sec: float
    peak_fast_bytes: int
    per_block_latencies_s: list
    total_time_s: float
    iterations: int
    h2d_bytes: int


def block_latencies(events: list) -> tuple[list, float]:
    """Per-block latencies of one iteration from its timeline, and its span."""
    dense = sorted((e for e in events if e["label"] == "non_moe"), key=lambda e: e["block"])
    start = min(e["start_s"] for e in events)
    end = max(e["end_s"] for e in events)
    lats, prev = [], start
    for e in dense:
        lats.append(e["end_s"] - prev)
        prev = e["end_s"]
    return lats, end - start


def measure(model: DeviceModel, x: torch.Tensor, iterations: int, include_first_block: bool = False,
            warmup: int = 1) -> tuple[Metrics, list]:
    for _ in range(warmup):
        model.decoder_iteration(x)
    torch.cuda.synchronize()
    per_block, total, h2d, peak, timelines = [], 0.0, 0, 0, []
    for _ in range(iterations):
        model.set_timeline(True)
        model.reset_stats()
        model.decoder_iteration(x)
        torch.cuda.synchronize()
        ev = model.timeline()
        st = model.stats()
        lats, span = block_latencies(ev)
        per_block.append(lats)
        total += span
        h2d += st["h2d_bytes"]
        if model.placement == "resident":
            peak = max(peak, st["pinned_hbm_bytes"] + _resident_expert_bytes(model))
        else:
            peak = max(peak, st["ledger_peak_bytes"])
        timelines.append(ev)
    model.set_timeline(False)
    flat = [v for lats in per_block for v in (lats if include_first_block or len(lats) == 1 else lats[1:])]
    T = x.shape[0]
    m = Metrics(avg_moe_block_latency_s=sum(flat) / len(flat), tokens_per_sec=iterations * T / total,
                peak_fast_bytes=int(peak), per_block_latencies_s=per_block, total_time_s=total,
                iterations=iterations, h2d_bytes=h2d)
    return m, timelines


def _resident_expert_bytes(model: DeviceModel) -> int:
    c = model.config
    sw = 2 if model.dtype in ("bf16", "bfloat16") else 4
    rec = (2 * c.d_model * c.d_ff * sw + 255) // 256 * 256
    return c.num_blocks * c.num_experts * rec


def write_csv(rows: list, out_dir: str) -> list:
    """harness.py:227-282 CSV trio (model, strategy, sweep_value, value)."""
    os.makedirs(out_dir, exist_ok=True)
    files = {"block_lats.csv": ("avg_block_latency_s", "avg_moe_block_latency_s"),
             "throughputs.csv": ("tokens_per_sec", "tokens_per_sec"),
             "peak_mems.csv": ("peak_bytes", "peak_fast_bytes")}
    paths = []
    for fname, (col, attr) in files.items():
        lines = [f"model,strategy,sweep_value,{col}"]
        for r in rows:
            lines.append(",".join((r["model"], r["strategy"], r["sweep_value"], repr(r[attr]))))
        path = os.path.join(out_dir, fname)
        with open(path, "w") as fh:
            fh.write("\n".join(lines) + "\n")
        paths.append(path)
    return paths


def run(config: ModelConfig, T: int, iterations: int, out_dir: str | None = None, label: str = "model",
        strategies=STRATEGIES, dtype: str = "bf16") -> dict:
    x = token_inputs(config, T)
    results, rows = {}, []
    offl = None
    for strat in strategies:
        if strat == "resident_only":
            model = DeviceModel(config, dtype=dtype, placement="resident", max_tokens=T)
        else:
            if offl is None:
                offl = DeviceModel(config, dtype=dtype, placement="offloaded", max_tokens=T)
            model = offl
            model.set_strategy(strat)
        metrics, timelines = measure(model, x, iterations)
        results[strat] = metrics
        rows.append({"model": label, "strategy": strat, "sweep_value": str(T), **metrics.__dict__})
        if out_dir:
            os.makedirs(out_dir, exist_ok=True)
            with open(os.path.join(out_dir, f"timeline_{strat}.jsonl"), "w") as fh:
                for ev in timelines[-1]:
                    fh.write(json.dumps(ev) + "\n")
        if model is not offl:
            model.close()
    if offl is not None:
        offl.close()
    if out_dir:
        write_csv(rows, out_dir)
    return results


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--preset", choices=sorted(PRESETS), default="base128")
    ap.add_argument("--tokens", type=int, default=1)
    ap.add_argument("--iterations", type=int, default=4)
    ap.add_argument("--out", default=None)
    ap.add_argument("--strategies", default=",".join(STRATEGIES))
    args = ap.parse_args()
    cfg = ModelConfig(top_k=1, activation_level=1, **PRESETS[args.preset])
    res = run(cfg, args.tokens, args.iterations, args.out, label=args.preset,
              strategies=tuple(args.strategies.split(",")))
    summary = {s: {"avg_block_ms": m.avg_moe_block_latency_s * 1e3, "tokens_per_sec": m.tokens_per_sec,
                   "peak_gb": m.peak_fast_bytes / 1e9, "h2d_gb_per_iter": m.h2d_bytes / m.iterations / 1e9}
               for s, m in res.items()}
    if "pre_gated" in res:
        pg = res["pre_gated"].avg_moe_block_latency_s
        for s in ("on_demand", "prefetch_all", "resident_only"):
            if s in res:
                summary[s]["block_latency_vs_pre_gated"] = res[s].avg_moe_block_latency_s / pg
    print(json.dumps({"preset": args.preset, "tokens": args.tokens, "iterations": args.iterations,
                      "strategies": summary}))


if __name__ == "__main__":
    main()
