"""Summarise a gpu_quick.sh output directory (bench lines + probe timelines)."""
import json
import os
import sys

d = sys.argv[1]
for f in sorted(os.listdir(d)):
    if f.startswith("bench") and f.endswith(".json"):
        try:
            b = json.load(open(os.path.join(d, f)))
        except Exception as e:  # noqa: BLE001
            print(f, "unreadable", e)
            continue
        r = b.get("roofline", {})
        print(f"{f:34s} value={b.get('value')} block_ms={b.get('per_block_latency_ms')} "
              f"block_frac={b.get('block_roofline', {}).get('frac')} k2_frac={r.get('frac')} "
              f"k2_us={r.get('avg_launch_us')} phases={b.get('per_block_phase_ms')}")
p = os.path.join(d, "probe.jsonl")
if os.path.exists(p):
    for line in open(p):
        x = json.loads(line)
        print(x["preset"], "T", x["T"], "iteration_us", x["iteration_us"])
        for e in x["launches"]:
            if "kind" in e:
                keys = ["pdl", "logits", "sel0", "selred", "ranked", "sel1", "perm1"] if e["kind"] == "route" else \
                    ["entry", "gate0", "ph0", "gate1", "ph1", "r_pdl", "r_logits", "r_sel0", "r_sel1", "r_perm",
                     "gate2", "ph2", "exit"]
                print("   ", e["kind"], e["block"], " ".join(f"{k}={e[k][2] if k not in ('entry',) else e[k][0]}"
                                                         for k in keys if k in e))
