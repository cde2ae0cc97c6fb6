"""Summarise a tools/gpu/gpu_r2_ll.sh output directory."""
import glob
import json
import sys

d = sys.argv[1]
print(open(f"{d}/t_ll.log").read().strip().splitlines()[-2:])
for fn in sorted(glob.glob(f"{d}/bench_*.json")):
    try:
        b = json.loads(open(fn).read().strip().splitlines()[-1])
    except Exception as e:
        print(fn, "ERR", e)
        continue
    print(fn.split("/")[-1], "us/blk", round(b["per_block_latency_all_blocks_ms"] * 1e3, 2), "tok/s", b["value"],
          "kfrac", b["roofline"]["frac"], "fallbacks", b["routing"]["serial_fallbacks"])
try:
    for ln in open(f"{d}/probe.jsonl"):
        p = json.loads(ln)
        print(p["preset"], p["T"], "launch_us", p["launch_us_events"])
        for blk in p["blocks"][1:3]:
            print("   blk", blk["block"], " ".join(f"{k}={v[1]}/{v[2]}" for k, v in blk.items() if k != "block"))
        print("   fine2", {k: v[1] for k, v in p["block2_fine"].items()})
except FileNotFoundError:
    pass
