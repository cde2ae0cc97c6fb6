"""Copy the gpu_evidence_{a,b,c}.sh outputs (gpurun_out/ev, evb, evc) into
profiles/ under the round-1 names, tagging the ncu summaries with the
workload bench.py looks them up by."""
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

A, B, C = (os.path.join(ROOT, "gpurun_out", x) for x in ("ev", "evb", "evc"))
P = os.path.join(ROOT, "profiles")


def last_json(path):
    return [l for l in open(path).read().strip().splitlines() if l.strip().startswith("{")][-1]


copies = {os.path.join(A, "bench_default.json"): "r1_bench_default.json",
          os.path.join(A, "bench_reference.json"): "r1_bench_reference.json"}
for T in (1, 256):
    copies[os.path.join(C, f"bench_ep1_large128_T{T}.json")] = f"r1_bench_ep1_large128_T{T}.json"
    for pre in ("base64", "large128"):
        copies[os.path.join(C, f"bench_res_{pre}_T{T}.json")] = f"r1_bench_resident_{pre}_T{T}.json"
for src, dst in copies.items():
    open(os.path.join(P, dst), "w").write(last_json(src) + "\n")
for s in ("base64_resident", "large128_resident", "base128_offloaded", "large128_offloaded"):
    shutil.copy(os.path.join(A, f"sweep_{s}.jsonl"), os.path.join(P, f"r1_sweep_{s}.jsonl"))
shutil.copy(os.path.join(B, "launches_default.csv"), os.path.join(P, "r1_launches_default.csv"))
d = json.load(open(os.path.join(B, "ncu_summary.json")))
d["workload"] = bench.workload_name("large128", "offloaded", 256)
d["note"] = ("Round 1 (final kernel: one persistent tcgen05 launch per block). Command: python bench.py --steps 1 "
             "--warmup 1 --no-cpu-baseline (Switch-Large-128, experts offloaded, pre-gated, T=256, bf16) - the default "
             "bench workload. Launch list: ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, "
             "serialised: compare shares; gen_kernel is the one-off weight generation before the timed region). Full "
             "captures: ncu --set full --clock-control none --import-source on -k regex:block_gemm -s 30 -c 1 (one "
             "block launch: up + down + dense phases) and -k regex:route_kernel -s 30 -c 1. ffn = the block launch "
             "bench.py times as 'experts'. tools/gpu_evidence_b.sh.")
json.dump(d, open(os.path.join(P, "r1_ncu_summary.json"), "w"), indent=1)
shutil.copy(os.path.join(B, "ncu_summary.md"), os.path.join(P, "r1_ncu_summary.md"))
for pre in ("base64", "large128"):
    for T in (1, 256):
        d = json.load(open(os.path.join(B, f"ncu_summary_resident_{pre}_T{T}.json")))
        d["workload"] = bench.workload_name(pre, "resident", T)
        d["note"] = (f"Round 1. python bench.py --preset {pre} --placement resident --tokens {T} --steps 1 --warmup 1 "
                     "--no-cpu-baseline under ncu --set full -k regex:block_gemm -s 20 -c 1: one block launch incl. "
                     "the fused routing role (serialised and cache-flushed by ncu: no PDL overlap, cold L2). "
                     "tools/gpu_evidence_b.sh.")
        json.dump(d, open(os.path.join(P, f"r1_ncu_summary_resident_{pre}_T{T}.json"), "w"), indent=1)
        shutil.copy(os.path.join(B, f"ncu_summary_resident_{pre}_T{T}.md"),
                    os.path.join(P, f"r1_ncu_summary_resident_{pre}_T{T}.md"))
print("collected")
