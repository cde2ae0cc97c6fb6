"""Summarise ncu captures into profiles/ (run here, on the CPU box).

    python tools/summarize_ncu.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
        --out profiles/r1_ncu_summary --label ffn=grouped_gemm --label route=route_kernel

Writes <out>.json (machine readable; bench.py reads `kernels.<label>.dram_bytes_per_launch`
for the roofline `traffic` field) and <out>.md (tables)."""

from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import subprocess

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
]


def _scale(v: float, unit: str) -> float:
    """ncu units -> bytes / seconds."""
    u = unit.lower().split("/")[0].strip()
    table = {"gbyte": 1e9, "mbyte": 1e6, "kbyte": 1e3, "byte": 1.0, "tbyte": 1e12,
             "s": 1.0, "second": 1.0, "ms": 1e-3, "msecond": 1e-3, "us": 1e-6, "usecond": 1e-6,
             "ns": 1e-9, "nsecond": 1e-9}
    return v * table.get(u, 1.0)


def read_rep(path: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                try:
                    d[m] = _scale(float(r[i].replace(",", "")), units[i])
                except ValueError:
                    d[m] = r[i]
        res.append(d)
    return res


def read_launches(path: str) -> dict:
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        agg[r[ki]].append(_scale(float(r[vi].replace(",", "")), r[ui]))
    return agg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--launches", default=None)
    ap.add_argument("--out", required=True)
    ap.add_argument("--label", action="append", default=[], help="label=substring of the kernel name")
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    labels = dict(x.split("=", 1) for x in args.label)
    caps = [c for r in args.rep for c in read_rep(r)]
    summary = {"note": args.note, "captures": caps, "kernels": {}, "launch_shares": {}}
    for lab, sub in labels.items():
        # "substr@0+1": one logical launch made of several captures (summed),
        # e.g. the expert FFN = the up- and the down-projection GEMM
        pick = None
        if "@" in sub:
            sub, idx = sub.split("@")
            pick = [int(i) for i in idx.split("+")]
        ks = [c for c in caps if sub in c["kernel"]]
        if not ks:
            continue
        if pick is not None:
            ks = [ks[i] for i in pick if i < len(ks)]
            rd = sum(c.get("dram__bytes_read.sum", 0) for c in ks)
            wr = sum(c.get("dram__bytes_write.sum", 0) for c in ks)
            n = 1
        else:
            n = len(ks)
            rd = sum(c.get("dram__bytes_read.sum", 0) for c in ks) / n
            wr = sum(c.get("dram__bytes_write.sum", 0) for c in ks) / n
        summary["kernels"][lab] = {
            "kernel": ks[0]["kernel"], "captures": n,
            "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
            "duration_us_cold": sum(c.get("gpu__time_duration.sum", 0) for c in ks) / n * 1e6,
            "captures_used": len(ks),
            "dram_pct_peak": sum(c.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0) for c in ks) / n,
            "tensor_pipe_pct": sum(c.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0)
                                   for c in ks) / n,
            "registers": ks[0].get("launch__registers_per_thread"),
            "smem_dynamic": ks[0].get("launch__shared_mem_per_block_dynamic"),
        }
    md = [f"# ncu summary — {args.out}", "", args.note, ""]
    if args.launches:
        agg = read_launches(args.launches)
        tot = sum(sum(v) for v in agg.values())
        md += ["## Launch list (ncu --metrics gpu__time_duration.sum; cold-cache, serialised — compare shares)", "",
               "| kernel | launches | avg us | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            share = sum(v) / tot
            summary["launch_shares"][k] = {"n": len(v), "avg_us": sum(v) / len(v) * 1e6, "share": share}
            md.append(f"| `{k[:90]}` | {len(v)} | {sum(v) / len(v) * 1e6:.2f} | {share * 100:.1f}% |")
        md.append("")
    md += ["## Full captures (ncu --set full)", "",
           "| kernel | us | DRAM read MB | DRAM write MB | DRAM % peak | tensor pipe % | regs | smem KB |",
           "|---|---|---|---|---|---|---|---|"]
    for c in caps:
        md.append("| `{}` | {:.1f} | {:.2f} | {:.2f} | {:.1f} | {:.2f} | {} | {:.1f} |".format(
            c["kernel"][:70], c.get("gpu__time_duration.sum", 0) * 1e6, c.get("dram__bytes_read.sum", 0) / 1e6,
            c.get("dram__bytes_write.sum", 0) / 1e6,
            c.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 0),
            c.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0),
            c.get("launch__registers_per_thread"), c.get("launch__shared_mem_per_block_dynamic", 0) / 1e3))
    with open(args.out + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)
    with open(args.out + ".md", "w") as fh:
        fh.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    main()
