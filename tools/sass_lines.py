"""Aggregate ncu per-SASS warp samples (tools/gpu/gpu_ncu_source.sh) by CUDA
source line, using nvdisasm --print-line-info of the same build.

  python tools/sass_lines.py SASS_CSV KERNEL_SYMBOL [--file route_common] [--top 40]
"""
import argparse
import collections
import csv
import glob
import os
import re
import subprocess
import tempfile

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("symbol")
ap.add_argument("--lib", default=os.path.join(os.path.dirname(__file__), "..", "paper_2308_12066_b200", "_build",
                                              "libpgmoe.so"))
ap.add_argument("--file", default="")
ap.add_argument("--top", type=int, default=40)
a = ap.parse_args()

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(a.lib)], cwd=tmp, capture_output=True)
lines = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    out = subprocess.run(["nvdisasm", "--print-line-info", cub], capture_output=True, text=True).stdout
    start = out.find(".text." + a.symbol + ":")
    if start < 0:
        continue
    end = out.find(".section", start)
    cur = None
    for l in out[start:end if end > 0 else None].splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
        if m:
            lines[int(m.group(1), 16)] = (cur, m.group(2).strip())
rows = list(csv.reader(open(a.csv)))
hdr = rows[0]
ia, iall, inot = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Warp Stall Sampling (Not-issued Samples)")
stalls = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_")]
base = min(int(r[ia], 16) for r in rows[1:])
# the first sampled instruction may not be offset 0: align on the first row's text
first = min(rows[1:], key=lambda r: int(r[ia], 16))
for off, (loc, txt) in sorted(lines.items()):
    if txt.split(";")[0].split() == first[1].split():
        base -= off
        break
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
total = 0
for r in rows[1:]:
    off = int(r[ia], 16) - base
    loc = lines.get(off, (None, ""))[0]
    n = int(r[iall] or 0)
    total += n
    e = agg[loc]
    e[0] += n
    e[1] += int(r[inot] or 0)
    for i, h in stalls:
        if i < len(r) and r[i] not in ("", "0"):
            e[2][h] += int(float(r[i]))
print(f"total samples {total}")
sel = [(k, v) for k, v in agg.items() if k and a.file in k[0]]
for k, v in sorted(sel, key=lambda kv: -kv[1][0])[:a.top]:
    print(f"{k[0]}:{k[1]:5d} {v[0]:7d} {v[1]:7d}  " + " ".join(f"{h[6:]}={c}" for h, c in v[2].most_common(3)))
