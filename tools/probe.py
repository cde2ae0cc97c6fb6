"""Device-side phase timeline of K1 (route) and the tcgen05 block kernel.

Installs probe buffers (pgmoe_debug_set_probe), captures one decoder
iteration, and prints every launch of it on one clock (%globaltimer, µs from
the first CTA entry): for each slot min / median / max over the launch's
CTAs.  Debug tool, not a benchmark.

  python tools/probe.py --preset base64 --placement resident --tokens 1
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_12066_b200 as P  # noqa: E402
from paper_2308_12066_b200 import _lib  # noqa: E402
from paper_2308_12066_b200._rng import token_batch  # noqa: E402

PRESETS = {
    "base64": dict(d_model=768, d_ff=3072, num_blocks=12, num_experts=64),
    "base128": dict(d_model=768, d_ff=3072, num_blocks=12, num_experts=128),
    "large128": dict(d_model=1024, d_ff=4096, num_blocks=24, num_experts=128),
}
ROUTE_SLOTS = {0: "entry", 1: "pdl", 2: "logits", 3: "sel0", 7: "selred", 8: "ranked", 4: "sel1", 5: "perm0",
               6: "perm1"}
BLOCK_SLOTS = {0: "entry", 1: "prolog", 2: "gate0", 3: "gate1", 4: "gate2", 5: "acc0", 6: "ph0", 7: "ph1",
               8: "ph2", 11: "lastld", 12: "accN", 13: "partN", 14: "fixN", 15: "endN",
               25: "r_pdl", 40: "r_xs", 41: "r_rows", 26: "r_logits", 27: "r_sel0", 35: "r_sx", 32: "r_red", 37: "s_load", 38: "s_cert", 39: "s_z", 33: "r_selt", 28: "r_sel1", 29: "r_perm",
               30: "r_trig", 9: "exit"}
ROWS = 1 << 15


def launches(buf, ctas_of):
    """Split the row buffer into launches (consecutive CTA groups)."""
    a = buf.cpu().numpy().astype(np.int64)
    out, r = [], 0
    for n in ctas_of:
        out.append(a[r:r + n])
        r += n
    return out


def stat(rows, slot, t0):
    v = rows[:, slot]
    v = v[v > 0]
    if not v.size:
        return None
    r = (v - t0) / 1e3
    return [round(float(r.min()), 2), round(float(np.median(r)), 2), round(float(r.max()), 2)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="base64", choices=sorted(PRESETS))
    ap.add_argument("--placement", default="resident")
    ap.add_argument("--tokens", type=int, default=1)
    ap.add_argument("--blocks", type=int, default=4, help="blocks of the iteration to print")
    ap.add_argument("--cta-detail", action="store_true")
    ap.add_argument("--no-fused-route", action="store_true", help="resident: separate K1 launches")
    args = ap.parse_args()
    L = _lib.load()
    cfg = P.ModelConfig(top_k=1, activation_level=1, seed=0, **PRESETS[args.preset])
    m = P.DeviceModel(cfg, dtype="bf16", placement=args.placement, max_tokens=args.tokens)
    if args.no_fused_route:
        m.set_fused_route(False)
    x = torch.from_numpy(token_batch(0, cfg.d_model, args.tokens)).cuda()
    y = torch.empty_like(x)
    pr = torch.zeros((ROWS, 48), dtype=torch.int64, device="cuda")
    pb = torch.zeros((ROWS, 48), dtype=torch.int64, device="cuda")
    for it in range(4):
        if it == 0 or args.placement != "resident":
            _lib.check(L.pgmoe_debug_set_probe(0, pr.data_ptr(), ROWS))
            _lib.check(L.pgmoe_debug_set_probe(1, pb.data_ptr(), ROWS))
        pr.zero_()
        pb.zero_()
        m.decoder_iteration(x, out=y)
        torch.cuda.synchronize()
    _lib.check(L.pgmoe_debug_set_probe(0, None, 0))
    _lib.check(L.pgmoe_debug_set_probe(1, None, 0))
    nb = cfg.num_blocks
    # route launches: block 0 conv gate + pre-gates of blocks 0..nb-2
    T = args.tokens
    tok = 1 if T < 64 else 2 if T < 128 else 4 if T < 256 else 8
    tiles = (T + tok - 1) / tok
    ra = pr.cpu().numpy().astype(np.int64)
    ba = pb.cpu().numpy().astype(np.int64)
    nr = int((ra[:, 0] > 0).sum())
    fused = m.stats()["fused_routes"] > 0
    n_route = 1 if fused else nb  # block 0's gate (+ every pre-gate unless fused into the block launch)
    route_ctas = nr // n_route
    rl = [ra[i * route_ctas:(i + 1) * route_ctas] for i in range(n_route)]
    bl = [ba[i * 148:(i + 1) * 148] for i in range(nb)]
    t0 = min(r[:, 0][r[:, 0] > 0].min() for r in rl + bl)
    res = {"preset": args.preset, "placement": args.placement, "T": T, "route_ctas": route_ctas,
           "iteration_us": round(float((max(b[:, 9].max() for b in bl) - t0) / 1e3), 2), "launches": []}
    order = [("route", 0, rl[0])]
    for b in range(nb):
        if b + 1 < nb and not fused:
            order.append(("route", b, rl[b + 1]))
        order.append(("block", b, bl[b]))
    res["fused_route"] = fused
    for kind, b, rows in order:
        if b >= args.blocks and b < nb - 1:
            continue
        slots = ROUTE_SLOTS if kind == "route" else BLOCK_SLOTS
        ent = {"kind": kind, "block": b}
        for s, name in slots.items():
            st = stat(rows, s, t0)
            if st:
                ent[name] = st
        res["launches"].append(ent)
        if args.cta_detail and kind == "block":
            # the slowest CTA of each phase
            for s in (6, 7, 8):
                v = rows[:, s]
                if (v > 0).any():
                    c = int(np.argmax(v))
                    res["launches"].append({"cta": c, "phase_slot": s, 
                                            "row": {BLOCK_SLOTS[k]: round(float((rows[c, k] - t0) / 1e3), 2)
                                                    for k in BLOCK_SLOTS if rows[c, k] > 0}})
    # effective SM clock over each block kernel CTA: d(clock64) / d(globaltimer)
    mhz = []
    for b in bl:
        ok = (b[:, 21] > 0) & (b[:, 22] > b[:, 21]) & (b[:, 9] > b[:, 0])
        if ok.any():
            mhz.append(float(np.median((b[ok, 22] - b[ok, 21]) / (b[ok, 9] - b[ok, 0]) * 1e3)))
    res["sm_mhz_in_block_kernel"] = [round(v) for v in mhz[:4]]
    # producer cycle counters of block 1's launch: gate waits / empty-stage waits / unit atomics / units
    b = bl[1]
    res["producer_us"] = {k: [round(float(np.percentile(b[:, s] / 1.86e3, q)), 1) for q in (0, 50, 100)]
                          for k, s in (("gate", 16), ("empty", 17), ("atomic", 18))}
    res["split_per_phase"] = [int(b[0, 23]), int(b[0, 24]), int(b[0, 31])]
    res["units_per_cta"] = [int(b[:, 19].min()), float(np.median(b[:, 19])), int(b[:, 19].max())]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
