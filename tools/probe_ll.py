"""Device-side timeline of the low-latency decode launch (decode_ll.cu probe
slots): per block, per event, [min, median, max] over the CTAs that stamp it,
in microseconds from the first CTA's entry.  Debug tool.

  make -C paper_2308_12066_b200/csrc EXTRA=-DPGMOE_LL_PROBE   # stamps exist only in a probe build
  python tools/probe_ll.py --preset base64 --tokens 1
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

PRESETS = {"base64": dict(d_model=768, d_ff=3072, num_blocks=12, num_experts=64),
           "large128": dict(d_model=1024, d_ff=4096, num_blocks=24, num_experts=128)}
EVENTS = ["decided", "up_in", "up_done", "dn_in", "dn_done", "selected", "dense_in", "dense_done"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--preset", default="base64", choices=sorted(PRESETS))
    ap.add_argument("--tokens", type=int, default=1)
    args = ap.parse_args()
    os.environ["PGMOE_NO_GRAPH"] = "1"  # eager launches: the probe pointer is read per launch
    L = _lib.load()
    cfg = P.ModelConfig(top_k=1, activation_level=1, seed=0, **PRESETS[args.preset])
    m = P.DeviceModel(cfg, dtype="bf16", placement="resident", max_tokens=args.tokens)
    x = torch.from_numpy(token_batch(0, cfg.d_model, args.tokens)).cuda()
    for _ in range(3):
        m.decoder_iteration(x)
    torch.cuda.synchronize()
    pb = torch.zeros((4096, 48), dtype=torch.int64, device="cuda")
    _lib.check(L.pgmoe_debug_set_probe(1, pb.data_ptr(), 4096))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    m.decoder_iteration(x)
    b.record()
    torch.cuda.synchronize()
    _lib.check(L.pgmoe_debug_set_probe(1, None, 0))
    arr = pb.cpu().numpy().astype(np.int64)
    rows = arr[arr[:, 0] > 0]
    t0 = rows[:, 0].min()
    out = {"preset": args.preset, "T": args.tokens, "ctas": int(rows.shape[0]),
           "launch_us_events": round(a.elapsed_time(b) * 1e3, 2),
           "entry_max": round(float((rows[:, 0].max() - t0) / 1e3), 2),
           "exit": [round(float((rows[:, 41][rows[:, 41] > 0].min() - t0) / 1e3), 2),
                    round(float((rows[:, 41].max() - t0) / 1e3), 2)],
           "blocks": []}
    for blk in range(4):
        ent = {"block": blk}
        for k, nm in enumerate(EVENTS):
            v = rows[:, 1 + 8 * blk + k]
            v = v[v > 0]
            if v.size:
                r = (v - t0) / 1e3
                ent[nm] = [round(float(r.min()), 2), round(float(np.median(r)), 2), round(float(r.max()), 2)]
        out["blocks"].append(ent)
    # block 2, compute group of each CTA: cycles waiting for the weight slice, staging, in the
    # GEMV, in the epilogue; pieces (medians / maxima over CTAs that had pieces)
    acc = {}
    for ph, nm in enumerate(["up", "dn"]):
        n = rows[:, 45 + ph]
        sel = n > 0
        acc[nm] = {"pieces_med": float(np.median(n[sel])) if sel.any() else 0}
        for k, q in enumerate(["wait", "stage", "gemv", "epi"]):
            v = rows[sel, 33 + 4 * ph + k]
            acc[nm][q] = [int(np.median(v)), int(v.max())] if v.size else None
    out["block2_cycles"] = acc
    print(json.dumps(out))


if __name__ == "__main__":
    main()
