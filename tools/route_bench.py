"""K1 (pgmoe_gate_forward) launch time, cluster form vs split-partials form.

`device_us`: first CTA entry -> permutation written (probe %globaltimer
stamps), launches separated by a synchronize; `graph_us_per_launch`: 200
back-to-back launches replayed from CUDA graphs, CUDA events (PDL lets each
launch stage its gate slice during the previous tail).  The gate is L2-resident
after the first launch in both forms.  Prints one JSON line per point.

  python tools/route_bench.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_12066_b200 as P  # noqa: E402
from paper_2308_12066_b200._rng import token_batch  # noqa: E402
from oracle import oracle as og  # noqa: E402

SLOTS = {0: "entry", 1: "pdl", 10: "x", 2: "partials", 7: "selred", 3: "sums", 8: "ranked", 4: "selected",
         5: "perm0", 11: "scan", 6: "perm1"}
SHAPES = {"large128": (1024, 128), "base64": (768, 64), "base128": (768, 128)}


def main():
    from paper_2308_12066_b200 import _lib
    L = _lib.load()
    torch.cuda.set_device(0)
    rows = 1 << 14
    pb = torch.zeros((rows, 48), dtype=torch.int64, device="cuda")
    for name, (d, E) in SHAPES.items():
        G = og.weights(og.derive_seed(0, og.TAG_PRE_GATE, 1, -1), d, E, "bf16")
        Gt = torch.from_numpy(G.view(np.int16)).view(torch.bfloat16).cuda()
        for T in (1, 8, 64, 256):
            x = torch.from_numpy(token_batch(0, d, T)).cuda()
            row = {"shape": name, "d": d, "E": E, "T": T}
            ids = {}
            for mode in ("cluster", "split"):
                os.environ["PGMOE_ROUTE_KERNEL"] = mode
                r = P.route(x, Gt, 1)
                for _ in range(5):
                    P.route(x, Gt, 1, out=r)
                torch.cuda.synchronize()
                # device duration of one launch: first CTA entry -> permutation written
                # (probe stamps, %globaltimer), launches separated by a synchronize
                dur, slots = [], []
                for _ in range(30):
                    pb.zero_()
                    _lib.check(L.pgmoe_debug_set_probe(0, pb.data_ptr(), rows))
                    P.route(x, Gt, 1, out=r)
                    torch.cuda.synchronize()
                    _lib.check(L.pgmoe_debug_set_probe(0, None, 0))
                    a = pb.cpu().numpy()
                    ent = a[:, 0][a[:, 0] > 0]
                    fin = a[:, 6][a[:, 6] > 0]
                    dur.append((fin.max() - ent.min()) / 1e3)
                    sl = {}
                    for k, nm in SLOTS.items():
                        v = a[:, k][a[:, k] > 0]
                        if v.size:
                            sl[nm] = (v.max() - ent.min()) / 1e3
                    c = np.nonzero(a[:, 13] > 0)[0]
                    if c.size:
                        c = c[0]
                        sl["sm_mhz"] = (a[c, 13] - a[c, 12]) / max(1, a[c, 6] - a[c, 0]) * 1e3
                    slots.append(sl)
                # back-to-back launches replayed from a CUDA graph (no host gaps; PDL overlap)
                g = torch.cuda.CUDAGraph()
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    P.route(x, Gt, 1, out=r)
                    torch.cuda.synchronize()
                    with torch.cuda.graph(g, stream=s):
                        for _ in range(50):
                            P.route(x, Gt, 1, out=r)
                g.replay()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(4):
                    g.replay()
                b.record()
                torch.cuda.synchronize()
                row[mode + "_device_us"] = round(float(np.median(dur)), 2)
                row[mode + "_slots_us"] = {nm: round(float(np.median([x[nm] for x in slots if nm in x])), 2)
                                           for nm in list(SLOTS.values()) + ["sm_mhz"] if any(nm in x for x in slots)}
                row[mode + "_graph_us_per_launch"] = round(a.elapsed_time(b) * 1e3 / 200, 2)
                ids[mode] = r.ids.clone()
            row["ids_equal"] = bool(torch.equal(ids["cluster"], ids["split"]))
            print(json.dumps(row), flush=True)
    os.environ.pop("PGMOE_ROUTE_KERNEL", None)


if __name__ == "__main__":
    main()
