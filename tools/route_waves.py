"""K1 cluster form at one shape: per-CTA probe stamps -> entry / partials /
sums spread (two waves show as a bimodal entry time).  Debug tool."""
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
from oracle import oracle as og  # noqa: E402


def main():
    d, E = int(sys.argv[1]), int(sys.argv[2])
    L = _lib.load()
    pb = torch.zeros((1 << 14, 48), dtype=torch.int64, device="cuda")
    G = og.weights(og.derive_seed(0, og.TAG_PRE_GATE, 1, -1), d, E, "bf16")
    Gt = torch.from_numpy(G.view(np.int16)).view(torch.bfloat16).cuda()
    for T in [int(t) for t in sys.argv[3:]]:
        x = torch.from_numpy(token_batch(0, d, T)).cuda()
        r = P.route(x, Gt, 1)
        for _ in range(5):
            P.route(x, Gt, 1, out=r)
        torch.cuda.synchronize()
        pb.zero_()
        _lib.check(L.pgmoe_debug_set_probe(0, pb.data_ptr(), 1 << 14))
        P.route(x, Gt, 1, out=r)
        torch.cuda.synchronize()
        _lib.check(L.pgmoe_debug_set_probe(0, None, 0))
        a = pb.cpu().numpy()
        rows = a[a[:, 0] > 0]
        t0 = rows[:, 0].min()
        out = {"d": d, "E": E, "T": T, "ctas": int(rows.shape[0])}
        for k, nm in {0: "entry", 1: "pdl", 10: "x", 2: "partials", 3: "sums", 4: "selected", 6: "perm1"}.items():
            v = rows[:, k][rows[:, k] > 0]
            if v.size:
                q = np.percentile((v - t0) / 1e3, [0, 25, 50, 75, 100])
                out[nm] = [round(float(z), 2) for z in q]
        print(json.dumps(out))


if __name__ == "__main__":
    main()
