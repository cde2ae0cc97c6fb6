"""A few K1 launches at one shape (ncu target): python tools/route_one.py <shape> <T> [split]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2308_12066_b200 as P  # noqa: E402
from paper_2308_12066_b200._rng import token_batch  # noqa: E402
from oracle import oracle as og  # noqa: E402

d, E = {"large128": (1024, 128), "base64": (768, 64)}[sys.argv[1]]
T = int(sys.argv[2])
if len(sys.argv) > 3:
    os.environ["PGMOE_ROUTE_KERNEL"] = sys.argv[3]
G = og.weights(og.derive_seed(0, og.TAG_PRE_GATE, 1, -1), d, E, "bf16")
Gt = torch.from_numpy(G.view(np.int16)).view(torch.bfloat16).cuda()
x = torch.from_numpy(token_batch(0, d, T)).cuda()
r = P.route(x, Gt, 1)
for _ in range(5):
    P.route(x, Gt, 1, out=r)
torch.cuda.synchronize()
print("ok", r.ids[:4].flatten().tolist())
