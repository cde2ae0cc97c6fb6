python - <<'PY'
import sys, os, json, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2308_12066_b200 as P
from paper_2308_12066_b200 import _lib
from paper_2308_12066_b200._rng import token_batch
L = _lib.load()
cfg = P.ModelConfig(top_k=1, activation_level=1, seed=0, d_model=768, d_ff=3072, num_blocks=12, num_experts=64)
m = P.DeviceModel(cfg, dtype="bf16", placement="resident", max_tokens=1)
x = torch.from_numpy(token_batch(0, 768, 1)).cuda(); y = torch.empty_like(x)
pr = torch.zeros((1 << 15, 32), dtype=torch.int64, device="cuda"); pb = torch.zeros((1 << 15, 32), dtype=torch.int64, device="cuda")
_lib.check(L.pgmoe_debug_set_probe(0, pr.data_ptr(), 1 << 15)); _lib.check(L.pgmoe_debug_set_probe(1, pb.data_ptr(), 1 << 15))
for it in range(4):
    pb.zero_(); m.decoder_iteration(x, out=y); torch.cuda.synchronize()
b = pb.cpu().numpy()
t0 = b[148:296, 0][b[148:296, 0] > 0].min()
rows = b[148:296]
for c in list(range(0, 14)) + [24, 60, 100, 147]:
    r = rows[c]
    print(c, " ".join(f"{n}={(r[s]-t0)/1e3:.2f}" for s, n in [(0,'entry'),(1,'prolog'),(2,'gate0'),(25,'r_pdl'),(26,'r_log'),(27,'sel0'),(23,'sums'),(24,'stored'),(28,'sel1'),(29,'perm'),(30,'trig'),(6,'ph0'),(7,'ph1'),(4,'gate2'),(8,'ph2'),(9,'exit')] if r[s] > 0))
PY
