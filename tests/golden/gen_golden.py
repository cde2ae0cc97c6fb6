"""Generate the golden fixtures by running the REFERENCE itself.

Run in the development container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/gen_golden.py

It imports ``moesim`` (the unmodified reference package, read-only) and
records its outputs for fixed seeds.  Weights are produced by the
reference's own generator (rng.py / core.py:200-211) where that is cheap,
and for Switch-scale shapes they are fed through the reference's
``BlockParams(loaded=...)`` hook (core.py:185-211) after rounding to the
storage precision, exactly as the north star prescribes ("the reference is
fed the rounded values").  Floats are stored as ``float.hex`` strings so
the fixtures are bit-exact.
"""

from __future__ import annotations

import hashlib
import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", ".."))
sys.path.insert(0, "/root/reference/pkg/src")

import moesim  # noqa: E402  (the reference)
from moesim import core as mcore  # noqa: E402
from moesim.rng import SplitMix64, Xoshiro256StarStar, derive_seed  # noqa: E402

from oracle import oracle as og  # noqa: E402  (only for the rounded-weight feed)


def hx(v) -> str:
    return float(v).hex()


def hxl(vs) -> list[str]:
    return [float(v).hex() for v in vs]


def rng_fixture():
    sm = SplitMix64(0)
    out = {"splitmix_seed0": [hex(sm.next_u64()) for _ in range(4)]}
    xs = {}
    for seed in (0, 1, 42, 2**63, 0xDEADBEEF):
        g = Xoshiro256StarStar(seed)
        xs[hex(seed)] = [hex(g.next_u64()) for _ in range(50)]
    out["xoshiro"] = xs
    ds = []
    for base in (0, 7, 2**64 - 1):
        for tags in ((), (0,), (1, 2), (2, 1), (2, 3, 5), (4, 11, -1), (5,), (5, 255), (2, 23, 127)):
            ds.append({"base": hex(base), "tags": list(tags), "seed": hex(derive_seed(base, *tags))})
    out["derive_seed"] = ds
    out["fill_123"] = hxl(Xoshiro256StarStar(123).fill(64))
    out["fill_9_lohi"] = hxl(Xoshiro256StarStar(9).fill(32, -2.0, 2.0))
    # Full-scale generator pin: block 0 / expert 0 W1 of Switch-Base dims,
    # seed 0, straight from the reference generator (core.py:207-209).
    seed = derive_seed(0, mcore._TAG_W1, 0, 0)
    flat = Xoshiro256StarStar(seed).fill(3072 * 768)
    out["base_w1_b0_e0_sha256_f64le"] = hashlib.sha256(struct.pack(f"<{len(flat)}d", *flat)).hexdigest()
    f32 = np.asarray(flat, dtype=np.float64).astype(np.float32)
    out["base_w1_b0_e0_sha256_f32le"] = hashlib.sha256(f32.tobytes()).hexdigest()
    # default_input for the Switch dims (core.py:274-277)
    cfg = moesim.ModelConfig(d_model=1024, d_ff=4096, num_blocks=24, num_experts=128, top_k=1, seed=0)
    out["default_input_large"] = hxl(mcore.default_input(cfg))
    return out


def linalg_fixture():
    from moesim import linalg
    rng = Xoshiro256StarStar(12)
    cases = []
    for rows, cols in [(1, 1), (2, 7), (16, 3), (9, 33), (64, 24)]:
        mat = rng.fill_matrix(rows, cols, -1.0, 1.0)
        x = rng.fill(cols, -1.0, 1.0)
        xt = rng.fill(rows, -1.0, 1.0)
        cases.append({"mat": [hxl(r) for r in mat], "x": hxl(x), "xt": hxl(xt),
                      "matvec": hxl(linalg.matvec(mat, x)),
                      "matvec_columns": hxl(linalg.matvec_columns(mat, xt))})
    sm = []
    for n in (2, 3, 8, 100, 128):
        logits = rng.fill(n, -5.0, 5.0)
        sm.append({"logits": hxl(logits), "probs": hxl(linalg.softmax(logits))})
    return {"matvec": cases, "softmax": sm}


def gate_fixture():
    out = {}
    d = moesim.gate_forward([1.0], [[1.0, 0.0]], 1)
    out["hand_softmax"] = {"ids": list(d.expert_ids), "w": hxl(d.combine_weights)}
    d = moesim.gate_forward([1.0], [[0.5, 0.5, 0.5, 0.5]], 2)
    out["tie"] = {"ids": list(d.expert_ids), "w": hxl(d.combine_weights)}
    rng = Xoshiro256StarStar(21)
    cases = []
    for i in range(50):
        rows = 6 if i < 25 else 1 + int(rng.uniform() * 16)
        E = 8 if i < 25 else 2 + int(rng.uniform() * 40)
        k = 2 if i < 25 else 1 + int(rng.uniform() * min(E, 4))
        gate = rng.fill_matrix(rows, E, -1.0, 1.0)
        x = rng.fill(rows, -1.0, 1.0)
        r = moesim.gate_forward(x, gate, k)
        cases.append({"gate": [hxl(row) for row in gate], "x": hxl(x), "k": k,
                      "ids": list(r.expert_ids), "w": hxl(r.combine_weights)})
    out["random"] = cases
    # exact-tie rows: duplicated gate columns give bit-equal logits
    ties = []
    for i in range(10):
        E = 6 + i
        base = rng.fill_matrix(5, E, -1.0, 1.0)
        for row in base:
            row[E - 1] = row[1]
            row[3] = row[0]
        x = rng.fill(5, -1.0, 1.0)
        r = moesim.gate_forward(x, base, 2)
        ties.append({"gate": [hxl(row) for row in base], "x": hxl(x), "k": 2,
                     "ids": list(r.expert_ids), "w": hxl(r.combine_weights)})
    out["ties"] = ties
    return out


class RoundedLoaded(dict):
    """Lazy ``loaded`` mapping for BlockParams (core.py:204-205): matrices
    produced by the reference generator recipe, rounded to `dtype`, handed
    to the reference as Python floats."""

    def __init__(self, cfg, block, dtype):
        super().__init__()
        self.cfg, self.block, self.dtype = cfg, block, dtype

    def __missing__(self, key):
        name, expert = key
        c = self.cfg
        tag, rows, cols = {
            "gate": (mcore._TAG_GATE, c.d_model, c.num_experts),
            "pre_gate": (mcore._TAG_PRE_GATE, c.d_model, c.num_experts),
            "w1": (mcore._TAG_W1, c.d_ff, c.d_model),
            "w2": (mcore._TAG_W2, c.d_model, c.d_ff),
            "non_moe": (mcore._TAG_DENSE, c.d_model, c.d_model),
        }[name]
        m = og.as_f64(og.weights(derive_seed(c.seed, tag, self.block, expert), rows, cols, self.dtype))
        v = m.tolist()
        self[key] = v
        return v


def rounded_params(cfg, dtype):
    return mcore.ModelParams(cfg, [mcore.BlockParams(cfg, b, loaded=RoundedLoaded(cfg, b, dtype))
                                   for b in range(cfg.num_blocks)])


def small_decoder_fixture():
    """decoder_iteration on small configs, weights from the reference's own
    generator (fp64, no rounding) and also fp32-rounded via `loaded`."""
    out = []
    rng = Xoshiro256StarStar(99)
    for trial in range(24):
        dims = dict(
            d_model=2 + int(rng.uniform() * 30), d_ff=2 + int(rng.uniform() * 40),
            num_blocks=2 + int(rng.uniform() * 5), num_experts=2 + int(rng.uniform() * 15),
            top_k=1 + int(rng.uniform() * 2), activation_level=1 + int(rng.uniform() * 2) if trial % 3 else 1,
            seed=trial)
        if dims["top_k"] > dims["num_experts"] or dims["activation_level"] >= dims["num_blocks"]:
            continue
        cfg = moesim.ModelConfig(**dims)
        for dtype in ("f64", "f32", "bf16"):
            params = mcore.init_model(cfg) if dtype == "f64" else rounded_params(cfg, dtype)
            x = mcore.default_input(cfg)
            iters = []
            for _ in range(2):
                x, consumed = moesim.decoder_iteration(x, params)
                iters.append({"y": hxl(x), "ids": [list(d.expert_ids) for d in consumed],
                              "w": [hxl(d.combine_weights) for d in consumed]})
            out.append({"cfg": {"d_model": cfg.d_model, "d_ff": cfg.d_ff, "num_blocks": cfg.num_blocks,
                                "num_experts": cfg.num_experts, "top_k": cfg.top_k,
                                "activation_level": cfg.activation_level, "seed": cfg.seed},
                        "dtype": dtype, "iterations": iters})
    return out


def switch_fixture():
    """Teacher-forced Switch-scale samples: the reference's gate on the
    Large-128 shape and one full block of Base-8 (d=768, f=3072) per dtype."""
    out = {"gate_large": [], "block_base8": []}
    large = moesim.ModelConfig(d_model=1024, d_ff=4096, num_blocks=24, num_experts=128, top_k=1, seed=0)
    for dtype in ("f32", "bf16"):
        params = rounded_params(large, dtype)
        for b in (0, 5, 22):
            blk = params.blocks[b]
            G = blk.gate if b == 0 else blk.pre_gate
            for t in range(4):
                x = og.token_input(og.Dims(1024, 4096, 24, 128, 1), t + 7 * b).astype(np.float32).astype(np.float64)
                r = moesim.gate_forward(x.tolist(), G, 1)
                out["gate_large"].append({"dtype": dtype, "block": b, "which": "gate" if b == 0 else "pre_gate",
                                          "x": hxl(x), "ids": list(r.expert_ids), "w": hxl(r.combine_weights)})
    base8 = moesim.ModelConfig(d_model=768, d_ff=3072, num_blocks=12, num_experts=8, top_k=1, seed=0)
    for dtype in ("f32", "bf16"):
        params = rounded_params(base8, dtype)
        for b, t in ((0, 0), (3, 1)):
            x = og.token_input(og.Dims(768, 3072, 12, 8, 1), t).astype(np.float32).astype(np.float64).tolist()
            blk = params.blocks[b]
            dec = moesim.gate_forward(x, blk.gate if b == 0 else params.blocks[b - 1].pre_gate, 1)
            y, rout = moesim.moe_block_forward(x, blk, dec)
            out["block_base8"].append({"dtype": dtype, "block": b, "token": t, "x": hxl(x),
                                       "ids_in": list(dec.expert_ids), "w_in": hxl(dec.combine_weights),
                                       "y": hxl(y), "ids_out": list(rout.expert_ids) if rout else None,
                                       "w_out": hxl(rout.combine_weights) if rout else None})
    return out


def gate_f64_fixture():
    """The reference's gate at ITS OWN precision: moesim's unrounded fp64
    init_model weights and fp64 inputs (core.py:200-211, :274-277), Switch
    Large-128 shapes, plus planted exact and 1-ulp near ties.  Pins the
    drop-in's fp64 routing (pgmoe_gate_forward_f64)."""
    out = []
    large = moesim.ModelConfig(d_model=1024, d_ff=4096, num_blocks=24, num_experts=128, top_k=1, seed=0)
    params = mcore.init_model(large)
    dims = og.Dims(1024, 4096, 24, 128, 1)
    for b in (0, 5, 22):
        blk = params.blocks[b]
        which = "gate" if b == 0 else "pre_gate"
        G = blk.gate if b == 0 else blk.pre_gate
        for t in range(6):
            x = og.token_input(dims, t + 7 * b).tolist()  # fp64, unrounded
            for k in (1, 2):
                r = moesim.gate_forward(x, G, k)
                out.append({"block": b, "which": which, "token": t + 7 * b, "k": k, "tie": None,
                            "ids": list(r.expert_ids), "w": hxl(r.combine_weights)})
    # near ties: column 9 := column 3 (exact tie), column 40 := column 3 with one
    # element moved by one ulp; x chosen so that column 3 wins
    G = [list(row) for row in params.blocks[5].pre_gate]
    for i, row in enumerate(G):
        row[9] = row[3]
        row[40] = row[3] if i != 100 else float(np.nextafter(row[3], 1.0))
    x = [0.05 if row[3] >= 0 else -0.05 for row in G]
    for k in (1, 2, 3):
        r = moesim.gate_forward(x, G, k)
        out.append({"block": 5, "which": "pre_gate", "token": -1, "k": k, "tie": [3, 9, 40],
                    "x": hxl(x), "ids": list(r.expert_ids), "w": hxl(r.combine_weights)})
    return out


def pgmoe1_fixture():
    """A PGMOE1 file written by the reference's own save_model (model_io.py:39-60)."""
    from moesim.model_io import save_model
    cfg = moesim.ModelConfig(d_model=16, d_ff=24, num_blocks=3, num_experts=4, top_k=1, seed=11)
    save_model(mcore.init_model(cfg), os.path.join(HERE, "small_d16_f24_b3_e4.pgmoe1"))


def cache_fixture():
    """moesim.ExpertCache (cache.py:49-103) on Zipf and uniform traces."""
    from moesim.cache import ExpertCache
    cfg = moesim.ModelConfig(d_model=4, d_ff=8, num_blocks=6, num_experts=32, top_k=1, seed=0)
    out = []
    for skew, seed in ((1.0, 1), (0.0, 2), (1.4, 3)):
        trace = mcore.gen_routing_trace(cfg, 400, skew, seed)
        keys = [(b, d.expert_ids[0]) for it in trace.decisions for b, d in enumerate(it)]
        for policy in ("lifo", "lfu", "lru"):
            for cap in (0, 1, 7, 40, 120):
                c = ExpertCache(cap * 100, policy)
                res = [c.access(k, 100, i) for i, k in enumerate(keys)]
                out.append({"skew": skew, "policy": policy, "capacity_records": cap,
                            "blocks": [k[0] for k in keys], "experts": [k[1] for k in keys],
                            "hit": [int(r.hit) for r in res], "n_evicted": [len(r.evicted) for r in res]})
    return out


def main():
    only = sys.argv[1:]  # optional: names of the fixtures to (re)generate
    if not only:
        pgmoe1_fixture()
    fixtures = {
        "rng.json": rng_fixture,
        "linalg.json": linalg_fixture,
        "gate.json": gate_fixture,
        "decoder_small.json": small_decoder_fixture,
        "switch.json": switch_fixture,
        "cache.json": cache_fixture,
        "gate_f64.json": gate_f64_fixture,
    }
    if only:
        fixtures = {k: v for k, v in fixtures.items() if k in only}
    meta = {"generator": "tests/golden/gen_golden.py", "reference": "moesim " + moesim.__version__,
            "python": sys.version.split()[0]}
    for name, fn in fixtures.items():
        data = fn()
        data = {"meta": meta, "data": data}
        with open(os.path.join(HERE, name), "w") as fh:
            json.dump(data, fh, separators=(",", ":"))
        print("wrote", name, os.path.getsize(os.path.join(HERE, name)), "bytes")


if __name__ == "__main__":
    main()
