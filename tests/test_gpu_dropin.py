"""The drop-in boundary on the GPU: the reference signatures
(core.py:284-383) on the reference's own types and precision, and
dropin.install() patching a moesim-shaped package.

The reference itself is not on the GPU box, so its inputs come from the
golden fixtures it produced (tests/golden/gate*.json, gen_golden.py) and from
the oracle's RNG (pinned bit-for-bit to moesim by tests/test_oracle.py);
the block-level objects are minimal stand-ins with moesim's BlockParams /
ModelParams interface (core.py:175-263)."""

import json
import os
import sys
import types

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as og  # noqa: E402

sys.path.insert(0, os.path.dirname(__file__))
from test_oracle import fxa, gate_f64_case, load  # noqa: E402

pytestmark = pytest.mark.gpu


def P():
    import paper_2308_12066_b200 as p
    return p


def test_fp64_gate_dropin_matches_reference_golden():
    """Unrounded fp64 inputs (what moesim feeds gate_forward) route through
    pgmoe_gate_forward_f64: ids equal moesim's, including exact ties and
    1-ulp near ties at Switch-Large scale; weights within fp32 rounding."""
    p = P()
    g = load("gate.json")
    for c in g["random"] + g["ties"]:
        G = [[float.fromhex(v) for v in row] for row in c["gate"]]
        x = [float.fromhex(v) for v in c["x"]]
        d = p.gate_forward(x, G, c["k"])
        assert list(d.expert_ids) == c["ids"]
        assert np.allclose(d.combine_weights, fxa(c["w"]), rtol=1e-6, atol=0)
    for c in load("gate_f64.json"):
        x, G, k = gate_f64_case(c)
        d = p.gate_forward(x.tolist(), G.tolist(), k)
        assert list(d.expert_ids) == c["ids"], c
        assert np.allclose(d.combine_weights, fxa(c["w"]), rtol=1e-6, atol=0)
    # batched fp64 route: 700 unrounded tokens, ids vs the oracle's serial fp64
    dims = og.Dims(1024, 4096, 24, 128, 1)
    G = og.weights(og.derive_seed(0, og.TAG_PRE_GATE, 7, -1), 1024, 128, "f64")
    X = np.stack([og.token_input(dims, t) for t in range(700)])
    r = p.route(torch.from_numpy(X).cuda(), torch.from_numpy(G).cuda(), 2)
    r.check()
    ids_ref, w_ref = og.gate_batch(X, G, 2, nthreads=16)
    assert np.array_equal(r.ids.cpu().numpy(), ids_ref)
    assert np.max(np.abs(r.w.cpu().numpy() - w_ref) / w_ref) <= 1e-6


def test_gate_dropin_errors_mirror_reference():
    p = P()
    with pytest.raises(p.ConfigError, match="exceeds expert count"):
        p.gate_forward([0.1, 0.2], [[1.0, 2.0], [3.0, 4.0]], 3)
    with pytest.raises(p.ShapeError, match="gate expects input of width 2, got 3"):
        p.gate_forward([0.1, 0.2, 0.3], [[1.0, 2.0], [3.0, 4.0]], 1)
    with pytest.raises(p.GateOverflowError, match="numerical overflow in gate"):
        p.gate_forward([1e300, 1e300], [[1e300, 1.0], [1e300, 1.0]], 1)
    with pytest.raises(p.GateOverflowError, match="underflowed to zero"):
        p.gate_forward([1.0], [[0.0, -1000.0]], 2)


# ------------------------------------------- moesim-shaped stand-ins ----

class Cfg:
    def __init__(self, d, f, nb, E, k, L=1, seed=0):
        self.d_model, self.d_ff, self.num_blocks, self.num_experts, self.top_k = d, f, nb, E, k
        self.activation_level, self.seed = L, seed

    def has_conv_gate(self, b):
        return True if self.activation_level == 0 else b < self.activation_level

    def has_pre_gate(self, b):
        return False if self.activation_level == 0 else b < self.num_blocks - self.activation_level


class Expert:
    def __init__(self, w1, w2):
        self.w1, self.w2 = w1, w2


class Block:
    """BlockParams' interface (core.py:175-240): unrounded fp64 matrices as
    lists, from the oracle's RNG (== moesim's generator)."""

    def __init__(self, cfg, b):
        self.config, self.index = cfg, b
        self.materialized = set()

    def _m(self, tag, rows, cols, e=-1):
        self.materialized.add((tag, e))
        return og.weights(og.derive_seed(self.config.seed, tag, self.index, e), rows, cols, "f64").tolist()

    has_conv_gate = property(lambda s: s.config.has_conv_gate(s.index))
    has_pre_gate = property(lambda s: s.config.has_pre_gate(s.index))
    gate = property(lambda s: s._m(og.TAG_GATE, s.config.d_model, s.config.num_experts))
    pre_gate = property(lambda s: s._m(og.TAG_PRE_GATE, s.config.d_model, s.config.num_experts))
    non_moe = property(lambda s: s._m(og.TAG_DENSE, s.config.d_model, s.config.d_model))

    def expert(self, e):
        c = self.config
        return Expert(self._m(og.TAG_W1, c.d_ff, c.d_model, e), self._m(og.TAG_W2, c.d_model, c.d_ff, e))


class Params:
    def __init__(self, cfg):
        self.config = cfg
        self.blocks = [Block(cfg, b) for b in range(cfg.num_blocks)]


def _normwise(y, ref):
    y, ref = np.asarray(y, np.float64), np.asarray(ref, np.float64)
    return float(np.max(np.abs(y - ref)) / np.max(np.abs(ref)))


def test_moe_block_forward_dropin_contract():
    """core.py:319-339: pre-gate on the block input, dry_run touches no
    expert, a missing decision raises RoutingError with the reference
    message, outputs within the fp32 bar of the oracle (fp64 reference)."""
    p = P()
    cfg = Cfg(64, 96, 3, 8, 2)
    params = Params(cfg)
    dims = og.Dims(64, 96, 3, 8, 2)
    om = og.OracleModel(dims, "f64")
    x = og.token_input(dims, 0).tolist()
    blk = params.blocks[0]
    y, rout = p.moe_block_forward(x, blk, None, dry_run=True)
    assert y is None and not any(tag in (og.TAG_W1, og.TAG_W2) for tag, _ in blk.materialized)
    ids_ref, w_ref, _ = og.gate_forward(np.array(x), om.pre_gate(0), 2)
    assert rout.expert_ids == ids_ref
    with pytest.raises(p.RoutingError, match="no routing decision available"):
        p.moe_block_forward(x, blk, None)
    dec = p.gate_forward(x, blk.gate, 2)
    y, rout2 = p.moe_block_forward(x, blk, dec)
    y_ref, _ = og.block_forward(om, 0, np.array(x), (dec.expert_ids, dec.combine_weights))
    assert _normwise(y, y_ref) <= 1e-4
    assert rout2.expert_ids == rout.expert_ids
    _, none_out = p.moe_block_forward(x, blk, dec, want_routing_out=False)
    assert none_out is None
    with pytest.raises(p.RoutingError):
        p.moe_block_forward(x, blk, p.RoutingDecision((1,), (1.0,)))  # top_k mismatch (validate_for)


def test_decoder_iteration_dropin_routed_and_supplied():
    """core.py:342-383 on the reference's fp64 weights: routing ids equal the
    oracle's at every block, outputs within the fp32 bar; supplied decisions
    bypass the gates; the reference's RoutingErrors."""
    p = P()
    cfg = Cfg(48, 80, 4, 6, 1)
    params = Params(cfg)
    dims = og.Dims(48, 80, 4, 6, 1)
    om = og.OracleModel(dims, "f64")
    x = og.token_input(dims, 0)
    y, consumed = p.decoder_iteration(x.tolist(), params)
    y_ref, consumed_ref = og.decoder_iteration(om, x)
    assert [d.expert_ids for d in consumed] == [c[0] for c in consumed_ref]
    assert _normwise(y, y_ref) <= 1e-4
    sup = [p.RoutingDecision(((b + 1) % 6,), (0.5,)) for b in range(4)]
    ys, cs = p.decoder_iteration(x.tolist(), params, supplied_decisions=sup)
    assert cs == sup
    fresh = Params(cfg)  # supplied decisions: no gate is ever materialised
    p.decoder_iteration(x.tolist(), fresh, supplied_decisions=sup)
    assert not any(tag in (og.TAG_GATE, og.TAG_PRE_GATE) for blk in fresh.blocks for tag, _ in blk.materialized)
    with pytest.raises(p.RoutingError, match="supplied 3 decisions for 4 blocks"):
        p.decoder_iteration(x.tolist(), params, supplied_decisions=sup[:3])


def test_install_patches_a_moesim_shaped_package():
    """dropin.install() on a package with moesim's layout (core, errors,
    scheduler and harness binding decoder_iteration by name): the patched
    names run on the GPU, return the package's own RoutingDecision type and
    raise its own exception classes; uninstall() restores everything."""
    from paper_2308_12066_b200 import dropin
    name = "fake_moesim_for_dropin"
    pkg = types.ModuleType(name)
    core = types.ModuleType(name + ".core")
    errs = types.ModuleType(name + ".errors")
    sched = types.ModuleType(name + ".scheduler")
    harness = types.ModuleType(name + ".harness")

    class MoESimError(Exception):
        pass

    for n, base in (("ConfigError", ValueError), ("ShapeError", ValueError), ("GateOverflowError", ArithmeticError),
                    ("RoutingError", RuntimeError), ("OomError", MemoryError), ("WeightFileError", ValueError),
                    ("InvariantError", AssertionError)):
        setattr(errs, n, type(n, (MoESimError, base), {}))
    errs.MoESimError = MoESimError

    class RoutingDecision:
        def __init__(self, ids, w):
            self.expert_ids, self.combine_weights = tuple(ids), tuple(w)

        def validate_for(self, cfg):
            if len(self.expert_ids) != cfg.top_k:
                raise errs.RoutingError("bad k")

    core.RoutingDecision = RoutingDecision
    orig = {}
    for n in dropin.HOT_PATH:
        f = (lambda n: (lambda *a, **k: ("cpu", n)))(n)
        setattr(core, n, f)
        orig[n] = f
    sched.decoder_iteration = core.decoder_iteration
    harness.decoder_iteration = core.decoder_iteration
    for m in (pkg, core, errs, sched, harness):
        sys.modules[m.__name__] = m
    try:
        h = dropin.install(name)
        assert sched.decoder_iteration is not orig["decoder_iteration"]
        d = core.gate_forward([0.3, -0.2, 0.1], [[0.1, 0.9], [0.4, -0.3], [0.2, 0.2]], 1)
        assert type(d) is RoutingDecision and d.expert_ids == (1,)  # logits -0.03, 0.35
        with pytest.raises(errs.ShapeError, match="gate expects input of width 3, got 2"):
            core.gate_forward([0.3, -0.2], [[0.1, 0.9], [0.4, -0.3], [0.2, 0.2]], 1)
        params = Params(Cfg(32, 40, 3, 4, 1))
        y, consumed = harness.decoder_iteration(og.token_input(og.Dims(32, 40, 3, 4, 1), 0).tolist(), params)
        assert len(y) == 32 and all(type(c) is RoutingDecision for c in consumed)
        h.uninstall()
        for n in dropin.HOT_PATH:
            assert getattr(core, n) is orig[n]
        assert sched.decoder_iteration is orig["decoder_iteration"]
    finally:
        for m in (pkg, core, errs, sched, harness):
            sys.modules.pop(m.__name__, None)
