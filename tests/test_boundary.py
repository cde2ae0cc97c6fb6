"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every symbol include/pgmoe.h declares; host logic mirrors the
reference (wiring, validation, errors) without touching a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pgmoe.h")


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"PGMOE_API[^;(]*?\b(pgmoe_\w+)\s*\(", txt)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("pgmoe_gate_forward", "pgmoe_expert_forward", "pgmoe_dense_forward",
                 "pgmoe_moe_block_forward", "pgmoe_decoder_iteration", "pgmoe_decoder_iteration_host",
                 "pgmoe_model_create", "pgmoe_last_error"):
        assert must in syms


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2308_12066_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2308_12066_b200.build import build
        build()
    L = ctypes.CDLL(_lib.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(L, s), s
    assert set(_lib.EXPORTS) == set(declared_symbols())
    v = _lib.load().pgmoe_version()
    assert v.startswith(b"pgmoe-b200") and b"sm_100a" in v


def test_status_codes_map_onto_reference_exceptions():
    from paper_2308_12066_b200 import _lib, errors
    with pytest.raises(errors.GateOverflowError, match="numerical overflow in gate"):
        _lib.check(_lib.E_GATE_OVERFLOW)
    with pytest.raises(errors.GateOverflowError, match="underflowed to zero"):
        _lib.check(_lib.E_GATE_UNDERFLOW)
    for code, exc in ((_lib.E_CONFIG, errors.ConfigError), (_lib.E_SHAPE, errors.ShapeError),
                      (_lib.E_ROUTING, errors.RoutingError), (_lib.E_OOM, errors.OomError)):
        with pytest.raises(exc):
            _lib.check(code)
    assert issubclass(errors.ConfigError, ValueError) and issubclass(errors.GateOverflowError, ArithmeticError)


def test_model_config_mirrors_reference_wiring_and_validation():
    from paper_2308_12066_b200.core import ModelConfig
    from paper_2308_12066_b200.errors import ConfigError
    cfg = ModelConfig(d_model=4, d_ff=8, num_blocks=3, num_experts=4, top_k=2, activation_level=1, seed=7)
    assert [cfg.has_pre_gate(b) for b in range(3)] == [True, True, False]
    assert [cfg.has_conv_gate(b) for b in range(3)] == [True, False, False]
    assert [cfg.decision_origin(b) for b in range(3)] == [0, 0, 1]
    lvl2 = ModelConfig(d_model=4, d_ff=8, num_blocks=5, num_experts=4, top_k=2, activation_level=2)
    assert [lvl2.has_conv_gate(b) for b in range(5)] == [True, True, False, False, False]
    assert lvl2.decision_origin(4) == 2
    for bad in (dict(top_k=5), dict(activation_level=3), dict(d_model=0), dict(seed=-1)):
        kw = dict(d_model=4, d_ff=8, num_blocks=3, num_experts=4, top_k=2, activation_level=1, seed=7)
        kw.update(bad)
        with pytest.raises(ConfigError):
            ModelConfig(**kw)
    assert cfg.gate_count == 3


def test_routing_decision_validation():
    from paper_2308_12066_b200.core import ModelConfig, RoutingDecision
    from paper_2308_12066_b200.errors import RoutingError
    with pytest.raises(RoutingError):
        RoutingDecision((0, 0), (0.5, 0.5))
    with pytest.raises(RoutingError):
        RoutingDecision((), ())
    with pytest.raises(RoutingError):
        RoutingDecision((1,), (0.0,))
    cfg = ModelConfig(d_model=4, d_ff=8, num_blocks=3, num_experts=4, top_k=1)
    with pytest.raises(RoutingError):
        RoutingDecision((7,), (0.5,)).validate_for(cfg)


def test_host_token_generator_matches_oracle():
    from oracle import oracle as og
    from paper_2308_12066_b200._rng import token_batch
    dims = og.Dims(768, 3072, 12, 64, 1, seed=3)
    got = token_batch(3, 768, 9)
    ref = np.stack([og.token_input(dims, t) for t in range(9)]).astype(np.float32)
    assert np.array_equal(got, ref)


def test_ep_slot_layout_is_host_computable():
    """pgmoe_ep_slot_rows: each peer slot is cap routed rows plus the header
    rows that carry the sender's per-expert int32 counts in-band (one
    all-to-all for rows and counts).  Pure host arithmetic: no GPU needed."""
    from paper_2308_12066_b200 import _lib
    L = _lib.load()
    assert L.pgmoe_ep_slot_rows(256, 16, 1024) == 257     # Large-128 over 8 ranks
    assert L.pgmoe_ep_slot_rows(48, 8, 256) == 49
    assert L.pgmoe_ep_slot_rows(4, 600, 256) == 4 + 5     # 2400 B of counts in 512-byte rows
