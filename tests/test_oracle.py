"""The CPU oracle is pinned bit-for-bit against fixtures produced by running
the reference itself (tests/golden/gen_golden.py imports moesim)."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle as og

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)["data"]


def fx(s):
    return float.fromhex(s)


def fxa(lst):
    return np.array([float.fromhex(v) for v in lst], dtype=np.float64)


# ---- rng.py ----------------------------------------------------------------

def test_splitmix_published_vectors():
    g = load("rng.json")
    assert [hex(v) for v in og.splitmix64(0, 4)] == g["splitmix_seed0"]


def test_xoshiro_streams_and_frozen_first_outputs():
    g = load("rng.json")
    for seed, vals in g["xoshiro"].items():
        assert [hex(v) for v in og.xoshiro_u64(int(seed, 16), 50)] == vals
    # tests/test_rng.py:134-137 of the reference
    assert og.xoshiro_u64(0, 2) == [0x99EC5F36CB75F2B4, 0xBF6E1F784956452A]


def test_derive_seed_including_negative_tag():
    for case in load("rng.json")["derive_seed"]:
        assert hex(og.derive_seed(int(case["base"], 16), *case["tags"])) == case["seed"]


def test_fill_bit_exact():
    g = load("rng.json")
    assert og.fill(123, 64).tolist() == fxa(g["fill_123"]).tolist()
    assert og.fill(9, 32, -2.0, 2.0).tolist() == fxa(g["fill_9_lohi"]).tolist()


def test_full_scale_generator_pin():
    g = load("rng.json")
    seed = og.derive_seed(0, og.TAG_W1, 0, 0)
    w64 = og.weights(seed, 3072, 768, "f64")
    assert hashlib.sha256(w64.astype("<f8").tobytes()).hexdigest() == g["base_w1_b0_e0_sha256_f64le"]
    w32 = og.weights(seed, 3072, 768, "f32")
    assert hashlib.sha256(w32.astype("<f4").tobytes()).hexdigest() == g["base_w1_b0_e0_sha256_f32le"]
    dims = og.Dims(1024, 4096, 24, 128, 1)
    assert og.default_input(dims).tolist() == fxa(g["default_input_large"]).tolist()


def test_bf16_rounding_is_rne_of_f32():
    seed = og.derive_seed(3, og.TAG_W2, 1, 2)
    w32 = og.weights(seed, 64, 48, "f32")
    wb = og.weights(seed, 64, 48, "bf16")
    u = w32.view(np.uint32).astype(np.uint64)
    rne = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    assert np.array_equal(wb, rne)


# ---- linalg.py -------------------------------------------------------------

def test_matvec_and_columns_bit_exact():
    for c in load("linalg.json")["matvec"]:
        mat = np.array([[fx(v) for v in r] for r in c["mat"]])
        assert og.matvec(mat, fxa(c["x"])).tolist() == fxa(c["matvec"]).tolist()
        assert og.matvec_columns(mat, fxa(c["xt"])).tolist() == fxa(c["matvec_columns"]).tolist()


def test_softmax_bit_exact():
    for c in load("linalg.json")["softmax"]:
        assert og.softmax(fxa(c["logits"])).tolist() == fxa(c["probs"]).tolist()


# ---- core.py gate ----------------------------------------------------------

def test_gate_hand_softmax_and_tie_rule():
    g = load("gate.json")
    ids, w, _ = og.gate_forward([1.0], np.array([[1.0, 0.0]]), 1)
    assert list(ids) == g["hand_softmax"]["ids"] and list(w) == fxa(g["hand_softmax"]["w"]).tolist()
    ids, w, _ = og.gate_forward([1.0], np.array([[0.5, 0.5, 0.5, 0.5]]), 2)
    assert list(ids) == g["tie"]["ids"] == [0, 1] and list(w) == [0.25, 0.25]


@pytest.mark.parametrize("group", ["random", "ties"])
def test_gate_random_and_exact_ties(group):
    for c in load("gate.json")[group]:
        G = np.array([[fx(v) for v in r] for r in c["gate"]])
        ids, w, _ = og.gate_forward(fxa(c["x"]), G, c["k"])
        assert list(ids) == c["ids"]
        assert list(w) == fxa(c["w"]).tolist()


def test_gate_errors_mirror_reference():
    with pytest.raises(og.OracleError) as e:
        og.gate_forward([1e308], np.array([[2.0, 1.0]]), 1)
    assert e.value.code == og.E_GATE_OVERFLOW
    with pytest.raises(og.OracleError) as e:
        og.gate_forward([1.0, 2.0], np.array([[1.0, 0.0]]), 1)
    assert e.value.code == og.E_SHAPE
    with pytest.raises(og.OracleError) as e:
        og.gate_forward([1.0], np.array([[1.0, 0.0]]), 3)
    assert e.value.code == og.E_CONFIG


# ---- core.py decoder -------------------------------------------------------

def test_small_decoder_iterations_bit_exact():
    cases = load("decoder_small.json")
    assert len(cases) >= 30
    for c in cases:
        dims = og.Dims(**c["cfg"])
        model = og.OracleModel(dims, c["dtype"])
        x = og.default_input(dims)
        for it in c["iterations"]:
            x, consumed = og.decoder_iteration(model, x)
            assert [list(ids) for ids, _ in consumed] == it["ids"]
            assert [list(w) for _, w in consumed] == [fxa(w).tolist() for w in it["w"]]
            assert x.tolist() == fxa(it["y"]).tolist()


def test_switch_large_gate_teacher_forced():
    for c in load("switch.json")["gate_large"]:
        dims = og.Dims(1024, 4096, 24, 128, 1)
        model = og.OracleModel(dims, c["dtype"])
        G = model.gate(0) if c["which"] == "gate" else model.pre_gate(c["block"])
        ids, w, _ = og.gate_forward(fxa(c["x"]), G, 1)
        assert list(ids) == c["ids"] and list(w) == fxa(c["w"]).tolist()


def test_switch_base8_block_teacher_forced():
    for c in load("switch.json")["block_base8"]:
        dims = og.Dims(768, 3072, 12, 8, 1)
        model = og.OracleModel(dims, c["dtype"])
        x = fxa(c["x"])
        routing = (tuple(c["ids_in"]), tuple(fxa(c["w_in"]).tolist()))
        y, rout = og.block_forward(model, c["block"], x, routing)
        assert y.tolist() == fxa(c["y"]).tolist()
        assert list(rout[0]) == c["ids_out"]


def test_permutation_is_stable_counting_sort():
    rng = np.random.default_rng(0)
    ids = rng.integers(0, 16, size=(37, 2)).astype(np.int32)
    hist, off, perm, act = og.permute(ids, 16)
    flat = ids.reshape(-1)
    expect = sorted(range(flat.size), key=lambda i: (flat[i], i))
    assert perm.tolist() == expect
    assert hist.tolist() == np.bincount(flat, minlength=16).tolist()
    assert act.tolist() == [e for e in range(16) if hist[e] > 0]
    assert off[-1] == flat.size


def gate_f64_case(c):
    """(x fp64, G fp64, k) of a gate_f64.json case: moesim's unrounded
    init_model weights (core.py:200-211) regenerated by the oracle's RNG."""
    dims = og.Dims(1024, 4096, 24, 128, 1)
    tag = og.TAG_GATE if c["which"] == "gate" else og.TAG_PRE_GATE
    G = og.weights(og.derive_seed(0, tag, c["block"], -1), 1024, 128, "f64")
    if c["tie"]:
        G = G.copy()
        G[:, 9] = G[:, 3]
        G[:, 40] = G[:, 3]
        G[100, 40] = np.nextafter(G[100, 3], 1.0)
        x = fxa(c["x"])
    else:
        x = og.token_input(dims, c["token"])
    return x, G, c["k"]


def test_gate_fp64_switch_matches_reference():
    """The reference's gate at its own precision (fp64 weights and inputs,
    never rounded), Switch-Large shapes and planted near ties."""
    for c in load("gate_f64.json"):
        x, G, k = gate_f64_case(c)
        ids, w, _ = og.gate_forward(x, G, k)
        assert list(ids) == c["ids"]
        assert [v.hex() for v in w] == c["w"]
