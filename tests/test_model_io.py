"""PGMOE1 weight files (model_io.py:1-105): the reference wrote the golden file
(tests/golden/gen_golden.py calls moesim's save_model)."""

import os
import struct

import numpy as np
import pytest

from oracle import oracle as og

GOLD = os.path.join(os.path.dirname(__file__), "golden", "small_d16_f24_b3_e4.pgmoe1")


def test_header_read_without_gpu():
    from paper_2308_12066_b200 import weight_file_config
    cfg = weight_file_config(GOLD, seed=11)
    assert (cfg.d_model, cfg.d_ff, cfg.num_blocks, cfg.num_experts, cfg.top_k, cfg.activation_level) == \
        (16, 24, 3, 4, 1, 1)
    # header is 30 bytes, first float at offset 30 (test_model_io.py:378-388 of the reference)
    raw = open(GOLD, "rb").read()
    assert raw[:6] == b"PGMOE1" and struct.unpack_from("<6i", raw, 6) == (16, 24, 3, 4, 1, 1)


@pytest.mark.parametrize("corrupt,msg", [(lambda r: b"XXXXXX" + r[6:], "bad magic"),
                                         (lambda r: r[:20], "truncated header")])
def test_header_errors_are_weight_file_errors(tmp_path, corrupt, msg):
    from paper_2308_12066_b200 import WeightFileError, weight_file_config
    p = tmp_path / "bad.pgmoe1"
    p.write_bytes(corrupt(open(GOLD, "rb").read()))
    with pytest.raises(WeightFileError, match=msg):
        weight_file_config(str(p))


@pytest.mark.gpu
def test_load_reference_file_matches_generator_and_roundtrips(tmp_path):
    import paper_2308_12066_b200 as p
    m = p.DeviceModel.load(GOLD, dtype="f32", max_tokens=4, seed=11)
    dims = og.Dims(16, 24, 3, 4, 1, seed=11)
    om = og.OracleModel(dims, "f32")
    assert np.array_equal(m.get_matrix("gate", 0), om.gate(0))
    assert np.array_equal(m.get_matrix("pre_gate", 1), om.pre_gate(1))
    assert np.array_equal(m.get_matrix("w2", 2, 3), om.w2(2, 3))
    assert np.array_equal(m.get_matrix("non_moe", 2), om.dense(2))
    # same weights as the device generator -> identical decoder outputs
    ref = p.DeviceModel(m.config, dtype="f32", max_tokens=4)
    x = p.token_inputs(m.config, 4)
    assert np.array_equal(m.decoder_iteration(x)[0].cpu().numpy(), ref.decoder_iteration(x)[0].cpu().numpy())
    out = tmp_path / "rt.pgmoe1"
    m.save(str(out))
    assert open(out, "rb").read() == open(GOLD, "rb").read()
    # bf16 model: RNE of the file's fp32 values
    mb = p.DeviceModel.load(GOLD, dtype="bf16", max_tokens=4, seed=11)
    assert np.array_equal(mb.get_matrix("w1", 1, 2), og.OracleModel(dims, "bf16").w1(1, 2))


@pytest.mark.gpu
@pytest.mark.parametrize("corrupt,msg", [
    (lambda r: r[:-10], "file ends inside block 2"),
    (lambda r: r + b"\0\0\0\0", "4 trailing bytes"),
    (lambda r: r[:30] + struct.pack("<f", float("nan")) + r[34:], "non-finite value in block 0 matrix 'gate'"),
])
def test_body_errors_are_weight_file_errors(tmp_path, corrupt, msg):
    import paper_2308_12066_b200 as p
    f = tmp_path / "bad.pgmoe1"
    f.write_bytes(corrupt(open(GOLD, "rb").read()))
    with pytest.raises(p.WeightFileError, match=msg):
        p.DeviceModel.load(str(f), dtype="f32", max_tokens=2)
