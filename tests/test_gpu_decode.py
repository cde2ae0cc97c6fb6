"""The persistent small-batch decoder (csrc/decode_tc.cu): one launch per
decoder iteration, 8-CTA clusters splitting K with DSMEM partial sums.

Bars (north star): consumed routing ids bit-exact against the reference gate
on the kernel's own block inputs (teacher forced, traced from inside the
launch), combine weights 1e-6, block outputs normwise <= 2e-2 (bf16).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as og  # noqa: E402

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _model(dims, T, placement="resident"):
    import paper_2308_12066_b200 as p
    cfg = p.ModelConfig(d_model=dims.d_model, d_ff=dims.d_ff, num_blocks=dims.num_blocks,
                        num_experts=dims.num_experts, top_k=1, activation_level=1, seed=dims.seed)
    m = p.DeviceModel(cfg, dtype="bf16", placement=placement, max_tokens=T)
    m.set_ll_decode(False)  # this file tests decode_tc.cu (the LL decoder: test_gpu_lldecode.py)
    m.set_decode(True, min(T, 64))  # the kernel serves up to 64 tokens (default threshold: 1)
    return m


def _tokens(d, T, seed=0):
    from paper_2308_12066_b200._rng import token_batch
    return token_batch(seed, d, T)


def _normwise(y, ref):
    ref = np.asarray(ref, dtype=np.float64)
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(np.asarray(y, np.float64) - ref)) / (den if den > 0 else 1.0))


def _traced(m, x):
    c = m.config
    T = x.shape[0]
    xt = torch.empty((c.num_blocks, T, c.d_model), dtype=torch.float32, device="cuda")
    y, ids, w = m.decoder_iteration(x, trace=True, x_trace=xt)
    torch.cuda.synchronize()
    return y, ids, w, xt


@pytest.mark.parametrize("shape", [(256, 512, 4, 64), (768, 3072, 12, 64), (1024, 4096, 5, 128), (256, 1024, 3, 256)])
@pytest.mark.parametrize("T", [1, 3, 16])
def test_decode_kernel_teacher_forced(shape, T):
    d, f, nb, E = shape
    dims = og.Dims(d, f, nb, E, 1, seed=1)
    m = _model(dims, T)
    om = og.OracleModel(dims, "bf16")
    x = torch.from_numpy(_tokens(d, T, seed=T)).cuda()
    n0 = m.decode_iterations
    y, ids, w, xt = _traced(m, x)
    assert m.decode_iterations == n0 + 1, "the persistent decode launch must serve this call"
    ids, w, xt = ids.cpu().numpy(), w.cpu().numpy().astype(np.float64), xt.cpu().numpy().astype(np.float64)
    yl = y.cpu().numpy()
    for b in range(nb):
        # consumed decision == reference gate on the block input that produced it
        G, xin = (om.gate(0), xt[0]) if b == 0 else (om.pre_gate(b - 1), xt[b - 1])
        ids_ref, w_ref = og.gate_batch(xin, G, 1, nthreads=8)
        assert np.array_equal(ids[b], ids_ref), f"block {b}: routing differs from the reference"
        assert np.max(np.abs(w[b] - w_ref) / w_ref) <= 1e-6
        w1 = {e: om.w1(b, e) for e in np.unique(ids[b])}
        w2 = {e: om.w2(b, e) for e in np.unique(ids[b])}
        y_ref = og.block_batch(xt[b], ids[b], w[b], w1, w2, om.dense(b), E, nthreads=8)
        out = xt[b + 1] if b + 1 < nb else yl
        err = _normwise(out, y_ref)
        assert err <= TOL, f"block {b}: normwise error {err:.3g}"
    m.close()


def test_decode_deterministic_graph_replay_and_close_to_block_launches():
    dims = og.Dims(768, 3072, 6, 64, 1, seed=3)
    T = 8
    x = torch.from_numpy(_tokens(768, T, seed=5)).cuda()
    m = _model(dims, T)
    outs = []
    for _ in range(3):  # eager (traced) then graph replays (plain)
        y, ids, w, _ = _traced(m, x)
        outs.append((y.clone(), ids.clone(), w.clone()))
    yg = torch.empty_like(x)
    for _ in range(3):
        m.decoder_iteration(x, out=yg)
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert all(torch.equal(a, b) for a, b in zip(outs[0], o)), "decode launch not deterministic"
    assert torch.equal(yg, outs[0][0]), "graph replay differs from the eager launch"
    m.set_decode(False)
    y2, ids2, w2, _ = _traced(m, x)
    assert torch.equal(ids2, outs[0][1])  # same routing (certified, inputs equal within bf16)
    assert _normwise(outs[0][0].cpu().numpy(), y2.cpu().numpy()) <= 1e-2
    m.close()


def test_decode_threshold_and_switch():
    dims = og.Dims(256, 512, 3, 64, 1, seed=2)
    m = _model(dims, 32)
    x = torch.from_numpy(_tokens(256, 32)).cuda()
    m.set_decode(True, 16)
    n0 = m.decode_iterations
    m.decoder_iteration(x)  # above the threshold: per-block launches
    torch.cuda.synchronize()
    assert m.decode_iterations == n0
    m.set_decode(True, 32)
    m.decoder_iteration(x)
    torch.cuda.synchronize()
    assert m.decode_iterations == n0 + 1
    m.close()
