"""The low-latency small-batch decoder (csrc/decode_ll.cu): one persistent
launch per decoder iteration; row-split phases exchange flag-in-word (LL)
stores; the dense CTAs produce the next pre-gate's partial fp64 logits and T
reducer CTAs certify and select.

Bars (north star): consumed routing ids bit-exact against the reference gate
on the kernel's own block inputs (teacher forced, traced from inside the
launch), combine weights 1e-6, block outputs normwise <= 2e-2 (bf16); the
launch is deterministic, graph replays equal eager launches, and
back-to-back launches (the epoch-tagged flags) never read a stale word.
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
    m.set_ll_decode(True, min(T, 8))
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


def _check_teacher_forced(dims, om, ids, w, xt, yl):
    nb, E = dims.num_blocks, dims.num_experts
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


@pytest.mark.parametrize("shape", [(256, 512, 4, 64), (768, 3072, 12, 64), (1024, 4096, 5, 128),
                                   (768, 3072, 4, 128)])
@pytest.mark.parametrize("T", [1, 3, 8])
def test_ll_decode_teacher_forced(shape, T):
    d, f, nb, E = shape
    dims = og.Dims(d, f, nb, E, 1, seed=1)
    m = _model(dims, T)
    om = og.OracleModel(dims, "bf16")
    x = torch.from_numpy(_tokens(d, T, seed=T)).cuda()
    n0 = m.ll_decode_iterations
    y, ids, w, xt = _traced(m, x)
    assert m.ll_decode_iterations == n0 + 1, "the LL decode launch must serve this call"
    _check_teacher_forced(dims, om, ids.cpu().numpy(), w.cpu().numpy().astype(np.float64),
                          xt.cpu().numpy().astype(np.float64), y.cpu().numpy())
    m.close()


def test_ll_decode_deterministic_graph_replay_and_back_to_back():
    """Eager (traced) launches, then graph replays, then a different batch
    size on the same buffers: every launch must read only its own epoch's
    words — equal outputs for equal inputs, no stale data after T changes."""
    dims = og.Dims(768, 3072, 6, 64, 1, seed=3)
    m = _model(dims, 8)
    x8 = torch.from_numpy(_tokens(768, 8, seed=5)).cuda()
    outs = []
    for _ in range(3):
        y, ids, w, _ = _traced(m, x8)
        outs.append((y.clone(), ids.clone(), w.clone()))
    yg = torch.empty_like(x8)
    for _ in range(5):
        m.decoder_iteration(x8, out=yg)
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert all(torch.equal(a, b) for a, b in zip(outs[0], o)), "LL decode launch not deterministic"
    assert torch.equal(yg, outs[0][0]), "graph replay differs from the eager launch"
    # a smaller batch (first 2 tokens) then the full one again
    y2, ids2, _, _ = _traced(m, x8[:2].contiguous())
    assert torch.equal(ids2, outs[0][1][:, :2]), "token 0/1 routing must not depend on the batch"
    y8, ids8, _, _ = _traced(m, x8)
    assert torch.equal(y8, outs[0][0]) and torch.equal(ids8, outs[0][1])
    # against the per-block tcgen05 launches: same routing, outputs within bf16
    m.set_ll_decode(False)
    m.set_decode(False)
    y3, ids3, _, _ = _traced(m, x8)
    assert torch.equal(ids3, outs[0][1])
    assert _normwise(outs[0][0].cpu().numpy(), y3.cpu().numpy()) <= 1e-2
    m.close()


def test_ll_decode_serial_fallback_on_planted_tie():
    """A pre-gate with two identical columns: every token's top logits tie
    exactly, so certification fails and the reducers recompute the tied
    candidates in the reference's serial order (ties -> lower id)."""
    dims = og.Dims(256, 512, 3, 64, 1, seed=4)
    m = _model(dims, 4)
    om = og.OracleModel(dims, "bf16")
    x = torch.from_numpy(_tokens(256, 4, seed=9)).cuda()
    ids0, _ = og.gate_batch(x.cpu().numpy().astype(np.float64), om.pre_gate(0), 1, nthreads=4)
    top = int(ids0[0, 0])
    twin = 7 if top != 7 else 9
    g = m.get_matrix("pre_gate", 0)  # bf16 bit patterns
    g[:, twin] = g[:, top]           # token 0's two best logits now tie exactly
    m.set_matrix("pre_gate", 0, -1, g)
    Gref = (g.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    m.reset_stats()
    y, ids, w, xt = _traced(m, x)
    ids_ref, _ = og.gate_batch(xt[0].cpu().numpy().astype(np.float64), Gref, 1, nthreads=4)
    assert np.array_equal(ids.cpu().numpy()[1], ids_ref)
    assert int(ids_ref[0, 0]) == min(top, twin)  # the reference tie rule: lower id
    assert m.stats()["route_fallbacks"] > 0, "the tie must take the serial recompute"
    m.check_routing()
    m.close()


def test_ll_decode_gate_overflow_surfaces_as_reference_error():
    """A non-finite pre-gate logit inside the launch (core.py:297): the
    reducer flags it on the routing buffer and check_routing raises the
    reference's GateOverflowError with its message; the next clean launch
    runs normally."""
    from paper_2308_12066_b200 import errors
    dims = og.Dims(256, 512, 3, 64, 1, seed=6)
    m = _model(dims, 2)
    x = torch.from_numpy(_tokens(256, 2, seed=3)).cuda()
    m.decoder_iteration(x)
    torch.cuda.synchronize()
    m.check_routing()
    g = m.get_matrix("pre_gate", 1)
    g_bad = g.copy()
    g_bad[:, 5] = 0x7F80  # +inf (bf16)
    m.set_matrix("pre_gate", 1, -1, g_bad)
    m.decoder_iteration(x)  # a graph replay of the LL launch (counted once, at capture)
    torch.cuda.synchronize()
    assert m.ll_decode_iterations >= 1
    with pytest.raises(errors.GateOverflowError, match="numerical overflow in gate"):
        m.check_routing()
    m.set_matrix("pre_gate", 1, -1, g)
    m.decoder_iteration(x)
    torch.cuda.synchronize()
    m.check_routing()
    m.close()
