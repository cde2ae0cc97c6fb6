"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle,
which is itself pinned bit-for-bit to the reference (tests/test_oracle.py).

Bars (north star): routing ids / permutation bit-exact; combine weights
fp32-relative 1e-6; block outputs normwise ||y - y_ref||_inf/||y_ref||_inf
<= 1e-4 (fp32 weights) and <= 2e-2 (bf16 weights), teacher-forced per block
(the oracle runs on the GPU's own block input promoted to fp64).
"""

import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as og  # noqa: E402

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2}
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def P():
    import paper_2308_12066_b200 as p
    return p


def as_torch_w(a: np.ndarray) -> "torch.Tensor":
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(a).cuda()


def normwise(y, ref):
    ref = np.asarray(ref, dtype=np.float64)
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(np.asarray(y, dtype=np.float64) - ref)) / (den if den > 0 else 1.0))


def tokens(d, T, seed=0, scale=1.0):
    from paper_2308_12066_b200._rng import token_batch
    return token_batch(seed, d, T) * np.float32(scale)


# ---------------------------------------------------------------- rng ----

@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_device_weight_generator_bit_exact(dtype):
    p = P()
    for (rows, cols, tag, b, e) in [(3072, 768, og.TAG_W1, 0, 0), (768, 128, og.TAG_PRE_GATE, 5, -1),
                                    (13, 7, og.TAG_W2, 1, 2)]:
        t = p.fill_weights(rows, cols, seed=0, tag=tag, block=b, expert=e, dtype=dtype)
        got = t.view(torch.int16).cpu().numpy().view(np.uint16) if dtype == "bf16" else t.cpu().numpy()
        ref = og.weights(og.derive_seed(0, tag, b, e), rows, cols, dtype)
        assert np.array_equal(got, ref)


# -------------------------------------------------------------- route ----

def _check_route(x, G, k, r):
    ids_ref, w_ref = og.gate_batch(x.astype(np.float64), G, k, nthreads=8)
    ids = r.ids.cpu().numpy()
    assert np.array_equal(ids, ids_ref), "routing ids differ from the reference"
    w = r.w.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(w - w_ref) / w_ref) <= 1e-6
    hist, off, perm, act = og.permute(ids_ref, G.shape[1])
    assert np.array_equal(r.hist.cpu().numpy(), hist)
    assert np.array_equal(r.off.cpu().numpy(), off)
    assert np.array_equal(r.perm.cpu().numpy()[: ids.size], perm)
    assert np.array_equal(r.act.cpu().numpy(), act)
    assert np.array_equal(r.w_perm.cpu().numpy()[: ids.size], r.w.cpu().numpy().reshape(-1)[perm])
    return ids_ref


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("shape", [(1024, 128), (768, 64), (768, 8)])
@pytest.mark.parametrize("T", [1, 37, 300, 700])
def test_route_bit_exact_switch_shapes(dtype, shape, T):
    p = P()
    d, E = shape
    G = og.weights(og.derive_seed(0, og.TAG_PRE_GATE, 3, -1), d, E, dtype)
    x = tokens(d, T, seed=T)
    r = p.route(torch.from_numpy(x).cuda(), as_torch_w(G), 1)
    r.check()
    _check_route(x, G, 1, r)  # flips measured: ids compared with the reference's serial fp64 ranking


@pytest.mark.parametrize("k", [1, 2, 3])
def test_route_topk_and_exact_ties_take_the_serial_path(k):
    """Duplicated gate columns give bit-equal logits: the certified fast path
    cannot separate them, the serial fallback must rank them by id."""
    p = P()
    rng = np.random.default_rng(k)
    d, E, T = 256, 24, 64
    G = rng.uniform(-0.1, 0.1, size=(d, E)).astype(np.float32)
    G[:, 7] = G[:, 3]
    G[:, 20] = G[:, 3]
    G[:, 11] = G[:, 0]
    x = rng.uniform(-0.1, 0.1, size=(T, d)).astype(np.float32)
    # make column 3 the winner for half the tokens
    x[::2] = np.sign(G[:, 3])[None, :] * 0.05
    r = p.route(torch.from_numpy(x).cuda(), torch.from_numpy(G).cuda(), k)
    st = r.check()
    assert st["fallbacks"] >= T // 2
    ids_ref = _check_route(x, G, k, r)
    assert (ids_ref[::2, 0] == 3).all()


def test_route_near_ties_one_ulp_apart():
    p = P()
    rng = np.random.default_rng(5)
    d, E, T = 512, 16, 32
    G = rng.uniform(-0.1, 0.1, size=(d, E)).astype(np.float32)
    G[:, 9] = G[:, 2]
    G[100, 9] = np.nextafter(G[100, 2], np.float32(1))  # logits differ in the last bits
    x = np.tile(np.sign(G[:, 2]) * 0.03, (T, 1)).astype(np.float32)
    x += rng.uniform(-1e-7, 1e-7, size=x.shape).astype(np.float32)
    r = p.route(torch.from_numpy(x).cuda(), torch.from_numpy(G).cuda(), 2)
    r.check()
    _check_route(x, G, 2, r)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("d,E,T", [(768, 64, 1), (768, 64, 3), (1024, 128, 8), (1024, 128, 9), (768, 128, 256),
                                   (1024, 256, 65), (768, 8, 700), (512, 24, 64)])
def test_route_cluster_kernel_equals_split_kernel(monkeypatch, dtype, d, E, T):
    """K1's two forms (thread-block clusters reducing over DSMEM; split-K
    partials through global memory) give identical routing buffers, and
    both equal the reference (ties planted so the serial path runs too)."""
    p = P()
    G = og.weights(og.derive_seed(0, og.TAG_PRE_GATE, 7, -1), d, E, dtype)
    x = tokens(d, T, seed=d + T)
    if E > 16:  # duplicated columns: bit-equal logits the certified path cannot separate
        G = G.copy()
        G[:, 11] = G[:, 5]
        x[::3] = (np.sign(G[:, 5].astype(np.float32) if G.dtype != np.uint16 else
                          (G[:, 5].astype(np.uint32) << 16).view(np.float32)) * 0.05)[None, :]
    xt = torch.from_numpy(x).cuda()
    outs = []
    for mode in ("cluster", "split"):
        monkeypatch.setenv("PGMOE_ROUTE_KERNEL", mode)
        r = p.route(xt, as_torch_w(G), 1)
        st = r.check()
        outs.append((r, st))
    a, b = outs[0][0], outs[1][0]
    for name in ("ids", "w", "hist", "off", "act"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    n = T
    assert torch.equal(a.perm[:n], b.perm[:n]) and torch.equal(a.w_perm[:n], b.w_perm[:n])
    assert outs[0][1]["fallbacks"] == outs[1][1]["fallbacks"]
    _check_route(x, G, 1, a)


def test_route_golden_reference_gate_large():
    """Reference outputs (moesim.gate_forward) on the Large-128 gate shape."""
    p = P()
    with open(os.path.join(GOLD, "switch.json")) as fh:
        cases = json.load(fh)["data"]["gate_large"]
    for c in cases:
        model = og.OracleModel(og.Dims(1024, 4096, 24, 128, 1), c["dtype"])
        G = model.gate(0) if c["which"] == "gate" else model.pre_gate(c["block"])
        x = np.array([float.fromhex(v) for v in c["x"]], dtype=np.float32)[None, :]
        r = p.route(torch.from_numpy(x).cuda(), as_torch_w(G), 1)
        r.check()
        assert r.ids.cpu().tolist() == [c["ids"]]
        assert abs(float(r.w[0, 0]) - float.fromhex(c["w"][0])) <= 1e-6 * float.fromhex(c["w"][0])


def test_route_errors_surface_as_reference_exceptions():
    p = P()
    G = torch.zeros((4, 2), device="cuda")
    G[0, 0], G[0, 1] = 1.0, -1.0
    x = torch.full((1, 4), float("inf"), device="cuda")
    with pytest.raises(p.GateOverflowError, match="numerical overflow in gate"):
        p.route(x, G, 1).check()
    x = torch.zeros((1, 4), device="cuda")
    x[0, 0] = 1000.0
    with pytest.raises(p.GateOverflowError, match="underflowed to zero"):
        p.route(x, G, 2).check()
    with pytest.raises(p.ConfigError):
        p.route(torch.zeros((1, 4), device="cuda"), G, 3)
    with pytest.raises(p.ShapeError):
        p.route(torch.zeros((1, 5), device="cuda"), G, 1)


def test_route_empty_batch():
    p = P()
    G = torch.rand((64, 8), device="cuda")
    r = p.route(torch.zeros((0, 64), device="cuda"), G, 1)
    torch.cuda.synchronize()
    assert r.n_act == 0 and int(r.hist.sum()) == 0


# ---------------------------------------------------- block / decoder ----

def _device_model(dims: og.Dims, dtype: str, placement="resident", max_tokens=64, kernel="auto"):
    p = P()
    cfg = p.ModelConfig(d_model=dims.d_model, d_ff=dims.d_ff, num_blocks=dims.num_blocks,
                        num_experts=dims.num_experts, top_k=dims.top_k,
                        activation_level=dims.activation_level, seed=dims.seed)
    return p.DeviceModel(cfg, dtype=dtype, placement=placement, max_tokens=max_tokens, kernel=kernel)


def _teacher_forced_chain(m, oracle_model, x0, tol, check_blocks=None):
    """Runs moe_block_forward block by block on the device and checks each
    block against the oracle on the device's own block input."""
    p = P()
    c = m.config
    x = torch.from_numpy(x0).cuda()
    T = x.shape[0]
    pending = {}
    outs = []
    for b in range(c.num_blocks):
        if c.has_conv_gate(b):
            r_in = p.route(x, m.matrix("gate", b), c.top_k)
        else:
            r_in = pending.pop(b)
        r_in.check()
        y, r_out = m.moe_block_forward(b, x, r_in)
        torch.cuda.synchronize()
        if check_blocks is None or b in check_blocks:
            xb = x.cpu().numpy().astype(np.float64)
            ids_in = r_in.ids.cpu().numpy()
            w_in = r_in.w.cpu().numpy().astype(np.float64)
            # consumed routing == reference gate on the same input
            G = oracle_model.gate(b) if c.has_conv_gate(b) else None
            if G is not None:
                ids_ref, _ = og.gate_batch(xb, G, c.top_k, nthreads=8)
                assert np.array_equal(ids_in, ids_ref)
            w1 = {e: oracle_model.w1(b, e) for e in np.unique(ids_in)}
            w2 = {e: oracle_model.w2(b, e) for e in np.unique(ids_in)}
            y_ref = og.block_batch(xb, ids_in, w_in, w1, w2, oracle_model.dense(b), c.num_experts, nthreads=8)
            err = normwise(y.cpu().numpy(), y_ref)
            assert err <= tol, f"block {b}: normwise error {err:.3g} > {tol}"
            if r_out is not None:
                r_out.check()
                ids_ref, w_ref = og.gate_batch(xb, oracle_model.pre_gate(b), c.top_k, nthreads=8)
                assert np.array_equal(r_out.ids.cpu().numpy(), ids_ref)
        if r_out is not None:
            pending[b + c.activation_level] = r_out
        outs.append(y)
        x = y
    return outs


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_block_parity_base8_teacher_forced(dtype):
    dims = og.Dims(768, 3072, 12, 8, 1)
    m = _device_model(dims, dtype, max_tokens=16)
    om = og.OracleModel(dims, dtype)
    x0 = tokens(768, 16)
    _teacher_forced_chain(m, om, x0, TOL[dtype], check_blocks={0, 1, 5, 11})
    m.close()


def test_block_matches_reference_golden_outputs():
    """moesim.moe_block_forward outputs captured by gen_golden.py."""
    p = P()
    with open(os.path.join(GOLD, "switch.json")) as fh:
        cases = json.load(fh)["data"]["block_base8"]
    for dtype in ("f32", "bf16"):
        m = _device_model(og.Dims(768, 3072, 12, 8, 1), dtype, max_tokens=4)
        for c in (c for c in cases if c["dtype"] == dtype):
            x = torch.tensor([[float.fromhex(v) for v in c["x"]]], dtype=torch.float32, device="cuda")
            r_in = p.DeviceRouting.from_host(np.array([c["ids_in"]]), np.array([[float.fromhex(c["w_in"][0])]]), 8)
            y, r_out = m.moe_block_forward(c["block"], x, r_in)
            y_ref = [float.fromhex(v) for v in c["y"]]
            assert normwise(y[0].cpu().numpy(), y_ref) <= TOL[dtype]
            r_out.check()
            assert r_out.ids.cpu().tolist() == [c["ids_out"]]
        m.close()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_decoder_iteration_equals_block_chain_and_small_configs(dtype):
    rng = np.random.default_rng(11)
    for trial in range(6):
        dims = og.Dims(d_model=int(rng.integers(2, 40)), d_ff=int(rng.integers(2, 50)),
                       num_blocks=int(rng.integers(2, 6)), num_experts=int(rng.integers(2, 17)),
                       top_k=int(rng.integers(1, 3)), activation_level=1, seed=trial)
        if dims.top_k > dims.num_experts:
            continue
        m = _device_model(dims, dtype, max_tokens=8)
        om = og.OracleModel(dims, dtype)
        x0 = tokens(dims.d_model, 8, seed=trial)
        outs = _teacher_forced_chain(m, om, x0, TOL[dtype])
        y, ids, w = m.decoder_iteration(torch.from_numpy(x0).cuda(), trace=True)
        torch.cuda.synchronize()
        assert torch.equal(y, outs[-1]), "decoder_iteration must equal the moe_block_forward chain bitwise"
        m.close()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_offloaded_equals_resident_and_ledger(dtype):
    dims = og.Dims(256, 512, 6, 16, 1, seed=4)
    T = 24
    x0 = torch.from_numpy(tokens(256, T)).cuda()
    res = _device_model(dims, dtype, "resident", max_tokens=T)
    off = _device_model(dims, dtype, "offloaded", max_tokens=T)
    y0, ids0, w0 = res.decoder_iteration(x0, trace=True)
    off.reset_stats()
    y1, ids1, w1 = off.decoder_iteration(x0, trace=True)
    torch.cuda.synchronize()
    assert torch.equal(ids0, ids1) and torch.equal(w0, w1)
    assert torch.equal(y0, y1)
    st = off.stats()
    rec = 2 * 256 * 512 * (2 if dtype == "bf16" else 4)
    n_act = [len(np.unique(ids1[b].cpu().numpy())) for b in range(dims.num_blocks)]
    assert st["h2d_bytes"] == sum(n_act) * rec
    eq1 = st["pinned_hbm_bytes"] + max(rec * (n_act[i] + (n_act[i + 1] if i + 1 < len(n_act) else 0))
                                       for i in range(len(n_act)))
    assert st["eq1_peak_bytes"] == eq1
    assert st["ledger_peak_bytes"] <= eq1
    # host-buffer entry point gives the same answer
    yh, idh, wh = off.decoder_iteration_host(x0.cpu().numpy(), trace=True)
    assert np.array_equal(yh, y1.cpu().numpy()) and np.array_equal(idh, ids1.cpu().numpy())
    res.close()
    off.close()


@pytest.mark.parametrize("L", [2, 3])
def test_fused_routing_with_deeper_lookahead(L):
    """Lookahead L >= 2 (core.py:73-89: block b's pre-gate decides block b+L):
    the routing computed inside block b's launch goes to ring entry (b+L) %
    (L+1) while the dense epilogue packs block b+1's operand from the entry
    an earlier launch filled.  Outputs and decisions equal the separate-K1
    schedule and the offloaded one bitwise, and the teacher-forced oracle."""
    dims = og.Dims(256, 2048, 6, 64, 1, activation_level=L, seed=11)
    T = 24
    xn = tokens(256, T, seed=L)
    x0 = torch.from_numpy(xn).cuda()
    fused = _device_model(dims, "bf16", "resident", max_tokens=T)
    sep = _device_model(dims, "bf16", "resident", max_tokens=T)
    sep.set_fused_route(False)
    off = _device_model(dims, "bf16", "offloaded", max_tokens=T)
    outs = []
    for m in (fused, sep, off):
        m.reset_stats()
        for _ in range(2):
            y, ids, w = m.decoder_iteration(x0, trace=True)
        torch.cuda.synchronize()
        outs.append((y.clone(), ids.clone(), w.clone()))
    assert fused.stats()["fused_routes"] > 0 and sep.stats()["fused_routes"] == 0
    for y, ids, w in outs[1:]:
        assert torch.equal(outs[0][1], ids) and torch.equal(outs[0][2], w)
        assert torch.equal(outs[0][0], y)
    om = og.OracleModel(dims, "bf16")
    _teacher_forced_chain(fused, om, xn, TOL["bf16"])
    for m in (fused, sep, off):
        m.close()


@pytest.mark.parametrize("E,T", [(64, 1), (64, 10), (64, 40), (128, 33), (128, 256), (256, 17)])
def test_fused_routing_equals_separate_launch_and_offloaded(E, T):
    """Resident top-1 decoding computes each pre-gate inside the block's
    tcgen05 launch (route_common.cuh).  Routing ids, weights and block
    outputs must equal the separate-K1 schedule and the offloaded one bitwise,
    including tokens whose ranking needs the serial-fp64 recompute (exact
    ties planted in block 0's pre-gate)."""
    dims = og.Dims(256, 2048, 5, E, 1, seed=7)  # the routing role is fused while T <= d_ff / 8
    x0 = torch.from_numpy(tokens(256, T)).cuda()
    fused = _device_model(dims, "bf16", "resident", max_tokens=T)
    fused.set_ll_decode(False)
    fused.set_decode(False)  # the per-block launches (the persistent small-batch launch: test_gpu_decode.py)
    sep = _device_model(dims, "bf16", "resident", max_tokens=T)
    sep.set_fused_route(False)
    off = _device_model(dims, "bf16", "offloaded", max_tokens=T)
    g = fused.get_matrix("pre_gate", 0)
    g[:, 1] = g[:, 0]  # exact ties between experts 0, 1 and 2
    g[:, 2] = g[:, 0]
    for m in (fused, sep, off):
        m.set_matrix("pre_gate", 0, -1, g)
    outs = []
    for m in (fused, sep, off):
        m.reset_stats()
        for _ in range(2):  # the second call replays the captured graph (resident)
            y, ids, w = m.decoder_iteration(x0, trace=True)
        torch.cuda.synchronize()
        outs.append((y.clone(), ids.clone(), w.clone()))
    nf = fused.stats()["fused_routes"]  # counted per host pass (a graph capture is one pass)
    assert nf > 0 and nf % (dims.num_blocks - 1) == 0
    assert sep.stats()["fused_routes"] == 0
    for y, ids, w in outs[1:]:
        assert torch.equal(outs[0][1], ids) and torch.equal(outs[0][2], w)
        assert torch.equal(outs[0][0], y)
    st_f, st_s = fused.stats(), sep.stats()
    assert st_f["route_fallbacks"] == st_s["route_fallbacks"]
    for m in (fused, sep, off):
        m.close()


def test_chained_block_launches_equal_pdl_chain(monkeypatch):
    """Chained launches (the default; PGMOE_CHAIN=0 turns them off): each
    resident block launch waits for its predecessor's dense phase through a
    device counter (parity-buffered counters) instead of its completion;
    outputs and routing must be identical, eagerly and from the graph."""
    dims = og.Dims(256, 512, 6, 128, 1, seed=9)
    x0 = torch.from_numpy(tokens(256, 48)).cuda()
    monkeypatch.setenv("PGMOE_CHAIN", "0")
    base = _device_model(dims, "bf16", "resident", max_tokens=48)
    monkeypatch.setenv("PGMOE_CHAIN", "1")
    chained = _device_model(dims, "bf16", "resident", max_tokens=48)
    outs = []
    for m in (base, chained):
        for _ in range(3):
            y, ids, w = m.decoder_iteration(x0, trace=True)
        torch.cuda.synchronize()
        outs.append((y.clone(), ids.clone(), w.clone()))
        yg = torch.empty_like(x0)
        for _ in range(3):  # captured once, then replayed (persistent buffers)
            m.decoder_iteration(x0, out=yg)
        torch.cuda.synchronize()
        outs[-1] = outs[-1] + (yg.clone(),)
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)
    assert torch.equal(outs[1][0], outs[1][3])
    base.close()
    chained.close()


def test_timeline_schema_and_causality():
    dims = og.Dims(128, 256, 4, 8, 1)
    m = _device_model(dims, "bf16", "offloaded", max_tokens=8)
    m.set_timeline(True)
    m.decoder_iteration(torch.from_numpy(tokens(128, 8)).cuda())
    ev = m.timeline()
    assert {e["lane"] for e in ev} == {"compute", "transfer"}
    for e in ev:
        assert set(e) == {"lane", "label", "block", "start_s", "end_s"} and e["end_s"] >= e["start_s"]
    fetch = {e["block"]: e for e in ev if e["lane"] == "transfer"}
    experts = {e["block"]: e for e in ev if e["label"] == "experts"}
    for b, e in experts.items():  # no expert runs before its transfer ends
        assert e["start_s"] >= fetch[b]["end_s"] - 1e-6
    m.close()


# ------------------------------------------------- reference drop-ins ----

def test_dropin_single_token_api_matches_oracle():
    p = P()
    rng = np.random.default_rng(3)
    G = rng.uniform(-1, 1, size=(6, 8)).astype(np.float32).astype(np.float64)
    x = rng.uniform(-1, 1, size=6).astype(np.float32).astype(np.float64)
    d = p.gate_forward(x.tolist(), G.tolist(), 2)
    ids, w, _ = og.gate_forward(x, G, 2)
    assert d.expert_ids == ids
    assert np.allclose(d.combine_weights, w, rtol=1e-6)

    class Ex:
        pass
    ex = Ex()
    ex.w1 = rng.uniform(-1, 1, size=(12, 6)).astype(np.float32).tolist()
    ex.w2 = rng.uniform(-1, 1, size=(6, 12)).astype(np.float32).tolist()
    y = p.expert_forward(x.tolist(), ex)
    y_ref = og.expert_forward(x, np.array(ex.w1, np.float32), np.array(ex.w2, np.float32))
    assert normwise(y, y_ref) <= 1e-5
    with pytest.raises(p.ShapeError):
        p.expert_forward([1.0, 2.0], ex)


# ------------------------------------------------- tcgen05 vs SIMT / oracle

@pytest.mark.parametrize("T,E,k", [(1, 128, 1), (5, 8, 1), (37, 64, 1), (256, 128, 1), (600, 2, 1), (64, 16, 2),
                                   (300, 8, 2)])
def test_tcgen05_grouped_ffn_matches_oracle(T, E, k):
    """K2 on tcgen05 (split-K at small T, multi N-tiles for hot experts) vs
    the oracle's fp64 experts+combine, and vs the SIMT kernel."""
    p = P()
    d, f = 256, 512
    rng = np.random.default_rng(T * 7 + E)
    G = og.weights(og.derive_seed(1, og.TAG_GATE, 0, -1), d, E, "bf16")
    x = tokens(d, T, seed=E)
    xt = torch.from_numpy(x).cuda()
    r = p.route(xt, as_torch_w(G), k)
    r.check()
    recs = np.stack([np.concatenate([og.weights(og.derive_seed(1, og.TAG_W1, 0, e), f, d, "bf16").reshape(-1),
                                     og.weights(og.derive_seed(1, og.TAG_W2, 0, e), d, f, "bf16").reshape(-1)])
                     for e in range(E)])
    recs_t = as_torch_w(recs)
    yw_tc = p.expert_ffn(xt, r, recs_t, f, kernel="tcgen05")
    yw_simt = p.expert_ffn(xt, r, recs_t, f, kernel="simt")
    torch.cuda.synchronize()
    ids = r.ids.cpu().numpy()
    w = r.w.cpu().numpy().astype(np.float64)
    ref = np.zeros((T * k, d))
    for t in range(T):
        for s in range(k):
            e = ids[t, s]
            ref[t * k + s] = w[t, s] * og.expert_forward(x[t].astype(np.float64), recs[e, : f * d].reshape(f, d),
                                                         recs[e, f * d:].reshape(d, f))
    assert normwise(yw_simt.cpu().numpy(), ref) <= 1e-4
    assert normwise(yw_tc.cpu().numpy(), ref) <= TOL["bf16"]
    # dense on tcgen05 (split-K, k-slot sum) vs oracle
    D = og.weights(og.derive_seed(1, og.TAG_DENSE, 0, -1), d, d, "bf16")
    y_tc = p.dense(yw_tc, T, k, as_torch_w(D), kernel="tcgen05")
    mix = yw_tc.cpu().numpy().astype(np.float64).reshape(T, k, d).sum(1)
    y_ref = np.stack([og.matvec(D, mix[t]) for t in range(T)])
    assert normwise(y_tc.cpu().numpy(), y_ref) <= TOL["bf16"]


def test_tcgen05_deterministic_across_runs():
    p = P()
    d, f, E, T = 256, 512, 4, 3
    x = torch.from_numpy(tokens(d, T)).cuda()
    G = as_torch_w(og.weights(og.derive_seed(2, og.TAG_GATE, 0, -1), d, E, "bf16"))
    r = p.route(x, G, 1)
    recs = torch.randn((E, 2 * f * d), device="cuda").to(torch.bfloat16) * 0.05
    a = p.expert_ffn(x, r, recs, f, kernel="tcgen05")
    b = p.expert_ffn(x, r, recs, f, kernel="tcgen05")
    torch.cuda.synchronize()
    assert torch.equal(a, b)


@pytest.mark.parametrize("placement", ["resident", "offloaded"])
def test_model_tcgen05_equals_teacher_forced_oracle_large_dims(placement):
    dims = og.Dims(1024, 4096, 3, 128, 1)
    m = _device_model(dims, "bf16", placement, max_tokens=64, kernel="tcgen05")
    om = og.OracleModel(dims, "bf16")
    _teacher_forced_chain(m, om, tokens(1024, 64), TOL["bf16"], check_blocks={0, 2})
    m.close()


# ------------------------------------------------------ expert parallel ----

@pytest.mark.parametrize("k", [1, 2])
def test_ep_decoder_single_rank_nccl_equals_single_gpu(k):
    """EP plumbing on one rank (NCCL world of 1): dispatch/combine over NCCL,
    receiver routing and un-permute must reproduce the single-GPU decoder
    bit-for-bit."""
    import socket
    import torch.distributed as dist
    p = P()
    from paper_2308_12066_b200.ep import EPDecoder
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        cfg = p.ModelConfig(d_model=256, d_ff=512, num_blocks=4, num_experts=16, top_k=k, activation_level=1)
        x = p.token_inputs(cfg, 24)
        ep = EPDecoder(cfg, dtype="bf16", max_tokens=24)
        y_ep, ids_ep = ep.decoder_iteration(x, trace=True)
        ref = p.DeviceModel(cfg, dtype="bf16", max_tokens=24)
        y, ids, _ = ref.decoder_iteration(x, trace=True)
        torch.cuda.synchronize()
        assert torch.equal(ids_ep, ids)
        assert torch.equal(y_ep, y)
        # without a trace the iteration is captured once and replayed
        for _ in range(3):
            y_g, _ = ep.decoder_iteration(x)
        torch.cuda.synchronize()
        assert ep.replayed_kernels > 0 and torch.equal(y_g, y)
        ep.close()
        ref.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("Pn", [2, 4])
def test_ep_ranks_in_one_process_equal_single_gpu(monkeypatch, Pn):
    """The P > 1 device path of the fixed-size EP exchange (slots per peer,
    in-band counts, receiver routing over P sources, un-permute) on one GPU:
    P EPDecoder ranks in P threads (one stream: stream-ordered like P
    processes), the all-to-all replaced by a copy of the peers' slots.  Every
    rank's outputs and routing must equal the single-GPU decoder on the
    concatenated batch bit-for-bit."""
    import threading
    import paper_2308_12066_b200.ep as epm
    p = P()
    T = 24
    cfg = p.ModelConfig(d_model=256, d_ff=512, num_blocks=4, num_experts=16, top_k=2, activation_level=1)

    class Hub:
        barrier = threading.Barrier(Pn, timeout=120)  # a stuck rank fails the test instead of hanging it
        bufs: dict = {}

    class SlotExchange:  # what all_to_all_single does with equal splits
        def __init__(self, rank):
            self.P, self.rank = Pn, rank

        def fixed(self, send, recv):
            torch.cuda.synchronize()
            Hub.bufs[self.rank] = send
            Hub.barrier.wait()
            c = send.shape[0] // Pn
            for q in range(Pn):
                recv[q * c:(q + 1) * c].copy_(Hub.bufs[q][self.rank * c:(self.rank + 1) * c])
            torch.cuda.synchronize()
            Hub.barrier.wait()
            return recv

    monkeypatch.setattr(epm, "Exchange", lambda group: group)
    from paper_2308_12066_b200._rng import token_batch
    xs = [torch.from_numpy(token_batch(0, 256, T, offset=r * T)).cuda() for r in range(Pn)]
    out, errs = {}, []

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            ep = epm.EPDecoder(cfg, dtype="bf16", max_tokens=T, group=SlotExchange(r))
            ep.use_graph = False
            y, ids = ep.decoder_iteration(xs[r], trace=True)
            torch.cuda.synchronize()
            out[r] = (y.clone(), ids.clone())
            ep.close()
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            Hub.barrier.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(Pn)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    assert len(out) == Pn
    ref = p.DeviceModel(cfg, dtype="bf16", max_tokens=Pn * T)
    y, ids, _ = ref.decoder_iteration(torch.cat(xs), trace=True)
    torch.cuda.synchronize()
    for r in range(Pn):
        assert torch.equal(out[r][1], ids[:, r * T:(r + 1) * T])
        assert torch.equal(out[r][0], y[r * T:(r + 1) * T])
    ref.close()


# ------------------------------------------------- migration strategies ----

@pytest.mark.parametrize("strategy", ["pre_gated", "on_demand", "prefetch_all"])
def test_strategies_change_the_schedule_not_the_math(strategy):
    """scheduler.py:220-410: outputs are identical under every strategy; the
    copy schedule follows the strategy (checked on the real event timeline)."""
    dims = og.Dims(256, 512, 5, 8, 1, seed=2)
    T = 16
    x0 = torch.from_numpy(tokens(256, T)).cuda()
    res = _device_model(dims, "bf16", "resident", max_tokens=T)
    y_ref, ids_ref, _ = res.decoder_iteration(x0, trace=True)
    m = _device_model(dims, "bf16", "offloaded", max_tokens=T)
    m.set_strategy(strategy)
    m.set_timeline(True)
    m.reset_stats()
    y, ids, _ = m.decoder_iteration(x0, trace=True)
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref) and torch.equal(ids, ids_ref)
    ev = m.timeline()
    fetch = {e["block"]: e for e in ev if e["lane"] == "transfer"}
    experts = {e["block"]: e for e in ev if e["label"] == "experts"}
    dense = {e["block"]: e for e in ev if e["label"] == "non_moe"}
    rec = 2 * 256 * 512 * 2
    st = m.stats()
    n_act = [len(np.unique(ids[b].cpu().numpy())) for b in range(dims.num_blocks)]
    for b in range(dims.num_blocks):
        assert experts[b]["start_s"] >= fetch[b]["end_s"] - 1e-6
    if strategy == "prefetch_all":
        assert st["h2d_bytes"] == dims.num_blocks * dims.num_experts * rec
        for b in range(1, dims.num_blocks):  # block b's set streams while block b-1 computes
            assert fetch[b]["start_s"] <= dense[b - 1]["end_s"]
    else:
        assert st["h2d_bytes"] == sum(n_act) * rec
    if strategy == "on_demand":
        for b in range(1, dims.num_blocks):  # serial: no transfer before the previous block finished
            assert fetch[b]["start_s"] >= dense[b - 1]["end_s"] - 1e-6
    res.close()
    m.close()


@pytest.mark.parametrize("strategy", ["pre_gated", "prefetch_all"])
@pytest.mark.parametrize("policy", ["lru", "lfu", "lifo"])
def test_expert_cache_saves_pcie_not_math(strategy, policy):
    """cache.py: with the whole expert set cacheable, a repeated iteration
    moves nothing over PCIe; a small cache moves less; outputs unchanged."""
    dims = og.Dims(256, 512, 4, 8, 1, seed=6)
    T = 8
    x0 = torch.from_numpy(tokens(256, T)).cuda()
    ref = _device_model(dims, "bf16", "resident", max_tokens=T)
    y_ref, _, _ = ref.decoder_iteration(x0)
    m = _device_model(dims, "bf16", "offloaded", max_tokens=T)
    m.set_strategy(strategy)
    m.set_cache(policy, 1.0)
    m.decoder_iteration(x0)
    m.reset_stats()
    y, _, _ = m.decoder_iteration(x0)
    torch.cuda.synchronize()
    st = m.stats()
    assert torch.equal(y, y_ref)
    assert st["h2d_bytes"] == 0 and st["cache_hits"] > 0
    m.set_cache(policy, 0.3)
    m.reset_stats()
    m.decoder_iteration(x0)
    y2, _, _ = m.decoder_iteration(x0)
    torch.cuda.synchronize()
    assert torch.equal(y2, y_ref)
    m.set_cache("none", 0.0)
    ref.close()
    m.close()


@pytest.mark.parametrize("level", [0, 2])
@pytest.mark.parametrize("placement", ["resident", "offloaded"])
def test_activation_levels_wiring_and_migration(level, placement):
    """core.py:73-89: level 0 = conventional gating (every block its own gate,
    on-demand fetch when offloaded), level 2 = decisions two blocks ahead
    (three expert slots).  Device decisions equal the oracle's decoder run on
    the device's own block inputs; offloaded equals resident."""
    p = P()
    dims = og.Dims(128, 256, 5, 8, 2, activation_level=level, seed=9)
    T = 12
    x0 = tokens(128, T, seed=3)
    res = _device_model(dims, "f32", "resident", max_tokens=T)
    om = og.OracleModel(dims, "f32")
    outs = _teacher_forced_chain(res, om, x0, TOL["f32"])
    y, ids, w = res.decoder_iteration(torch.from_numpy(x0).cuda(), trace=True)
    torch.cuda.synchronize()
    assert torch.equal(y, outs[-1])
    if placement == "offloaded":
        off = _device_model(dims, "f32", "offloaded", max_tokens=T)
        if level == 0:
            off.set_strategy("on_demand")
        y2, ids2, _ = off.decoder_iteration(torch.from_numpy(x0).cuda(), trace=True)
        torch.cuda.synchronize()
        assert torch.equal(ids2, ids) and torch.equal(y2, y)
        off.close()
    res.close()


@pytest.mark.parametrize("Pn,El", [(1, 128), (3, 16), (8, 16)])
def test_ep_recv_route_pack_equals_two_launches(Pn, El):
    """pgmoe_ep_recv_route_pack (receiver routing + packing in one launch) ==
    pgmoe_ep_local_routing_padded then pgmoe_ep_pack_recv, bit for bit, on a
    received slot buffer with random in-band counts (empty experts and empty
    sources included)."""
    import ctypes
    p = P()
    from paper_2308_12066_b200 import _lib
    L = _lib.load()
    d, cap = 256, 40
    slot = int(L.pgmoe_ep_slot_rows(cap, El, d))
    g = torch.Generator().manual_seed(7 + Pn)
    recv = torch.randn((Pn * slot, d), generator=g).to(torch.bfloat16)
    for q in range(Pn):
        cnt = torch.zeros(El, dtype=torch.int32)
        n = 0 if q == 1 else int(torch.randint(0, cap + 1, (1,), generator=g))
        for _ in range(n):
            cnt[int(torch.randint(0, El // 2 if El > 2 else El, (1,), generator=g)) * 2 % El] += 1
        hdr = recv[q * slot + cap:(q + 1) * slot].contiguous().view(torch.int32).view(-1)
        hdr[:El] = cnt
        recv[q * slot + cap:(q + 1) * slot] = hdr.view(torch.bfloat16).view(-1, d)
    recv = recv.cuda()
    outs = []
    for fused in (False, True):
        lr = p.DeviceRouting(Pn * slot, El, 1)
        xb = torch.zeros((Pn * cap, d), dtype=torch.bfloat16, device="cuda")
        if fused:
            _lib.check(L.pgmoe_ep_recv_route_pack(recv.data_ptr(), Pn, El, cap, d, ctypes.byref(lr.c),
                                                  xb.data_ptr(), None))
        else:
            _lib.check(L.pgmoe_ep_local_routing_padded(recv.data_ptr(), Pn, El, cap, d, ctypes.byref(lr.c), None))
            _lib.check(L.pgmoe_ep_pack_recv(recv.data_ptr(), ctypes.byref(lr.c), El, Pn * cap, d, xb.data_ptr(),
                                            None))
        torch.cuda.synchronize()
        outs.append((lr, xb))
    (a, xa), (b, xb2) = outs
    total = int(a.off[El].item())
    assert total > 0
    for name in ("hist", "off", "act_n", "ids", "w"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    assert torch.equal(a.perm[:total], b.perm[:total]) and torch.equal(a.w_perm[:total], b.w_perm[:total])
    assert torch.equal(xa[:total], xb2[:total])
