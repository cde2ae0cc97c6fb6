"""Parity at the benchmark's own shapes.

DeviceModel runs exactly as bench.py runs it — default kernels, routing
fused into the block launch (resident), chained block launches, CUDA-graph
replay, offloaded slots — at T=256 on every block of the Switch configs, two
chained decoder iterations.  The traced run (block inputs copied out between
launches) must equal the plain run bitwise; then every block is checked
against the oracle teacher-forced on the GPU's own block inputs
(oracle/parity.py): routing ids of all 256 tokens bit-exact at every block,
combine weights within 1e-6, and block outputs of 16 sampled tokens at >= 4
blocks (including the last) within the bf16 bar 2e-2 normwise.

Also here: the chained (not teacher-forced) flip measurement, supplied
decisions in the batched path, prefetch_all with lookahead 0, and the
persistent kernel on a reduced-SM context.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import oracle as og  # noqa: E402
from oracle import parity  # noqa: E402

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PRESETS = {  # presets.py:64-70 full-size dims
    "base64": (768, 3072, 12, 64),
    "base128": (768, 3072, 12, 128),
    "large128": (1024, 4096, 24, 128),
}
BF16_TOL = 2e-2


def P():
    import paper_2308_12066_b200 as p
    return p


def run_traced(m, x, iterations):
    """`iterations` chained decoder iterations through the bench's call, once
    plain (graph replay / the default launch sequence) and once with block
    inputs and decisions traced.  Returns per iteration (x_trace, y, ids, w)
    on the host, after checking traced == plain bitwise."""
    c = m.config
    T = x.shape[0]
    y_plain = torch.empty_like(x)
    y_tr = torch.empty_like(x)
    xt = torch.empty((c.num_blocks, T, c.d_model), dtype=torch.float32, device="cuda")
    ids = torch.empty((c.num_blocks, T, c.top_k), dtype=torch.int32, device="cuda")
    w = torch.empty((c.num_blocks, T, c.top_k), dtype=torch.float32, device="cuda")
    out = []
    cur = x
    for _ in range(iterations):
        for _ in range(2):  # the second call replays the captured graph (resident)
            m.decoder_iteration(cur, out=y_plain)
        m.decoder_iteration(cur, out=y_tr, x_trace=xt, trace_out=(ids, w))
        torch.cuda.synchronize()
        m.check_routing()
        assert torch.equal(y_plain, y_tr), "tracing block inputs changed the result"
        assert torch.equal(xt[0], cur)
        out.append((xt.cpu().numpy(), y_tr.cpu().numpy(), ids.cpu().numpy(), w.cpu().numpy()))
        cur = y_tr.clone()
    return out


@pytest.mark.parametrize("preset,placement", [("large128", "offloaded"), ("large128", "resident"),
                                              ("base64", "resident"), ("base128", "offloaded")])
def test_bench_shape_teacher_forced_parity(preset, placement):
    p = P()
    d, f, nb, E = PRESETS[preset]
    T = 256
    cfg = p.ModelConfig(d_model=d, d_ff=f, num_blocks=nb, num_experts=E, top_k=1, activation_level=1, seed=0)
    dims = og.Dims(d, f, nb, E, 1, 1, 0)
    m = p.DeviceModel(cfg, dtype="bf16", placement=placement, max_tokens=T)
    x = p.token_inputs(cfg, T)
    runs = run_traced(m, x, 2)
    st = m.stats()
    m.close()
    if placement == "resident":
        assert st["fused_routes"] > 0, "the bench's resident path routes inside the block launch"
    sample = np.linspace(0, T - 1, 16).astype(int)
    om = og.OracleModel(dims, "bf16")
    for it, (xt, y, ids, w) in enumerate(runs):
        # iteration 2 starts ~1e-29 (Large) and leaves the fp32 range after
        # a few blocks: check the blocks whose input is still normal
        blocks = {0, 1, nb // 2, nb - 1} if it == 0 else {0, 1, 2, 3}
        r = parity.teacher_forced(dims, "bf16", xt, y, ids, w, sample, blocks, model=om)
        assert r["ids_mismatch_tokens"] == 0, f"iteration {it}: routing ids differ from the reference"
        assert r["ids_blocks_checked"] >= (nb if it == 0 else 4)
        assert r["w_max_rel"] <= 1e-6
        checked = [b["block"] for b in r["blocks"]]
        assert len(checked) >= 4 and (it > 0 or nb - 1 in checked), r
        assert r["max_err"] <= BF16_TOL, r["blocks"]


def test_chained_flip_measurement_runs_and_starts_clean():
    """The GPU's own chain beside the oracle's fp64 chain (no teacher
    forcing).  Blocks 0 and 1 consume decisions computed from the identical
    fp32 input, so they cannot flip; later flips are counted, not assumed."""
    p = P()
    d, f, nb, E = PRESETS["base64"]
    T, S = 64, 6
    cfg = p.ModelConfig(d_model=d, d_ff=f, num_blocks=nb, num_experts=E, top_k=1, activation_level=1, seed=0)
    dims = og.Dims(d, f, nb, E, 1, 1, 0)
    m = p.DeviceModel(cfg, dtype="bf16", placement="resident", max_tokens=T)
    x = p.token_inputs(cfg, T)
    runs = run_traced(m, x, 3)
    m.close()
    sample = np.arange(S) * 10
    gx = [xt[:, sample] for xt, _, _, _ in runs]
    gi = [ids[:, sample] for _, _, ids, _ in runs]
    r = parity.chained(dims, "bf16", runs[0][0][0][sample], gx, gi)
    assert r["iterations"] == 3 and len(r["per_block"]) == 3 * nb
    first = r["per_block"][:2]
    assert first[0]["flips"] == 0 and first[1]["flips"] == 0
    assert first[0]["input_err"] == 0.0
    # the first block's output drifts only by bf16 rounding
    assert r["per_block"][1]["input_err"] <= BF16_TOL


@pytest.mark.parametrize("placement", ["resident", "offloaded"])
def test_supplied_decisions_equal_routed_run(placement):
    """core.py:342-364 supplied_decisions in the batched C ABI: replaying the
    decisions the gates produced reproduces the routed run bitwise (same
    kernels, same migration); a synthetic skewed trace runs too; invalid
    decisions raise RoutingError and leave the model usable."""
    p = P()
    d, f, nb, E, T = 256, 512, 6, 32, 40
    cfg = p.ModelConfig(d_model=d, d_ff=f, num_blocks=nb, num_experts=E, top_k=1, activation_level=1, seed=3)
    m = p.DeviceModel(cfg, dtype="bf16", placement=placement, max_tokens=T)
    x = p.token_inputs(cfg, T)
    y0, ids, w = m.decoder_iteration(x, trace=True)
    torch.cuda.synchronize()
    m.reset_stats()
    y1, ids1, w1 = m.decoder_iteration(x, trace=True, supplied=(ids.clone(), w.clone()))
    torch.cuda.synchronize()
    m.check_routing()
    assert torch.equal(ids, ids1) and torch.equal(w, w1)
    assert torch.equal(y0, y1)
    if placement == "offloaded":
        rec = 2 * d * f * 2
        n_act = sum(len(np.unique(ids[b].cpu().numpy())) for b in range(nb))
        assert m.stats()["h2d_bytes"] == n_act * rec
    # a skewed synthetic trace: every token on experts 0..3
    sid = (torch.arange(nb * T, device="cuda", dtype=torch.int32) % 4).reshape(nb, T, 1)
    sw = torch.full((nb, T, 1), 0.5, device="cuda")
    y2, ids2, _ = m.decoder_iteration(x, trace=True, supplied=(sid, sw))
    torch.cuda.synchronize()
    m.check_routing()
    assert torch.equal(ids2, sid) and torch.isfinite(y2).all()
    bad = sid.clone()
    bad[2, 5, 0] = E  # out of range
    m.decoder_iteration(x, supplied=(bad, sw))
    with pytest.raises(p.RoutingError):
        m.check_routing()
    y3, _, _ = m.decoder_iteration(x, trace=True, supplied=(ids, w))
    torch.cuda.synchronize()
    m.check_routing()
    assert torch.equal(y3, y0)
    m.close()


def test_prefetch_all_with_lookahead_zero():
    """activation_level 0 (conventional gates everywhere): prefetch_all needs
    two whole-block slots, or block b+1's set overwrites block b's."""
    p = P()
    d, f, nb, E, T = 256, 512, 5, 16, 24
    cfg = p.ModelConfig(d_model=d, d_ff=f, num_blocks=nb, num_experts=E, top_k=1, activation_level=0, seed=5)
    x = p.token_inputs(cfg, T)
    res = p.DeviceModel(cfg, dtype="bf16", placement="resident", max_tokens=T)
    y_ref, ids_ref, _ = res.decoder_iteration(x, trace=True)
    torch.cuda.synchronize()
    res.close()
    for strategy in ("prefetch_all", "on_demand"):
        off = p.DeviceModel(cfg, dtype="bf16", placement="offloaded", max_tokens=T)
        off.set_strategy(strategy)
        for _ in range(2):
            y, ids, _ = off.decoder_iteration(x, trace=True)
        torch.cuda.synchronize()
        assert torch.equal(ids, ids_ref) and torch.equal(y, y_ref), strategy
        off.close()


_REDUCED_SM = r'''
import os, sys, numpy as np
sys.path.insert(0, os.environ["ROOT"])
mode = sys.argv[1]
if mode == "green":
    import ctypes
    from paper_2308_12066_b200 import _lib
    n = ctypes.c_int32(0)
    _lib.check(_lib.load().pgmoe_debug_green_context(int(sys.argv[2]), ctypes.byref(n)))
    print("green context SMs:", n.value, flush=True)
import paper_2308_12066_b200 as p
cfg = p.ModelConfig(d_model=256, d_ff=2048, num_blocks=4, num_experts=64, top_k=1, activation_level=1, seed=2)
m = p.DeviceModel(cfg, dtype="bf16", placement="resident", max_tokens=32)
from paper_2308_12066_b200._rng import token_batch
y, ids, w = m.decoder_iteration_host(token_batch(2, 256, 32), trace=True)
np.save(sys.argv[3], y)
np.save(sys.argv[3] + ".ids.npy", ids)
print("done", flush=True)
'''


@pytest.mark.parametrize("mode", ["limit", "green"])
def test_persistent_kernel_on_fewer_sms(tmp_path, mode):
    """The persistent block kernel spins on grid-wide counters, so its grid
    must be what is co-resident.  On a context with fewer SMs (a green
    context carved out with cuGreenCtxCreate, or PGMOE_SM_LIMIT) it sizes its
    grid from the context and must run to the same routing and outputs
    within the bf16 bar — never hang (the subprocess has a hard timeout)."""
    script = tmp_path / "run.py"
    script.write_text(_REDUCED_SM)
    env = dict(os.environ, ROOT=ROOT)
    ref = tmp_path / "ref.npy"
    r0 = subprocess.run([sys.executable, str(script), "full", "0", str(ref)], env=env, timeout=300,
                        capture_output=True, text=True)
    assert r0.returncode == 0, r0.stderr[-2000:]
    out = tmp_path / "out.npy"
    if mode == "limit":
        env["PGMOE_SM_LIMIT"] = "37"
    r = subprocess.run([sys.executable, str(script), mode, "24", str(out)], env=env, timeout=300,
                       capture_output=True, text=True)
    if mode == "green" and r.returncode != 0 and "green context SMs" not in r.stdout:
        pytest.skip("green contexts unavailable here: " + r.stderr[-300:])
    assert r.returncode == 0, r.stderr[-2000:]
    assert np.array_equal(np.load(str(ref) + ".ids.npy"), np.load(str(out) + ".ids.npy"))
    a, b = np.load(ref), np.load(out)
    assert np.max(np.abs(a - b)) <= BF16_TOL * np.max(np.abs(a))


def test_block_end_stamps_of_chained_launches():
    """Chained resident block launches stamp when each block's dense layer
    completes (pgmoe_model_block_stamps); the bench derives the reference's
    block latency (scheduler.py:374-397) from them on graph-replayed
    iterations.  Stamps are per block, increasing, and span less than the
    event-timed iteration."""
    import ctypes
    p = P()
    from paper_2308_12066_b200 import _lib
    cfg = p.ModelConfig(d_model=256, d_ff=2048, num_blocks=5, num_experts=64, top_k=1, activation_level=1)
    m = p.DeviceModel(cfg, dtype="bf16", placement="resident", max_tokens=24)
    x = p.token_inputs(cfg, 24)
    y = torch.empty_like(x)
    for _ in range(3):  # eager, capture, replay
        m.decoder_iteration(x, out=y)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    m.decoder_iteration(x, out=y)
    b.record()
    torch.cuda.synchronize()
    st = np.zeros(cfg.num_blocks + 1, dtype=np.int64)
    _lib.check(_lib.load().pgmoe_model_block_stamps(m._h, ctypes.c_void_p(st.ctypes.data), cfg.num_blocks + 1))
    d = np.diff(st[1:])
    assert (st[1:] > 0).all() and (d > 0).all(), st
    assert (st[-1] - st[1]) / 1e6 < a.elapsed_time(b)
    m.close()
