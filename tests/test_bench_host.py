"""Host-side checks of bench.py's contract pieces (no GPU): workload naming
by BASELINE config, the ncu-traffic lookup keyed by workload, and the
reference arm's JSON line."""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_workload_names_follow_baseline_configs():
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"]
    assert len(base) == 5
    assert bench.workload_name("large128", "offloaded", 256).endswith("(BASELINE configs[3])")
    assert bench.workload_name("base64", "resident", 256).endswith("(BASELINE configs[1])")
    assert bench.workload_name("base128", "offloaded", 1).endswith("(BASELINE configs[2])")
    assert "configs[" not in bench.workload_name("large128", "resident", 256)


def test_default_workload_has_committed_ncu_traffic():
    """The default bench line reports roofline.traffic from the committed
    ncu capture of the SAME workload, and nothing for other workloads."""
    wl = bench.workload_name("large128", "offloaded", 256)
    t = bench.ncu_traffic("ffn", wl)
    assert t is not None and 1.5e9 < t < 2.5e9  # ~1.9 GB per block launch
    assert bench.ncu_traffic("ffn", "no such workload") is None


def test_reference_arm_line(monkeypatch):
    """--impl reference: rank 0 runs the oracle port on host cores and
    prints the contract keys; other ranks print nothing."""
    class A:
        preset, steps, warmup, cpu_sample = "base8", 1, 0, 1
    monkeypatch.setattr(bench, "cpu_reference_run", lambda *a, **k: [0.5])
    out = bench.run_reference(A(), 0, 1)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "impl", "cpu_baseline",
                "e2e", "config"):
        assert key in out
    assert out["impl"] == "reference" and out["value"] == 2.0
    assert out["e2e"]["h2d_bytes_per_step"] == 0 and out["cpu_baseline"]["kind"] == "port"
    assert bench.run_reference(A(), 1, 2) is None


def test_block_latencies_follow_reference_definition():
    """scheduler.py:374-397: a block's latency runs from the end of the
    previous block's dense layer; block 0 from its iteration's start."""
    ev = []
    t = 0.0
    for it in range(2):
        for b in range(3):
            ev.append({"lane": "compute", "label": "experts", "block": b, "start_s": t, "end_s": t + 1.0})
            ev.append({"lane": "compute", "label": "non_moe", "block": b, "start_s": t + 1.0,
                       "end_s": t + 1.5 + b})
            t += 1.5 + b
    lats = bench.block_latencies(ev, 3)
    assert lats == [[1.5, 2.5, 3.5], [1.5, 2.5, 3.5]]


def test_parity_measurements_on_oracle_traces():
    """oracle/parity.py on traces produced by the oracle itself (fp32-rounded
    block inputs): no id mismatches, no flips, errors at fp32 rounding."""
    import numpy as np
    from oracle import oracle as og
    from oracle import parity
    dims = og.Dims(16, 24, 4, 8, 1, 1, 3)
    om = og.OracleModel(dims, "f32")
    T = 10
    x0 = np.stack([og.token_input(dims, t) for t in range(T)]).astype(np.float32)
    traces = []
    x = x0.astype(np.float64)
    for it in range(2):
        xt, ids_t, w_t = [], [], []
        pending = {}
        for b in range(dims.num_blocks):
            xt.append(x.astype(np.float32))
            xb = xt[-1].astype(np.float64)
            if dims.has_conv_gate(b):
                ids, w = og.gate_batch(xb, om.gate(b), 1)
            else:
                ids, w = pending.pop(b)
            if dims.has_pre_gate(b):
                pending[b + 1] = og.gate_batch(xb, om.pre_gate(b), 1)
            ids_t.append(ids)
            w_t.append(w.astype(np.float32))
            w1 = {int(e): om.w1(b, int(e)) for e in np.unique(ids)}
            w2 = {int(e): om.w2(b, int(e)) for e in np.unique(ids)}
            x = og.block_batch(xb, ids, w, w1, w2, om.dense(b), dims.num_experts)
        traces.append((np.stack(xt), x.astype(np.float32), np.stack(ids_t), np.stack(w_t)))
    xt, y, ids, w = traces[0]
    r = parity.teacher_forced(dims, "f32", xt, y, ids, w, np.arange(T), {0, 1, 3})
    assert r["ids_mismatch_tokens"] == 0 and r["ids_blocks_checked"] == 4
    assert len(r["blocks"]) == 3 and r["max_err"] < 1e-6 and r["w_max_rel"] < 1e-6
    ch = parity.chained(dims, "f32", x0, [t[0] for t in traces], [t[2] for t in traces])
    assert ch["flips_total"] == 0 and len(ch["per_block"]) == 8
    assert ch["per_block"][0]["input_err"] == 0.0
