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
