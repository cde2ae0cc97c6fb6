"""Host logic of the measured strategy comparison (no GPU): metric
definitions and the reference's CSV schema (harness.py:227-282)."""

import os

from paper_2308_12066_b200.strategies import block_latencies, write_csv


def test_block_latency_is_dense_end_to_dense_end():
    ev = [{"lane": "compute", "label": "gate", "block": 0, "start_s": 0.0, "end_s": 1.0},
          {"lane": "transfer", "label": "fetch[1]", "block": 0, "start_s": 1.0, "end_s": 4.0},
          {"lane": "compute", "label": "experts", "block": 0, "start_s": 4.0, "end_s": 5.0},
          {"lane": "compute", "label": "non_moe", "block": 0, "start_s": 5.0, "end_s": 6.0},
          {"lane": "compute", "label": "experts", "block": 1, "start_s": 6.0, "end_s": 8.0},
          {"lane": "compute", "label": "non_moe", "block": 1, "start_s": 8.0, "end_s": 9.5}]
    lats, span = block_latencies(ev)
    assert lats == [6.0, 3.5] and span == 9.5


def test_csv_trio_schema(tmp_path):
    rows = [{"model": "base8", "strategy": "pre_gated", "sweep_value": "1", "avg_moe_block_latency_s": 0.001,
             "tokens_per_sec": 100.0, "peak_fast_bytes": 1234}]
    paths = write_csv(rows, str(tmp_path))
    names = sorted(os.path.basename(p) for p in paths)
    assert names == ["block_lats.csv", "peak_mems.csv", "throughputs.csv"]
    assert (tmp_path / "block_lats.csv").read_text() == \
        "model,strategy,sweep_value,avg_block_latency_s\nbase8,pre_gated,1,0.001\n"
    assert (tmp_path / "peak_mems.csv").read_text().splitlines()[1] == "base8,pre_gated,1,1234"
