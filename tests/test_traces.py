"""Synthetic routing traces (gen_routing_trace, core.py:436-479): at T = 1
the batched generator reproduces the reference's trace value for value."""

import os
import sys

import numpy as np
import pytest

from paper_2308_12066_b200.core import ModelConfig
from paper_2308_12066_b200.errors import ConfigError
from paper_2308_12066_b200.traces import routing_trace

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present (GPU box)")
@pytest.mark.parametrize("E,k,skew,seed", [(8, 1, 0.0, 0), (128, 1, 1.2, 3), (64, 2, 0.8, 1), (16, 3, 2.0, 7)])
def test_single_token_trace_equals_reference(E, k, skew, seed):
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import moesim
    from moesim.core import gen_routing_trace
    rc = moesim.ModelConfig(d_model=8, d_ff=16, num_blocks=5, num_experts=E, top_k=k, activation_level=1)
    ref = gen_routing_trace(rc, 3, skew, seed)
    ids, w = routing_trace(ModelConfig(d_model=8, d_ff=16, num_blocks=5, num_experts=E, top_k=k,
                                       activation_level=1), 3, skew, seed)
    for it in range(3):
        for b in range(5):
            d = ref.decisions[it][b]
            assert list(ids[it, b, 0]) == list(d.expert_ids)
            assert np.allclose(w[it, b, 0], d.combine_weights)


def test_batched_trace_shape_and_invariants():
    cfg = ModelConfig(d_model=8, d_ff=16, num_blocks=4, num_experts=32, top_k=2, activation_level=1)
    ids, w = routing_trace(cfg, 2, 1.5, 0, tokens=50)
    assert ids.shape == (2, 4, 50, 2) and w.shape == ids.shape
    assert (np.diff(ids, axis=-1) > 0).all() and ids.min() >= 0 and ids.max() < 32
    assert np.all(w == np.float32(0.5))
    # skew concentrates the traffic on the low expert ids
    assert np.mean(ids[..., 0] < 4) > 0.5
    with pytest.raises(ConfigError):
        routing_trace(cfg, 0, 1.0, 0)
    with pytest.raises(ConfigError):
        routing_trace(cfg, 1, -1.0, 0)
