#!/bin/bash
# round 2: the GPU test suite (no -x: every failure listed)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -rf 2>&1 | tail -60 > gpurun_out/t_b.log
