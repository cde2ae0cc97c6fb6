#!/bin/bash
# round 2: GPU test suite + a short default bench (parity object included)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
(free -g; nproc; nvidia-smi --query-gpu=name,clocks.max.sm --format=csv) > gpurun_out/host.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu --timeout 900 -x 2>&1 | tail -40 > gpurun_out/t_a.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/b_a.json 2> gpurun_out/b_a.err
echo "bench rc=$?" >> gpurun_out/b_a.err
