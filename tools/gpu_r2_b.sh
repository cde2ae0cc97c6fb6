#!/bin/bash
# round 2: full GPU test suite (every failure listed) + smoke + default bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
(free -g; nproc; nvidia-smi --query-gpu=name,clocks.max.sm --format=csv) > gpurun_out/host.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -rfs --durations=15 2>&1 | tail -80 > gpurun_out/t_b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/b_b.json 2> gpurun_out/b_b.err
echo "bench rc=$?" >> gpurun_out/b_b.err
