#!/bin/bash
# round 2: the GPU test suite (no -x: every failure listed); optional test selection in $1
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 2400 python -m pytest ${1:-tests} -q -m gpu --timeout 900 -rfs 2>&1 | tail -80 > gpurun_out/t_b.log
