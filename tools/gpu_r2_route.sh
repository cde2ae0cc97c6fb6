#!/bin/bash
# K1 forms: route parity tests + launch timing (probe stamps, graph replay)
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2route; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "route" -rfs 2>&1 | tail -30 > $OUT/tests${1}.log
timeout 400 python tools/route_bench.py > $OUT/route_bench${1}.jsonl 2> $OUT/route_bench${1}.err
