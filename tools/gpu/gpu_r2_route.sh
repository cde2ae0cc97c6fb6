#!/bin/bash
# K1: routing parity tests, then per-CTA timing (route_waves) and the forms benchmark
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2route${TAG}; rm -rf $OUT; mkdir -p $OUT
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -k "route or fused_routing or golden" -p no:cacheprovider > $OUT/t_route.log 2>&1
echo "rc=$?" >> $OUT/t_route.log
timeout -s KILL 120 python tools/route_waves.py 1024 128 1 8 64 128 256 > $OUT/waves_large128.jsonl 2>&1
timeout -s KILL 120 python tools/route_waves.py 768 64 1 8 64 256 > $OUT/waves_base64.jsonl 2>&1
timeout -s KILL 600 python tools/route_bench.py > $OUT/k1_route_forms.jsonl 2> $OUT/route_bench.err
