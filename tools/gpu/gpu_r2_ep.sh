#!/bin/bash
# EP: device tests, then the one-GPU EP bench (P=1) at T=256 / T=1
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2ep${TAG}; rm -rf $OUT; mkdir -p $OUT
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ep_multi.py -q --timeout 300 -k "ep" -rfs -p no:cacheprovider > $OUT/t_ep.log 2>&1
echo "rc=$?" >> $OUT/t_ep.log
for T in 256 1; do
  timeout -s KILL 600 python bench.py --mode ep --tokens $T --steps 10 --warmup 3 > $OUT/bench_ep1_large128_T$T.json 2>> $OUT/bench.err
done
