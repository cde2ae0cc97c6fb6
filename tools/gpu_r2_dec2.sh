#!/bin/bash
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2dec; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q --timeout 240 -rfs > $OUT/t_decode${TAG}.log 2>&1
echo "rc=$?" >> $OUT/t_decode${TAG}.log
if grep -q "passed" $OUT/t_decode${TAG}.log && ! grep -q "failed\|error" $OUT/t_decode${TAG}.log; then
  bash tools/gpu_r2_dprobe.sh
  for T in 1 2 4 8; do
    timeout 300 python bench.py --preset base64 --placement resident --tokens $T --steps 50 --warmup 5 --no-cpu-baseline --no-parity > $OUT/bench${TAG}_b64_T$T.json 2>> $OUT/bench.err
    timeout 300 python bench.py --preset large128 --placement resident --tokens $T --steps 30 --warmup 5 --no-cpu-baseline --no-parity > $OUT/bench${TAG}_l128_T$T.json 2>> $OUT/bench.err
  done
fi
