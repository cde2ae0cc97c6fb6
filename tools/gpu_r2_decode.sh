#!/bin/bash
# persistent small-batch decode kernel: tests first (short timeouts), then the full suite and quick benches
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2dec; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q --timeout 240 -rfs > $OUT/t_decode.log 2>&1
echo "rc=$?" >> $OUT/t_decode.log
if grep -q "passed" $OUT/t_decode.log && ! grep -q "failed\|error" $OUT/t_decode.log; then
  for T in 1 8 16; do
    timeout 300 python bench.py --preset base64 --placement resident --tokens $T --steps 50 --warmup 5 --no-cpu-baseline --no-parity > $OUT/bench_b64_T$T.json 2>> $OUT/bench.err
    timeout 300 python bench.py --preset large128 --placement resident --tokens $T --steps 30 --warmup 5 --no-cpu-baseline --no-parity > $OUT/bench_l128_T$T.json 2>> $OUT/bench.err
  done
  timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -rfs 2>&1 | tail -30 > $OUT/t_all.log
fi
