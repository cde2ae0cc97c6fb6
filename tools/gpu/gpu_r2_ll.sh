#!/bin/bash
# LL decoder: its tests under short timeouts first, then probes and quick resident benches.
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2ll${TAG}; rm -rf $OUT; mkdir -p $OUT
timeout -s KILL 240 python -m pytest tests/test_gpu_lldecode.py -x -q --timeout 60 -rfs -p no:cacheprovider > $OUT/t_ll.log 2>&1
echo "rc=$?" >> $OUT/t_ll.log
if grep -q " passed" $OUT/t_ll.log && ! grep -qE "failed|error|rc=[1-9]" $OUT/t_ll.log; then
  for c in "base64 1" "base64 8" "large128 1"; do set -- $c
    timeout -s KILL 60 python tools/probe_ll.py --preset $1 --tokens $2 >> $OUT/probe.jsonl 2>> $OUT/probe.err; done
  for c in "base64 1" "base64 2" "base64 4" "base64 8" "large128 1" "large128 8"; do set -- $c
    timeout -s KILL 120 python bench.py --preset $1 --placement resident --tokens $2 --steps 50 --warmup 5 --no-cpu-baseline --no-parity > $OUT/bench_$1_T$2.json 2>> $OUT/bench.err
  done
  if [ -n "$REG" ]; then
    timeout -s KILL 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity.py tests/test_gpu_bench_shapes.py -q --timeout 300 -rfs -p no:cacheprovider > $OUT/t_reg.log 2>&1
    echo "rc=$?" >> $OUT/t_reg.log
  fi
fi
