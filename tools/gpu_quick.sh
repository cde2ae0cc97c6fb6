#!/bin/bash
# Quick iteration: GPU parity tests, probes, headline + resident benches.
OUT=gpurun_out/q; rm -rf $OUT; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for c in "base64 resident 1" "base64 resident 256" "large128 resident 256"; do set -- $c
  timeout 300 python tools/probe.py --preset $1 --placement $2 --tokens $3 --cta-detail --blocks 2 >> $OUT/probe.jsonl 2>> $OUT/probe.err; done
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_default.json 2> $OUT/bench_default.err
for c in "base64 1" "base64 256" "large128 1" "large128 256"; do set -- $c
  timeout 300 python bench.py --placement resident --preset $1 --tokens $2 --no-cpu-baseline > $OUT/bench_res_$1_T$2.json 2> $OUT/bench_res_$1_T$2.err
done
python tools/summ.py $OUT
