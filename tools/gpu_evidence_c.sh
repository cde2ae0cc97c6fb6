#!/bin/bash
# Evidence, part C: EP x1 lines (with the FFN roofline pass) and the resident
# lines (clock samples).
OUT=gpurun_out/evc; rm -rf $OUT; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q -k "ep or EP" > $OUT/pytest_ep.log 2>&1; tail -1 $OUT/pytest_ep.log
for T in 1 256; do
  timeout 300 python bench.py --mode ep --preset large128 --tokens $T --no-cpu-baseline > $OUT/bench_ep1_large128_T$T.json 2> $OUT/bench_ep1_T$T.err
done
for c in "base64 1" "base64 256" "large128 1" "large128 256"; do set -- $c
  timeout 300 python bench.py --placement resident --preset $1 --tokens $2 --no-cpu-baseline > $OUT/bench_res_$1_T$2.json 2> $OUT/bench_res_$1_T$2.err
done
