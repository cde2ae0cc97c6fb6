#!/bin/bash
# Quick GPU check: parity tests, smoke, default bench, resident small/large-T benches.
OUT=gpurun_out/chk
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for T in 1 256; do
  timeout 300 python bench.py --placement resident --tokens $T --no-cpu-baseline > $OUT/bench_res_large_T$T.json 2> $OUT/bench_res_large_T$T.err
  timeout 300 python bench.py --placement resident --preset base64 --tokens $T --no-cpu-baseline > $OUT/bench_res_base64_T$T.json 2> $OUT/bench_res_base64_T$T.err
done
ls -la $OUT
