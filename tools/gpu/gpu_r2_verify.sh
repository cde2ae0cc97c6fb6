#!/bin/bash
# Round-2 state check: the full GPU suite, smoke, the headline bench and resident points.
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2v${TAG}; rm -rf $OUT; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rfs -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for c in "base64 1" "base64 8" "base64 64" "base64 256" "large128 1" "large128 8" "large128 256"; do set -- $c
  timeout 300 python bench.py --placement resident --preset $1 --tokens $2 --no-cpu-baseline > $OUT/bench_res_$1_T$2.json 2> $OUT/bench_res_$1_T$2.err
done
