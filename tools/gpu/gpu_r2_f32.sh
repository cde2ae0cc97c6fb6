#!/bin/bash
# fp32-weight path: parity tests, then Base-8 (configs[0]) resident/offloaded benches
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2f32${TAG}; rm -rf $OUT; mkdir -p $OUT
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -k "f32 or simt or offloaded_equals or decoder_iteration_equals or activation_levels" -rfs -p no:cacheprovider > $OUT/t_f32.log 2>&1
echo "rc=$?" >> $OUT/t_f32.log
for T in 256 64 8; do
  timeout -s KILL 600 python bench.py --preset base8 --placement resident --dtype f32 --tokens $T --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_base8_f32_resident_T$T.json 2>> $OUT/bench.err
done
