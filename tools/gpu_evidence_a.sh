#!/bin/bash
# Evidence, part A: GPU tests + smoke, the headline bench (+ reference arm),
# resident and EP bench lines, batch sweeps.  Part B (ncu): gpu_evidence_b.sh
OUT=gpurun_out/ev; rm -rf $OUT; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 900 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for c in "base64 1" "base64 256" "large128 1" "large128 256"; do set -- $c
  timeout 300 python bench.py --placement resident --preset $1 --tokens $2 --no-cpu-baseline > $OUT/bench_res_$1_T$2.json 2> $OUT/bench_res_$1_T$2.err
done
for T in 1 256; do
  timeout 300 python bench.py --mode ep --preset large128 --tokens $T --no-cpu-baseline > $OUT/bench_ep1_large128_T$T.json 2> $OUT/bench_ep1_T$T.err
done
timeout 900 python tools/sweep.py --preset base64 --placement resident --tokens 1,2,4,8,16,32,64,128,256 --steps 5 > $OUT/sweep_base64_resident.jsonl 2> $OUT/sweep.err
timeout 900 python tools/sweep.py --preset large128 --placement resident --tokens 1,8,32,64,128,256 --steps 5 > $OUT/sweep_large128_resident.jsonl 2>> $OUT/sweep.err
timeout 1200 python tools/sweep.py --preset base128 --tokens 1,2,4,8,16,32,64,128,256 --steps 3 > $OUT/sweep_base128_offloaded.jsonl 2>> $OUT/sweep.err
timeout 1500 python tools/sweep.py --preset large128 --tokens 1,2,4,8,16,32,64,128,256 --steps 2 > $OUT/sweep_large128_offloaded.jsonl 2>> $OUT/sweep.err
tail -2 $OUT/pytest_gpu.log; tail -1 $OUT/smoke.log; du -sh $OUT
