#!/bin/bash
# Batch sweeps (BASELINE configs[1]-[3]) and the reference's four strategies measured on hardware.
OUT=gpurun_out/sw; rm -rf $OUT; mkdir -p $OUT
timeout 900 python tools/sweep.py --preset base64 --placement resident --tokens 1,2,4,8,16,32,64,128,256 --steps 5 > $OUT/sweep_base64_resident.jsonl 2> $OUT/err
timeout 900 python tools/sweep.py --preset large128 --placement resident --tokens 1,8,32,64,128,256 --steps 5 > $OUT/sweep_large128_resident.jsonl 2>> $OUT/err
timeout 1200 python tools/sweep.py --preset base128 --tokens 1,2,4,8,16,32,64,128,256 --steps 3 > $OUT/sweep_base128_offloaded.jsonl 2>> $OUT/err
timeout 1500 python tools/sweep.py --preset large128 --tokens 1,2,4,8,16,32,64,128,256 --steps 2 > $OUT/sweep_large128_offloaded.jsonl 2>> $OUT/err
for P in "base128 1" "large128 1" "large128 32"; do
  set -- $P
  timeout 900 python -m paper_2308_12066_b200.strategies --preset $1 --tokens $2 --iterations 3 --out $OUT/strategies/$1_T$2 > $OUT/strategies_$1_T$2.json 2>> $OUT/err
done
du -sh $OUT; tail -3 $OUT/err
