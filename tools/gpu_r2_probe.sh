#!/bin/bash
# round 2: device-side timelines (probe) of the small-T resident chain and K1, plus the headline bench at driver-like steps
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2probe; rm -rf $OUT; mkdir -p $OUT
for c in "base64 resident 1" "base64 resident 8" "large128 resident 1" "base64 resident 256" "large128 offloaded 256" "large128 offloaded 1"; do set -- $c
timeout 300 python tools/probe.py --preset $1 --placement $2 --tokens $3 --cta-detail --blocks 3 >> $OUT/probe.jsonl 2>> $OUT/probe.err; done
python tools/summ.py $OUT > $OUT/summary.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_default.json 2> $OUT/bench_default.err
for T in 1 8 256; do
timeout 300 python bench.py --preset base64 --placement resident --tokens $T --steps 50 --warmup 5 --no-cpu-baseline --no-parity > $OUT/bench_b64_T$T.json 2>> $OUT/bench.err
done
