#!/bin/bash
# LL decoder evidence: resident small-T bench lines (with parity) and ncu captures of one LL launch.
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2llev${TAG}; rm -rf $OUT; mkdir -p $OUT
for c in base64:1 base64:2 base64:4 base64:8 large128:1 large128:2 large128:4 large128:8; do set -- ${c/:/ }
  timeout -s KILL 300 python bench.py --preset $1 --placement resident --tokens $2 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_resident_$1_T$2.json 2>> $OUT/bench.err
done
export PGMOE_NO_GRAPH=1
for c in base64:1 large128:1 base64:8; do set -- ${c/:/ }
  timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:ll_decode -s 6 -c 1 -o $OUT/ll_$1_T$2 \
    python bench.py --preset $1 --placement resident --tokens $2 --steps 1 --warmup 3 --no-cpu-baseline --no-parity > $OUT/ncu_$1_T$2.out 2>&1
  python tools/summarize_ncu.py --rep $OUT/ll_$1_T$2.ncu-rep --out $OUT/r2_ncu_summary_ll_$1_T$2 --label ffn=ll_decode > /dev/null 2>&1
  rm -f $OUT/ll_$1_T$2.ncu-rep
done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches_base64_T1.csv \
  python bench.py --preset base64 --placement resident --tokens 1 --steps 2 --warmup 1 --no-cpu-baseline --no-parity > /dev/null 2>&1
