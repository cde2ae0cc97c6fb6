#!/bin/bash
# ncu --set full of one resident block launch (fused routing role) for the
# resident bench workloads; summaries only (reports are too big to bring back).
OUT=gpurun_out/ncures; rm -rf $OUT; mkdir -p $OUT
for c in "large128 256" "large128 1" "base64 1"; do set -- $c
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_gemm -s 20 -c 1 -o $OUT/prof_$1_T$2 \
    python bench.py --preset $1 --placement resident --tokens $2 --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_$1_T$2.out 2>&1
  python tools/summarize_ncu.py --rep $OUT/prof_$1_T$2.ncu-rep --out $OUT/ncu_summary_resident_$1_T$2 --label ffn=block_gemm > /dev/null 2>&1
  ncu -i $OUT/prof_$1_T$2.ncu-rep --page details --csv > $OUT/prof_$1_T$2.details.csv 2>/dev/null
  rm -f $OUT/prof_$1_T$2.ncu-rep
done
ls -la $OUT
