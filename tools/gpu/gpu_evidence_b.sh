#!/bin/bash
# Evidence, part B: ncu launch list of the default bench command, --set full
# captures of its block launch and K1 route launch, and of one resident block
# launch per resident workload; text summaries only (reports are too big).
OUT=gpurun_out/evb; rm -rf $OUT; mkdir -p $OUT
for T in 1 256; do
  timeout 300 python bench.py --mode ep --preset large128 --tokens $T --no-cpu-baseline > $OUT/bench_ep1_large128_T$T.json 2> $OUT/bench_ep1_T$T.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_default.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_launch.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:block_gemm -s 30 -c 1 -o $OUT/prof_block \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_block.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_kernel -s 30 -c 1 -o $OUT/prof_route \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_route.out 2>&1
python tools/summarize_ncu.py --rep $OUT/prof_block.ncu-rep --rep $OUT/prof_route.ncu-rep \
   --launches $OUT/launches_default.csv --out $OUT/ncu_summary --label ffn=block_gemm --label route=route_kernel \
   > $OUT/summ.log 2>&1
for c in "base64 256" "base64 1" "large128 256" "large128 1"; do set -- $c
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_gemm -s 20 -c 1 -o $OUT/prof_$1_T$2 \
    python bench.py --preset $1 --placement resident --tokens $2 --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_$1_T$2.out 2>&1
  python tools/summarize_ncu.py --rep $OUT/prof_$1_T$2.ncu-rep --out $OUT/ncu_summary_resident_$1_T$2 --label ffn=block_gemm >> $OUT/summ.log 2>&1
done
for r in $OUT/*.ncu-rep; do rm -f $r; done
ls -la $OUT; du -sh $OUT
