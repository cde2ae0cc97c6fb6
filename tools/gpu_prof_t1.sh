#!/bin/bash
# Small-T latency investigation: launch list + full captures at resident T=1.
OUT=gpurun_out/t1
mkdir -p $OUT
timeout 300 python tools/micro.py > $OUT/micro.json 2> $OUT/micro.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches_base64_T1.csv \
   python bench.py --preset base64 --placement resident --tokens 1 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>> $OUT/ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_gemm -s 40 -c 1 -o $OUT/prof_block_T1 \
   python bench.py --preset base64 --placement resident --tokens 1 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>> $OUT/ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_kernel -s 40 -c 1 -o $OUT/prof_route_T1 \
   python bench.py --preset base64 --placement resident --tokens 1 --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>> $OUT/ncu.err
ls -la $OUT
