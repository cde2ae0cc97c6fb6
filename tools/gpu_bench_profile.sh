#!/bin/bash
# One GPU session: benches + ncu launch list + one full ncu capture of the grouped GEMM.
set -x
OUT=gpurun_out
python bench.py --preset base64 --placement resident --no-cpu-baseline > $OUT/b_base64_res.json 2> $OUT/b.err
python bench.py --preset large128 --placement resident --no-cpu-baseline > $OUT/b_large_res.json 2>> $OUT/b.err
python bench.py > $OUT/b_large_off.json 2>> $OUT/b.err
python bench.py --tokens 1 --no-cpu-baseline > $OUT/b_large_off_t1.json 2>> $OUT/b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_base64.csv \
   python bench.py --preset base64 --placement resident --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>> $OUT/b.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 30 -c 3 -o $OUT/prof_tc \
   python bench.py --preset base64 --placement resident --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>> $OUT/b.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_kernel -s 4 -c 1 -o $OUT/prof_route \
   python bench.py --preset base64 --placement resident --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>> $OUT/b.err
ls -la $OUT
