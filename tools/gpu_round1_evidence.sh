#!/bin/bash
# Round-1 evidence session: tests, headline bench, strategy comparison, ncu.
OUT=gpurun_out/r1
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $OUT/pytest_gpu.log
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
for P in "base128 1" "large128 1" "large128 32"; do
  set -- $P
  timeout 900 python -m paper_2308_12066_b200.strategies --preset $1 --tokens $2 --iterations 3 --out $OUT/strategies_$1_T$2 > $OUT/strategies_$1_T$2.json 2>> $OUT/strategies.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_default.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>> $OUT/ncu.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm -s 150 -c 3 -o $OUT/prof_ffn \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>> $OUT/ncu.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route -s 60 -c 2 -o $OUT/prof_route \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>> $OUT/ncu.err
ls -la $OUT
