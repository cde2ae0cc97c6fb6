#!/bin/bash
# The reference's four strategies measured on hardware (CSV trio + timelines).
OUT=gpurun_out/strat; rm -rf $OUT; mkdir -p $OUT
for P in "base128 1" "large128 1" "large128 32"; do
  set -- $P
  timeout 900 python -m paper_2308_12066_b200.strategies --preset $1 --tokens $2 --iterations 3 --out $OUT/$1_T$2 > $OUT/strategies_$1_T$2.json 2>> $OUT/err
done
tail -3 $OUT/err; du -sh $OUT
