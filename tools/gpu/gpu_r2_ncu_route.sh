#!/bin/bash
# ncu source-level capture of one K1 cluster-form launch (Large-128; T from $TS, default "256 1")
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2ncu${TAG}; rm -rf $OUT; mkdir -p $OUT
for T in ${TS:-256 1}; do
  timeout -s KILL 300 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --warp-sampling-interval 0 --clock-control none --import-source on -k regex:route_cluster -s 3 -c 1 -o $OUT/route_T$T python tools/route_one.py large128 $T > $OUT/log_T$T.txt 2>&1
  ncu -i $OUT/route_T$T.ncu-rep --page source --csv --print-source cuda,sass > $OUT/source_T$T.csv 2>> $OUT/log_T$T.txt
  rm -f $OUT/route_T$T.ncu-rep
done
