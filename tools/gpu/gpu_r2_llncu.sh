#!/bin/bash
# ncu source-level stall sampling of one LL decode launch at the finest interval
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2llncu${TAG}; rm -rf $OUT; mkdir -p $OUT
export PGMOE_NO_GRAPH=1
timeout -s KILL 300 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --warp-sampling-max-passes 20 --warp-sampling-buffer-size 268435456 \
  --clock-control none --import-source on -k regex:ll_decode -s 3 -c 1 \
  -o $OUT/ll_base64_T1 python tools/probe_ll.py --preset base64 --tokens 1 > $OUT/ncu.log 2>&1
ncu -i $OUT/ll_base64_T1.ncu-rep --page source --csv > $OUT/source.csv 2>> $OUT/ncu.log
ncu -i $OUT/ll_base64_T1.ncu-rep --page raw --csv > $OUT/raw.csv 2>> $OUT/ncu.log
