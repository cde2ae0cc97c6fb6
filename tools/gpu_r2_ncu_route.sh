#!/bin/bash
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2ncu; mkdir -p $OUT
for c in "large128 1" "large128 256"; do set -- $c
timeout 300 ncu --set full --clock-control none --import-source on -k regex:route -s 3 -c 1 -o $OUT/route_$1_T$2 python tools/route_one.py $1 $2 > $OUT/route_$1_T$2.log 2>&1
done
