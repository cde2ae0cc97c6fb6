#!/bin/bash
# K1 cluster size sweep (PGMOE_ROUTE_S) with tools/route_bench.py on the _build_B library.
# (historical: the PGMOE_ROUTE_S override was removed from route.cu after this sweep — no effect)
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2routeS; rm -rf $OUT; mkdir -p $OUT
for S in 0 2 4 8 16; do
  if [ $S = 0 ]; then ev=""; else ev="PGMOE_ROUTE_S=$S"; fi
  env $ev PGMOE_LIB_PATH=paper_2308_12066_b200/_build_B/libpgmoe.so timeout -s KILL 300 python tools/route_bench.py > $OUT/S$S.jsonl 2>> $OUT/err.txt
done
