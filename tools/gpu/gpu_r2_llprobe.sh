#!/bin/bash
# Device-side timelines of the LL decoder from probe builds (-DPGMOE_LL_PROBE): _build_P and, if present, _build_PB.
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2llp${TAG}; rm -rf $OUT; mkdir -p $OUT
for v in P PB; do
  L=paper_2308_12066_b200/_build_$v/libpgmoe.so; [ -f $L ] || continue
  for c in ${SHAPES:-base64:1 base64:8 large128:8}; do set -- ${c/:/ }
    PGMOE_LIB_PATH=$L timeout -s KILL 60 python tools/probe_ll.py --preset $1 --tokens $2 >> $OUT/probe_$v.jsonl 2>> $OUT/probe.err; done
done
