#!/bin/bash
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2llp${TAG}; rm -rf $OUT; mkdir -p $OUT
for c in "base64 1" "base64 8" "large128 1"; do set -- $c
  timeout -s KILL 60 python tools/probe_ll.py --preset $1 --tokens $2 >> $OUT/probe.jsonl 2>> $OUT/probe.err; done
for c in "base64 1" "large128 1"; do set -- $c
  PGMOE_LL_EXCL=1 timeout -s KILL 60 python tools/probe_ll.py --preset $1 --tokens $2 >> $OUT/probe_excl.jsonl 2>> $OUT/probe.err; done
