#!/bin/bash
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2dec; mkdir -p $OUT
for c in "base64 1" "base64 8" "large128 1"; do set -- $c
timeout 300 python tools/probe_decode.py --preset $1 --tokens $2 >> $OUT/dprobe${TAG}.jsonl 2>> $OUT/dprobe.err; done
