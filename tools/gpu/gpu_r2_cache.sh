#!/bin/bash
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2cache; mkdir -p $OUT
timeout 1500 python tools/cache_study.py --preset large128 --tokens 1 > $OUT/cache_large128_T1.jsonl 2> $OUT/err1.log
timeout 1500 python tools/cache_study.py --preset large128 --tokens 32 > $OUT/cache_large128_T32.jsonl 2> $OUT/err32.log
