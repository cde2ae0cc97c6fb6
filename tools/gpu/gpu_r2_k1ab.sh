#!/bin/bash
# K1 A/B: route tests on the candidate build (B), then tools/route_bench.py on A and B.
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2k1ab${TAG}; rm -rf $OUT; mkdir -p $OUT
PGMOE_LIB_PATH=paper_2308_12066_b200/_build_${TV:-B}/libpgmoe.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "route or cluster or gate" > $OUT/t_B.log 2>&1
for v in ${VARIANTS:-A B}; do
  PGMOE_LIB_PATH=paper_2308_12066_b200/_build_$v/libpgmoe.so timeout -s KILL 300 python tools/route_bench.py > $OUT/rb_$v.jsonl 2>> $OUT/err.txt
done
