#!/bin/bash
# LL decoder A/B: parity tests on the candidate build (B), then resident small-T benches of A and B.
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2llab${TAG}; rm -rf $OUT; mkdir -p $OUT
PGMOE_LIB_PATH=paper_2308_12066_b200/_build_B/libpgmoe.so timeout -s KILL 400 python -m pytest tests/test_gpu_lldecode.py -x -q -p no:cacheprovider > $OUT/t_B.log 2>&1
tail -2 $OUT/t_B.log
VARIANTS="${VARIANTS:-A B}" SHAPES="${SHAPES:-base64:1 large128:1 base64:4 base64:8 large128:8}" TAG=${TAG} bash tools/gpu/gpu_r2_libab.sh
