#!/bin/bash
# Block launch with narrow N tiles (PGMOE_BN=16/32 on a _build_B carrying those instantiations).
# (historical: measured no gain and removed; results in profiles/r2/l2_prefetch/narrow_n_tiles.txt)
cd "$GRAFT_REPO_ROOT"
export PGMOE_LIB_PATH=paper_2308_12066_b200/_build_B/libpgmoe.so
mkdir -p gpurun_out/bnab
for bn in 32 16; do PGMOE_BN=$bn timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_shapes.py -x -q -p no:cacheprovider -k "not ep_ranks" > gpurun_out/bnab/t_bn$bn.log 2>&1; done
ENVS="-;PGMOE_BN=32;PGMOE_BN=16" SHAPES="base64:256 large128:256 base64:64 base64:32" bash tools/gpu/gpu_r2_envblk.sh
