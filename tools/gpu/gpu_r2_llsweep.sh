#!/bin/bash
# LL decoder ring / row-group / partition sweep on one build (PGMOE_LIB_PATH=_build_B): env combos x shapes.
# (historical: PGMOE_LL_GROUP / PGMOE_LL_ALIGN existed only in the measured variant, see profiles/r2/ll_chunk/attempt.diff)
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2lls${TAG}; rm -rf $OUT; mkdir -p $OUT
L=paper_2308_12066_b200/_build_${V:-B}/libpgmoe.so
for combo in ${COMBOS:-"0 0 0"}; do
  IFS=, read -r slot grp al <<< "$combo"
  for c in ${SHAPES:-base64:1 base64:8 large128:8}; do set -- ${c/:/ }
    PGMOE_LIB_PATH=$L PGMOE_LL_SLOT_KB=$slot PGMOE_LL_GROUP=$grp PGMOE_LL_ALIGN=$al timeout -s KILL 90 python bench.py --preset $1 --placement resident --tokens $2 --steps 30 --warmup 3 --no-cpu-baseline --no-parity > $OUT/b_s${slot}_g${grp}_a${al}_$1_T$2.json 2>> $OUT/bench.err
  done
done
python - <<'PY' > $OUT/summary.txt
import glob, json, os
for fn in sorted(glob.glob("gpurun_out/r2lls*/b_*.json")):
    try:
        d = json.loads(open(fn).read().strip().splitlines()[-1])
        print(os.path.basename(fn), round(d["per_block_latency_all_blocks_ms"] * 1e3, 2))
    except Exception as e:
        print(os.path.basename(fn), "ERR", e)
PY
