#!/bin/bash
# A/B of library builds (PGMOE_LIB_PATH = paper_2308_12066_b200/_build_<V>/libpgmoe.so) on resident small-T benches.
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2libab${TAG}; rm -rf $OUT; mkdir -p $OUT
for rep in 1 2; do
  for v in ${VARIANTS:-A B C D}; do
    L=paper_2308_12066_b200/_build_$v/libpgmoe.so
    for c in ${SHAPES:-base64:1 large128:1 base64:8}; do set -- ${c/:/ }
      PGMOE_LIB_PATH=$L $ENVV timeout -s KILL 90 python bench.py --preset $1 --placement resident --tokens $2 --steps 30 --warmup 3 --no-cpu-baseline --no-parity > $OUT/b_${v}_$1_T$2_r$rep.json 2>> $OUT/bench.err
    done
  done
done
python - <<'PY' > $OUT/summary.txt
import glob, json, os
for fn in sorted(glob.glob("gpurun_out/r2libab*/b_*.json")):
    try:
        d = json.loads(open(fn).read().strip().splitlines()[-1])
        print(os.path.basename(fn), round(d["per_block_latency_all_blocks_ms"] * 1e3, 2))
    except Exception as e:
        print(os.path.basename(fn), "ERR", e)
PY
