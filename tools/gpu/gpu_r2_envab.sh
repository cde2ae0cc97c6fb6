#!/bin/bash
# A/B of one library under several environment settings (ENVS="A=1 B=2;A=2 ..."), resident benches
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2envab${TAG}; rm -rf $OUT; mkdir -p $OUT
IFS=';' read -ra SETS <<< "${ENVS}"
for e in "${SETS[@]}"; do
  tag=$(echo "$e" | tr ' =' '_-')
  for c in ${SHAPES:-base64:1 large128:1 base64:8 large128:8}; do set -- ${c/:/ }
    env $e timeout -s KILL 90 python bench.py --preset $1 --placement resident --tokens $2 --steps 30 --warmup 3 --no-cpu-baseline --no-parity > $OUT/b_${tag}_$1_T$2.json 2>> $OUT/bench.err
  done
done
python - <<'PY' > $OUT/summary.txt
import glob, json, os
for fn in sorted(glob.glob("gpurun_out/r2envab*/b_*.json")):
    try:
        d = json.loads(open(fn).read().strip().splitlines()[-1])
        print(os.path.basename(fn), round(d["per_block_latency_all_blocks_ms"] * 1e3, 2), d["roofline"]["kernel"][:14])
    except Exception as e:
        print(os.path.basename(fn), "ERR", e)
PY
