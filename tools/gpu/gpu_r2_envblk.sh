#!/bin/bash
# Env A/B of the tcgen05 block launch at resident T >= 64 (ENVS="A=1;B=2 C=3", "-" = defaults): per-block latency
# (reference definition, block 0 excluded) and block-roofline fraction, two repeats.
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2envblk${TAG}; rm -rf $OUT; mkdir -p $OUT
IFS=';' read -ra SETS <<< "${ENVS:--}"
for rep in 1 2; do
for e in "${SETS[@]}"; do
  tag=$(echo "$e" | tr ' =' '_-')
  for c in ${SHAPES:-base64:256 large128:256 base64:64}; do set -- ${c/:/ }
    if [ "$e" = "-" ]; then ev=""; else ev="$e"; fi
    env $ev timeout -s KILL 120 python bench.py --preset $1 --placement resident --tokens $2 --steps 20 --warmup 3 --no-cpu-baseline --no-parity > $OUT/b_${tag}_$1_T$2_r$rep.json 2>> $OUT/bench.err
  done
done
done
python - <<'PY' > $OUT/summary.txt
import glob, json, os
for fn in sorted(glob.glob("gpurun_out/r2envblk*/b_*.json")):
    try:
        d = json.loads(open(fn).read().strip().splitlines()[-1])
        print(os.path.basename(fn), round(d["per_block_latency_ms"] * 1e3, 2), d["block_roofline"]["frac"], d["roofline"]["frac"])
    except Exception as e:
        print(os.path.basename(fn), "ERR", e)
PY
