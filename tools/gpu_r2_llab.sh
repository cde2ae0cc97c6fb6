#!/bin/bash
# A/B of the LL decoder's waiting strategies (env knobs), resident benches.
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2llab${TAG}; rm -rf $OUT; mkdir -p $OUT
timeout -s KILL 120 python -m pytest tests/test_gpu_lldecode.py -x -q --timeout 60 -k "teacher_forced and shape1" -p no:cacheprovider > $OUT/t_ll.log 2>&1
echo "rc=$?" >> $OUT/t_ll.log
grep -q "rc=0" $OUT/t_ll.log || exit 0
for v in ${VARIANTS:-"1 1 64" "0 1 64" "0 0 0" "0 1 0" "1 1 0" "0 0 64"}; do set -- $v
  for c in "base64 1" "large128 1" "base64 8"; do set -- $v $c
    PGMOE_LL_SENT=$1 PGMOE_LL_POLL=$2 PGMOE_LL_SLEEP=$3 timeout -s KILL 90 python bench.py --preset $4 --placement resident --tokens $5 --steps 30 --warmup 3 --no-cpu-baseline --no-parity > $OUT/b_s$1_p$2_z$3_$4_T$5.json 2>> $OUT/bench.err
  done
done
python - <<'PY' > $OUT/summary.txt
import glob, json, os
for fn in sorted(glob.glob(os.environ.get("GRAFT_REPO_ROOT", ".") + "/gpurun_out/r2llab*/b_*.json")):
    try:
        d = json.loads(open(fn).read().strip().splitlines()[-1])
        print(os.path.basename(fn), round(d["per_block_latency_all_blocks_ms"] * 1e3, 2))
    except Exception as e:
        print(os.path.basename(fn), "ERR", e)
PY
