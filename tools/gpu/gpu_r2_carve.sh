#!/bin/bash
# A/B: route-kernel shared-memory carveout (PGMOE_ROUTE_CARVEOUT=0 restores the driver's choice) on the default bench.
# (historical: the PGMOE_ROUTE_CARVEOUT knob was measured identical and removed; results in profiles/r2/launch_gap/)
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2carve${TAG}; rm -rf $OUT; mkdir -p $OUT
for rep in 1 2; do for cv in 0 1; do
  PGMOE_ROUTE_CARVEOUT=$cv timeout -s KILL 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-parity > $OUT/b_cv${cv}_r$rep.json 2>> $OUT/bench.err
done; done
python - <<'PY' > $OUT/summary.txt
import glob, json, os
for fn in sorted(glob.glob("gpurun_out/r2carve*/b_*.json")):
    d = json.loads(open(fn).read().strip().splitlines()[-1])
    print(os.path.basename(fn), d["value"], d["roofline"]["avg_launch_us"], d["roofline"]["frac"], d["per_block_latency_ms"])
PY
