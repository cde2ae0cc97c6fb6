# per-block latency (bench clock, graph replay) vs split-K cap
OUT=gpurun_out/split2; rm -rf $OUT; mkdir -p $OUT
for S in ${SPLITS:-0 1 2 4}; do
PGMOE_MAX_SPLIT=$S timeout 300 python tools/sweep.py --preset base64 --placement resident --tokens 1,2,4,8,16,32,64,128,256 --steps 10 > $OUT/b64_$S.jsonl 2>> $OUT/err
PGMOE_MAX_SPLIT=$S timeout 300 python tools/sweep.py --preset large128 --placement resident --tokens 1,8,32,64,128,256 --steps 10 > $OUT/l128_$S.jsonl 2>> $OUT/err
done
python - <<'PY'
import json, os
for m in ("b64","l128"):
    rows={}
    for S in [int(v) for v in os.environ.get("SPLITS","0 1 2 4").split()]:
        for l in open(f"gpurun_out/split2/{m}_{S}.jsonl"):
            d=json.loads(l); rows.setdefault(d["tokens"],{})[S]=round(d["per_block_ms"]*1e3,1)
    for t,v in sorted(rows.items()): print(m,t,v)
PY
