# per-block latency (bench clock, graph replay) vs one knob:
#   VAR=PGMOE_INFLIGHT VALS="6 8" bash tools/gpu/gpu_env_sweep.sh
OUT=gpurun_out/envsw; rm -rf $OUT; mkdir -p $OUT
B64=${B64:-1,8,64,128,256}; L128=${L128:-1,64,256}
for v in $VALS; do
env $VAR=$v timeout 300 python tools/sweep.py --preset base64 --placement resident --tokens $B64 --steps 10 > $OUT/b64_$v.jsonl 2>> $OUT/err
[ -n "$L128" ] && env $VAR=$v timeout 300 python tools/sweep.py --preset large128 --placement resident --tokens $L128 --steps 10 > $OUT/l128_$v.jsonl 2>> $OUT/err
done
python - <<'PY'
import json, os
for m in ("b64","l128"):
    rows={}
    for v in os.environ["VALS"].split():
        f=f"gpurun_out/envsw/{m}_{v}.jsonl"
        if not os.path.exists(f): continue
        for l in open(f):
            d=json.loads(l); rows.setdefault(d["tokens"],{})[v]=round(d["per_block_ms"]*1e3,1)
    for t,v in sorted(rows.items()): print(os.environ["VAR"], m,t,v)
PY
