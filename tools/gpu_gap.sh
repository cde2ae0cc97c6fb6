python tools/probe.py --preset base64 --placement resident --tokens 256 --blocks 12 > gpurun_out/gap.json 2>/dev/null
python - <<'PY'
import json
d=json.load(open('gpurun_out/gap.json'))
prev=None
for e in d['launches']:
    if e.get('kind')!='block': continue
    g={k:e[k] for k in ['entry','gate0','ph0','ph1','gate2','ph2','exit'] if k in e}
    print(e['block'], {k:(v[0],v[2]) for k,v in g.items()})
PY
