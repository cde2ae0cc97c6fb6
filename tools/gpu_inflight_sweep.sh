OUT=gpurun_out/infl; rm -rf $OUT; mkdir -p $OUT
for L in 8 5 4; do for c in "base64 256" "large128 256" "base64 1"; do set -- $c
PGMOE_INFLIGHT=$L timeout 120 python tools/probe.py --preset $1 --placement resident --tokens $2 --blocks 2 > $OUT/p_${L}_$1_$2.jsonl 2>> $OUT/err; done; done
for f in $OUT/p_*.jsonl; do echo "$f $(python -c "import json,sys; d=json.load(open('$f')); b=[e for e in d['launches'] if e.get('kind')=='block' and e['block']==1][0]; print(d['iteration_us'], {k:b[k][2] for k in ['gate0','ph0','ph1','r_logits','r_sel1','r_perm','gate2','ph2'] if k in b})")"; done
