OUT=gpurun_out/ab; rm -rf $OUT; mkdir -p $OUT
for dbg in 0 1 2 3 4; do
PGMOE_DBG=$dbg timeout 300 python tools/probe.py --preset base64 --placement resident --tokens 256 --cta-detail --blocks 2 > $OUT/p$dbg.jsonl 2>> $OUT/probe.err
PGMOE_DBG=$dbg timeout 300 python tools/probe.py --preset base64 --placement resident --tokens 1 --cta-detail --blocks 2 > $OUT/q$dbg.jsonl 2>> $OUT/probe.err
done
