OUT=gpurun_out/probe; rm -rf $OUT; mkdir -p $OUT
for c in ${PROBE_CFGS:-"base64 resident 1" "base64 resident 256"}; do set -- $c
timeout 300 python tools/probe.py --preset $1 --placement $2 --tokens $3 --cta-detail --blocks 2 >> $OUT/probe.jsonl 2>> $OUT/probe.err; done
python tools/summ.py $OUT
