OUT=gpurun_out/infl; rm -rf $OUT; mkdir -p $OUT
for L in 8 6 4; do for c in "base64 256" "base64 128" "base64 64"; do set -- $c
PGMOE_INFLIGHT=$L timeout 120 python tools/probe.py --preset $1 --placement resident --tokens $2 --blocks 2 > $OUT/p_${L}_$1_$2.jsonl 2>> $OUT/err
echo "L=$L $1 T=$2 $(python -c "import json; print(json.load(open('$OUT/p_${L}_$1_$2.jsonl'))['iteration_us'])")"; done; done
