# iteration time (probe clock) vs split-K cap, resident Base-64 / Large-128
OUT=gpurun_out/split; rm -rf $OUT; mkdir -p $OUT
for c in "base64 1" "base64 8" "base64 32" "base64 64" "large128 8" "large128 32"; do set -- $c
for S in 0 1 2 4; do
PGMOE_MAX_SPLIT=$S timeout 120 python tools/probe.py --preset $1 --placement resident --tokens $2 --blocks 2 > $OUT/p_${S}_$1_$2.json 2>> $OUT/err
echo "S<=$S $1 T=$2 $(python -c "import json; d=json.load(open('$OUT/p_${S}_$1_$2.json')); print(d['iteration_us'], d['units_per_cta'])")"; done; done
