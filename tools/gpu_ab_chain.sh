OUT=gpurun_out/ab; rm -rf $OUT; mkdir -p $OUT
for i in 1 2; do for C in 0 1; do for c in "base64 1" "large128 1" "base64 256"; do set -- $c
PGMOE_NO_CHAIN=$C timeout 120 python tools/probe.py --preset $1 --placement resident --tokens $2 --blocks 2 > $OUT/p_${C}_$1_$2_$i.json 2>> $OUT/err
echo "nochain=$C $1 T=$2 run$i $(python -c "import json; print(json.load(open('$OUT/p_${C}_$1_$2_$i.json'))['iteration_us'])")"
done; done; done
