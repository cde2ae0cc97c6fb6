for c in "base64 512" "base64 1024" "large128 512" "large128 1024"; do set -- $c
for F in "" "--no-fused-route"; do timeout 200 python tools/probe.py --preset $1 --placement resident --tokens $2 --blocks 2 $F > gpurun_out/pc.json 2>/dev/null
echo "$1 T=$2 fused=${F:-yes} $(python -c "import json; print(json.load(open('gpurun_out/pc.json'))['iteration_us'])")"; done; done
