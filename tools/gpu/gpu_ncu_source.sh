#!/bin/bash
# ncu per-SASS-instruction warp-state samples of one resident block launch
# (rows with samples only); map addresses to source lines here with
# nvdisasm --print-line-info.  Usage: gpu_ncu_source.sh PRESET T
OUT=gpurun_out/ncusrc; mkdir -p $OUT
P=${1:-base64}; T=${2:-8}
timeout 600 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:block_gemm -s 20 -c 1 -o $OUT/src_${P}_T${T} \
  python bench.py --preset $P --placement resident --tokens $T --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_${P}_T${T}.out 2>&1
ncu -i $OUT/src_${P}_T${T}.ncu-rep --page source --csv --print-source sass > $OUT/sass_full.csv 2> $OUT/src.err
python - "$OUT/sass_full.csv" "$OUT/sass_${P}_T${T}.csv" <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r or "# Address" in r)
hdr = rows[hdr_i]
print(hdr[:40])
w = csv.writer(open(sys.argv[2], "w"))
w.writerow(hdr)
samp = [i for i, h in enumerate(hdr) if "Sampling" in h]
for r in rows[hdr_i + 1:]:
    if any(i < len(r) and r[i] not in ("", "0") for i in samp):
        w.writerow(r)
PY
rm -f $OUT/src_${P}_T${T}.ncu-rep $OUT/sass_full.csv; ls -la $OUT
