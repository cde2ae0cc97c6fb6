#!/bin/bash
# Round-1 evidence session: tests, headline bench (+ reference arm), resident
# points, ncu launch list + full captures of the dominant kernels.
OUT=gpurun_out/r1
rm -rf $OUT; mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 900 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for c in "base64 1" "base64 256" "large128 1" "large128 256"; do set -- $c
  timeout 300 python bench.py --placement resident --preset $1 --tokens $2 --no-cpu-baseline > $OUT/bench_res_$1_T$2.json 2> $OUT/bench_res_$1_T$2.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_default.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_launch.out 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:block_gemm -s 30 -c 1 -o $OUT/prof_block \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_block.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_kernel -s 30 -c 1 -o $OUT/prof_route \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_route.out 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_gemm -s 20 -c 1 -o $OUT/prof_block_res_base64_T256 \
  python bench.py --preset base64 --placement resident --tokens 256 --steps 1 --warmup 1 --no-cpu-baseline > $OUT/ncu_block_res.out 2>&1
ls -la $OUT
# bring back text exports, not the 40 MB reports (gpurun merges <= 64 MiB)
python tools/summarize_ncu.py --rep $OUT/prof_block.ncu-rep --rep $OUT/prof_route.ncu-rep \
   --launches $OUT/launches_default.csv --out $OUT/ncu_summary --label ffn=block_gemm --label route=route_kernel \
   > /dev/null 2>&1
python tools/summarize_ncu.py --rep $OUT/prof_block_res_base64_T256.ncu-rep --out $OUT/ncu_summary_res_base64_T256 \
   --label ffn=block_gemm > /dev/null 2>&1
for r in $OUT/*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  rm -f $r
done
du -sh $OUT
