#!/bin/bash
# round-2 evidence: the default bench line (20 steps, CPU baseline), the reference arm,
# resident / EP / fp32 lines, the ncu launch list of the default command and a full capture of its block launch.
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2final${TAG}; rm -rf $OUT; mkdir -p $OUT
timeout -s KILL 1200 python bench.py --steps 20 --warmup 5 > $OUT/bench_default_20steps.json 2> $OUT/bench_default.err
timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
for c in base64:1 base64:8 base64:64 base64:256 large128:1 large128:8 large128:256; do set -- ${c/:/ }
  timeout -s KILL 300 python bench.py --preset $1 --placement resident --tokens $2 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_resident_$1_T$2.json 2>> $OUT/bench.err
done
timeout -s KILL 900 python bench.py --preset base128 --placement offloaded --tokens 256 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_offloaded_base128_T256.json 2>> $OUT/bench.err
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_default.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parity > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:block_gemm -s 30 -c 1 -o $OUT/prof_default python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity > $OUT/ncu_default.out 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:route_cluster -s 5 -c 1 -o $OUT/prof_route python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-parity > $OUT/ncu_route.out 2>&1
python tools/summarize_ncu.py --rep $OUT/prof_default.ncu-rep --rep $OUT/prof_route.ncu-rep --launches $OUT/launches_default.csv --out $OUT/r2_ncu_summary --label ffn=block_gemm --label route=route_cluster > /dev/null 2>&1
rm -f $OUT/*.ncu-rep
