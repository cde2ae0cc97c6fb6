OUT=gpurun_out/ncusrc; mkdir -p $OUT
timeout 600 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --warp-sampling-interval 0 --clock-control none --import-source on -k regex:block_gemm -s 30 -c 1 -o $OUT/blk_b64_T256 \
   python bench.py --preset base64 --placement resident --tokens 256 --steps 1 --warmup 1 --no-cpu-baseline >> $OUT/ncu.out 2>&1
timeout 600 ncu --section SourceCounters --section WarpStateStats --section SpeedOfLight --warp-sampling-interval 0 --clock-control none --import-source on -k regex:route_kernel -s 30 -c 1 -o $OUT/route_b64_T1 \
   python bench.py --preset base64 --placement resident --tokens 1 --steps 1 --warmup 1 --no-cpu-baseline >> $OUT/ncu.out 2>&1
ls -la $OUT
