#!/bin/bash
# compute-sanitizer passes over representative GPU tests (memcheck, synccheck, racecheck on the route kernel).
OUT=gpurun_out/sanitizer
rm -rf $OUT; mkdir -p $OUT
K='route_bit_exact_switch_shapes and 37 and 1024 or tcgen05_grouped_ffn_matches_oracle or offloaded_equals_resident or strategies_change or expert_cache_saves and lru or fused_routing and 64-40 or fused_routing and 256-17 or chained_block or ep_ranks or ep_decoder'
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests -m gpu -q -x -k "$K" > $OUT/memcheck.log 2>&1; echo "memcheck rc=$?" >> $OUT/summary.txt
timeout 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests -m gpu -q -x -k "route_bit_exact_switch_shapes and 37 and 1024 or tcgen05_grouped_ffn_matches_oracle and 37 or fused_routing and 64-40" > $OUT/synccheck.log 2>&1; echo "synccheck rc=$?" >> $OUT/summary.txt
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests -m gpu -q -x -k "route_bit_exact_switch_shapes and 37 and 1024 or route_topk_and_exact_ties or fused_routing and 64-10 or fused_routing and 256-17" > $OUT/racecheck.log 2>&1; echo "racecheck rc=$?" >> $OUT/summary.txt
for f in $OUT/*.log; do echo "== $f" >> $OUT/summary.txt; tail -n 4 $f >> $OUT/summary.txt; done
