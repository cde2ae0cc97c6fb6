#!/bin/bash
# compute-sanitizer over the round-2 kernels: the LL decoder (memcheck, synccheck, racecheck),
# K1 cluster form, the tcgen05 decoder and the EP receiver routing / fused receiver (memcheck, racecheck).
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/sanitizer_r2; rm -rf $OUT; mkdir -p $OUT
K_LL='ll_decode_teacher_forced and (1-shape0 or 8-shape0 or 3-shape3) or planted_tie'
timeout -s KILL 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_lldecode.py -q -x -k "$K_LL" -p no:cacheprovider > $OUT/memcheck_ll.log 2>&1; echo "memcheck_ll rc=$?" >> $OUT/summary.txt
timeout -s KILL 1200 compute-sanitizer --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_lldecode.py -q -x -k "ll_decode_teacher_forced and 1-shape0" -p no:cacheprovider > $OUT/synccheck_ll.log 2>&1; echo "synccheck_ll rc=$?" >> $OUT/summary.txt
timeout -s KILL 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_lldecode.py -q -x -k "ll_decode_teacher_forced and 3-shape0" -p no:cacheprovider > $OUT/racecheck_ll.log 2>&1; echo "racecheck_ll rc=$?" >> $OUT/summary.txt
timeout -s KILL 1200 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py tests/test_gpu_decode.py -q -x -k "cluster_kernel_equals_split or ep_ranks or ep_decoder or recv_route_pack or decode_kernel_teacher_forced and 1-shape0" -p no:cacheprovider > $OUT/memcheck_other.log 2>&1; echo "memcheck_k1_ep_decode rc=$?" >> $OUT/summary.txt
timeout -s KILL 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "recv_route_pack" -p no:cacheprovider > $OUT/racecheck_ep_recv.log 2>&1; echo "racecheck_ep_recv rc=$?" >> $OUT/summary.txt
for f in $OUT/*.log; do echo "== $f" >> $OUT/summary.txt; tail -n 3 $f >> $OUT/summary.txt; done
