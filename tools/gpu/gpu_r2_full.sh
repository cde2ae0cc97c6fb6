#!/bin/bash
# the whole GPU suite + smoke (as the driver runs them)
cd "$GRAFT_REPO_ROOT"
OUT=gpurun_out/r2full${TAG}; rm -rf $OUT; mkdir -p $OUT
timeout -s KILL 1500 python -m pytest tests -m gpu -q --timeout 600 -rfs -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
