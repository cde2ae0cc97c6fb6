cd "$GRAFT_REPO_ROOT"
for spec in "PGMOE_INFLIGHT=4" "PGMOE_INFLIGHT=6" "PGMOE_INFLIGHT=8" "PGMOE_MAX_SPLIT=1" "PGMOE_MAX_SPLIT=2" "PGMOE_CHAIN=0" "PGMOE_FUSED_ROUTE=0" "NONE=0"; do
  env $spec timeout -s KILL 200 python tools/sweep.py --preset base64 --placement resident --tokens 64,256 --steps 20 > gpurun_out/env_${spec%%=*}_${spec##*=}.jsonl 2>> gpurun_out/env.err
done
