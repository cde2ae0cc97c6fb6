VAR=PGMOE_FUSED_ROUTE VALS="1 0" B64=8,16 L128=6,8,12,16,24 bash tools/gpu_env_sweep.sh
mv gpurun_out/envsw gpurun_out/envsw_fr
VAR=PGMOE_INFLIGHT VALS="5 6 7 8" B64=8,16,32,64,128,256 L128=64,256 bash tools/gpu_env_sweep.sh
