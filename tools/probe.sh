nproc; free -g; lscpu | head -20; nvidia-smi; nvidia-smi topo -m; 
python - <<'PY'
import torch, time
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))
for nb in [16<<20, 256<<20, 1<<30]:
    h = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(nb, dtype=torch.uint8, device='cuda')
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    print("H2D", nb, nb*10/(s.elapsed_time(e)*1e-3)/1e9, "GB/s")
t=time.time(); h = torch.empty(8<<30, dtype=torch.uint8, pin_memory=True); print("pin 8GiB", time.time()-t)
PY
