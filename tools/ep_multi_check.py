"""Expert parallelism over NCCL on every GPU of the node (launched by
torchrun, one rank per GPU): each rank decodes its own tokens with its expert
shard; rank r's outputs and routing must equal a single-GPU decoder on the
concatenated batch bit for bit.  tests/test_gpu_ep_multi.py runs it (skipped
on a one-GPU box).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/ep_multi_check.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    import paper_2308_12066_b200 as p
    from paper_2308_12066_b200._rng import token_batch
    from paper_2308_12066_b200.ep import EPDecoder
    T = 24
    cfg = p.ModelConfig(d_model=256, d_ff=512, num_blocks=4, num_experts=16, top_k=2, activation_level=1)
    x = torch.from_numpy(token_batch(0, 256, T, offset=rank * T)).cuda()
    ep = EPDecoder(cfg, dtype="bf16", max_tokens=T)
    y_ep, ids_ep = ep.decoder_iteration(x, trace=True)
    for _ in range(3):  # graph-captured iterations (NCCL collectives inside the graph)
        y_g, _ = ep.decoder_iteration(x)
    torch.cuda.synchronize()
    ok = torch.equal(y_g, y_ep)
    if rank == 0:
        ref = p.DeviceModel(cfg, dtype="bf16", max_tokens=world * T)
        xs = torch.cat([torch.from_numpy(token_batch(0, 256, T, offset=r * T)).cuda() for r in range(world)])
        y, ids, _ = ref.decoder_iteration(xs, trace=True)
        torch.cuda.synchronize()
        ref_y, ref_ids = y, ids
    # every rank checks its slice against rank 0's single-GPU reference
    buf = torch.empty((world * T, cfg.d_model), device="cuda")
    bids = torch.empty((cfg.num_blocks, world * T, cfg.top_k), dtype=torch.int32, device="cuda")
    if rank == 0:
        buf.copy_(ref_y)
        bids.copy_(ref_ids)
    dist.broadcast(buf, 0)
    dist.broadcast(bids, 0)
    ok &= torch.equal(y_ep, buf[rank * T:(rank + 1) * T]) and torch.equal(ids_ep, bids[:, rank * T:(rank + 1) * T])
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    ep.close()
    dist.destroy_process_group()
    if rank == 0:
        print("EP_MULTI_OK" if flag.item() == 1 else "EP_MULTI_MISMATCH")
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
