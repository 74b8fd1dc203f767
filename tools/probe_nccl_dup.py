import os, torch, torch.distributed as dist, sys
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
r = dist.get_rank()
t = torch.ones(4, device="cuda") * (r + 1)
try:
    dist.all_reduce(t)
    torch.cuda.synchronize()
    print("rank", r, "allreduce ok", t.tolist(), flush=True)
except Exception as e:
    print("rank", r, "allreduce failed", repr(e)[:300], flush=True)
dist.destroy_process_group()
