import os, sys, torch, torch.distributed as dist
print("rank env", os.environ.get("RANK"), {k: v for k, v in os.environ.items() if k.startswith("NCCL")}, file=sys.stderr)
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
t = torch.ones(4, device="cuda")
dist.all_reduce(t)
torch.cuda.synchronize()
dist.destroy_process_group()
