# two NCCL ranks on one GPU: does NCCL accept it?
import os, sys, torch, torch.distributed as dist
r = int(os.environ["RANK"])
torch.cuda.set_device(0)
try:
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    t = torch.ones(1, device="cuda")
    dist.all_reduce(t)
    torch.cuda.synchronize()
    print("rank", r, "allreduce ok", t.item(), flush=True)
    dist.destroy_process_group()
except Exception as e:
    print("rank", r, "NCCL error:", repr(e)[:400], flush=True)
