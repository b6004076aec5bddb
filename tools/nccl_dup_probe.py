"""Probe: can two ranks share one GPU under NCCL (all_gather)?  Run with torchrun --nproc-per-node 2."""
import os, torch, torch.distributed as dist
dist.init_process_group("nccl")
r = dist.get_rank()
torch.cuda.set_device(0)
x = torch.full((4,), r, device="cuda", dtype=torch.int32)
out = torch.empty(8, device="cuda", dtype=torch.int32)
dist.all_gather_into_tensor(out, x)
torch.cuda.synchronize()
print("rank", r, out.tolist(), flush=True)
dist.destroy_process_group()
