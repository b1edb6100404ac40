"""Does gloo all_gather / all_reduce on CUDA tensors work with two ranks on
one GPU? (test-hook sanity for VS_BENCH_ONE_GPU)"""
import os
import torch
import torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("gloo")
r = dist.get_rank()
t = torch.full((4,), float(r), device="cuda")
parts = [torch.empty_like(t) for _ in range(2)]
print(r, "allgather...", flush=True)
dist.all_gather(parts, t)
print(r, "allgather ok", [p.tolist() for p in parts], flush=True)
dist.all_reduce(t, op=dist.ReduceOp.MIN)
print(r, "allreduce ok", t.tolist(), flush=True)
dist.barrier()
print(r, "barrier ok", flush=True)
