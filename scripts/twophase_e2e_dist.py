"""Two ranks on one GPU (gloo) running the bench's config-2 two-phase flow:
device steps, then host-input steps. Usage (torchrun, VS_BENCH_ONE_GPU-style):
python -m torch.distributed.run --nproc-per-node 2 scripts/twophase_e2e_dist.py [n_rows]"""
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2605_15957_b200.distributed import ShardSearch, TorchComm, two_phase_search  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    cfg = dict(bench.CONFIGS[2])
    cfg["n"] = n
    W = bench.build_cfg2(rank, world, cfg)
    import paper_2605_15957_b200 as vs
    shard = ShardSearch(vs.EmbeddingColumn.from_device(W["data"]))
    comm = TorchComm()
    q, bits, lo = W["queries"], W["bits"], W["lo"]
    qh, bh = q.cpu().pin_memory(), bits.cpu().pin_memory()
    for s in range(3):
        r = two_phase_search(shard, comm, q, 100, "squared_l2", row_filter=bits, id_offset=lo)
        torch.cuda.synchronize()
        print(rank, "device step", s, int(r[2].min()), flush=True)
    for s in range(3):
        qq = qh.to(dev, non_blocking=True)
        bb = bh.to(dev, non_blocking=True)
        r = two_phase_search(shard, comm, qq, 100, "squared_l2", row_filter=bb, id_offset=lo)
        torch.cuda.synchronize()
        print(rank, "e2e step", s, int(r[2].min()), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
