"""Single-process reproduction of the bench's N > 1 config-2 flow (two-phase
protocol) with a world-1 communicator: device steps, then host-input (e2e)
steps. Usage: python scripts/twophase_e2e_repro.py [n_rows]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2605_15957_b200.distributed import ShardSearch, two_phase_search  # noqa: E402


class One:
    def size(self):
        return 1

    def rank(self):
        return 0

    def allreduce_min(self, t):
        return t

    def allgather(self, t):
        return t.unsqueeze(0)

    def allgather_topk(self, i, d, c):
        return i.unsqueeze(0), d.unsqueeze(0), c.unsqueeze(0)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
    dev = torch.device("cuda", 0)
    cfg = dict(bench.CONFIGS[2])
    cfg["n"] = n
    W = bench.build_cfg2(0, 1, cfg)
    import paper_2605_15957_b200 as vs
    col = vs.EmbeddingColumn.from_device(W["data"])
    shard = ShardSearch(col)
    q, bits = W["queries"], W["bits"]
    qh, bh = q.cpu().pin_memory(), bits.cpu().pin_memory()
    for s in range(4):
        r = two_phase_search(shard, One(), q, 100, "squared_l2", row_filter=bits)
        torch.cuda.synchronize()
        print("device step", s, int(r[2].min()), flush=True)
    mode = sys.argv[2] if len(sys.argv) > 2 else "both"
    for s in range(3):
        qq = qh.to(dev, non_blocking=True) if mode in ("both", "q") else q
        bb = bh.to(dev, non_blocking=True) if mode in ("both", "b") else bits
        r = two_phase_search(shard, One(), qq, 100, "squared_l2", row_filter=bb)
        torch.cuda.synchronize()
        print("e2e step", mode, s, int(r[2].min()), flush=True)


if __name__ == "__main__":
    main()
