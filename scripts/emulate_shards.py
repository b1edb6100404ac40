"""Per-rank cost of the row-sharded exact search at G GPUs, emulated on one
B200: the config-2 collection split into G row shards (one library context
each); every shard runs phase A + the k-th keys (vs_enn_search_begin), the
bound T = MIN over shards, then each shard's bounded re-rank
(vs_enn_search_finish) is timed; compared with the one-phase shard search
(vs_enn_search: local top-k, full re-rank). Prints one JSON line per G.

    python scripts/emulate_shards.py [G ...]
"""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2605_15957_b200 as vs  # noqa: E402
from paper_2605_15957_b200 import _native as N  # noqa: E402
from paper_2605_15957_b200.distributed import ShardSearch, row_shard  # noqa: E402
from paper_2605_15957_b200.vecindex import enn_search_raw  # noqa: E402


def timed(fn, reps=3, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    gs = [int(a) for a in sys.argv[1:]] or [2, 4, 8]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    cfg = bench.CONFIGS[2]
    W = bench.build_cfg2(0, 1, cfg)
    data, bits, q = W["data"], W["bits"], W["queries"]
    mask = None
    n, k = cfg["n"], cfg["k"]
    words = bits
    for G in gs:
        shards, kths = [], []
        for r in range(G):
            lo, hi = row_shard(n, r, G)
            ctx = N.Context(0)
            col = vs.EmbeddingColumn.from_device(data[lo:hi])
            sb = bench.pack_bits_torch(W["mask"][lo:hi].contiguous())
            shards.append((ShardSearch(col, ctx), ctx, col, sb, lo))
        # phase A + local top-k keys per shard
        t_begin = []
        for sh, ctx, col, sb, lo in shards:
            t_begin.append(timed(lambda: sh.begin(q, k, "squared_l2", sb)))
            kths.append(sh.begin(q, k, "squared_l2", sb).clone())
        T = shards[0][0].union_kth(torch.stack(kths))
        sh0, ctx0, _, sb0, _ = shards[0]
        ctx0.set_option(N.OPT_TIMING, 1)
        ctx0.kernel_times(reset=True)
        sh0.begin(q, k, "squared_l2", sb0)
        torch.cuda.synchronize()
        kt_begin = {c: round(v[0] / 1e6, 3) for c, v in ctx0.kernel_times(reset=True).items() if v[1]}
        ctx0.set_option(N.OPT_TIMING, 0)
        t_finish, surv = [], []
        for (sh, ctx, col, sb, lo) in shards:
            tot = 0.0
            for rep in range(4):
                sh.begin(q, k, "squared_l2", sb)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                sh.finish(T, lo)
                e1.record()
                torch.cuda.synchronize()
                if rep:
                    tot += e0.elapsed_time(e1)
            t_finish.append(tot / 3)
            surv.append(ctx.stats()[N.STAT_SURVIVORS] / q.shape[0])
        # one-phase shard search (local top-k, full re-rank)
        t_plain = []
        for (sh, ctx, col, sb, lo) in shards[:2]:
            out = (torch.empty((q.shape[0], k), dtype=torch.int64, device=dev),
                   torch.empty((q.shape[0], k), dtype=torch.float64, device=dev),
                   torch.empty((q.shape[0],), dtype=torch.int32, device=dev))
            t_plain.append(timed(lambda: enn_search_raw(q, col, k, row_filter=sb, id_offset=lo,
                                                       device=ctx, out=out)))
        print(json.dumps({"G": G, "begin_ms_max": round(max(t_begin), 3),
                          "finish_ms_max": round(max(t_finish), 3),
                          "two_phase_ms_per_rank": round(max(b + f for b, f in zip(t_begin, t_finish)), 3),
                          "one_phase_ms_per_rank": round(max(t_plain), 3),
                          "survivors_per_query_per_shard": [round(s, 1) for s in surv],
                          "begin_kernel_ms_shard0": kt_begin}), flush=True)
        del shards, kths
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
