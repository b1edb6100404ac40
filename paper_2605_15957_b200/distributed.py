"""Data placement across GPUs of one box: one process per GPU,
`torch.distributed` (NCCL over NVLink/NVSwitch) as plumbing for the single
exchange step, and the library's merge kernel for the global top-k.

Exact search (configs 2/5): contiguous row ranges [r*N/G, (r+1)*N/G), the
bitmap sliced identically, queries broadcast; each rank searches its shard
with ids offset to global rows, the [Q, k] (id, distance, count) triples are
all-gathered, and `vs_topk_merge` selects the global top-k under the tie rule.
Per-pair arithmetic does not depend on the shard, so results are identical
for every world size.

IVF (config 4): centroids replicated (coarse probes identical everywhere),
lists assigned to ranks by greedy size balancing (LPT); each rank scans the
probed lists it owns; same exchange + merge.

The search and merge callables are injectable so the exchange logic is
tested on CPU with the gloo backend and the oracle (tests/test_dist_gloo.py).
"""

from __future__ import annotations

import numpy as np


def row_shard(n: int, rank: int, world: int) -> tuple:
    """Contiguous row range of `rank` (balanced to within one row)."""
    lo = (n * rank) // world
    hi = (n * (rank + 1)) // world
    return lo, hi


def slice_bitmap_words(mask_bool: np.ndarray, lo: int, hi: int) -> np.ndarray:
    from .vecindex import pack_bitmap
    return pack_bitmap(np.asarray(mask_bool, bool)[lo:hi])


def lpt_assign(sizes, world: int) -> np.ndarray:
    """Greedy longest-processing-time list assignment: lists in decreasing
    size (ties by list id) each go to the currently lightest rank (ties by
    rank). Deterministic, so every rank computes the same map."""
    sizes = np.asarray(sizes, np.int64)
    order = np.lexsort((np.arange(len(sizes)), -sizes))
    load = np.zeros(world, np.int64)
    owner = np.empty(len(sizes), np.int32)
    for li in order:
        r = int(np.argmin(load))
        owner[li] = r
        load[r] += sizes[li]
    return owner


def all_gather_topk(ids, dist, counts, group=None):
    """All-gather per-rank [Q, k] results -> [G, Q, k] (torch tensors on the
    process's device; NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist_

    world = dist_.get_world_size(group)
    outs = []
    for t in (ids, dist, counts):
        t = t.contiguous()
        if dist_.get_backend(group) == "nccl":
            o = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            dist_.all_gather_into_tensor(o, t, group=group)
        else:  # gloo (CPU tests): list form
            parts = [torch.empty_like(t) for _ in range(world)]
            dist_.all_gather(parts, t, group=group)
            o = torch.stack(parts)
        outs.append(o)
    return tuple(outs)


def gpu_merge(ids, dist, counts, k: int, metric: str, device=None, out=None):
    """Global top-k of [G, Q, k_in] shard results with the library's merge
    kernel (vs_topk_merge)."""
    import ctypes as C  # noqa: F401

    import torch

    from . import _native as N
    from .vecindex import _Stream, _ctx

    G, Q, k_in = ids.shape
    ctx = _ctx(device)
    if out is None:
        out = (torch.empty((Q, k), dtype=torch.int64, device=ids.device),
               torch.empty((Q, k), dtype=torch.float64, device=ids.device),
               torch.empty((Q,), dtype=torch.int32, device=ids.device))
    oi, od, oc = out
    with _Stream(ctx, ids, oi):
        N.check(N.load().vs_topk_merge(ctx.handle, G, Q, k_in, N.ptr(ids), N.ptr(dist), N.ptr(counts),
                                       int(k), N.METRIC_CODE[metric], N.ptr(oi), N.ptr(od),
                                       N.ptr(oc)), "topk_merge")
    return oi, od, oc


def sharded_search(local_search, k: int, metric: str, merge=None, group=None):
    """One exchange step: run this rank's search, all-gather, merge.

    local_search() -> (ids [Q,k] int64, dist [Q,k] float64, counts [Q] int32)
    torch tensors with GLOBAL ids. merge(ids, dist, counts, k, metric) over
    [G, Q, k] defaults to the GPU merge kernel."""
    ids, dist, cnt = local_search()
    gi, gd, gc = all_gather_topk(ids, dist, cnt, group)
    merge = merge or gpu_merge
    return merge(gi, gd, gc, k, metric)
