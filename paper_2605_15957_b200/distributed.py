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
        else:  # gloo (CPU tests): list form over host copies
            h = t.cpu()
            parts = [torch.empty_like(h) for _ in range(world)]
            dist_.all_gather(parts, h, group=group)
            o = torch.stack(parts).to(t.device)
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


# ---- two-phase exact search over row shards ----------------------------------------------------
#
# Plain row sharding re-ranks every shard's full local top-k (k + margin band
# survivors per query per shard), so the exact float64 work per GPU does not
# shrink with the shard count. The two-phase protocol first exchanges, per
# query, k floats per shard: upper bounds on the exact keys of the shard's k
# smallest APPROXIMATE keys (approx + that shard's margin/2, rounded up). The
# k-th smallest of their union, U*, bounds the global k-th exact key from
# above (k rows have exact key <= U*), so a row of the global top-k has approx
# key <= U* + m_s/2 on its shard s whatever the other shards' margins (their
# max norms or phase-A kernels may differ). Each shard re-ranks only those
# candidates: the single-GPU survivor set, split across the shards. Rows a
# shard dropped in phase A (local top-k mode) have exact key > that shard's
# bound, which is checked against the merged k-th key; a failing query is
# re-run with the one-phase search on every shard.


class TorchComm:
    """Collectives of the protocol over torch.distributed (NCCL on GPUs)."""

    def __init__(self, group=None):
        self.group = group

    def size(self):
        import torch.distributed as dist_
        return dist_.get_world_size(self.group) if dist_.is_initialized() else 1

    def rank(self):
        import torch.distributed as dist_
        return dist_.get_rank(self.group) if dist_.is_initialized() else 0

    def allreduce_min(self, t):
        import torch.distributed as dist_
        if dist_.get_backend(self.group) != "nccl" and t.is_cuda:
            # gloo: reduce a host copy (device tensors only via NCCL)
            h = t.cpu()
            dist_.all_reduce(h, op=dist_.ReduceOp.MIN, group=self.group)
            t.copy_(h)
            return t
        dist_.all_reduce(t, op=dist_.ReduceOp.MIN, group=self.group)
        return t

    def allgather(self, t):
        import torch
        import torch.distributed as dist_
        world = dist_.get_world_size(self.group)
        t = t.contiguous()
        if dist_.get_backend(self.group) == "nccl":
            o = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
            dist_.all_gather_into_tensor(o, t, group=self.group)
            return o
        h = t.cpu()
        parts = [torch.empty_like(h) for _ in range(world)]
        dist_.all_gather(parts, h, group=self.group)
        return torch.stack(parts).to(t.device)

    def allgather_topk(self, ids, dist, counts):
        return all_gather_topk(ids, dist, counts, self.group)


def _merged_is_exact(md, mc, bound, k: int, metric: str):
    """Per query: the merged top-k is provably complete (torch, on device)."""
    import torch
    inf = torch.full_like(bound, float("inf"))
    kidx = (mc.clamp(min=1) - 1).long().unsqueeze(1)
    kth = md.gather(1, kidx).squeeze(1)
    key = -kth if metric == "inner_product" else kth
    full = mc >= k
    ok = torch.where(full, key < bound, bound >= inf)
    return ok


def two_phase_search(shard, comm, queries, k: int, metric: str = "squared_l2", row_filter=None,
                     id_offset: int = 0, merge=None):
    """Exact filtered top-k over row shards (one call per rank, collectively).

    `shard` is this rank's ShardSearch (begin / finish / plain); `comm`
    provides allreduce_min and allgather_topk. Returns (ids, dist, counts) of
    the global result on every rank (torch tensors on the shard's device)."""
    import torch

    from . import _native as N
    merge = merge or gpu_merge
    if k > N.topk_cap():
        # k' above the candidate buffers (device-wide large-k' path): one phase,
        # every shard's exact local top-k', all-gather + merge
        ri, rd, rc = shard.plain(queries, k, metric, row_filter, id_offset)
        gi, gd, gc = comm.allgather_topk(ri, rd, rc)
        shard.reruns = 0
        return merge(gi, gd, gc, k, metric)
    keys = shard.begin(queries, k, metric, row_filter)        # [Q, k] upper bounds on exact keys
    T = shard.union_kth(comm.allgather(keys))               # [Q] >= global k-th exact key
    ids, dist, cnt, bound = shard.finish(T, id_offset)
    gi, gd, gc = comm.allgather_topk(ids, dist, cnt)
    mi, md, mc = merge(gi, gd, gc, k, metric)
    comm.allreduce_min(bound)
    # the re-run set is agreed collectively (MIN of the per-rank verdicts), so
    # every rank takes part in the same collectives even if a verdict differed
    ok = _merged_is_exact(md, mc, bound, k, metric).to(torch.int32)
    comm.allreduce_min(ok)
    bad = torch.nonzero(ok == 0).flatten()
    if bad.numel():
        sub_q = queries[bad] if hasattr(queries, "index_select") else queries[bad.cpu().numpy()]
        ri, rd, rc = shard.plain(sub_q, k, metric, row_filter, id_offset)
        gi, gd, gc = comm.allgather_topk(ri, rd, rc)
        si, sd, sc = merge(gi, gd, gc, k, metric)
        mi[bad], md[bad], mc[bad] = si, sd, sc
    shard.reruns = int(bad.numel())
    return mi, md, mc


class ShardSearch:
    """This rank's row shard for two_phase_search (vs_enn_search_begin/finish
    through ctypes; CUDA torch tensors in and out)."""

    def __init__(self, column, ctx=None):
        from . import _native as N
        from .vecindex import _as_column, _ctx, device_column
        self.col = _as_column(column)
        self.ctx = ctx or _ctx()
        self.dc = device_column(self.col, self.ctx)
        self.N = N
        self.reruns = 0

    def begin(self, queries, k, metric, row_filter):
        import ctypes as C

        import torch

        from .vecindex import _query_buffer, _Stream, filter_bitmap
        N = self.N
        q, nq, d = _query_buffer(queries)
        self._q, self._nq, self._k = q, nq, int(k)
        self._bm = filter_bitmap(row_filter, self.col.count)
        dev = q.device if N.is_torch(q) and q.is_cuda else torch.device("cuda", self.ctx.device)
        self._dev = dev
        keys = torch.empty((nq, self._k), dtype=torch.float32, device=dev)
        vis = C.c_int64(0)
        with _Stream(self.ctx, q, self._bm, keys):
            N.check(N.load().vs_enn_search_begin(
                self.ctx.handle, self.dc.handle, N.ptr(q), nq, d, N.ptr(self._bm),
                self.col.count if self._bm is not None else 0, self._k, N.METRIC_CODE[metric],
                N.ptr(keys), C.byref(vis)), "enn_search_begin")
        return keys

    def union_kth(self, all_keys):
        """[G, Q, k] gathered shard keys -> [Q] k-th smallest of the union."""
        import torch

        from .vecindex import _Stream
        N = self.N
        G, nq, k = all_keys.shape
        out = torch.empty(nq, dtype=torch.float32, device=all_keys.device)
        with _Stream(self.ctx, all_keys, out):
            N.check(N.load().vs_union_kth(self.ctx.handle, int(G), int(nq), int(k),
                                          N.ptr(all_keys.contiguous()), N.ptr(out)), "union_kth")
        return out

    def finish(self, thresholds, id_offset):
        import torch

        from .vecindex import _Stream
        N = self.N
        nq, k, dev = self._nq, self._k, self._dev
        ids = torch.empty((nq, k), dtype=torch.int64, device=dev)
        dist = torch.empty((nq, k), dtype=torch.float64, device=dev)
        cnt = torch.empty((nq,), dtype=torch.int32, device=dev)
        bound = torch.empty((nq,), dtype=torch.float64, device=dev)
        with _Stream(self.ctx, thresholds, ids):
            N.check(N.load().vs_enn_search_finish(
                self.ctx.handle, N.ptr(thresholds.contiguous()), int(id_offset), N.ptr(ids), N.ptr(dist),
                N.ptr(cnt), N.ptr(bound)), "enn_search_finish")
        return ids, dist, cnt, bound

    def plain(self, queries, k, metric, row_filter, id_offset):
        import torch

        from .vecindex import enn_search_raw
        nq = queries.shape[0]
        out = (torch.empty((nq, k), dtype=torch.int64, device=self._dev),
               torch.empty((nq, k), dtype=torch.float64, device=self._dev),
               torch.empty((nq,), dtype=torch.int32, device=self._dev))
        from .errors import EmptyInputError
        try:
            enn_search_raw(queries, self.col, k, metric, row_filter=row_filter, id_offset=id_offset,
                           device=self.ctx, out=out)
        except EmptyInputError:   # this shard selects no rows: it contributes nothing
            out[0].fill_(-1)
            out[1].fill_(float("nan"))
            out[2].zero_()
        return out


# ---- IVF over list shards --------------------------------------------------------------------


def ivf_sharded_search(index, queries, k: int, nprobe: int, row_filter=None, list_owned=None, comm=None,
                       merge=None, device=None):
    """IVF search with lists sharded across ranks (LPT `list_owned`).

    The coarse quantizer is split by QUERIES instead of replicated: rank r
    probes its slice of the batch, the [Q, nprobe] probes are all-gathered
    (every rank then holds the probes of the reference's coarse step), each
    rank scans the probed lists it owns, and the per-rank top-k are
    all-gathered and merged (tie rule). Returns (ids, dist, counts) on every
    rank."""
    import torch
    comm = comm or TorchComm()
    merge = merge or gpu_merge
    world, rank = comm.size(), comm.rank()
    nq = queries.shape[0]
    per = (nq + world - 1) // world
    lo, hi = min(nq, rank * per), min(nq, (rank + 1) * per)
    mine = index.probe(queries[lo:hi], nprobe, device=device) if hi > lo else None
    pad = torch.full((per, nprobe), -1, dtype=torch.int32, device=queries.device)
    if mine is not None:
        pad[: hi - lo] = mine if N_is_torch(mine) else torch.from_numpy(mine).to(queries.device)
    probes = comm.allgather(pad).reshape(world * per, nprobe)[:nq].contiguous()
    dev = queries.device
    out = (torch.empty((nq, k), dtype=torch.int64, device=dev),
           torch.empty((nq, k), dtype=torch.float64, device=dev),
           torch.empty((nq,), dtype=torch.int32, device=dev))
    index.search_raw(queries, k, nprobe, row_filter=row_filter, device=device, list_owned=list_owned,
                     out=out, probes_in=probes)
    gi, gd, gc = comm.allgather_topk(*out)
    return merge(gi, gd, gc, k, index.metric)


def N_is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")
