"""Two-phase exact search over row shards (distributed.two_phase_search,
vs_enn_search_begin/finish): G shards emulated on one GPU by G library
contexts driven from G threads with in-process collectives. The merged result
must equal the unsharded search bit for bit (ids, float64 distances), which
itself equals the reference composition."""

import threading
from functools import partial

import numpy as np
import pytest
import torch

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O
from paper_2605_15957_b200 import _native as N
from paper_2605_15957_b200.distributed import ShardSearch, gpu_merge, row_shard, two_phase_search

pytestmark = pytest.mark.gpu


class ThreadComm:
    """allreduce(MIN) / all-gather between threads of one process."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def rank(self, r):
        comm = self

        class _R:
            def size(self):
                return comm.world

            def rank(self):
                return r

            def allreduce_min(self, t):
                comm.slots[r] = t.clone()
                comm.barrier.wait()
                m = torch.stack(comm.slots).min(0).values
                comm.barrier.wait()
                t.copy_(m)
                return t

            def allgather(self, t):
                comm.slots[r] = t
                comm.barrier.wait()
                out = torch.stack(list(comm.slots))
                comm.barrier.wait()
                return out

            def allgather_topk(self, ids, dist, cnt):
                comm.slots[r] = (ids, dist, cnt)
                comm.barrier.wait()
                out = tuple(torch.stack([s[j] for s in comm.slots]) for j in range(3))
                comm.barrier.wait()
                return out

        return _R()


def _run(world, data, q, mask, k, metric, shard_cls=ShardSearch, kernels=None):
    n = data.shape[0]
    xd = torch.from_numpy(data).cuda()
    qd = torch.from_numpy(q).cuda()
    comm = ThreadComm(world)
    results, shards, errors = [None] * world, [None] * world, []

    def rank(r):
        try:
            lo, hi = row_shard(n, r, world)
            ctx = N.Context(0)
            if kernels is not None:
                ctx.set_option(N.OPT_ENN_KERNEL, kernels[r])
            shard = shard_cls(vs.EmbeddingColumn.from_device(xd[lo:hi].contiguous()), ctx)
            shards[r] = shard
            results[r] = two_phase_search(shard, comm.rank(r), qd, k, metric,
                                          row_filter=None if mask is None else mask[lo:hi],
                                          id_offset=lo, merge=partial(gpu_merge, device=ctx))
            torch.cuda.synchronize()
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)
            comm.barrier.abort()

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    return results, shards


def _flat(res):
    ids, dist, cnt = (t.cpu().numpy() for t in res)
    m = np.arange(ids.shape[1])[None, :] < cnt[:, None]
    return ids[m], dist[m], cnt


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
def test_two_phase_equals_unsharded(world, metric):
    rng = np.random.default_rng(world * 10 + (metric == "inner_product"))
    n, d, k = 40000, 128, 50
    data = rng.standard_normal((n, d)).astype(np.float32)
    q = rng.standard_normal((300, d)).astype(np.float32)   # >= 256: tensor-core phase A
    mask = rng.random(n) < 0.4
    results, shards = _run(world, data, q, mask, k, metric)
    whole = vs.enn_search(q, data, vs.SearchParams(k=k), metric=metric, row_filter=mask)
    for r in range(world):
        ids, dist, _ = _flat(results[r])
        assert np.array_equal(ids, whole.data_row)
        assert np.array_equal(dist, whole.distance)


@pytest.mark.parametrize("kernels", [(2, 2), (2, 1, 2), (1, 2, 1, 2)])
@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
def test_two_phase_forced_and_mixed_phase_a_kernels(kernels, metric):
    """Every shard on the tensor-core phase A (local top-k + verification
    bounds at world > 1), and shards mixing tensor-core (bf16, wide margin) and
    SIMT (fp32, narrow margin) phase A at small d, with shards of very
    different max norms: the exchanged bounds must hold across margins."""
    world = len(kernels)
    rng = np.random.default_rng(70 + world + 10 * (metric == "inner_product"))
    n, d, k = 24000, 64, 40
    data = rng.standard_normal((n, d)).astype(np.float32)
    for r in range(world):                     # shard r's rows scaled by 1 + 2r
        lo, hi = row_shard(n, r, world)
        data[lo:hi] *= np.float32(1 + 2 * r)
    q = rng.standard_normal((150, d)).astype(np.float32)
    mask = rng.random(n) < 0.5
    results, shards = _run(world, data, q, mask, k, metric, kernels=list(kernels))
    for r in range(world):
        assert shards[r].ctx.stats()[N.STAT_LAST_ENN_KERNEL] == kernels[r]
    ref = O.enn_filtered(q, data, mask, k, metric)
    ids, dist, _ = _flat(results[0])
    assert np.array_equal(ids, ref.data_row)
    assert np.array_equal(dist, ref.distance)


def test_two_phase_rerun_path_and_empty_shard():
    rng = np.random.default_rng(5)
    n, d, k = 20000, 64, 30
    data = rng.standard_normal((n, d)).astype(np.float32)
    q = rng.standard_normal((280, d)).astype(np.float32)
    mask = rng.random(n) < 0.5
    mask[: n // 3] = False                   # shard 0 of 3 selects nothing

    class Pessimist(ShardSearch):            # bounds below every key: every query re-runs
        def finish(self, thresholds, id_offset):
            ids, dist, cnt, bound = super().finish(thresholds, id_offset)
            return ids, dist, cnt, torch.full_like(bound, -1e30)

    for cls in (ShardSearch, Pessimist):
        results, shards = _run(3, data, q, mask, k, "squared_l2", cls)
        ref = O.enn_filtered(q, data, mask, k)
        ids, dist, _ = _flat(results[1])
        assert np.array_equal(ids, ref.data_row)
        assert np.array_equal(dist, ref.distance)
        if cls is Pessimist:
            assert shards[0].reruns == q.shape[0]


@pytest.mark.parametrize("world", [2, 3])
def test_ivf_list_sharded_query_sliced_probing(world):
    """IVF with LPT list shards: each rank probes a slice of the queries, the
    probes are all-gathered, each rank scans its own lists, merge == one GPU."""
    from paper_2605_15957_b200.distributed import ivf_sharded_search, lpt_assign
    rng = np.random.default_rng(40 + world)
    n, d, nlist = 30000, 64, 40
    data = rng.standard_normal((n, d)).astype(np.float32)
    cen = data[rng.choice(n, nlist, replace=False)].copy()
    assign = np.argmin(O.pairwise_sq_l2_fast(data, cen), axis=1)
    parts = [np.flatnonzero(assign == c).astype(np.int64) for c in range(nlist)]
    payload = [data[p] for p in parts]
    q = rng.standard_normal((101, d)).astype(np.float32)
    mask = rng.random(n) < 0.6
    owner = lpt_assign([len(p) for p in parts], world)
    qd = torch.from_numpy(q).cuda()
    comm = ThreadComm(world)
    results, errors = [None] * world, []

    def rank(r):
        try:
            ctx = N.Context(0)
            idx = vs.IvfIndex(nlist, d, n, "squared_l2", "owning", cen, parts, payload)
            results[r] = ivf_sharded_search(idx, qd, 15, 7, row_filter=mask,
                                            list_owned=(owner == r).astype(np.uint8), comm=comm.rank(r),
                                            merge=partial(gpu_merge, device=ctx), device=ctx)
            torch.cuda.synchronize()
        except Exception as e:  # pragma: no cover
            errors.append(e)
            comm.barrier.abort()

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errors:
        raise errors[0]
    ref = O.ivf_search(q, cen, parts, lambda c: payload[c], 7, 15, mask=mask)
    for r in range(world):
        ids, dist, _ = _flat(results[r])
        assert np.array_equal(ids, ref.data_row)
        assert np.array_equal(dist, ref.distance)


def test_inputs_from_async_copies_on_the_default_stream():
    """Device inputs produced by non_blocking host->device copies on torch's
    default stream (handle 0) right before the call: the library must be
    ordered after them (it runs on cudaStreamLegacy then, not its own stream)."""
    rng = np.random.default_rng(11)
    n, d, nq, k = 200000, 256, 3000, 10
    data = rng.standard_normal((n, d)).astype(np.float32)
    q = rng.standard_normal((nq, d)).astype(np.float32)
    mask = rng.random(n) < 0.2
    col = vs.EmbeddingColumn.from_device(torch.from_numpy(data).cuda())
    qh = torch.from_numpy(q).pin_memory()
    bh = torch.from_numpy(vs.vecindex.pack_bitmap(mask).view(np.int32)).pin_memory()
    shard = ShardSearch(col)

    class One:
        def size(self):
            return 1

        def rank(self):
            return 0

        def allreduce_min(self, t):
            return t

        def allgather(self, t):
            return t.unsqueeze(0)

        def allgather_topk(self, i, dd, c):
            return i.unsqueeze(0), dd.unsqueeze(0), c.unsqueeze(0)

    ref = O.enn_filtered(q[::97], data, mask, k)
    for _ in range(3):
        qq = qh.to("cuda", non_blocking=True)
        bb = bh.to("cuda", non_blocking=True)
        ids, dist, cnt = two_phase_search(shard, One(), qq, k, "squared_l2", row_filter=bb)
        ids, dist = ids.cpu().numpy()[::97].reshape(-1), dist.cpu().numpy()[::97].reshape(-1)
        assert np.array_equal(ids, ref.data_row)
        assert np.array_equal(dist, ref.distance)
