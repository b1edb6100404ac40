"""Parity at the BASELINE scales, part A: the 10M x 1024 float32 collection
of configs 2 and 3 (BASELINE.json configs[1], configs[2]), built exactly as
bench.py builds it, searched through the same entry points, and compared with
`==` (ids and float64 distances) against the oracle on sampled queries spread
over the whole batch (so over every query tile and split of phase A).

- config 2: exact filtered top-100, 10% Bernoulli bitmap, 10k queries
  (enn_search_raw, the tcgen05 phase A); oracle = oracle.enn_pruned over the
  host copy of the selected rows (reference arithmetic, vecindex.py:109-132).
- config 2, two-phase: two row shards as two library contexts (threads,
  in-process collectives); merged result == the one-GPU result for all 10k.
- config 3: IVF-Flat nlist=16384 built on the GPU, nprobe=32, top-10, 1%
  bitmap; probes, ids and distances vs oracle.ivf_search (vecindex.py:230-258).
"""

import threading

import numpy as np
import pytest
import torch

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O
from paper_2605_15957_b200 import _native as N
from paper_2605_15957_b200 import synth
from paper_2605_15957_b200.vecindex import enn_search_raw

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N_ROWS, D, NQ = 10_000_000, 1024, 10_000


def sample_rows(nq, m):
    """m query indices spread over the batch (first and last included)."""
    return np.unique(np.linspace(0, nq - 1, m).round().astype(np.int64))


def assert_rows_equal(ids, dist, cnt, ref, qidx):
    for j, qi in enumerate(qidx):
        want_ids, want_d = ref.per_query(j)
        c = int(cnt[qi])
        assert c == len(want_ids), f"query {qi}: {c} results, oracle {len(want_ids)}"
        assert np.array_equal(ids[qi, :c], want_ids), f"query {qi}: ids differ from the oracle"
        assert np.array_equal(dist[qi, :c], want_d), f"query {qi}: distances differ from the oracle"


@pytest.fixture(scope="module")
def coll():
    dev = torch.device("cuda", 0)
    data, centers = synth.device_rows(N_ROWS, D, 0, N_ROWS, dev)
    queries = synth.device_queries(centers, NQ, seed=7)
    torch.cuda.synchronize()
    yield {"data": data, "queries": queries, "dev": dev}
    del data
    torch.cuda.empty_cache()


@pytest.fixture(scope="module")
def cfg2(coll):
    dev = coll["dev"]
    mask = synth.device_bernoulli(N_ROWS, 0.10, 4242, dev)
    bits = synth.pack_bits_torch(mask)
    ctx = N.Context(0)
    col = vs.EmbeddingColumn.from_device(coll["data"])
    out = (torch.empty((NQ, 100), dtype=torch.int64, device=dev),
           torch.empty((NQ, 100), dtype=torch.float64, device=dev),
           torch.empty((NQ,), dtype=torch.int32, device=dev))
    enn_search_raw(coll["queries"], col, 100, "squared_l2", row_filter=bits, device=ctx, out=out)
    kern = ctx.stats()[N.STAT_LAST_ENN_KERNEL]
    torch.cuda.synchronize()
    res = tuple(t.cpu().numpy() for t in out)
    yield {"mask": mask, "bits": bits, "res": res, "kernel": kern, "ctx": ctx}
    ctx.close()


def test_config2_sampled_queries_equal_oracle(coll, cfg2):
    assert cfg2["kernel"] == 2, "config 2 must run the tcgen05 phase A"
    ids, dist, cnt = cfg2["res"]
    mask = cfg2["mask"]
    n_sel = int(mask.sum())
    assert (cnt == 100).all()
    qidx = sample_rows(NQ, 16)
    rows = torch.nonzero(mask).flatten()
    xs = coll["data"][rows].cpu().numpy()                 # the selected rows, ascending (4 GB)
    q = coll["queries"][torch.from_numpy(qidx).to(coll["dev"])].cpu().numpy()
    ref = O.enn_pruned(q, xs, 100, "squared_l2", row_ids=rows.cpu().numpy())
    assert xs.shape[0] == n_sel
    assert_rows_equal(ids, dist, cnt, ref, qidx)


def test_config2_two_phase_two_shards_equal_one_gpu(coll, cfg2):
    from functools import partial

    from paper_2605_15957_b200.distributed import ShardSearch, gpu_merge, row_shard, two_phase_search
    from test_gpu_two_phase import ThreadComm
    world = 2
    comm = ThreadComm(world)
    results, errors = [None] * world, []
    mask = cfg2["mask"]

    def rank(r):
        try:
            lo, hi = row_shard(N_ROWS, r, world)
            ctx = N.Context(0)
            shard = ShardSearch(vs.EmbeddingColumn.from_device(coll["data"][lo:hi]), ctx)
            bits = synth.pack_bits_torch(mask[lo:hi].contiguous())
            results[r] = two_phase_search(shard, comm.rank(r), coll["queries"], 100, "squared_l2",
                                          row_filter=bits, id_offset=lo, merge=partial(gpu_merge, device=ctx))
            torch.cuda.synchronize()
            results[r] = tuple(t.cpu().numpy() for t in results[r]) + (shard.reruns,)
            ctx.close()
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
    ids, dist, cnt = cfg2["res"]
    for r in range(world):
        gi, gd, gc, _ = results[r]
        assert np.array_equal(gc, cnt)
        assert np.array_equal(gi, ids)
        assert np.array_equal(gd, dist)


def test_config3_ivf_sampled_queries_equal_oracle(coll):
    dev = coll["dev"]
    mask = synth.device_bernoulli(N_ROWS, 0.01, 4243, dev)
    bits = synth.pack_bits_torch(mask)
    ctx = N.Context(0)
    col = vs.EmbeddingColumn.from_device(coll["data"])
    index = vs.IvfIndex.build(col, 16384, seed=0, device=ctx)
    out = (torch.empty((NQ, 10), dtype=torch.int64, device=dev),
           torch.empty((NQ, 10), dtype=torch.float64, device=dev),
           torch.empty((NQ,), dtype=torch.int32, device=dev))
    stats0 = ctx.stats()[N.STAT_OVERFLOW_QUERIES]
    _, _, _, probes, _ = index.search_raw(coll["queries"], 10, 32, row_filter=bits, device=ctx, out=out,
                                          want_probes=True)
    torch.cuda.synchronize()
    overflows = ctx.stats()[N.STAT_OVERFLOW_QUERIES] - stats0
    ids, dist, cnt = (t.cpu().numpy() for t in out)
    qidx = sample_rows(NQ, 16)
    q = coll["queries"][torch.from_numpy(qidx).to(dev)].cpu().numpy()
    lists = {int(c): coll["data"][torch.from_numpy(index.partitions[int(c)]).to(dev)].cpu().numpy()
             for c in np.unique(probes[qidx])}
    mask_h = mask.cpu().numpy()

    def vectors_of(c):
        if c not in lists:
            raise AssertionError(f"oracle probes list {c}, not among the GPU probes")
        return lists[c]

    ref = O.ivf_search(q, index.centroids, index.partitions, vectors_of, 32, 10, mask=mask_h)
    assert np.array_equal(np.asarray(ref.probes), probes[qidx]), "probes differ from the oracle"
    assert_rows_equal(ids, dist, cnt, ref, qidx)
    print(f"config 3: overflow re-runs in the search: {overflows}")
    del index, col
    ctx.close()
