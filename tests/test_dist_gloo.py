"""World-size-2 process group on CPU (gloo): the sharded exchange step
(row shards with global ids -> all-gather -> tie-rule merge) reproduces the
unsharded exact search; IVF list sharding (LPT) likewise. The per-shard
search is the oracle here (no GPU); on the B200 it is the library kernel."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sqlvs_oracle as O
from paper_2605_15957_b200.distributed import all_gather_topk, lpt_assign, row_shard, sharded_search


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_merge(gi, gd, gc, k, metric):
    G, Q, _ = gi.shape
    ids = np.full((Q, k), -1, np.int64)
    dd = np.full((Q, k), np.nan)
    cnt = np.zeros(Q, np.int32)
    for q in range(Q):
        parts = [(gi[g, q, :gc[g, q]].numpy(), gd[g, q, :gc[g, q]].numpy()) for g in range(G)]
        a, b = O.merge_topk(parts, k, metric)
        ids[q, :len(a)], dd[q, :len(a)], cnt[q] = a, b, len(a)
    return torch.from_numpy(ids), torch.from_numpy(dd), torch.from_numpy(cnt)


def _padded(res, nq, k):
    ids = np.full((nq, k), -1, np.int64)
    dd = np.full((nq, k), np.nan)
    cnt = np.zeros(nq, np.int32)
    for q in range(nq):
        a, b = res.per_query(q)
        ids[q, :len(a)], dd[q, :len(a)], cnt[q] = a, b, len(a)
    return torch.from_numpy(ids), torch.from_numpy(dd), torch.from_numpy(cnt)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    data = rng.standard_normal((3000, 16)).astype(np.float32)
    q = rng.standard_normal((7, 16)).astype(np.float32)
    mask = rng.random(3000) < 0.4
    k = 25
    lo, hi = row_shard(3000, rank, world)

    def local():
        rows = lo + np.flatnonzero(mask[lo:hi])
        res = O.enn_search(q, data[rows], k, row_ids=rows)
        return _padded(res, 7, k)

    mi, md, mc = sharded_search(local, k, "squared_l2", merge=_oracle_merge)
    # IVF: replicated centroids, LPT-owned lists
    cen, parts, payload = O.ivf_build(data[:500], 12, 0)
    assign = np.argmin(O.pairwise_sq_l2_fast(data, cen), axis=1)
    parts = [np.flatnonzero(assign == c).astype(np.int64) for c in range(12)]
    owner = lpt_assign([len(p) for p in parts], world)
    mine = [p if owner[c] == rank else np.empty(0, np.int64) for c, p in enumerate(parts)]
    r = O.ivf_search(q, cen, mine, lambda c: data[mine[c]], 4, k)
    gi, gd, gc = all_gather_topk(*_padded(r, 7, k))
    ii, id_, ic = _oracle_merge(gi, gd, gc, k, "squared_l2")
    if rank == 0:
        out["enn"] = (mi.numpy(), md.numpy(), mc.numpy())
        out["ivf"] = (ii.numpy(), id_.numpy(), ic.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_world2_exchange_matches_unsharded():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        enn, ivf = out["enn"], out["ivf"]
    rng = np.random.default_rng(0)
    data = rng.standard_normal((3000, 16)).astype(np.float32)
    q = rng.standard_normal((7, 16)).astype(np.float32)
    mask = rng.random(3000) < 0.4
    ref = O.enn_filtered(q, data, mask, 25)
    ids, dd, cnt = enn
    m = np.arange(25)[None, :] < cnt[:, None]
    assert np.array_equal(ids[m], ref.data_row)
    assert np.array_equal(dd[m], ref.distance)
    cen, parts, payload = O.ivf_build(data[:500], 12, 0)
    assign = np.argmin(O.pairwise_sq_l2_fast(data, cen), axis=1)
    parts = [np.flatnonzero(assign == c).astype(np.int64) for c in range(12)]
    ref = O.ivf_search(q, cen, parts, lambda c: data[parts[c]], 4, 25)
    ids, dd, cnt = ivf
    m = np.arange(25)[None, :] < cnt[:, None]
    assert np.array_equal(ids[m], ref.data_row)
    assert np.array_equal(dd[m], ref.distance)
