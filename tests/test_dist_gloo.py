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


class _OracleShard:
    """CPU stand-in for ShardSearch: phase A keys are the exact float64 keys
    (margin 0), so the protocol's choreography is what is tested here."""

    def __init__(self, data, mask, lo, hi, pessimist=False):
        self.data, self.mask, self.lo, self.hi, self.pessimist = data, mask, lo, hi, pessimist
        self.reruns = 0

    def _scores(self, q):
        rows = self.lo + np.flatnonzero(self.mask[self.lo:self.hi])
        return rows, (O.pairwise(q, self.data[rows]) if rows.size else np.zeros((len(q), 0)))

    def begin(self, q, k, metric, row_filter):
        self.q, self.k = q, k
        rows, s = self._scores(q)
        keys = np.full((len(q), k), np.inf, np.float32)
        if rows.size:
            srt = np.sort(s, axis=1)[:, :k].astype(np.float32)
            keys[:, :srt.shape[1]] = srt
        return torch.from_numpy(keys)

    def union_kth(self, all_keys):
        G, nq, k = all_keys.shape
        u = all_keys.permute(1, 0, 2).reshape(nq, G * k)
        return torch.sort(u, dim=1).values[:, k - 1]

    def finish(self, thr, id_offset):
        rows, s = self._scores(self.q)
        nq, k = len(self.q), self.k
        ids = torch.full((nq, k), -1, dtype=torch.int64)
        dd = torch.full((nq, k), float("nan"), dtype=torch.float64)
        cnt = torch.zeros(nq, dtype=torch.int32)
        for i in range(nq):
            keep = s[i] <= float(thr[i]) * (1 + 1e-6) + 1e-6
            if keep.any():
                top = O.select_top(s[i][keep], rows[keep], min(k, int(keep.sum())), "squared_l2")
                r_ = rows[keep][top]
                ids[i, :len(r_)] = torch.from_numpy(r_)
                dd[i, :len(r_)] = torch.from_numpy(s[i][keep][top])
                cnt[i] = len(r_)
        bound = torch.full((nq,), -1e30 if self.pessimist else float("inf"), dtype=torch.float64)
        return ids, dd, cnt, bound

    def plain(self, q, k, metric, row_filter, id_offset):
        rows = self.lo + np.flatnonzero(self.mask[self.lo:self.hi])
        res = O.enn_search(np.asarray(q), self.data[rows], k, row_ids=rows)
        return _padded(res, len(q), k)


def _worker_two_phase(rank, world, port, out):
    from paper_2605_15957_b200.distributed import TorchComm, two_phase_search
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(1)
    data = rng.standard_normal((2400, 16)).astype(np.float32)
    q = rng.standard_normal((9, 16)).astype(np.float32)
    mask = rng.random(2400) < 0.5
    lo, hi = row_shard(2400, rank, world)
    for pess in (False, True):
        shard = _OracleShard(data, mask, lo, hi, pessimist=pess)
        mi, md, mc = two_phase_search(shard, TorchComm(), torch.from_numpy(q), 20, "squared_l2",
                                      id_offset=lo, merge=_oracle_merge)
        if rank == 0:
            out[f"tp{int(pess)}"] = (mi.numpy(), md.numpy(), mc.numpy(), shard.reruns)
    dist.barrier()
    dist.destroy_process_group()


def test_world3_two_phase_protocol_matches_unsharded():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker_two_phase, args=(3, port, out), nprocs=3, join=True)
        res = dict(out)
    rng = np.random.default_rng(1)
    data = rng.standard_normal((2400, 16)).astype(np.float32)
    q = rng.standard_normal((9, 16)).astype(np.float32)
    mask = rng.random(2400) < 0.5
    ref = O.enn_filtered(q, data, mask, 20)
    for key, reruns in (("tp0", 0), ("tp1", 9)):
        ids, dd, cnt, rr = res[key]
        m = np.arange(20)[None, :] < cnt[:, None]
        assert np.array_equal(ids[m], ref.data_row)
        assert np.array_equal(dd[m], ref.distance)
        assert rr == reruns
