"""Parity at the BASELINE scales, part C: config 5 variant B (BASELINE.json
configs[4]) — one 12.5M x 768 float32 row shard (1/8 of 100M) in pinned host
memory, only the filter-selected rows streamed over PCIe in chunks, 10%
Bernoulli bitmap, top-100, 10k queries; sampled queries vs the oracle over the
host copy of the selected rows (vecindex.py:109-132 + the filtered
composition of SURVEY §8c)."""

import numpy as np
import pytest
import torch

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O
from paper_2605_15957_b200 import _native as N
from paper_2605_15957_b200 import synth
from paper_2605_15957_b200.vecindex import enn_search_raw
from test_gpu_scale_a import assert_rows_equal, sample_rows

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_config5b_host_resident_shard_sampled_queries_equal_oracle():
    n_all, shards, d, nq, k = 100_000_000, 8, 768, 10_000, 100
    n = n_all // shards
    dev = torch.device("cuda", 0)
    host = torch.empty((n, d), dtype=torch.float32).pin_memory()
    chunk = 1 << 20
    centers = None
    for a in range(0, n, chunk):                      # shard 0 of the global collection
        b = min(n, a + chunk)
        part, centers = synth.device_rows(n_all, d, a, b, dev)
        host[a:b].copy_(part)
        del part
    mask = synth.device_bernoulli(n_all, 0.10, 4242, dev)[:n].contiguous()
    bits = synth.pack_bits_torch(mask)
    queries = synth.device_queries(centers, nq, seed=7)
    torch.cuda.synchronize()
    ctx = N.Context(0)
    col = vs.EmbeddingColumn.host_resident(host)
    out = (torch.empty((nq, k), dtype=torch.int64, device=dev),
           torch.empty((nq, k), dtype=torch.float64, device=dev),
           torch.empty((nq,), dtype=torch.int32, device=dev))
    enn_search_raw(queries, col, k, "squared_l2", row_filter=bits, device=ctx, out=out)
    torch.cuda.synchronize()
    ids, dist, cnt = (t.cpu().numpy() for t in out)
    assert (cnt == k).all()
    qidx = sample_rows(nq, 8)
    rows = np.flatnonzero(mask.cpu().numpy())
    xs = host.numpy()[rows]
    q = queries[torch.from_numpy(qidx).to(dev)].cpu().numpy()
    ref = O.enn_pruned(q, xs, k, "squared_l2", row_ids=rows)
    assert_rows_equal(ids, dist, cnt, ref, qidx)
    del col
    ctx.close()
