"""Host-resident columns (config 5 B): only filter-selected rows cross PCIe,
in chunks merged with the cross-shard merge kernel. Results must be identical
to the device-resident search and to the oracle (enn_search over the gathered
rows, vecindex.py:109-132 + the filtered composition of SURVEY §8c)."""

import numpy as np
import pytest
import torch

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O
from paper_2605_15957_b200 import _native as N
from paper_2605_15957_b200.vecindex import enn_search_raw

pytestmark = pytest.mark.gpu


def _chunked(rows):
    ctx = N.Context.get()
    ctx.set_option(N.OPT_STREAM_CHUNK, rows)
    return ctx


@pytest.mark.parametrize("chunk", [0, 997, 4096])
@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
def test_host_resident_equals_device_and_oracle(chunk, metric):
    rng = np.random.default_rng(3 + chunk)
    n, d = 20000, 128
    data = rng.standard_normal((n, d)).astype(np.float32)
    q = rng.standard_normal((37, d)).astype(np.float32)
    mask = rng.random(n) < 0.3
    pinned = torch.from_numpy(data).pin_memory()
    host_col = vs.EmbeddingColumn.host_resident(pinned)
    ctx = _chunked(chunk)
    try:
        got = vs.enn_search(q, host_col, vs.SearchParams(k=25), metric=metric, row_filter=mask)
    finally:
        ctx.set_option(N.OPT_STREAM_CHUNK, 0)
    dev = vs.enn_search(q, data, vs.SearchParams(k=25), metric=metric, row_filter=mask)
    ref = O.enn_filtered(q, data, mask, 25, metric)
    for nt in (dev, ref):
        assert np.array_equal(got.query_row, nt.query_row)
        assert np.array_equal(got.data_row, nt.data_row)
        assert np.array_equal(got.distance, nt.distance)


def test_host_resident_unpinned_numpy_is_registered():
    rng = np.random.default_rng(8)
    data = rng.standard_normal((5000, 64)).astype(np.float32)
    q = rng.standard_normal((9, 64)).astype(np.float32)
    col = vs.EmbeddingColumn.host_resident(data)       # plain pageable numpy: cudaHostRegister
    got = vs.enn_search(q, col, vs.SearchParams(k=7))
    ref = O.enn_search(q, data, 7)
    assert np.array_equal(got.data_row, ref.data_row)
    assert np.array_equal(got.distance, ref.distance)


def test_host_resident_bf16_and_id_offset():
    rng = np.random.default_rng(12)
    n, d = 9000, 96
    x = torch.from_numpy(rng.standard_normal((n, d)).astype(np.float32)).to(torch.bfloat16)
    q = rng.standard_normal((21, d)).astype(np.float32)
    mask = rng.random(n) < 0.5
    host_col = vs.EmbeddingColumn.host_resident(x.pin_memory())
    ctx = _chunked(1500)
    try:
        ids, dist, cnt, _ = enn_search_raw(q, host_col, 12, row_filter=mask, id_offset=1000)
    finally:
        ctx.set_option(N.OPT_STREAM_CHUNK, 0)
    ref = O.enn_filtered(q, x.float().numpy(), mask, 12)
    m = np.arange(12)[None, :] < cnt[:, None]
    assert np.array_equal(ids[m], ref.data_row + 1000)
    assert np.array_equal(dist[m], ref.distance)
