"""Single-process device groups (vs_group_*, group.DeviceGroup; SURVEY §5,
§8b, §8e): a group over [0, 0] (two members on the one GPU of the pool: the
peer-copy exchange) and over [0] (a one-rank NCCL clique: ncclCommInitAll,
ncclGroupStart/End, ncclAllGather) must return exactly the one-GPU search,
which equals the oracle. use_devices() makes the group the default placement
of the drop-in API (vector_search_operator unchanged)."""

import numpy as np
import pytest

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O
from paper_2605_15957_b200.table import Schema, Table, embedding
from paper_2605_15957_b200.vecsearch import vector_search_operator

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[[0, 0], [0], [0, 0, 0]], ids=["peer2", "nccl1", "peer3"])
def group(request):
    g = vs.DeviceGroup(request.param)
    assert g.uses_nccl == (len(request.param) == 1)
    return g


def _eq(a, b):
    assert np.array_equal(a.query_row, b.query_row)
    assert np.array_equal(a.data_row, b.data_row)
    assert np.array_equal(a.distance, b.distance)


@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
@pytest.mark.parametrize("k", [10, 300, 2600])
def test_group_enn_equals_one_gpu(group, metric, k):
    rng = np.random.default_rng(k)
    n, d = 25_003, 96
    data = rng.standard_normal((n, d)).astype(np.float32)
    q = rng.standard_normal((300, d)).astype(np.float32)      # tensor-core phase A per member
    mask = rng.random(n) < 0.4
    col = vs.EmbeddingColumn(data)
    got = vs.enn_search(q, col, vs.SearchParams(k=k), metric=metric, row_filter=mask, device=group)
    one = vs.enn_search(q, col, vs.SearchParams(k=k), metric=metric, row_filter=mask)
    _eq(got, one)
    assert got.visited_rows == one.visited_rows
    if k == 10:
        _eq(got, O.enn_filtered(q, data, mask, k, metric))


def test_group_enn_empty_shards(group):
    rng = np.random.default_rng(1)
    data = rng.standard_normal((4000, 16)).astype(np.float32)
    q = rng.standard_normal((5, 16)).astype(np.float32)
    mask = np.zeros(4000, bool)
    mask[-3:] = True                                             # only the last shard selects rows
    got = vs.enn_search(q, data, vs.SearchParams(k=8), row_filter=mask, device=group)
    _eq(got, O.enn_filtered(q, data, mask, 8))
    with pytest.raises(vs.EmptyInputError):
        vs.enn_search(q, data, vs.SearchParams(k=8), row_filter=np.zeros(4000, bool), device=group)


@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
def test_group_ivf_equals_one_gpu(group, metric):
    rng = np.random.default_rng(7)
    n, d, nlist = 30_000, 32, 48
    data = rng.standard_normal((n, d)).astype(np.float32)
    cen, parts, payload = O.ivf_build(data, nlist, 0)
    idx = vs.IvfIndex(nlist, d, n, metric, "owning", cen, parts, payload)
    q = rng.standard_normal((77, d)).astype(np.float32)
    mask = rng.random(n) < 0.5
    got = idx.search(q, vs.SearchParams(k=15, nprobe=6), row_filter=mask, device=group)
    ref = O.ivf_search(q, cen, parts, lambda c: payload[c], 6, 15, metric, mask=mask)
    _eq(got, ref)
    assert got.visited_rows == ref.visited_rows


def test_use_devices_makes_the_operator_span_the_group():
    rng = np.random.default_rng(3)
    d = 24
    data = rng.standard_normal((9000, d)).astype(np.float32)
    qv = rng.standard_normal((6, d)).astype(np.float32)
    dt = Table(Schema([("id", "int64"), ("e", embedding(d))]), {"id": np.arange(9000), "e": data})
    qt = Table(Schema([("q", embedding(d))]), {"q": qv})
    try:
        g = vs.use_devices([0, 0])
        out, stats = vector_search_operator(qt, "q", dt, "e", vs.SearchParams(k=5, k_prime=40))
        assert len(g._cols) == 1                                 # the data column was sharded on the group
    finally:
        vs.use_devices(None)
    ref = O.enn_search(qv, data, 40)
    assert np.array_equal(np.asarray(out.column("vs_data_row")), ref.data_row)
    assert np.array_equal(np.asarray(out.column("vs_distance")), ref.distance)
    assert stats.visited_rows == 6 * 9000
