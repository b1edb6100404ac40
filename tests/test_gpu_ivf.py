"""IVF search on the B200: identical probe lists, exact ids, bit-exact
distances versus the reference goldens and the oracle composition."""

import numpy as np
import pytest

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O
from paper_2605_15957_b200 import _native as N

pytestmark = pytest.mark.gpu


def _golden_index(g, name):
    seed0, n, dim, nlist, seed, ip = g[f"{name}_spec"].tolist()
    r = np.random.default_rng(seed0)
    data = r.standard_normal((n, dim)).astype(np.float32)
    queries = r.standard_normal((9, dim)).astype(np.float32)
    parts = np.split(g[f"{name}_ids"], np.cumsum(g[f"{name}_sizes"])[:-1])
    payload = [data[p] for p in parts]
    metric = "inner_product" if ip else "squared_l2"
    idx = vs.IvfIndex(nlist, dim, n, metric, "owning", g[f"{name}_centroids"], parts, payload)
    return idx, data, queries, nlist, metric


@pytest.mark.parametrize("name", ["a", "b"])
def test_ivf_matches_reference_goldens(golden, name):
    g = golden("ivf_small.npz")
    idx, data, queries, nlist, metric = _golden_index(g, name)
    for nprobe in (1, 4, nlist):
        nt = idx.search(queries, vs.SearchParams(k=7, k_prime=11, nprobe=nprobe))
        assert np.array_equal(nt.query_row, g[f"{name}_np{nprobe}_qrow"])
        assert np.array_equal(nt.data_row, g[f"{name}_np{nprobe}_ids"])
        assert np.array_equal(nt.distance, g[f"{name}_np{nprobe}_dist"])
        ref_probes = O.ivf_probes(queries, idx.centroids, nprobe)
        assert np.array_equal(nt.probes, ref_probes)


def test_owning_and_non_owning_identical(golden):
    g = golden("ivf_small.npz")
    idx, data, queries, nlist, metric = _golden_index(g, "a")
    non = idx.as_layout("non_owning", base=vs.EmbeddingColumn(data))
    for nprobe in (1, 3, 10):
        a = idx.search(queries, vs.SearchParams(k=4, nprobe=nprobe))
        b = non.search(queries, vs.SearchParams(k=4, nprobe=nprobe))
        assert np.array_equal(a.data_row, b.data_row) and np.array_equal(a.distance, b.distance)


@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
def test_filtered_ivf_vs_oracle(metric):
    rng = np.random.default_rng(11)
    data = rng.standard_normal((20000, 64)).astype(np.float32)
    queries = rng.standard_normal((50, 64)).astype(np.float32)
    centroids, parts, payload = O.ivf_build(data[:4000], 40, 0)
    # assign all rows to the nearest centroid (a valid IVF structure)
    assign = np.argmin(O.pairwise_sq_l2_fast(data, centroids), axis=1)
    parts = [np.flatnonzero(assign == c).astype(np.int64) for c in range(40)]
    payload = [data[p] for p in parts]
    idx = vs.IvfIndex(40, 64, 20000, metric, "owning", centroids, parts, payload)
    mask = rng.random(20000) < 0.05
    for nprobe in (1, 7, 40):
        nt = idx.search(queries, vs.SearchParams(k=10, nprobe=nprobe), row_filter=mask)
        ref = O.ivf_search(queries, centroids, parts, lambda c: payload[c], nprobe, 10, metric, mask=mask)
        assert np.array_equal(nt.probes, ref.probes)
        assert np.array_equal(nt.query_row, ref.query_row)
        assert np.array_equal(nt.data_row, ref.data_row)
        assert np.array_equal(nt.distance, ref.distance)
        assert nt.visited_rows == ref.visited_rows
    # full probe == filtered exhaustive search
    full = idx.search(queries, vs.SearchParams(k=10, nprobe=40), row_filter=mask)
    enn = vs.enn_search(queries, data, vs.SearchParams(k=10), metric=metric, row_filter=mask)
    assert np.array_equal(full.data_row, enn.data_row)
    assert np.array_equal(full.distance, enn.distance)


def test_list_sharding_plus_merge_equals_unsharded():
    from paper_2605_15957_b200 import _native as N
    from paper_2605_15957_b200.distributed import lpt_assign
    rng = np.random.default_rng(12)
    data = rng.standard_normal((8000, 32)).astype(np.float32)
    q = rng.standard_normal((25, 32)).astype(np.float32)
    centroids, parts, payload = O.ivf_build(data[:2000], 16, 1)
    assign = np.argmin(O.pairwise_sq_l2_fast(data, centroids), axis=1)
    parts = [np.flatnonzero(assign == c).astype(np.int64) for c in range(16)]
    payload = [data[p] for p in parts]
    idx = vs.IvfIndex(16, 32, 8000, "squared_l2", "owning", centroids, parts, payload)
    owner = lpt_assign([len(p) for p in parts], 3)
    ids_l, dist_l, cnt_l = [], [], []
    for r in range(3):
        ids, dist, cnt, probes, _ = idx.search_raw(q, 12, 5, list_owned=(owner == r).astype(np.uint8))
        ids_l.append(ids), dist_l.append(dist), cnt_l.append(cnt)
    ids = np.ascontiguousarray(np.stack(ids_l))
    dist = np.ascontiguousarray(np.stack(dist_l))
    cnt = np.ascontiguousarray(np.stack(cnt_l))
    oi, od, oc = np.empty((25, 12), np.int64), np.empty((25, 12)), np.empty(25, np.int32)
    ctx = N.Context.get()
    N.check(N.load().vs_topk_merge(ctx.handle, 3, 25, 12, N.ptr(ids), N.ptr(dist), N.ptr(cnt), 12, 0,
                                   N.ptr(oi), N.ptr(od), N.ptr(oc)))
    whole = idx.search(q, vs.SearchParams(k=12, nprobe=5))
    mask = np.arange(12)[None, :] < oc[:, None]
    assert np.array_equal(oi[mask], whole.data_row)
    assert np.array_equal(od[mask], whole.distance)


@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
@pytest.mark.parametrize("coarse", [1, 2])
def test_coarse_quantizer_modes_equal_oracle(metric, coarse):
    """The coarse quantizer with candidate buffers (VS_OPT_COARSE=1) and with
    dense tensor-core keys + per-query margin-band select (2): identical
    probes (the reference's select_top over float64 centroid distances)."""
    rng = np.random.default_rng(17 + coarse)
    n, d, nlist = 40000, 128, 2048
    data = rng.standard_normal((n, d)).astype(np.float32)
    cen = data[np.sort(rng.choice(n, nlist, replace=False))].copy()
    cen[7] = cen[3]                                     # tied centroids: the lower list id wins
    assign = np.argmin(O.pairwise_sq_l2_fast(data, cen), axis=1)
    parts = [np.flatnonzero(assign == c).astype(np.int64) for c in range(nlist)]
    payload = [data[p] for p in parts]
    q = rng.standard_normal((400, d)).astype(np.float32)
    ctx = N.Context.get()
    ctx.set_option(N.OPT_COARSE, coarse)
    try:
        idx = vs.IvfIndex(nlist, d, n, metric, "owning", cen, parts, payload)
        got = idx.search(q, vs.SearchParams(k=10, nprobe=40))
    finally:
        ctx.set_option(N.OPT_COARSE, 0)
    ref = O.ivf_search(q, cen, parts, lambda c: payload[c], 40, 10, metric)
    assert np.array_equal(got.probes, ref.probes)
    assert np.array_equal(got.data_row, ref.data_row)
    assert np.array_equal(got.distance, ref.distance)


@pytest.mark.parametrize("full_select", [False, True])
@pytest.mark.parametrize("dups", [0, 700])
def test_coarse_dense_select_variants(monkeypatch, full_select, dups):
    """Dense coarse keys: the chunk-minima select (k_coarse_select) and the
    whole-row select give the reference's probes; 700 identical centroids put
    more keys inside the margin than the chunk select holds (its whole-row
    fallback) and than the band buffer holds (overflow re-run)."""
    if full_select:
        monkeypatch.setenv("VS_COARSE_FULLSELECT", "1")
    rng = np.random.default_rng(5 + dups)
    n, d, nlist = 30000, 64, 3000
    data = rng.standard_normal((n, d)).astype(np.float32)
    cen = data[np.sort(rng.choice(n, nlist, replace=False))].copy()
    if dups:
        cen[100:100 + dups] = cen[99]
    assign = np.argmin(O.pairwise_sq_l2_fast(data, cen), axis=1)
    parts = [np.flatnonzero(assign == c).astype(np.int64) for c in range(nlist)]
    payload = [data[p] for p in parts]
    q = rng.standard_normal((300, d)).astype(np.float32)
    q[:20] = cen[99] + 1e-3 * rng.standard_normal((20, d)).astype(np.float32)
    ctx = N.Context.get()
    ctx.set_option(N.OPT_COARSE, 2)
    try:
        idx = vs.IvfIndex(nlist, d, n, "squared_l2", "owning", cen, parts, payload)
        got = idx.search(q, vs.SearchParams(k=5, nprobe=48))
    finally:
        ctx.set_option(N.OPT_COARSE, 0)
    ref = O.ivf_search(q, cen, parts, lambda c: payload[c], 48, 5)
    assert np.array_equal(got.probes, ref.probes)
    assert np.array_equal(got.data_row, ref.data_row)
    assert np.array_equal(got.distance, ref.distance)
