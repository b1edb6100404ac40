"""k' above the candidate-buffer top-k (vs_topk_cap() = 2048): the
device-wide select / exact re-rank / segmented sort of vs_wide.cu, and the
operator's placement contract (vecsearch.py:86-87): CapExceededError only for
device="device" with an explicit cap; otherwise every k' runs on the GPU.

Reference tests mirrored: tests/test_vs_operator.py:65-95 (cap on device,
host path uncapped, chunking invariance, index full probe == exact),
tests/test_enn.py (k = N, ties), and the reference's own Q15 'ivf' plan call
(k' = 500 k = 50,000, plans.py:256, 571) from the golden q15_ivf.npz."""

import numpy as np
import pytest
import torch

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O
from paper_2605_15957_b200 import _native as N
from paper_2605_15957_b200.errors import CapExceededError
from paper_2605_15957_b200.table import Schema, Table, embedding
from paper_2605_15957_b200.vecsearch import oversample_postfilter, vector_search_operator

pytestmark = pytest.mark.gpu


def _eq(got, ref):
    assert np.array_equal(got.query_row, ref.query_row)
    assert np.array_equal(got.data_row, ref.data_row)
    assert np.array_equal(got.distance, ref.distance)


@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
@pytest.mark.parametrize("d,k", [(64, 2049), (384, 5000), (3, 4096)])
def test_enn_large_k_equals_oracle(metric, d, k):
    rng = np.random.default_rng(d + k)
    n = 20000
    data = rng.standard_normal((n, d)).astype(np.float32)
    data[17] = data[3]                       # duplicates: ties broken by row id
    data[900:1200] = data[50]
    q = np.concatenate([rng.standard_normal((6, d)), data[[3, 50]]]).astype(np.float32)
    mask = rng.random(n) < 0.7
    got = vs.enn_search(q, data, vs.SearchParams(k=10, k_prime=k), metric=metric, row_filter=mask)
    assert N.Context.get().stats()[N.STAT_LAST_ENN_KERNEL] == 3
    _eq(got, O.enn_filtered(q, data, mask, k, metric))


def test_enn_k_at_least_n_returns_every_row_sorted():
    rng = np.random.default_rng(4)
    data = rng.standard_normal((3000, 32)).astype(np.float32)
    q = rng.standard_normal((3, 32)).astype(np.float32)
    mask = rng.random(3000) < 0.5
    got = vs.enn_search(q, data, vs.SearchParams(k=1, k_prime=50000), row_filter=mask)
    ref = O.enn_filtered(q, data, mask, 50000)
    assert len(got) == 3 * int(mask.sum())
    _eq(got, ref)


def test_enn_large_k_bf16_and_device_column():
    rng = np.random.default_rng(8)
    data = rng.standard_normal((12000, 128)).astype(np.float32)
    t = torch.from_numpy(data).cuda().to(torch.bfloat16)
    col = vs.EmbeddingColumn.from_device(t)
    q = rng.standard_normal((5, 128)).astype(np.float32)
    got = vs.enn_search(q, col, vs.SearchParams(k=3000))
    ref = O.enn_search(q, t.float().cpu().numpy(), 3000)
    _eq(got, ref)


def test_large_k_chunked_queries_match():
    """Many queries at large k: key-matrix query chunks and survivor sub-ranges."""
    rng = np.random.default_rng(12)
    data = rng.standard_normal((9000, 16)).astype(np.float32)
    q = rng.standard_normal((300, 16)).astype(np.float32)
    got = vs.enn_search(q, data, vs.SearchParams(k=2500))
    _eq(got, O.enn_search(q, data, 2500))


@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
def test_ivf_large_k_equals_oracle(metric):
    rng = np.random.default_rng(31)
    n, d, nlist = 30000, 32, 50
    data = rng.standard_normal((n, d)).astype(np.float32)
    cen, parts, payload = O.ivf_build(data, nlist, 0)
    q = rng.standard_normal((7, d)).astype(np.float32)
    mask = rng.random(n) < 0.6
    idx = vs.IvfIndex(nlist, d, n, metric, "owning", cen, parts, payload)
    got = idx.search(q, vs.SearchParams(k=5, k_prime=4000, nprobe=9), row_filter=mask)
    ref = O.ivf_search(q, cen, parts, lambda c: payload[c], 9, 4000, metric, mask=mask)
    assert np.array_equal(got.probes, ref.probes)
    _eq(got, ref)
    assert got.visited_rows == ref.visited_rows


def test_ivf_nprobe_above_cap():
    """nprobe > 2048: the coarse quantizer itself takes the wide path."""
    rng = np.random.default_rng(5)
    n, d, nlist = 40000, 8, 3000
    data = rng.standard_normal((n, d)).astype(np.float32)
    cen = data[np.sort(rng.choice(n, nlist, replace=False))].copy()
    assign = np.argmin(O.pairwise_sq_l2_fast(data, cen), axis=1)
    parts = [np.flatnonzero(assign == c).astype(np.int64) for c in range(nlist)]
    payload = [data[p] for p in parts]
    q = rng.standard_normal((4, d)).astype(np.float32)
    idx = vs.IvfIndex(nlist, d, n, "squared_l2", "owning", cen, parts, payload)
    got = idx.search(q, vs.SearchParams(k=20, nprobe=2500))
    ref = O.ivf_search(q, cen, parts, lambda c: payload[c], 2500, 20)
    assert np.array_equal(got.probes, ref.probes)
    _eq(got, ref)


def test_merge_large_k():
    from paper_2605_15957_b200.distributed import gpu_merge
    rng = np.random.default_rng(2)
    G, Q, k_in, k = 3, 4, 3000, 5000
    ids = np.stack([np.sort(rng.choice(10**6, (Q, k_in), replace=True), axis=1) for _ in range(G)])
    dist = np.sort(rng.integers(0, 500, (G, Q, k_in)).astype(np.float64), axis=2)   # many ties
    cnt = rng.integers(1000, k_in + 1, (G, Q)).astype(np.int32)
    oi, od, oc = gpu_merge(*(torch.from_numpy(a).cuda() for a in (ids, dist, cnt)), k, "squared_l2")
    for q in range(Q):
        parts = [(ids[g, q, :cnt[g, q]], dist[g, q, :cnt[g, q]]) for g in range(G)]
        ri, rd = O.merge_topk(parts, k, "squared_l2")
        c = int(oc[q])
        assert c == len(ri)
        assert np.array_equal(oi[q, :c].cpu().numpy(), ri)
        assert np.array_equal(od[q, :c].cpu().numpy(), rd)


# ---- the operator (vecsearch.py:64-120) ---------------------------------------------------------


@pytest.fixture
def sides():
    """tests/test_vs_operator.py's fixture shape: 3 queries, 120 data rows."""
    rng = np.random.default_rng(0)
    d = 8
    data = rng.standard_normal((120, d)).astype(np.float32)
    qv = rng.standard_normal((3, d)).astype(np.float32)
    dt = Table(Schema([("id", "int64"), ("e", embedding(d))]), {"id": np.arange(120), "e": data})
    qt = Table(Schema([("qid", "int64"), ("e", embedding(d))]), {"qid": np.arange(3), "e": qv})
    return qt, dt


def test_topk_cap_on_device_only(sides):
    qt, dt = sides
    with pytest.raises(CapExceededError):
        vector_search_operator(qt, "e", dt, "e", vs.SearchParams(k=10, k_prime=5000),
                               device="device", gpu_topk_cap=2048)
    out, _ = vector_search_operator(qt, "e", dt, "e", vs.SearchParams(k=10, k_prime=5000),
                                    device="host", gpu_topk_cap=2048)
    assert out.row_count == 3 * 120
    out2, _ = vector_search_operator(qt, "e", dt, "e", vs.SearchParams(k=10, k_prime=5000), device="device")
    assert out2.row_count == 3 * 120
    ref = O.enn_search(qt.column("e").values, dt.column("e").values, 5000)
    assert np.array_equal(np.asarray(out.column("vs_data_row")), ref.data_row)
    assert np.array_equal(np.asarray(out.column("vs_distance")), ref.distance)


@pytest.mark.parametrize("kp", [7, 3000])
def test_chunking_invariance(sides, kp):
    qt, dt = sides
    full, _ = vector_search_operator(qt, "e", dt, "e", vs.SearchParams(k=7, k_prime=kp))
    chunked, _ = vector_search_operator(qt, "e", dt, "e", vs.SearchParams(k=7, k_prime=kp), chunk_queries=1)
    for c in ("vs_query_row", "vs_data_row", "vs_distance", "vs_rank", "id", "qid"):
        assert np.array_equal(np.asarray(full.column(c)), np.asarray(chunked.column(c)))


def test_with_index_full_probe_equals_exact(sides):
    qt, dt = sides
    idx = vs.IvfIndex.build(dt.column("e"), nlist=6, seed=0)
    out, stats = vector_search_operator(qt, "e", dt, "e", vs.SearchParams(k=3, nprobe=6), index=idx)
    exact, _ = vector_search_operator(qt, "e", dt, "e", vs.SearchParams(k=3))
    assert np.array_equal(np.asarray(out.column("vs_data_row")), np.asarray(exact.column("vs_data_row")))
    assert np.array_equal(np.asarray(out.column("vs_distance")), np.asarray(exact.column("vs_distance")))
    assert stats.index_kind == "ivf"


def test_flat_index(sides):
    qt, dt = sides
    fi = vs.FlatIndex.build(dt.column("e"), metric="inner_product")
    assert fi.layout == "non_owning" and fi.structure_nbytes() == 0 and fi.count == 120
    got = fi.search(qt.column("e"), vs.SearchParams(k=9))
    _eq(got, O.enn_search(qt.column("e").values, dt.column("e").values, 9, "inner_product"))
    mask = np.arange(120) % 3 == 0
    got = fi.search(qt.column("e"), vs.SearchParams(k=9), row_filter=mask)
    _eq(got, O.enn_filtered(qt.column("e").values, dt.column("e").values, mask, 9, "inner_product"))


def test_device_resident_data_side_operator():
    """A data table whose embedding column lives on the GPU: the result is
    flattened on the device and the output embedding column is gathered
    there (no host copy of the collection)."""
    rng = np.random.default_rng(21)
    d = 16
    data = rng.standard_normal((5000, d)).astype(np.float32)
    t = torch.from_numpy(data).cuda()
    dt = Table(Schema([("id", "int64"), ("e", embedding(d))]),
               {"id": np.arange(5000), "e": vs.EmbeddingColumn.from_device(t)})
    qv = rng.standard_normal((4, d)).astype(np.float32)
    qt = Table(Schema([("qid", "int64"), ("q", embedding(d))]), {"qid": np.arange(4), "q": qv})
    out, stats = vector_search_operator(qt, "q", dt, "e", vs.SearchParams(k=5, k_prime=2600))
    ref = O.enn_search(qv, data, 2600)
    assert np.array_equal(np.asarray(out.column("vs_data_row")), ref.data_row)
    assert np.array_equal(np.asarray(out.column("vs_distance")), ref.distance)
    assert np.array_equal(np.asarray(out.column("id")), ref.data_row)
    emb = out.column("e")
    assert emb._dev_tensor is not None                        # stayed on the device
    assert np.array_equal(emb.values, data[ref.data_row])
    assert stats.visited_rows == 4 * 5000


def test_q15_ivf_plan_vector_search_bit_exact(golden, sf001):
    """The reference's Q15 'ivf' plan call (plans.py:571-574, executor.py:222):
    k' = 50,000 over the reference's SF=0.01 IVF index, then the semi-join
    post-filter (vecsearch.py:155-202) — identical to the reference's output."""
    g = golden("q15_ivf.npz")
    parts = np.split(g["ids"], np.cumsum(g["sizes"])[:-1])
    reviews = sf001["reviews"]
    nlist, d = g["centroids"].shape
    idx = vs.IvfIndex(int(nlist), int(d), reviews.shape[0], "squared_l2", "non_owning", g["centroids"], parts,
                      None, base=vs.EmbeddingColumn(reviews))
    pk = sf001["review_partkeys"]
    dt = Table(Schema([("rv_partkey", "int64"), ("rv_embedding", embedding(int(d)))]),
               {"rv_partkey": pk, "rv_embedding": reviews})
    qt = Table(Schema([("qv_review", embedding(int(d)))]), {"qv_review": g["queries"]})
    params = vs.SearchParams(k=int(g["k"]), k_prime=int(g["k_prime"]), nprobe=int(g["nprobe"]))
    out, stats = vector_search_operator(qt, "qv_review", dt, "rv_embedding", params, index=idx)
    for c in ("vs_query_row", "vs_data_row", "vs_distance", "vs_rank"):
        assert np.array_equal(np.asarray(out.column(c)), g[c]), c
    assert stats.visited_rows == int(g["visited"])
    keep_set = Table(Schema([("ps_partkey", "int64")]), {"ps_partkey": g["keep_set"]})
    kept, short = oversample_postfilter(out, None, int(g["pf_k"]), keep_set=keep_set,
                                        semi_keys=(str(g["semi_left"]), "ps_partkey"))
    assert np.array_equal(np.asarray(kept.column("vs_data_row")), g["pf_data_row"])
    assert np.array_equal(np.asarray(kept.column("vs_distance")), g["pf_distance"])
    assert short.get(0, 0) == int(g["pf_short"][0])
