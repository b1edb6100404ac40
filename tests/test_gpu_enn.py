"""Exhaustive (ENN) search on the B200 against the CPU oracle and the
reference's golden vectors: ids exact, distances bit-exact (the library
reproduces the reference's float64 arithmetic and summation order)."""

import numpy as np
import pytest

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O
from paper_2605_15957_b200 import _native as N
from paper_2605_15957_b200 import synth

pytestmark = pytest.mark.gpu


def assert_same(nt, ref):
    assert np.array_equal(nt.query_row, ref.query_row)
    assert np.array_equal(nt.data_row, ref.data_row)
    assert np.array_equal(nt.distance, ref.distance)
    assert np.array_equal(nt.rank, ref.rank)


def test_random_instances_match_reference_goldens(golden):
    g = golden("random_enn.npz")
    for t in range(12):
        seed, nq, nx, dim, k, ip = g[f"t{t}_spec"].tolist()
        r = np.random.default_rng(seed)
        data = r.standard_normal((nx, dim)).astype(np.float32)
        queries = r.standard_normal((nq, dim)).astype(np.float32)
        nt = vs.enn_search(queries, data, vs.SearchParams(k=k),
                           metric="inner_product" if ip else "squared_l2")
        assert np.array_equal(nt.query_row, g[f"t{t}_qrow"]), t
        assert np.array_equal(nt.data_row, g[f"t{t}_ids"]), t
        assert np.array_equal(nt.distance, g[f"t{t}_dist"]), t


def test_tie_rule_duplicates():
    base = np.zeros((6, 4), np.float32)
    base[3] = 1.0
    base[5] = 1.0
    nt = vs.enn_search(np.zeros((1, 4), np.float32), base, vs.SearchParams(k=6))
    assert nt.data_row.tolist() == [0, 1, 2, 4, 3, 5]


def test_many_exact_duplicates_force_buffer_growth():
    # 3000 identical rows: every candidate ties; lowest row ids must win
    base = np.ones((3000, 8), np.float32)
    base[::7] = 2.0
    q = np.ones((3, 8), np.float32)
    nt = vs.enn_search(q, base, vs.SearchParams(k=50))
    ref = O.enn_search(q, base, 50)
    assert_same(nt, ref)


def test_self_match_and_k_equals_count():
    rng = np.random.default_rng(0)
    data = rng.standard_normal((50, 8)).astype(np.float32)
    nt = vs.enn_search(data[7:8], data, vs.SearchParams(k=1))
    assert nt.data_row[0] == 7 and nt.distance[0] == 0.0
    data = rng.standard_normal((12, 4)).astype(np.float32)
    q = rng.standard_normal((1, 4)).astype(np.float32)
    nt = vs.enn_search(q, data, vs.SearchParams(k=12))
    assert len(nt) == 12 and list(nt.rank) == list(range(12))
    nt = vs.enn_search(q, data, vs.SearchParams(k=4, k_prime=50))
    assert nt.per_query_counts().tolist() == [12]


@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
@pytest.mark.parametrize("dim", [3, 16, 61, 64, 100, 384])
def test_filtered_matches_composition(metric, dim):
    rng = np.random.default_rng(dim)
    data = rng.standard_normal((5000, dim)).astype(np.float32)
    queries = rng.standard_normal((37, dim)).astype(np.float32)
    mask = rng.random(5000) < 0.13
    for k in (1, 10, 100):
        nt = vs.enn_search(queries, data, vs.SearchParams(k=k), metric=metric, row_filter=mask)
        assert_same(nt, O.enn_filtered(queries, data, mask, k, metric))


def test_filter_forms_equivalent():
    rng = np.random.default_rng(1)
    data = rng.standard_normal((777, 32)).astype(np.float32)
    q = rng.standard_normal((5, 32)).astype(np.float32)
    mask = rng.random(777) < 0.4
    a = vs.enn_search(q, data, vs.SearchParams(k=9), row_filter=mask)
    b = vs.enn_search(q, data, vs.SearchParams(k=9), row_filter=synth.pack_mask(mask))
    c = vs.enn_search(q, data, vs.SearchParams(k=9), row_filter=np.flatnonzero(mask))
    for x in (b, c):
        assert np.array_equal(a.data_row, x.data_row) and np.array_equal(a.distance, x.distance)


def test_q15_prefiltered_golden(golden, sf001):
    g = golden("q15_enn.npz")
    mask = synth.unpack_bitmap(g["bitmap"], int(g["n"]))
    nt = vs.enn_search(g["query"], sf001["reviews"], vs.SearchParams(k=int(g["k"])),
                       row_filter=g["bitmap"])
    assert np.array_equal(nt.data_row, g["ids"])
    assert np.array_equal(nt.distance, g["dist"])
    assert nt.visited_rows == int(mask.sum())


@pytest.mark.parametrize("name", ["q11", "q2", "q18"])
def test_batched_and_large_k_goldens(golden, sf001, name):
    g = golden(f"{name}_enn.npz")
    data = sf001["images"] if str(g["data"]) == "im_embedding" else sf001["reviews"]
    nt = vs.enn_search(g["queries"], data, vs.SearchParams(k=int(g["k"])), metric=str(g["metric"]))
    assert np.array_equal(nt.query_row, g["query_row"])
    assert np.array_equal(nt.data_row, g["ids"])
    assert np.array_equal(nt.distance, g["dist"])


def test_config1_sample_golden(golden):
    g = golden("config1_sample.npz")
    emb, mask, q = synth.config1()
    nt = vs.enn_search(q[g["queries_idx"]], emb, vs.SearchParams(k=10), row_filter=mask)
    assert np.array_equal(nt.data_row.reshape(-1, 10), g["ids"])
    assert np.array_equal(nt.distance.reshape(-1, 10), g["dist"])


def test_config1_full_batch_vs_oracle_sample():
    emb, mask, q = synth.config1()
    nt = vs.enn_search(q, emb, vs.SearchParams(k=10), row_filter=mask)
    assert nt.per_query_counts().tolist() == [10] * 1000
    idx = np.arange(3, 1000, 97)
    ref = O.enn_filtered(q[idx], emb, mask, 10)
    ids = nt.data_row.reshape(1000, 10)[idx]
    dist = nt.distance.reshape(1000, 10)[idx]
    assert np.array_equal(ids, ref.data_row.reshape(-1, 10))
    assert np.array_equal(dist, ref.distance.reshape(-1, 10))


def test_errors():
    data = np.zeros((3, 4), np.float32)
    with pytest.raises(vs.ShapeError):
        vs.enn_search(np.zeros((1, 5), np.float32), data, vs.SearchParams(k=1))
    with pytest.raises(vs.EmptyInputError):
        vs.enn_search(np.zeros((1, 4), np.float32), np.zeros((0, 4), np.float32), vs.SearchParams(k=1))
    with pytest.raises(vs.EmptyInputError):
        vs.enn_search(np.zeros((1, 4), np.float32), data, vs.SearchParams(k=1),
                      row_filter=np.zeros(3, bool))
    # k' above vs_topk_cap() is not an error of the search (vecindex.py:109-132
    # has no cap): every row comes back; the cap is the operator's contract
    nt = vs.enn_search(np.zeros((1, 4), np.float32), data, vs.SearchParams(k=1, k_prime=5000))
    assert len(nt) == 3 and nt.data_row.tolist() == [0, 1, 2]


def test_visited_rows():
    rng = np.random.default_rng(3)
    data = rng.standard_normal((40, 4)).astype(np.float32)
    q = rng.standard_normal((3, 4)).astype(np.float32)
    assert vs.enn_search(q, data, vs.SearchParams(k=2)).visited_rows == 120


def test_forced_retry_path_is_identical():
    rng = np.random.default_rng(4)
    data = rng.standard_normal((20000, 48)).astype(np.float32)
    q = rng.standard_normal((300, 48)).astype(np.float32)
    mask = rng.random(20000) < 0.5
    a = vs.enn_search(q, data, vs.SearchParams(k=20), row_filter=mask)
    ctx = N.Context.get()
    ctx.set_option(N.OPT_FORCE_RETRY, 1)
    try:
        b = vs.enn_search(q, data, vs.SearchParams(k=20), row_filter=mask)
    finally:
        ctx.set_option(N.OPT_FORCE_RETRY, 0)
    assert_same(a, b)


def test_torch_device_inputs_and_bf16_storage():
    import torch
    rng = np.random.default_rng(5)
    data = rng.standard_normal((4000, 128)).astype(np.float32)
    q = rng.standard_normal((64, 128)).astype(np.float32)
    dt = torch.from_numpy(data).cuda()
    col = vs.EmbeddingColumn.from_device(dt)
    nt = vs.enn_search(torch.from_numpy(q).cuda(), col, vs.SearchParams(k=16))
    assert_same(nt, O.enn_search(q, data, 16))
    # bf16 storage: oracle fed the bf16-rounded values upcast to f32
    bcol = vs.EmbeddingColumn.from_device(dt.to(torch.bfloat16))
    data_b = dt.to(torch.bfloat16).float().cpu().numpy()
    nt = vs.enn_search(q, bcol, vs.SearchParams(k=16))
    assert_same(nt, O.enn_search(q, data_b, 16))


def test_merge_kernel_matches_oracle_merge():
    rng = np.random.default_rng(6)
    data = rng.standard_normal((6000, 24)).astype(np.float32)
    q = rng.standard_normal((40, 24)).astype(np.float32)
    parts = []
    ids_l, dist_l, cnt_l = [], [], []
    for lo, hi in ((0, 1000), (1000, 3500), (3500, 6000)):
        ids, dist, cnt, _ = vs.vecindex.enn_search_raw(q, data[lo:hi], 30, id_offset=lo)
        ids_l.append(ids), dist_l.append(dist), cnt_l.append(cnt)
    ids = np.ascontiguousarray(np.stack(ids_l))
    dist = np.ascontiguousarray(np.stack(dist_l))
    cnt = np.ascontiguousarray(np.stack(cnt_l))
    oi, od, oc = np.empty((40, 30), np.int64), np.empty((40, 30)), np.empty(40, np.int32)
    ctx = N.Context.get()
    N.check(N.load().vs_topk_merge(ctx.handle, 3, 40, 30, N.ptr(ids), N.ptr(dist), N.ptr(cnt), 30, 0,
                                   N.ptr(oi), N.ptr(od), N.ptr(oc)))
    ref = O.enn_search(q, data, 30)
    assert np.array_equal(oi.reshape(-1), ref.data_row)
    assert np.array_equal(od.reshape(-1), ref.distance)


@pytest.mark.parametrize("dim", [8, 127, 128, 129, 1000, 1152, 2048, 2100])
def test_exact_scores_across_dims(dim):
    # every summation-tree shape of the warp-cooperative float64 scorer
    rng = np.random.default_rng(dim)
    data = rng.standard_normal((700, dim)).astype(np.float32)
    q = rng.standard_normal((9, dim)).astype(np.float32)
    for metric in ("squared_l2", "inner_product"):
        nt = vs.enn_search(q, data, vs.SearchParams(k=25), metric=metric)
        assert_same(nt, O.enn_search(q, data, 25, metric))


def test_borrowed_column_mutation_invalidates_norms():
    """A from_device column modified in place between searches: the cached row
    norms must not survive (torch's version counter, or invalidate())."""
    import torch
    rng = np.random.default_rng(12)
    data = rng.standard_normal((20000, 64)).astype(np.float32)
    t = torch.from_numpy(data).cuda()
    col = vs.EmbeddingColumn.from_device(t)
    q = rng.standard_normal((300, 64)).astype(np.float32)
    vs.enn_search(q, col, vs.SearchParams(k=10))                 # norms cached
    t[::3] *= 3.0                                                # in place: _version bumps
    got = vs.enn_search(q, col, vs.SearchParams(k=10))
    ref = O.enn_search(q, t.cpu().numpy(), 10)
    assert np.array_equal(got.data_row, ref.data_row)
    assert np.array_equal(got.distance, ref.distance)
    # a write torch's version counter does not see: through a second view
    # object's storage (untracked), then the explicit invalidate()
    alias = torch.empty(0, device=t.device).set_(t.untyped_storage(), 0, t.shape, t.stride())
    alias[:500] = 0.0
    col.invalidate()
    got = vs.enn_search(q, col, vs.SearchParams(k=10))
    ref = O.enn_search(q, t.cpu().numpy(), 10)
    assert np.array_equal(got.data_row, ref.data_row)
    assert np.array_equal(got.distance, ref.distance)


@pytest.mark.parametrize("kernel", [1, 2])
def test_pinned_host_outputs_written_in_place(kernel):
    """Page-locked host output buffers are written by the kernels over PCIe
    (zero-copy final outputs): same results as the oracle, with tensor-core
    and SIMT phase A (their verification re-runs scatter into the same
    buffers)."""
    import torch
    from paper_2605_15957_b200.vecindex import enn_search_raw
    rng = np.random.default_rng(41 + kernel)
    data = rng.standard_normal((20000, 96)).astype(np.float32)
    q = rng.standard_normal((300, 96)).astype(np.float32)
    mask = rng.random(20000) < 0.2
    k = 24
    out = (torch.full((300, k), 7, dtype=torch.int64).pin_memory(),
           torch.zeros((300, k), dtype=torch.float64).pin_memory(),
           torch.zeros(300, dtype=torch.int32).pin_memory())
    ctx = N.Context.get()
    ctx.set_option(N.OPT_ENN_KERNEL, kernel)
    try:
        enn_search_raw(torch.from_numpy(q).pin_memory(), data, k, row_filter=mask, out=out)
    finally:
        ctx.set_option(N.OPT_ENN_KERNEL, 0)
    ref = O.enn_filtered(q, data, mask, k)
    assert np.array_equal(out[2].numpy(), np.full(300, k, np.int32))
    assert np.array_equal(out[0].numpy().reshape(-1), ref.data_row)
    assert np.array_equal(out[1].numpy().reshape(-1), ref.distance)


@pytest.mark.gpu
def test_large_pinned_host_outputs_staged(monkeypatch):
    """Page-locked output buffers above the zero-copy limit (VS_ZERO_COPY_MAX,
    here 2 MiB) are staged in device memory and copied back once: same results
    as the oracle."""
    import torch
    monkeypatch.setenv("VS_ZERO_COPY_MAX", str(2 << 20))
    from paper_2605_15957_b200.vecindex import enn_search_raw
    rng = np.random.default_rng(52)
    data = rng.standard_normal((20000, 32)).astype(np.float32)
    q = rng.standard_normal((3000, 32)).astype(np.float32)
    mask = rng.random(20000) < 0.3
    k = 100                                           # 3000 x 100 x 8 B = 2.4 MB per buffer
    out = (torch.full((3000, k), 7, dtype=torch.int64).pin_memory(),
           torch.zeros((3000, k), dtype=torch.float64).pin_memory(),
           torch.zeros(3000, dtype=torch.int32).pin_memory())
    enn_search_raw(torch.from_numpy(q).pin_memory(), data, k, row_filter=mask, out=out)
    ref = O.enn_filtered(q, data, mask, k)
    assert np.array_equal(out[2].numpy(), np.full(3000, k, np.int32))
    assert np.array_equal(out[0].numpy().reshape(-1), ref.data_row)
    assert np.array_equal(out[1].numpy().reshape(-1), ref.distance)
