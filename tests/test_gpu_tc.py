"""The tcgen05 (tensor-core) phase A must produce the same exact results as
the reference: bf16 candidate scores + rigorous margin + float64 re-rank."""

import numpy as np
import pytest

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O
from paper_2605_15957_b200 import _native as N
from paper_2605_15957_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture
def tc_kernel():
    ctx = N.Context.get()
    ctx.set_option(N.OPT_ENN_KERNEL, 2)
    yield ctx
    ctx.set_option(N.OPT_ENN_KERNEL, 0)


def assert_same(nt, ref):
    assert np.array_equal(nt.query_row, ref.query_row)
    assert np.array_equal(nt.data_row, ref.data_row)
    assert np.array_equal(nt.distance, ref.distance)


@pytest.mark.parametrize("dim", [64, 100, 384])
@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
def test_tc_random_filtered(tc_kernel, dim, metric):
    rng = np.random.default_rng(dim + (metric == "inner_product"))
    data = rng.standard_normal((9000, dim)).astype(np.float32)
    q = rng.standard_normal((150, dim)).astype(np.float32)
    mask = rng.random(9000) < 0.3
    for k in (1, 16, 100):
        nt = vs.enn_search(q, data, vs.SearchParams(k=k), metric=metric, row_filter=mask)
        assert N.Context.get().stats()[N.STAT_LAST_ENN_KERNEL] == 2
        assert_same(nt, O.enn_filtered(q, data, mask, k, metric))


def test_tc_mixture_d1024(tc_kernel):
    x = synth.mixture_chunked(40000, 1024, seed=9, chunk=1 << 14)
    rng = np.random.default_rng(3)
    c = np.random.default_rng(np.random.SeedSequence([9, 10])).standard_normal((64, 1024))
    c /= np.linalg.norm(c, axis=1, keepdims=True)
    q = synth.mixture(rng, c, rng.integers(0, 64, 300), 0.165)
    mask = rng.random(40000) < 0.1
    nt = vs.enn_search(q, x, vs.SearchParams(k=100), row_filter=mask)
    idx = np.arange(0, 300, 23)
    ref = O.enn_filtered(q[idx], x, mask, 100)
    got_ids = nt.data_row.reshape(300, 100)[idx].reshape(-1)
    got_d = nt.distance.reshape(300, 100)[idx].reshape(-1)
    assert np.array_equal(got_ids, ref.data_row)
    assert np.array_equal(got_d, ref.distance)


def test_tc_goldens(tc_kernel, golden, sf001):
    g = golden("q15_enn.npz")
    nt = vs.enn_search(g["query"], sf001["reviews"], vs.SearchParams(k=int(g["k"])), row_filter=g["bitmap"])
    assert np.array_equal(nt.data_row, g["ids"]) and np.array_equal(nt.distance, g["dist"])
    for name in ("q11", "q2"):
        g = golden(f"{name}_enn.npz")
        nt = vs.enn_search(g["queries"], sf001["images"], vs.SearchParams(k=int(g["k"])),
                           metric=str(g["metric"]))
        assert np.array_equal(nt.data_row, g["ids"]) and np.array_equal(nt.distance, g["dist"])


def test_tc_random_goldens(tc_kernel, golden):
    g = golden("random_enn.npz")
    for t in range(12):
        seed, nq, nx, dim, k, ip = g[f"t{t}_spec"].tolist()
        if dim < 8:
            continue
        r = np.random.default_rng(seed)
        data = r.standard_normal((nx, dim)).astype(np.float32)
        queries = r.standard_normal((nq, dim)).astype(np.float32)
        nt = vs.enn_search(queries, data, vs.SearchParams(k=k), metric="inner_product" if ip else "squared_l2")
        assert np.array_equal(nt.data_row, g[f"t{t}_ids"]), t
        assert np.array_equal(nt.distance, g[f"t{t}_dist"]), t


def test_tc_duplicates_and_retry(tc_kernel):
    base = np.ones((5000, 64), np.float32)
    base[::3] = 0.5
    q = np.ones((130, 64), np.float32)
    nt = vs.enn_search(q, base, vs.SearchParams(k=40))
    assert_same(nt, O.enn_search(q, base, 40))


@pytest.mark.parametrize("kernel", [0, 1, 2])
@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("force_retry", [0, 1])
def test_large_host_query_batch_async_upload(kernel, pinned, force_retry):
    """A >= 4 MB host query batch is copied in on the copy stream while the
    filter and the row staging run; every phase-A kernel (and the re-run of
    forced-overflow queries, which needs the deferred SIMT margins) must give
    the reference result."""
    import torch
    rng = np.random.default_rng(70 + kernel)
    n, d, nq, k = 12000, 1024, 1100, 20
    data = rng.standard_normal((n, d)).astype(np.float32)
    q = rng.standard_normal((nq, d)).astype(np.float32)
    mask = rng.random(n) < 0.5
    qin = torch.from_numpy(q).pin_memory() if pinned else q
    ctx = N.Context.get()
    ctx.set_option(N.OPT_ENN_KERNEL, kernel)
    ctx.set_option(N.OPT_FORCE_RETRY, force_retry)
    try:
        nt = vs.enn_search(qin, data, vs.SearchParams(k=k), row_filter=mask)
    finally:
        ctx.set_option(N.OPT_ENN_KERNEL, 0)
        ctx.set_option(N.OPT_FORCE_RETRY, 0)
    idx = np.arange(0, nq, 37)
    ref = O.enn_filtered(q[idx], data, mask, k)
    assert np.array_equal(nt.data_row.reshape(nq, k)[idx].reshape(-1), ref.data_row)
    assert np.array_equal(nt.distance.reshape(nq, k)[idx].reshape(-1), ref.distance)


@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
def test_adversarial_cancellation(tc_kernel, metric):
    """Rows whose dot products with the query cancel massively inside the fp32
    accumulation (a +8 half and a -8 half: partial sums reach 8 d/2 before
    falling back to ~0) and differ only by small perturbations that are added
    while the accumulator is large. The tensor-core keys then carry their
    largest accumulation error; the margin (E_acc, vs_tc.cu k_tc_margins)
    must still keep every true neighbour, so ids and distances equal the
    oracle's."""
    rng = np.random.default_rng(99)
    d, n = 2048, 3000
    base = np.concatenate([np.full(d // 2, 8.0), np.full(d // 2, -8.0)]).astype(np.float32)
    data = np.tile(base, (n, 1))
    cols = rng.integers(0, d // 2, (n, 6))
    vals = (rng.integers(-64, 65, (n, 6)) * 2.0 ** -10).astype(np.float32)    # bf16-exact
    np.put_along_axis(data, cols, np.take_along_axis(data, cols, 1) + vals, 1)
    data[::7] = rng.standard_normal((len(data[::7]), d)).astype(np.float32)   # ordinary rows too
    q = np.concatenate([np.ones((4, d)), rng.standard_normal((4, d))]).astype(np.float32)
    q[:4, : d // 2] += (rng.integers(-4, 5, (4, d // 2)) * 2.0 ** -8)
    nt = vs.enn_search(q, data, vs.SearchParams(k=25), metric=metric)
    assert tc_kernel.stats()[N.STAT_LAST_ENN_KERNEL] == 2
    assert_same(nt, O.enn_search(q, data, 25, metric))


@pytest.mark.parametrize("scale", [1e-15, 1e-6, 3e4, 1e12])
@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
def test_tc_fp16_operand_scaling(tc_kernel, scale, metric):
    """float32 rows run as power-of-two-scaled fp16 operands: magnitudes far
    outside fp16's range (overflow above 65504, subnormals below 6e-5) must
    still give the reference's exact answer, and mixed query magnitudes each
    get their own scale."""
    rng = np.random.default_rng(int(np.log10(scale)) + 50)
    data = (rng.standard_normal((6000, 96)) * scale).astype(np.float32)
    q = (rng.standard_normal((140, 96)) * scale).astype(np.float32)
    q[::7] *= np.float32(1e3)
    q[3] = 0.0
    data[5] = 0.0
    mask = rng.random(6000) < 0.5
    nt = vs.enn_search(q, data, vs.SearchParams(k=12), metric=metric, row_filter=mask)
    assert N.Context.get().stats()[N.STAT_LAST_ENN_KERNEL] == 2
    assert_same(nt, O.enn_filtered(q, data, mask, 12, metric))


@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
@pytest.mark.parametrize("dups", [False, True])
def test_tc_sampled_admission_seed(tc_kernel, monkeypatch, metric, dups):
    """Phase A seeded with the k-th smallest chunk minimum of a row sample
    (VS_TC_TAU_SAMPLE): exact results, also when the sample holds the
    whole top-k (the seed is then the k-th key itself) and with duplicated
    rows (ties across the sample boundary)."""
    monkeypatch.setenv("VS_TC_TAU_SAMPLE", "1024")
    rng = np.random.default_rng(90 + dups)
    data = rng.standard_normal((30000, 64)).astype(np.float32)
    q = rng.standard_normal((200, 64)).astype(np.float32)
    if dups:
        data[15000:15400] = data[:400]          # copies of sample rows later in the column
        q[:50] = data[:50] + 1e-3 * rng.standard_normal((50, 64)).astype(np.float32)
    mask = rng.random(30000) < 0.6
    for k in (10, 32):
        nt = vs.enn_search(q, data, vs.SearchParams(k=k), metric=metric, row_filter=mask)
        assert_same(nt, O.enn_filtered(q, data, mask, k, metric))


def test_tc_f16_shadow_repeated_searches_and_mutation(tc_kernel):
    """The column's fp16 shadow (built on its second tensor-core search):
    repeated searches, a new filter, an in-place update seen by torch's
    version counter and one behind its back (invalidate()) all stay exact."""
    import torch
    rng = np.random.default_rng(23)
    data = rng.standard_normal((24000, 96)).astype(np.float32)
    t = torch.from_numpy(data).cuda()
    col = vs.EmbeddingColumn.from_device(t)
    q = rng.standard_normal((260, 96)).astype(np.float32)

    def check(mask):
        nt = vs.enn_search(q, col, vs.SearchParams(k=20), row_filter=mask)
        assert_same(nt, O.enn_filtered(q, t.cpu().numpy(), mask, 20))

    m1 = rng.random(24000) < 0.4
    for _ in range(3):
        check(m1)
    check(rng.random(24000) < 0.1)
    t[::5] *= -2.0
    check(m1)
    alias = torch.empty(0, device=t.device).set_(t.untyped_storage(), 0, t.shape, t.stride())
    alias[100:900] = 0.5
    col.invalidate()
    check(m1)
