"""Both IVF list-scan kernels (query-major and list-major, VS_OPT_IVF_KERNEL
1 / 2) against the oracle restatement of IvfIndex.search (vecindex.py:230-258,
filtered extension of SURVEY §8c): identical probes, identical ids,
bit-identical float64 distances, identical visited counts."""

import numpy as np
import pytest
import torch

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O
from paper_2605_15957_b200 import _native as N

pytestmark = pytest.mark.gpu


def _index(rng, n, d, nlist, metric="squared_l2", skew=False):
    data = rng.standard_normal((n, d)).astype(np.float32)
    centroids = data[rng.choice(n, nlist, replace=False)].copy()
    if skew:  # one giant list (longer than a 2048-row selection segment)
        centroids[0] = 0.0
    assign = np.argmin(O.pairwise_sq_l2_fast(data, centroids), axis=1)
    parts = [np.flatnonzero(assign == c).astype(np.int64) for c in range(nlist)]
    payload = [data[p] for p in parts]
    idx = vs.IvfIndex(nlist, d, n, metric, "owning", centroids, parts, payload)
    return idx, data, centroids, parts, payload


def _check(idx, queries, centroids, parts, payload, nprobe, k, metric, mask, kernel):
    ctx = N.Context.get()
    ctx.set_option(N.OPT_IVF_KERNEL, kernel)
    try:
        nt = idx.search(queries, vs.SearchParams(k=k, nprobe=nprobe), row_filter=mask)
    finally:
        ctx.set_option(N.OPT_IVF_KERNEL, 0)
    ref = O.ivf_search(queries, centroids, parts, lambda c: payload[c], nprobe, k, metric, mask=mask)
    assert np.array_equal(nt.probes, ref.probes)
    assert np.array_equal(nt.query_row, ref.query_row)
    assert np.array_equal(nt.data_row, ref.data_row)
    assert np.array_equal(nt.distance, ref.distance)
    assert nt.visited_rows == ref.visited_rows
    return nt


@pytest.mark.parametrize("kernel", [1, 2])
@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
@pytest.mark.parametrize("d,sel", [(64, 0.05), (128, None), (100, 0.3), (384, 0.01), (1024, 0.02)])
def test_ivf_kernels_vs_oracle(kernel, metric, d, sel):
    rng = np.random.default_rng(d * 7 + (kernel if sel is None else 3))
    n, nlist = 12000, 48
    idx, data, centroids, parts, payload = _index(rng, n, d, nlist, metric)
    queries = rng.standard_normal((70, d)).astype(np.float32)
    mask = None if sel is None else rng.random(n) < sel
    for nprobe, k in ((1, 10), (6, 25), (nlist, 10)):
        _check(idx, queries, centroids, parts, payload, nprobe, k, metric, mask, kernel)


@pytest.mark.parametrize("kernel", [1, 2])
def test_ivf_kernels_long_list_and_many_queries_per_list(kernel):
    # a list longer than one selection segment, and > QT queries per list
    rng = np.random.default_rng(5)
    idx, data, centroids, parts, payload = _index(rng, 30000, 64, 8, skew=True)
    assert max(len(p) for p in parts) > 4096
    queries = rng.standard_normal((200, 64)).astype(np.float32) * 0.1
    for mask in (None, rng.random(30000) < 0.5):
        _check(idx, queries, centroids, parts, payload, 3, 40, "squared_l2", mask, kernel)


def test_ivf_kernels_empty_lists_and_empty_filter():
    rng = np.random.default_rng(9)
    idx, data, centroids, parts, payload = _index(rng, 3000, 32, 16)
    queries = rng.standard_normal((30, 32)).astype(np.float32)
    empty = np.zeros(3000, bool)
    for kernel in (1, 2):
        nt = _check(idx, queries, centroids, parts, payload, 4, 5, "squared_l2", empty, kernel)
        assert nt.data_row.size == 0
    # a filter that keeps a handful of rows: most queries get short results
    few = np.zeros(3000, bool)
    few[rng.choice(3000, 7, replace=False)] = True
    for kernel in (1, 2):
        _check(idx, queries, centroids, parts, payload, 16, 5, "squared_l2", few, kernel)


def _bf16_index(rng, n, d, nlist, metric="squared_l2"):
    import torch
    data = rng.standard_normal((n, d)).astype(np.float32)
    xb = torch.from_numpy(data).to(torch.bfloat16)
    rounded = xb.float().numpy()
    col = vs.EmbeddingColumn.from_device(xb.cuda())
    idx = vs.IvfIndex.build(col, nlist, metric=metric, seed=0)
    payload = [rounded[p] for p in idx.partitions]
    return idx, payload


@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
@pytest.mark.parametrize("d", [64, 96, 768])
def test_ivf_tensor_core_scan_vs_oracle(metric, d):
    """tcgen05 list-major scan (VS_OPT_IVF_KERNEL 3): bf16 payload as the B
    operand straight from the list-contiguous layout, queries grouped by list
    as the A operand; exact ids/distances/probes vs the oracle."""
    rng = np.random.default_rng(d + (metric == "inner_product"))
    n, nlist = 20000, 24          # ~830 rows per list: several 256-row tiles per list
    idx, payload = _bf16_index(rng, n, d, nlist, metric)
    queries = rng.standard_normal((300, d)).astype(np.float32)   # > 128 queries per list -> several units
    for mask in (None, rng.random(n) < 0.3):
        for nprobe, k in ((1, 10), (5, 64), (nlist, 10)):
            _check(idx, queries, idx.centroids, idx.partitions, payload, nprobe, k, metric, mask, 3)


def test_ivf_tensor_core_scan_forced_retry():
    rng = np.random.default_rng(77)
    idx, payload = _bf16_index(rng, 6000, 64, 12)
    queries = rng.standard_normal((40, 64)).astype(np.float32)
    ctx = N.Context.get()
    ctx.set_option(N.OPT_FORCE_RETRY, 1)
    try:
        _check(idx, queries, idx.centroids, idx.partitions, payload, 4, 20, "squared_l2", None, 3)
    finally:
        ctx.set_option(N.OPT_FORCE_RETRY, 0)


def test_ivf_lmajor_bf16_payload_matches_qmajor():
    """bf16-stored payload (cfg4 storage): both kernels return the same exact
    top-k over the bf16-rounded rows (the oracle is fed the rounded values)."""
    import torch
    rng = np.random.default_rng(21)
    n, d, nlist = 10000, 96, 32
    data = rng.standard_normal((n, d)).astype(np.float32)
    xb = torch.from_numpy(data).to(torch.bfloat16)
    rounded = xb.float().numpy()
    col = vs.EmbeddingColumn.from_device(xb.cuda())
    idx = vs.IvfIndex.build(col, nlist, seed=0)
    queries = rng.standard_normal((40, d)).astype(np.float32)
    mask = rng.random(n) < 0.2
    payload = [rounded[p] for p in idx.partitions]
    for kernel in (1, 2, 3):
        _check(idx, queries, idx.centroids, idx.partitions, payload, 5, 12, "squared_l2", mask, kernel)


def test_ivf_lmajor_list_sharding_plus_merge():
    from paper_2605_15957_b200.distributed import lpt_assign
    rng = np.random.default_rng(13)
    idx, data, centroids, parts, payload = _index(rng, 9000, 64, 24)
    q = rng.standard_normal((33, 64)).astype(np.float32)
    mask = rng.random(9000) < 0.4
    owner = lpt_assign([len(p) for p in parts], 4)
    outs = [idx.search_raw(q, 9, 6, row_filter=mask, list_owned=(owner == r).astype(np.uint8))
            for r in range(4)]
    ids = np.ascontiguousarray(np.stack([o[0] for o in outs]))
    dist = np.ascontiguousarray(np.stack([o[1] for o in outs]))
    cnt = np.ascontiguousarray(np.stack([o[2] for o in outs]))
    oi, od, oc = np.empty((33, 9), np.int64), np.empty((33, 9)), np.empty(33, np.int32)
    ctx = N.Context.get()
    N.check(N.load().vs_topk_merge(ctx.handle, 4, 33, 9, N.ptr(ids), N.ptr(dist), N.ptr(cnt), 9, 0,
                                   N.ptr(oi), N.ptr(od), N.ptr(oc)))
    whole = idx.search(q, vs.SearchParams(k=9, nprobe=6), row_filter=mask)
    m = np.arange(9)[None, :] < oc[:, None]
    assert np.array_equal(oi[m], whole.data_row)
    assert np.array_equal(od[m], whole.distance)
    # ownership reset: the same device copy scans every list again
    again = idx.search(q, vs.SearchParams(k=9, nprobe=6), row_filter=mask)
    assert np.array_equal(again.data_row, whole.data_row)


def test_sample_trained_index_assign_and_borrowed_payload():
    """Train on a sample (vs_ivf_build), assign every row (vs_ivf_assign,
    vecindex.py:303-304), build the list-contiguous payload in a caller-owned
    device buffer and borrow it (vs_ivf_wrap): searches equal the oracle on
    that structure (the tensor-core and list-major scans alike)."""
    rng = np.random.default_rng(31)
    n, d, nlist = 24000, 96, 20
    data = rng.standard_normal((n, d)).astype(np.float32)
    xd = torch.from_numpy(data).cuda()
    trained = vs.IvfIndex.build(vs.EmbeddingColumn.from_device(xd[:4000].contiguous()), nlist, seed=3)
    lists = trained.assign(vs.EmbeddingColumn.from_device(xd))
    assert lists.dtype == torch.int32 and lists.shape == (n,)
    ref_assign = np.argmin(O.pairwise(data, trained.centroids), axis=1)
    # tensor-core keys, then an exact float64 recheck of every row within the
    # keys' error bound of a second centroid: the reference's first-min argmin
    assert np.array_equal(lists.cpu().numpy(), ref_assign)
    order = torch.sort(lists, stable=True).indices
    sizes = torch.bincount(lists, minlength=nlist).cpu().numpy().astype(np.int64)
    payload = xd[order].to(torch.bfloat16).contiguous()
    idx = vs.IvfIndex.from_device_lists(trained.centroids, sizes, order.cpu().numpy(), payload, count=n)
    parts = np.split(order.cpu().numpy(), np.cumsum(sizes)[:-1])
    rounded = payload.float().cpu().numpy()
    offs = np.r_[0, np.cumsum(sizes)]
    q = rng.standard_normal((50, d)).astype(np.float32)
    mask = rng.random(n) < 0.5
    for kernel in (2, 3):
        _check(idx, q, trained.centroids, parts, [rounded[offs[c]:offs[c + 1]] for c in range(nlist)],
               4, 12, "squared_l2", mask, kernel)


@pytest.mark.parametrize("chunk_rows", [300, 1024])
def test_tensor_core_scan_long_lists_cut_into_row_chunks(chunk_rows):
    """Long lists split into row chunks (each its own work unit and candidate
    buffers, variable buffers per query in phase B): identical to the oracle,
    including a skewed index whose largest list spans many chunks."""
    rng = np.random.default_rng(chunk_rows)
    n, d, nlist = 16000, 64, 12
    data = rng.standard_normal((n, d)).astype(np.float32)
    xb = torch.from_numpy(data).to(torch.bfloat16)
    rounded = xb.float().numpy()
    cen = rounded[rng.choice(n, nlist, replace=False)].copy()
    cen[0] = 0.0                                            # one giant list
    assign = np.argmin(O.pairwise_sq_l2_fast(rounded, cen), axis=1)
    parts = [np.flatnonzero(assign == c).astype(np.int64) for c in range(nlist)]
    assert max(len(p) for p in parts) > 4 * chunk_rows
    order = torch.from_numpy(np.concatenate(parts))
    payload = xb[order].cuda().contiguous()
    idx = vs.IvfIndex.from_device_lists(cen, [len(p) for p in parts], order.numpy(), payload, count=n)
    q = rng.standard_normal((150, d)).astype(np.float32) * 0.2
    ctx = N.Context.get()
    ctx.set_option(N.OPT_IVF_CHUNK_ROWS, chunk_rows)
    try:
        for mask in (None, rng.random(n) < 0.4):
            for metric_k in ((3, 25), (nlist, 10)):
                _check(idx, q, cen, parts, [rounded[p] for p in parts], metric_k[0], metric_k[1],
                       "squared_l2", mask, 3)
    finally:
        ctx.set_option(N.OPT_IVF_CHUNK_ROWS, 0)


@pytest.mark.parametrize("simt", [False, True])
@pytest.mark.parametrize("metric", ["squared_l2", "inner_product"])
@pytest.mark.parametrize("scale", [1.0, 1e-6, 1e5])
def test_filtered_scan_tensor_core_and_simt(simt, metric, scale):
    """The filtered list-major scan over pre-selected rows: its tensor-core
    variant (mma.sync, fp16 operands with power-of-two scales, tensor-core
    margins) and the fp32 SIMT one (VS_OPT_ENN_KERNEL=1) both give the
    reference's exact result, also for magnitudes outside fp16's range and
    mixed query magnitudes; lists hold more selected rows than one 8-row chunk."""
    rng = np.random.default_rng(int(simt) * 10 + int(np.log10(scale)) + 20)
    n, d, nlist = 16000, 128, 24
    idx, data, centroids, parts, payload = _index(rng, n, d, nlist, metric)
    if scale != 1.0:
        data = (data * scale).astype(np.float32)
        centroids = (centroids * scale).astype(np.float32)
        payload = [p * np.float32(scale) for p in payload]
        idx = vs.IvfIndex(nlist, d, n, metric, "owning", centroids, parts, payload)
    queries = (rng.standard_normal((90, d)) * scale).astype(np.float32)
    queries[::5] *= np.float32(300.0)
    mask = rng.random(n) < 0.15
    ctx = N.Context.get()
    ctx.set_option(N.OPT_ENN_KERNEL, 1 if simt else 0)
    try:
        for nprobe, k in ((3, 10), (10, 40)):
            _check(idx, queries, centroids, parts, payload, nprobe, k, metric, mask, 2)
    finally:
        ctx.set_option(N.OPT_ENN_KERNEL, 0)


def test_ivf_pinned_host_outputs_written_in_place():
    """IVF search into page-locked host buffers (zero-copy final outputs)."""
    rng = np.random.default_rng(77)
    n, d, nlist = 12000, 64, 32
    idx, data, centroids, parts, payload = _index(rng, n, d, nlist)
    queries = rng.standard_normal((150, d)).astype(np.float32)
    mask = rng.random(n) < 0.3
    k, nprobe = 12, 5
    out = (torch.full((150, k), 7, dtype=torch.int64).pin_memory(),
           torch.zeros((150, k), dtype=torch.float64).pin_memory(),
           torch.zeros(150, dtype=torch.int32).pin_memory())
    idx.search_raw(torch.from_numpy(queries).pin_memory(), k, nprobe, row_filter=mask, out=out)
    ref = O.ivf_search(queries, centroids, parts, lambda c: payload[c], nprobe, k, mask=mask)
    cnt = out[2].numpy()
    ids = np.concatenate([out[0].numpy()[i, :cnt[i]] for i in range(150)])
    dist = np.concatenate([out[1].numpy()[i, :cnt[i]] for i in range(150)])
    assert np.array_equal(ids, ref.data_row)
    assert np.array_equal(dist, ref.distance)


@pytest.mark.parametrize("pinned", [False, True])
def test_ivf_large_host_query_batch_chunked_upload(pinned, monkeypatch):
    """A large host query batch is uploaded in chunks while the coarse
    quantizer runs on the chunks that have landed (opt-in, VS_Q_CHUNKS):
    identical to the same search with device-resident queries, and sampled
    queries equal the oracle."""
    monkeypatch.setenv("VS_Q_CHUNKS", "4")
    rng = np.random.default_rng(88)
    n, d, nlist = 20000, 512, 256
    idx, data, centroids, parts, payload = _index(rng, n, d, nlist)
    queries = rng.standard_normal((4200, d)).astype(np.float32)     # 8.6 MB: the chunked path
    mask = rng.random(n) < 0.25
    ctx = N.Context.get()
    ctx.set_option(N.OPT_COARSE, 2)
    try:
        hq = torch.from_numpy(queries).pin_memory() if pinned else queries
        host = idx.search(hq, vs.SearchParams(k=10, nprobe=12), row_filter=mask)
        dev = idx.search(torch.from_numpy(queries).cuda(), vs.SearchParams(k=10, nprobe=12), row_filter=mask)
    finally:
        ctx.set_option(N.OPT_COARSE, 0)
    assert np.array_equal(host.probes, dev.probes)
    assert np.array_equal(host.data_row, dev.data_row)
    assert np.array_equal(host.distance, dev.distance)
    sample = np.array([0, 1049, 1050, 2100, 4199])
    ref = O.ivf_search(queries[sample], centroids, parts, lambda c: payload[c], 12, 10, mask=mask)
    assert np.array_equal(host.probes[sample], ref.probes)
    sel = np.isin(host.query_row, sample)
    assert np.array_equal(host.data_row[sel], ref.data_row)
    assert np.array_equal(host.distance[sel], ref.distance)
