"""Native loaders: reference-written SVIX and .emb files
streamed through a pinned double buffer straight into device buffers
(vs_ivf_load, vs_file_to_device); searches over them equal the oracle."""

import numpy as np
import pytest
import torch

import paper_2605_15957_b200 as vs
from oracle import sqlvs_oracle as O

pytestmark = pytest.mark.gpu


def test_reference_svix_to_device_search_equals_oracle(golden):
    from conftest import GOLDEN
    data = np.random.default_rng(5).standard_normal((100, 4)).astype(np.float32)
    centroids, parts, payload = O.ivf_build(data, 4, 0)     # what the golden file holds
    idx = vs.load_index(GOLDEN / "svix_ivf_owning.bin", device=0)
    assert idx.layout == "owning" and idx.nlist == 4 and idx.count == 100
    assert np.array_equal(idx.centroids, centroids)
    for a, b in zip(idx.partitions, parts):
        assert np.array_equal(a, b)
    for a, b in zip(idx.payload, payload):                  # exported back from the device
        assert np.array_equal(a, b)
    q = np.random.default_rng(1).standard_normal((9, 4)).astype(np.float32)
    got = idx.search(q, vs.SearchParams(k=7, nprobe=2))
    ref = O.ivf_search(q, centroids, parts, lambda c: payload[c], 2, 7)
    assert np.array_equal(got.probes, ref.probes)
    assert np.array_equal(got.data_row, ref.data_row)
    assert np.array_equal(got.distance, ref.distance)


def test_svix_large_owning_and_non_owning_roundtrip(tmp_path):
    rng = np.random.default_rng(3)
    n, d, nlist = 300_000, 64, 40           # payload 77 MB: several 64 MiB staging chunks
    data = rng.standard_normal((n, d)).astype(np.float32)
    cen = data[np.sort(rng.choice(n, nlist, replace=False))].copy()
    assign = np.argmin(O.pairwise_sq_l2_fast(data, cen), axis=1)
    parts = [np.flatnonzero(assign == c).astype(np.int64) for c in range(nlist)]
    payload = [data[p] for p in parts]
    own = vs.IvfIndex(nlist, d, n, "inner_product", "owning", cen, parts, payload)
    vs.save_index(own, tmp_path / "own.idx")
    non = own.as_layout("non_owning", base=vs.EmbeddingColumn(data))
    vs.save_index(non, tmp_path / "non.idx")
    q = rng.standard_normal((33, d)).astype(np.float32)
    mask = rng.random(n) < 0.5
    ref = O.ivf_search(q, cen, parts, lambda c: payload[c], 5, 12, "inner_product", mask=mask)
    a = vs.load_index(tmp_path / "own.idx", device=0)
    b = vs.load_index(tmp_path / "non.idx", base=vs.EmbeddingColumn.from_device(torch.from_numpy(data).cuda()),
                      device=0)
    assert b.layout == "non_owning"
    for idx in (a, b):
        got = idx.search(q, vs.SearchParams(k=12, nprobe=5), row_filter=mask)
        assert np.array_equal(got.data_row, ref.data_row)
        assert np.array_equal(got.distance, ref.distance)
    with pytest.raises(vs.ParameterError):
        vs.load_index(tmp_path / "non.idx", device=0)       # non-owning needs its base


def test_reference_emb_to_device(golden, tmp_path):
    from conftest import GOLDEN
    host = vs.read_embeddings(GOLDEN / "ref_small.emb")
    dev = vs.read_embeddings(GOLDEN / "ref_small.emb", device=0)
    assert dev._dev_tensor is not None and dev._dev_tensor.is_cuda
    assert np.array_equal(dev.values, host.values)
    x = np.random.default_rng(17).standard_normal((500, 48)).astype(np.float32)
    assert np.array_equal(host.values, x)
    # a file larger than the staging ring, then an exact search over the device column
    big = np.random.default_rng(2).standard_normal((400_000, 96)).astype(np.float32)
    vs.write_embeddings(tmp_path / "big.emb", vs.EmbeddingColumn(big))
    col = vs.read_embeddings(tmp_path / "big.emb", device=0)
    assert torch.equal(col._dev_tensor.cpu(), torch.from_numpy(big))
    q = big[[5, 77, 399_999]]
    got = vs.enn_search(q, col, vs.SearchParams(k=4))
    assert np.array_equal(got.data_row.reshape(3, 4)[:, 0], [5, 77, 399_999])
    with pytest.raises(vs.ParameterError):
        (tmp_path / "bad.emb").write_bytes(b"NOPE" + b"\0" * 16)
        vs.read_embeddings(tmp_path / "bad.emb", device=0)
